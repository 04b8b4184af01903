export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/tr
timeout 900 python -m pytest tests -m gpu -x -q -k "units or tiny_end or 7b_width_c4 or full or ar_" 2>&1 | tail -1
SV_GTRACE=gpurun_out/tr/gtrace_c2.csv timeout 300 python tools/trace_step.py --layers 10 > gpurun_out/tr/c2.txt 2>&1
cat gpurun_out/tr/c2.txt
for v in X=1 X=1; do env $v timeout 300 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/tr/b.json 2>gpurun_out/tr/b.err; python -c "
import json; d=json.load(open('gpurun_out/tr/b.json')); k=d['roofline']['kernels']; print('$v C2 p50 %.4f ms frac %.4f' % (d['latency_p50_ms'], d['roofline']['frac']), d['exit_ready']['dev_ms_p50'], {kk: round(v['ms']*1e3/max(1,v['launches']),1) for kk,v in k.items()})" || tail -3 gpurun_out/tr/b.err; done
