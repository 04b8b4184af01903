# quick iteration: correctness subset + C2 bench + trace
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/it
timeout 900 python -m pytest tests -m gpu -x -q -k "units or 7b or tiny_end or graphs or exits or full or boundary or rollback" > gpurun_out/it/pytest.log 2>&1; tail -2 gpurun_out/it/pytest.log
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/it/c2_$i.json 2>gpurun_out/it/c2.err
python -c "
import json; d=json.load(open('gpurun_out/it/c2_$i.json')); k=d['roofline']['kernels']; print('C2 p50 %.4f ms tok/s %.0f frac %.4f step_frac %.4f' % (d['latency_p50_ms'], d['value'], d['roofline']['frac'], d['roofline']['step_frac_of_peak']), {kk: round(v['ms']*1e3/max(1,v['launches']),1) for kk,v in k.items()})" || tail -3 gpurun_out/it/c2.err; done
SV_GTRACE=gpurun_out/it/gtrace.csv timeout 300 python tools/trace_step.py --layers 10 > gpurun_out/it/trace.txt 2>&1; cat gpurun_out/it/trace.txt
