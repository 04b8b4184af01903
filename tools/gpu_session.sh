export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json')); r=d['roofline']; print(d['latency_p50_ms'], r['step_frac_of_peak'], {k:v['ms'] for k,v in r['kernels'].items()})" || tail -5 gpurun_out/b.err
for c in C5 C4; do timeout 600 python bench.py --config $c --no-cpu-baseline --steps 10 > gpurun_out/b_$c.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b_$c.json')); r=d['roofline']; print('$c', d['latency_p50_ms'], d['value'], r['step_frac_of_peak'], {k:v['ms'] for k,v in r['kernels'].items()})" || tail -5 gpurun_out/b.err; done
