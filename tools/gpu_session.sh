export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in C2 C5; do for cfg in "X=1" "SV_NO_BOX=1"; do env $cfg timeout 600 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/b_$c.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b_$c.json')); r=d['roofline']; print('$c $cfg', d['latency_p50_ms'], d['value'], r['step_frac_of_peak'], {k:v['ms'] for k,v in r['kernels'].items()})" || tail -5 gpurun_out/b.err; done; done
