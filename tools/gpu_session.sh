export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for cfg in "X=1" "SV_NO_ODD_TILES=1"; do env $cfg timeout 600 python bench.py --config C5 --no-cpu-baseline --steps 10 > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json')); r=d['roofline']; print('C5 $cfg', d['latency_p50_ms'], d['value'], r['step_frac_of_peak'], {k:v['ms'] for k,v in r['kernels'].items()})" || tail -3 gpurun_out/b.err; done
for cfg in "X=1" "SV_NO_ODD_TILES=1"; do env $cfg timeout 600 python bench.py --config C4 --batch 32 --no-cpu-baseline --steps 10 > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json')); r=d['roofline']; print('C4@8 $cfg', d['latency_p50_ms'], d['value'], r['step_frac_of_peak'], {k:v['ms'] for k,v in r['kernels'].items()})" || tail -3 gpurun_out/b.err; done
