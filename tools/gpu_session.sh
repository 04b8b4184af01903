export PYTHONUNBUFFERED=1
for cfg in "X=1" "SV_NO_WAVE=1"; do env $cfg timeout 900 python bench.py --config C4 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json')); r=d['roofline']; print('C4 $cfg', d['latency_p50_ms'], d['value'], r['step_frac_of_peak'], {k:v['ms'] for k,v in r['kernels'].items()})" || tail -3 gpurun_out/b.err; done
for b in 64 128; do for cfg in "X=1" "SV_NO_WAVE=1"; do env $cfg timeout 900 python bench.py --config C4 --batch $b --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json')); r=d['roofline']; print('C4 B=$b $cfg', d['latency_p50_ms'], d['value'], r['step_frac_of_peak'])" || tail -3 gpurun_out/b.err; done; done
