export PYTHONUNBUFFERED=1
for cfg in "X=1" "SV_PDL_LATE=1" "X=2" "SV_PDL_LATE=2"; do env $cfg timeout 600 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json')); r=d['roofline']; print('$cfg', d['latency_p50_ms'], d['value'], r['step_frac_of_peak'])" || tail -3 gpurun_out/b.err; done
