export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cfg in "X=1" "SV_O_RING=0" "X=2" "SV_O_RING=0"; do env $cfg timeout 900 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json')); r=d['roofline']; print('C2 $cfg', d['latency_p50_ms'], d['value'], r['step_frac_of_peak'])" || tail -3 gpurun_out/b.err; done
