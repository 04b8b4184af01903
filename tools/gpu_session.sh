export PYTHONUNBUFFERED=1
timeout 900 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json')); r=d['roofline']; print('C2', d['latency_p50_ms'], d['ms_per_step'], d['value'], r['step_frac_of_peak'])" || tail -3 gpurun_out/b.err
