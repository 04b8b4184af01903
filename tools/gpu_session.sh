export PYTHONUNBUFFERED=1
for c in C2 C5; do timeout 900 python bench.py --config $c --prefill --no-cpu-baseline --steps 10 > gpurun_out/b_pf_$c.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b_pf_$c.json')); r=d['roofline']; print('$c', d['latency_p50_ms'], d['value'], d['tokens_per_step'], r['step_frac_of_peak'], d['prefill'])" || tail -5 gpurun_out/b.err; done
