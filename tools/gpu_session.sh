export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cfg in "X=1" "SV_NO_ATTN_WARM=1" "X=2" "SV_NO_ATTN_WARM=2"; do env $cfg timeout 900 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json')); r=d['roofline']; print('C2 $cfg', d['latency_p50_ms'], d['value'], r['step_frac_of_peak'])" || tail -3 gpurun_out/b.err; done
SV_ATRACE=gpurun_out/at.csv SV_KTRACE=gpurun_out/kt.csv timeout 300 python tools/ncu_step.py --steps 3 > /dev/null 2>&1
python tools/atrace_report.py gpurun_out/at.csv gpurun_out/kt.csv 2>&1 | head -9
for c in C5 C4; do timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json')); r=d['roofline']; print('$c', d['latency_p50_ms'], d['value'], r['step_frac_of_peak'])" || tail -3 gpurun_out/b.err; done
