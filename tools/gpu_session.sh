export PYTHONUNBUFFERED=1
for cfg in "--batch 16 --ctx 2048" "--batch 1 --ctx 512"; do
SV_KTRACE=gpurun_out/kt.csv timeout 300 python tools/ncu_step.py $cfg --steps 3 > /dev/null 2>&1
echo "== $cfg"; python tools/ktrace_report.py gpurun_out/kt.csv 2>&1 | head -14
done
for cfg in "X=1" "SV_SPLIT_ANY=1"; do env $cfg timeout 600 python bench.py --config C5 --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json')); r=d['roofline']; print('C5 $cfg', d['latency_p50_ms'])" || tail -3 gpurun_out/b.err; done
