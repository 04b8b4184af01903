# refresh the round-2 lines the last commits changed: the C4 per-GPU shards, C4, C5, and the
# default C2 run (with also_measured)
export PYTHONUNBUFFERED=1
OUT=gpurun_out/refresh
mkdir -p $OUT
timeout 600 python bench.py > $OUT/c2.json 2> $OUT/c2.err
timeout 600 python bench.py --config C5 --steps 20 --warmup 3 --no-cpu-baseline --no-extra > $OUT/c5.json 2>/dev/null
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/c4.json 2>/dev/null
for b in 32 64 128; do timeout 600 python bench.py --config C4 --batch $b --steps 10 --warmup 3 --no-cpu-baseline > $OUT/c4_b$b.json 2>/dev/null; done
for f in $OUT/*.json; do python -c "
import json; d=json.load(open('$f')); print('$f', d['latency_p50_ms'], d['value'], d['roofline']['bound'], d['roofline']['frac'], d['roofline']['step_frac_of_peak'], d['clocks'])"; done
