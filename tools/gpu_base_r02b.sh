export PYTHONUNBUFFERED=1
OUT=gpurun_out/base
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt
timeout 300 python tools/trace_step.py --batch 16 --ctx 2048 --layers 10 > $OUT/tr_c5.txt 2>&1
timeout 300 python tools/trace_step.py --batch 32 --ctx 1024 --layers 10 > $OUT/tr_c4b32.txt 2>&1
timeout 300 python tools/trace_step.py --batch 1 --ctx 512 --layers 10 > $OUT/tr_c2.txt 2>&1
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $OUT/c2.json 2>$OUT/c2.err
timeout 300 python bench.py --config C5 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/c5.json 2>/dev/null
timeout 300 python bench.py --config C4 --batch 32 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/c4b32.json 2>/dev/null
for f in $OUT/*.json; do python -c "
import json; d=json.load(open('$f')); print('$f', d.get('latency_p50_ms'), d['value'], d['roofline']['frac'], d['clocks'])"; done
