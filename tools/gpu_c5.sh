export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/c5
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 600 python bench.py --config C5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/c5/c5.json 2>gpurun_out/c5/c5.err
timeout 600 python bench.py --config C4 --batch 32 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c5/c4_32.json 2>/dev/null
timeout 600 python bench.py --config C4 --batch 64 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c5/c4_64.json 2>/dev/null
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c5/c4.json 2>/dev/null
timeout 600 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/c5/c2.json 2>/dev/null
for c in c5 c4_32 c4_64 c4 c2; do python -c "
import json; d=json.load(open('gpurun_out/c5/$c.json')); k=d['roofline']['kernels']; print('$c', d['latency_p50_ms'], round(d['value']), d['roofline']['bound'], d['roofline']['frac'], {kk: round(v['ms']*1e3/max(1,v['launches']),1) for kk,v in k.items() if 'exit' not in kk})" || tail -2 gpurun_out/c5/c5.err; done
