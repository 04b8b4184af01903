export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_verify.py tests/test_gpu_full.py -m gpu -x -q 2>&1 | tail -1
for B in 64 32; do timeout 900 python bench.py --config C4 --batch $B --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('C4 B=$B', d['latency_p50_ms'])" || tail -3 gpurun_out/b.err; done
timeout 600 python bench.py --config C5 --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('C5', d['latency_p50_ms'])"
timeout 600 python bench.py > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json')); print('C2', d['latency_p50_ms'], d['value'], d['roofline']['frac'])"
