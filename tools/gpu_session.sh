export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_ar.py -x -q -s 2>&1 | tail -8
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --gamma 0 --no-cpu-baseline --steps 30 > gpurun_out/b_ar.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b_ar.json')); r=d['roofline']; print('AR', d['latency_p50_ms'], d['value'], d['tokens_per_step'], r['step_frac_of_peak'])" || tail -5 gpurun_out/b.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 | tail -c 400
