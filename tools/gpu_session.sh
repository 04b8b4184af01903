export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_exits.py -x -q 2>&1 | tail -8
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --no-cpu-baseline --steps 20 --all-exits > gpurun_out/b_allexits.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b_allexits.json')); r=d['roofline']; print('all-exits', d['latency_p50_ms'], d['value'], r['step_frac_of_peak'], d['config']['workload'])" || tail -5 gpurun_out/b.err
