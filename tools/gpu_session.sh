export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/b.json 2>gpurun_out/b.err
python -c "
import json; d=json.load(open('gpurun_out/b.json')); r=d['roofline']; print(d['latency_p50_ms'], r['step_frac_of_peak'], {k:v['ms'] for k,v in r['kernels'].items()})" || tail -5 gpurun_out/b.err
SV_ATRACE=gpurun_out/at.csv SV_KTRACE=gpurun_out/kt_at.csv timeout 300 python tools/ncu_step.py --steps 3 > gpurun_out/kt.log 2>&1
python tools/ktrace_report.py gpurun_out/kt_at.csv | tail -1
