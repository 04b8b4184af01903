export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err
python -c "
import json; d=json.load(open('gpurun_out/final_c2.json')); r=d['roofline']; print(d['latency_p50_ms'], d['value'], r['frac'], r['step_frac_of_peak'], d['cpu_baseline']['value'], d['cpu_baseline']['cores'], d['e2e'])"
