export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/full
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/full/pytest.log 2>&1; tail -2 gpurun_out/full/pytest.log
timeout 600 python bench.py > gpurun_out/full/c2.json 2> gpurun_out/full/c2.err
python -c "
import json; d=json.load(open('gpurun_out/full/c2.json')); print('C2', d['latency_p50_ms'], d['value'], d['tokens_per_step'], d['roofline']['frac'], d['roofline']['step_frac_of_peak'], d['exit_ready']['dev_ms_p50'], d['cpu_baseline']['value'] if d['cpu_baseline'] else None)" || tail -3 gpurun_out/full/c2.err
timeout 600 python bench.py --config C5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/full/c5.json 2>/dev/null
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/full/c4.json 2>/dev/null
for c in c5 c4; do python -c "
import json; d=json.load(open('gpurun_out/full/$c.json')); print('$c', d['latency_p50_ms'], d['value'], d['roofline']['bound'], d['roofline']['frac'])"; done
