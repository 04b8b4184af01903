export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/it
timeout 1200 python -m pytest tests -m gpu -x -q -k "units or tiny_end or 7b_width_c5 or full or rollback" > gpurun_out/it/pytest.log 2>&1; tail -2 gpurun_out/it/pytest.log
for i in 1 2; do for v in X=1 SV_NO_WARM=1; do env $v timeout 300 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/it/c2.json 2>gpurun_out/it/c2.err
python -c "
import json; d=json.load(open('gpurun_out/it/c2.json')); k=d['roofline']['kernels']; print('$v C2 p50 %.4f ms tok/s %.0f frac %.4f step_frac %.4f' % (d['latency_p50_ms'], d['value'], d['roofline']['frac'], d['roofline']['step_frac_of_peak']), {kk: round(v['ms']*1e3/max(1,v['launches']),1) for kk,v in k.items()})" || tail -3 gpurun_out/it/c2.err; done; done
