export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
run() { # tag config env...
  tag=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "
import json; d=json.load(open('gpurun_out/b.json')); r=d['roofline']; print('$tag', d['latency_p50_ms'], d['value'], r['step_frac_of_peak'], {k:v['ms'] for k,v in r['kernels'].items() if k.startswith('gemm') or k=='attention'})" || tail -3 gpurun_out/b.err
}
run "C4 t160" C4 X=1
run "C4 no-t160" C4 SV_NO_T160=1
run "C5 default" C5 X=1
run "C5 s2" C5 SV_ATTN_SPLITS=2
run "C5 s4" C5 SV_ATTN_SPLITS=4
run "C2 default" C2 X=1
run "C2 nst2" C2 SV_ATTN_NST=2
