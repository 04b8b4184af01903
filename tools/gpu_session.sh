export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
run() { # tag config env...
  tag=$1; c=$2; shift 2
  env "$@" timeout 900 python bench.py --config $c --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "
import json; d=json.load(open('gpurun_out/b.json')); r=d['roofline']; print('$tag', d['latency_p50_ms'], d['value'], r['step_frac_of_peak'], {k:v['ms'] for k,v in r['kernels'].items() if k in ('gemm_o','gemm_down')})" || tail -3 gpurun_out/b.err
}
ALT=SV_LIB=$PWD/paper_2505_21594_b200/libsv_alt.so
for c in C5 C5 C4 C2; do run "$c stash" $c X=1; run "$c old" $c $ALT; done
