# same-box A/B of variants on the C2 bench (VARS="name:ENV=.. name2:SV_LIB=..."), interleaved twice
export PYTHONUNBUFFERED=1
OUT=gpurun_out/abc2
mkdir -p $OUT
[ -n "$TESTS" ] && { timeout 900 python -m pytest tests -m gpu -q -x -k "$TESTS" > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log; }
run() { name=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --steps ${STEPS:-100} --warmup 5 > $OUT/$name.json 2>$OUT/$name.err;
  python -c "
import json; d=json.load(open('$OUT/$name.json')); k=d['roofline']['kernels']; print('%-12s p50 %.4f ms  qkv %.1f attn %.1f O %.1f gu %.1f dn %.1f us' % ('$name', d['latency_p50_ms'], *[k[x]['ms']*1e3/32 for x in ('gemm_qkv','attention','gemm_o','gemm_gate_up','gemm_down')]))" || tail -2 $OUT/$name.err; }
for rep in 1 2 3; do
for v in $VARS; do run ${v%%:*}$rep $(echo ${v#*:} | tr "," " "); done
done
