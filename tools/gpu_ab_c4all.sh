# same-box A/B at C5, the C4 per-GPU shards (32 / 64 / 128 requests) and C4 (VARS as gpu_ab_big.sh)
export PYTHONUNBUFFERED=1
OUT=gpurun_out/abc4
mkdir -p $OUT
[ -n "$TESTS" ] && { timeout 900 python -m pytest tests -m gpu -q -x -k "$TESTS" > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log; }
run() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --no-cpu-baseline --no-extra $cfg > $OUT/$name.json 2>$OUT/$name.err;
  python -c "
import json; d=json.load(open('$OUT/$name.json')); k=d['roofline']['kernels']; print('%-16s p50 %.4f ms  qkv %.1f O %.1f gu %.1f dn %.1f attn %.1f lm %.1f us' % ('$name', d['latency_p50_ms'], *[k[x]['ms']*1e3/32 for x in ('gemm_qkv','gemm_o','gemm_gate_up','gemm_down','attention')], k['gemm_lm_final']['ms']*1e3))" || tail -2 $OUT/$name.err; }
for rep in 1 2; do
for v in $VARS; do
  run c5_${v%%:*}$rep "--config C5 --steps 20 --warmup 3" ${v#*:}
  for b in 32 64 128; do run c4b${b}_${v%%:*}$rep "--config C4 --batch $b --steps 10 --warmup 3" ${v#*:}; done
  [ -n "$WITH_C4" ] && run c4_${v%%:*}$rep "--config C4 --steps 5 --warmup 3" ${v#*:}
done
done
