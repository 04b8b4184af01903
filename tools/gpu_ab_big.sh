# same-box A/B of the working build against libsv_prev.so at C5 / the C4 32-request shard / C4,
# with a 7B-width parity subset first; then persistent-GEMM phase traces (libsv_tr.so)
export PYTHONUNBUFFERED=1
OUT=gpurun_out/abb
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_verify.py -q -x -k "${TESTS:-c5_batch or c4_shard or c4_batch or tiny_large}" > $OUT/pytest.log 2>&1; tail -1 $OUT/pytest.log
run() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --no-cpu-baseline $cfg > $OUT/$name.json 2>$OUT/$name.err;
  python -c "
import json; d=json.load(open('$OUT/$name.json')); k=d['roofline']['kernels']; print('%-14s p50 %.4f ms  qkv %.1f O %.1f gu %.1f dn %.1f attn %.1f us' % ('$name', d['latency_p50_ms'], *[k[x]['ms']*1e3/32 for x in ('gemm_qkv','gemm_o','gemm_gate_up','gemm_down','attention')]))" || tail -2 $OUT/$name.err; }
C5="--config C5 --steps 20 --warmup 3"
C4S="--config C4 --batch 32 --steps 10 --warmup 3"
C4="--config C4 --steps 5 --warmup 3"
for rep in 1 2; do
for v in ${VARS:-prev:SV_LIB=$PWD/paper_2505_21594_b200/libsv_prev.so new:X=1}; do
  run c5_${v%%:*}$rep "$C5" ${v#*:}
  run c4s_${v%%:*}$rep "$C4S" ${v#*:}
  [ -n "$WITH_C4" ] && run c4_${v%%:*}$rep "$C4" ${v#*:}
done
done
if [ -n "$TRACE" ]; then
export SV_LIB=$PWD/paper_2505_21594_b200/libsv_tr.so
SV_GTRACE=$OUT/g_c4.csv timeout 300 python tools/trace_step.py --batch 32 --ctx 1024 --layers 10 > $OUT/tr_c4b32.txt 2>&1
SV_GTRACE=$OUT/g_c5.csv timeout 300 python tools/trace_step.py --batch 16 --ctx 2048 --layers 10 > $OUT/tr_c5.txt 2>&1
grep "layer 10 " $OUT/tr_*.txt
fi
