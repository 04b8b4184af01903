# distributed stream-K reduction: parity tests at 7B width (C5 batch, C4 shard, C4 batch),
# then same-box A/B against the previous build at C5 / C4 shard (SV_SK_FILL variants), + phase trace
export PYTHONUNBUFFERED=1
OUT=gpurun_out/sk2
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_verify.py -q -x -k "c5_batch or c4_shard or c4_batch or rollback or tiny_large" > $OUT/pytest.log 2>&1; tail -3 $OUT/pytest.log
run() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --no-cpu-baseline $cfg > $OUT/$name.json 2>$OUT/$name.err;
  python -c "
import json; d=json.load(open('$OUT/$name.json')); k=d['roofline']['kernels']; print('%-14s p50 %.4f ms  qkv %.1f O %.1f gu %.1f dn %.1f attn %.1f us' % ('$name', d['latency_p50_ms'], *[k[x]['ms']*1e3/32 for x in ('gemm_qkv','gemm_o','gemm_gate_up','gemm_down','attention')]))" || tail -2 $OUT/$name.err; }
C5="--config C5 --steps 20 --warmup 3"
C4S="--config C4 --batch 32 --steps 10 --warmup 3"
for rep in 1 2; do
run c5_prev$rep "$C5" SV_LIB=$PWD/paper_2505_21594_b200/libsv_prev.so
run c5_new$rep "$C5" X=1
run c5_new_f1$rep "$C5" SV_SK_FILL=1.01
run c4s_prev$rep "$C4S" SV_LIB=$PWD/paper_2505_21594_b200/libsv_prev.so
run c4s_new$rep "$C4S" X=1
run c4s_new_f1$rep "$C4S" SV_SK_FILL=1.01
done
export SV_LIB=$PWD/paper_2505_21594_b200/libsv_tr.so
SV_SK_FILL=1.01 SV_GTRACE=$OUT/g_c4.csv timeout 300 python tools/trace_step.py --batch 32 --ctx 1024 --layers 10 > $OUT/tr_c4b32.txt 2>&1
SV_SK_FILL=1.01 SV_GTRACE=$OUT/g_c5.csv timeout 300 python tools/trace_step.py --batch 16 --ctx 2048 --layers 10 > $OUT/tr_c5.txt 2>&1
