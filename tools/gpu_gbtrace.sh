# persistent-GEMM phase stamps (libsv_tr.so built with -DSV_GB_TRACE) at C5 and the C4 32-request shard
export PYTHONUNBUFFERED=1
OUT=gpurun_out/gbt
mkdir -p $OUT
export SV_LIB=$PWD/paper_2505_21594_b200/libsv_tr.so
SV_GTRACE=$OUT/g_c5.csv timeout 300 python tools/trace_step.py --batch 16 --ctx 2048 --layers 10 > $OUT/c5.txt 2>&1
SV_GTRACE=$OUT/g_c4.csv timeout 300 python tools/trace_step.py --batch 32 --ctx 1024 --layers 10 > $OUT/c4b32.txt 2>&1
