export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/tr
SV_GTRACE=gpurun_out/tr/gtrace_c5.csv timeout 300 python tools/trace_step.py --batch 16 --ctx 2048 --layers 10 > gpurun_out/tr/c5.txt 2>&1
cat gpurun_out/tr/c5.txt | grep "gemm_o (us\|gemm_down (us\|gemm_qkv (us\|charged\|  gemm\|traced"
