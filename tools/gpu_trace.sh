export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/tr
SV_GTRACE=gpurun_out/tr/gtrace_c2.csv SV_ATRACE=gpurun_out/tr/atrace_c2.csv timeout 300 python tools/trace_step.py --layers 10 > gpurun_out/tr/c2.txt 2>&1
cat gpurun_out/tr/c2.txt
