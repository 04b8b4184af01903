set -x
export PYTHONUNBUFFERED=1
./tools/tma_bw > gpurun_out/tma_bw_gu.txt 2>&1
./tools/tma_bw 12288 4096 > gpurun_out/tma_bw_qkv.txt 2>&1
./tools/tma_bw 4096 4096 > gpurun_out/tma_bw_o.txt 2>&1
SV_FUSED=1 timeout 600 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_c2_fused.json 2> gpurun_out/bench_c2_fused.err
SV_FUSED=1 SV_TRACE=gpurun_out/ftrace_c2.csv timeout 300 python tools/ncu_step.py --steps 3 > gpurun_out/ftrace.log 2>&1
python tools/trace_report.py gpurun_out/ftrace_c2.csv > gpurun_out/ftrace_report.txt 2>&1
cat gpurun_out/tma_bw_*.txt; tail -c 300 gpurun_out/bench_c2_fused.json; head -50 gpurun_out/ftrace_report.txt
