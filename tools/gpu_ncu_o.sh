mkdir -p gpurun_out/ncu
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:gemm_kernel -s 9 -c 1 -o gpurun_out/ncu/o_full -f python tools/ncu_step.py > gpurun_out/ncu/o.log 2>&1
ncu -i gpurun_out/ncu/o_full.ncu-rep --page source --csv > gpurun_out/ncu/o_source.csv 2>&1
ncu -i gpurun_out/ncu/o_full.ncu-rep --page details --csv > gpurun_out/ncu/o_details.csv 2>&1
tail -3 gpurun_out/ncu/o.log; wc -l gpurun_out/ncu/o_source.csv
