mkdir -p gpurun_out/ncu
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:gemm_big -s 4 -c 1 -o gpurun_out/ncu/big_full -f python tools/ncu_step.py --batch 64 --ctx 1024 > gpurun_out/ncu/big.log 2>&1
ncu -i gpurun_out/ncu/big_full.ncu-rep --page source --csv > gpurun_out/ncu/big_source.csv 2>&1
ncu -i gpurun_out/ncu/big_full.ncu-rep --page details --csv > gpurun_out/ncu/big_details.csv 2>&1
tail -3 gpurun_out/ncu/big.log
