# ncu --set full of one decoder layer's persistent GEMMs + attention at C5 (16 requests,
# ctx 2048) and the C4 8-GPU shard (32 requests, ctx 1024); raw metrics to CSV
export PYTHONUNBUFFERED=1
OUT=gpurun_out/ncu5
mkdir -p $OUT
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum"
for c in "c5:--batch 16 --ctx 2048" "c4s:--batch 32 --ctx 1024"; do
  n=${c%%:*}
  timeout 900 ncu --profile-from-start off --set full --clock-control none -k regex:"gemm_big|attn3" -s 5 -c 5 -o $OUT/$n -f python tools/ncu_step.py ${c#*:} > $OUT/ncu_$n.log 2>&1
  ncu -i $OUT/$n.ncu-rep --page raw --csv --metrics $M > $OUT/${n}_raw.csv 2>&1
done
ls -la $OUT
