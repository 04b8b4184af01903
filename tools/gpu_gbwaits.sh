export PYTHONUNBUFFERED=1
OUT=gpurun_out/gbw
mkdir -p $OUT
export SV_LIB=$PWD/paper_2505_21594_b200/libsv_tr.so
for c in "c4:--batch 256 --ctx 1024" "c4s:--batch 32 --ctx 1024" "c5:--batch 16 --ctx 2048"; do
  n=${c%%:*}; SV_GTRACE=$OUT/g_$n.csv timeout 300 python tools/trace_step.py ${c#*:} --layers 10 > $OUT/tr_$n.txt 2>&1
  echo "== $n"; grep "layer 10 " $OUT/tr_$n.txt; python tools/gb_waits.py $OUT/g_$n.csv
done
