# Round-2 measurement set: GPU tests, bench lines (C2 with the CPU oracle baseline, the
# reference arm, C3 sweeps, all-exits, AR, C5 (+prefill), C4 and its per-GPU shards),
# ncu launch list + full capture (C2), ncu capture of a C4 persistent GEMM, sanitizer.
export PYTHONUNBUFFERED=1
OUT=gpurun_out/final
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/gpu.txt
(nproc; lscpu | grep "Model name") >> $OUT/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; tail -1 $OUT/pytest_gpu.log
cp -r gpurun_out/parity $OUT/parity 2>/dev/null
timeout 900 python bench.py > $OUT/c2.json 2> $OUT/c2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/reference.json 2> $OUT/reference.err
for g in 1 2 3 4 5 6 7 8; do timeout 300 python bench.py --config C3 --gamma $g --steps 50 --warmup 5 --no-cpu-baseline > $OUT/c3_g$g.json 2>/dev/null; done
for e in 8 24; do timeout 300 python bench.py --config C3 --exit-layer $e --steps 50 --warmup 5 --no-cpu-baseline > $OUT/c3_e$e.json 2>/dev/null; done
timeout 300 python bench.py --all-exits --steps 50 --warmup 5 --no-cpu-baseline > $OUT/c2_all_exits.json 2>/dev/null
timeout 300 python bench.py --gamma 0 --steps 50 --warmup 5 --no-cpu-baseline > $OUT/c2_ar_gamma0.json 2>/dev/null
timeout 600 python bench.py --config C5 --steps 20 --warmup 3 --no-cpu-baseline > $OUT/c5.json 2>/dev/null
timeout 600 python bench.py --config C5 --prefill --steps 20 --warmup 3 --no-cpu-baseline > $OUT/c5_prefill.json 2>/dev/null
timeout 900 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/c4.json 2>/dev/null
for b in 32 64 128; do timeout 600 python bench.py --config C4 --batch $b --steps 10 --warmup 3 --no-cpu-baseline > $OUT/c4_b$b.json 2>/dev/null; done
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/c2_launches.csv python tools/ncu_step.py > $OUT/ncu_list.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"gemm_kernel|attn3" -c 10 -o $OUT/c2_full -f python tools/ncu_step.py > $OUT/ncu_full.log 2>&1
python tools/ncu_summarize.py --list $OUT/c2_launches.csv --full $OUT/c2_full.ncu-rep --out $OUT/ncu_summary.json --source "C2 (Llama2-7B shape, B=1, ctx 512, gamma 4, exit 16): ncu launch list of one step (cold-cache, serialised) + --set full on the first 10 gemm/attention launches" > /dev/null
ncu --profile-from-start off --set full --clock-control none -k regex:gemm_big -s 2 -c 4 -o $OUT/c4_gemm_full -f python tools/ncu_step.py --batch 256 --ctx 1024 > $OUT/ncu_c4.log 2>&1
ncu -i $OUT/c4_gemm_full.ncu-rep --page details --csv > $OUT/c4_gemm_details.csv 2>&1
ncu -i $OUT/c4_gemm_full.ncu-rep --page raw --csv --metrics sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed > $OUT/c4_gemm_raw.csv 2>&1
# (compute-sanitizer runs are closed on this GPU pool: tools/gpu_sanitizer.sh kept for pools that allow them)
for f in $OUT/*.json; do python -c "
import json,sys
d=json.load(open('$f'))
if 'roofline' in d and d['roofline']: print('$f', d.get('latency_p50_ms'), d['value'], d['roofline']['bound'], d['roofline']['frac'], d['roofline'].get('step_frac_of_peak'))
elif 'impl' in d: print('$f', d.get('value'), d.get('ms_per_step'))
" 2>/dev/null; done

