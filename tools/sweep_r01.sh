set -x
timeout 300 python -m pytest tests/test_gpu_verify.py -q -x -k "large_batch" > gpurun_out/large_batch.log 2>&1; tail -1 gpurun_out/large_batch.log
for g in 1 2 3 4 5 6 7 8; do timeout 200 python bench.py --config C3 --gamma $g --exit-layer 16 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/c3_g$g.json 2> gpurun_out/c3_g$g.err; done
for e in 8 24; do timeout 200 python bench.py --config C3 --gamma 4 --exit-layer $e --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/c3_e$e.json 2> gpurun_out/c3_e$e.err; done
timeout 300 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c5.json 2> gpurun_out/c5.err
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c4.json 2> gpurun_out/c4.err
echo done
