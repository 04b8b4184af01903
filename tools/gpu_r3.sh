export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/r3
timeout 900 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_multirank.py -x -q -s > gpurun_out/r3/pytest.log 2>&1
timeout 600 python bench.py > gpurun_out/r3/c2.json 2> gpurun_out/r3/c2.err
timeout 300 python bench.py --all-exits --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r3/c2_all.json 2> gpurun_out/r3/c2_all.err
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3/c4.json 2> gpurun_out/r3/c4.err
tail -3 gpurun_out/r3/pytest.log
