export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_verify.py -x -q -s -k "c4_batch" 2>&1 | tail -4
