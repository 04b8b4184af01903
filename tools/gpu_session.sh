export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_adapters.py -x -q -s 2>&1 | tail -15
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
