export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_units.py -x -q -k edge 2>&1 | tail -15
