export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
SV_A3_MINB=2 timeout 600 python -m pytest tests/test_gpu_verify.py tests/test_gpu_full.py -m gpu -x -q 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
bash tools/gpu_final.sh
