export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/it2
timeout 900 python -m pytest tests/test_gpu_units.py -q -s -k million 2>&1 | grep -E "trials|passed|failed"
timeout 900 python -m pytest tests -m gpu -x -q -k "7b or tiny_end or full" 2>&1 | tail -1
VARIANTS=("new:X=1" "prev:SV_LIB=$PWD/paper_2505_21594_b200/libsv_prev.so")
source tools/ab.sh
bash tools/gpu_sanitizer.sh 2>&1 | grep "rc="
