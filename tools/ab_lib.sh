# same-box A/B of the working build (libsv.so) against libsv_prev.so, + a GPU test subset
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/ab
timeout 1200 python -m pytest tests -m gpu -x -q -k "${TESTS:-units or tiny_end or 7b or full or rollback or exits or prefill}" 2>&1 | tail -1
VARIANTS=("new:X=1" "prev:SV_LIB=$PWD/paper_2505_21594_b200/libsv_prev.so")
source tools/ab.sh
