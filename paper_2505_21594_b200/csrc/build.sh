#!/usr/bin/env bash
# Builds libsv.so (all CUDA kernels + the C-ABI engine) for sm_100a, in-tree.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
OUT="${1:-$HERE/../libsv.so}"
shift || true
NVCC="${NVCC:-/usr/local/cuda/bin/nvcc}"
FLAGS=(-std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a
       -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -shared -cudart static
       -Xptxas -v --expt-relaxed-constexpr "$@")
"$NVCC" "${FLAGS[@]}" -o "$OUT" \
  "$HERE/engine.cu" "$HERE/gemm.cu" "$HERE/attn.cu" "$HERE/accept.cu" "$HERE/misc.cu" "$HERE/fused.cu" "$HERE/attn3.cu" "$HERE/gemm_big.cu" 2> "$HERE/../build.log" \
  || { cat "$HERE/../build.log"; exit 1; }
echo "built $OUT"
