#!/usr/bin/env bash
# Builds libsv.so (all CUDA kernels + the C-ABI engine) for sm_100a, in-tree.
# Each translation unit compiles in parallel into build/, then one link step.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
OUT="${1:-$HERE/../libsv.so}"
shift || true
NVCC="${NVCC:-/usr/local/cuda/bin/nvcc}"
OBJ="${SV_OBJ_DIR:-$HERE/../build}"
LOG="$HERE/../build.log"
mkdir -p "$OBJ"
FLAGS=(-std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a
       -Xcompiler -fPIC -Xcompiler -fvisibility=hidden
       -Xptxas -v --expt-relaxed-constexpr "$@")
SRCS=(engine gemm attn accept misc attn3 gemm_big)
: > "$LOG"
pids=()
for s in "${SRCS[@]}"; do
  "$NVCC" "${FLAGS[@]}" -c -o "$OBJ/$s.o" "$HERE/$s.cu" 2> "$OBJ/$s.log" &
  pids+=($!)
done
fail=0
for i in "${!pids[@]}"; do
  if ! wait "${pids[$i]}"; then fail=1; fi
  cat "$OBJ/${SRCS[$i]}.log" >> "$LOG"
done
if [ "$fail" != 0 ]; then cat "$LOG"; exit 1; fi
objs=()
for s in "${SRCS[@]}"; do objs+=("$OBJ/$s.o"); done
"$NVCC" -gencode arch=compute_100a,code=sm_100a -shared -cudart static -Xcompiler -fPIC -o "$OUT" "${objs[@]}" 2>> "$LOG" \
  || { cat "$LOG"; exit 1; }
echo "built $OUT"
