#!/usr/bin/env bash
# Builds paper_2601_22813_b200/libquartet2.so for sm_100a (cross-compiles without a GPU).
set -euo pipefail
cd "$(dirname "$0")"
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
OUT=paper_2601_22813_b200/libquartet2.so
SRC="paper_2601_22813_b200/csrc/quant_fwd.cu paper_2601_22813_b200/csrc/msed.cu paper_2601_22813_b200/csrc/gemm.cu paper_2601_22813_b200/csrc/helpers.cu paper_2601_22813_b200/csrc/sr.cu"
mkdir -p build
objs=""
for f in $SRC; do
  o=build/$(basename "${f%.cu}").o
  stale=0
  [ -f "$o" ] || stale=1
  for dep in "$f" paper_2601_22813_b200/csrc/*.cuh include/quartet2.h; do
    [ "$dep" -nt "$o" ] && stale=1
  done
  if [ "$stale" = 1 ]; then
    "$NVCC" -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 -Xcompiler -fPIC \
      -Xptxas -v -diag-suppress 128 ${Q2_NVCC_FLAGS:-} -c "$f" -o "$o" 2> "build/$(basename "${f%.cu}").ptxas.log" || { cat "build/$(basename "${f%.cu}").ptxas.log"; exit 1; }
  fi
  objs="$objs $o"
done
"$NVCC" -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC $objs -o "$OUT"
echo "built $OUT"
