#!/bin/bash
# Build a variant of libgk.so with extra nvcc defines for fill.cu (kernel A/B
# experiments on the same box).  Usage: scripts/build_variant.sh NAME -DFOO=1 ...
# Output: scripts/_variants/libgk_NAME.so (load with GK_LIB=<path>).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
OUT=$ROOT/scripts/_variants; mkdir -p "$OUT"
B=$ROOT/paper_1901_04162_b200/_build
python -m paper_1901_04162_b200.build >/dev/null
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
  -Xcompiler -ffp-contract=off -I "$ROOT/include" "$@" \
  -c "$ROOT/paper_1901_04162_b200/csrc/fill.cu" -o "$OUT/fill_$NAME.o"
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT/libgk_$NAME.so" \
  "$B/build.cu.o" "$OUT/fill_$NAME.o" "$B/eval.cu.o" "$B/abi.cu.o" "$B/host.cpp.o" -lcudart
echo "$OUT/libgk_$NAME.so"
