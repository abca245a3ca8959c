#!/bin/bash
# Build a variant of libgk.so with extra nvcc defines for the fill units
# (fill.cu, fill_mo*.cu, eval.cu; kernel A/B experiments on the same box, and
# the device-assert build: scripts/build_variant.sh asserts -DGK_DEVICE_ASSERTS).
# Usage: scripts/build_variant.sh NAME -DFOO=1 ...
# Output: scripts/_variants/libgk_NAME.so (load with GK_LIB=<path>).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
OUT=${TMPDIR:-/tmp}/gk_variants/$NAME; mkdir -p "$OUT" "$ROOT/scripts/_variants"
B=$ROOT/paper_1901_04162_b200/_build
C=$ROOT/paper_1901_04162_b200/csrc
python -m paper_1901_04162_b200.build >/dev/null
OBJS=()
for f in fill fill_mo1 fill_mo3 fill_mo4 fill_mo6 fill_mo7 eval; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
    -Xcompiler -ffp-contract=off -I "$ROOT/include" "$@" -c "$C/$f.cu" -o "$OUT/$f.o" &
  OBJS+=("$OUT/$f.o")
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$ROOT/scripts/_variants/libgk_$NAME.so" \
  "$B/build.cu.o" "${OBJS[@]}" "$B/abi.cu.o" "$B/host.cpp.o" "$B/edges.cu.o" "$B/comm.cu.o" \
  -lcudart -ldl
echo "$ROOT/scripts/_variants/libgk_$NAME.so"
