#!/bin/bash
# Debug build of the library with kernel printf in the fused stage 1 (not shipped).
set -e
cd "$(dirname "$0")/.."
OUT=/tmp/rbc_dbg; mkdir -p $OUT
for f in paper_1103_2635_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I include -DRBC_S1_DEBUG -c $f -o $OUT/$(basename $f .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/librbc_dbg.so $OUT/*.o
