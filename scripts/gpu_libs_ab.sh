#!/bin/bash
# A/B of library variants (scratch_so/*.so vs the in-tree build): tensor-core parity tests and
# quick device-resident bench lines for each library
mkdir -p gpurun_out/ab
for lib in paper_1103_2635_b200/librbc_b200.so scratch_so/*.so; do
  echo "== $lib"
  RBC_B200_LIB=$PWD/$lib timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc_bf.py -m gpu -x -q 2>&1 | tail -1
  RBC_B200_LIB=$PWD/$lib EXTRA="$EXTRA" bash scripts/quick_bench.sh 2>&1
done | tee gpurun_out/ab/bench.txt
