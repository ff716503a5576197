#!/bin/bash
# parity on the tensor-core paths (incl. full-size and large k), then quick device-resident bench lines
mkdir -p gpurun_out/c2
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc_bf.py tests/test_gpu_large_k.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/c2/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c2/pytest.log
tail -3 gpurun_out/c2/pytest.log
EXTRA="$EXTRA" bash scripts/quick_bench.sh 2>&1 | tee gpurun_out/c2/bench.txt
