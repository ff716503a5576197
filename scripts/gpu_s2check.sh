#!/bin/bash
# stage-2 change check: tensor-core parity tests, full-size cfg2/cfg3 vs the oracle, quick bench lines
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc_bf.py tests/test_gpu_sharded.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/pytest_s2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_s2.log
tail -4 gpurun_out/pytest_s2.log
bash scripts/quick_bench.sh
