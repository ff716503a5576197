#!/bin/bash
# quick stage-2 check: tensor-core parity tests (no full-size), then quick bench lines
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc_bf.py -m gpu -x -q 2>&1 | tail -2
bash scripts/quick_bench.sh
