#!/bin/bash
# round 2: tensor-core brute force -- parity tests, then the cfg2 bench line (includes the BF baseline)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc_bf.py tests/test_gpu_parity.py -m gpu -x -q --durations=10 > gpurun_out/pytest_tcbf.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tcbf.log
timeout 600 python bench.py --config cfg2 --steps 20 --warmup 5 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
tail -3 gpurun_out/pytest_tcbf.log
