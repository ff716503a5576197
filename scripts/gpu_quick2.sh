#!/bin/bash
# quick check of a stage-2 change: tensor-core parity tests, then device-resident bench lines
mkdir -p gpurun_out/q
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc_bf.py -m gpu -x -q > gpurun_out/q/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q/pytest.log
tail -3 gpurun_out/q/pytest.log
EXTRA="cfg5" bash scripts/quick_bench.sh 2>&1 | tee gpurun_out/q/bench.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('BF', d.get('gpu_bruteforce'))"
