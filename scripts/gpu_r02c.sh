#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc_bf.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c.log
tail -3 gpurun_out/pytest_c.log
RBC_DEBUG_CAND=1 python scripts/diag_bf.py 2>&1 | grep -v "^$" | grep "m=\|cap 96\|prepare" | head -20
timeout 600 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
python -c "import json;d=json.load(open('gpurun_out/bench_cfg3.json'));print('cfg3', d['value'], d['ms_per_step'], d['roofline']['phase_ms_per_step'])"
