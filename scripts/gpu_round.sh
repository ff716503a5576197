#!/bin/bash
# One gpurun call: GPU parity tests, bench line (with CPU baseline), device kernel timeline,
# ncu launch list, ncu --set full capture of the search kernels.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python scripts/kernel_timeline.py > gpurun_out/timeline.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 400 --csv \
   --log-file gpurun_out/launches.csv python scripts/prof_search.py --iters 4 > gpurun_out/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:'stage[12]_tc_kernel|stage1_fixup|rerank|tile_fill|pilot_key' -s 7 -c 6 \
   -o gpurun_out/prof_round -f python scripts/prof_search.py --iters 3 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
