#!/bin/bash
# ncu --set full of kernels matching $1 (regex) in one cfg2 exact search; report to gpurun_out/$2.ncu-rep
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${3:-2} -c ${4:-2} \
   -o gpurun_out/$2 -f python scripts/prof_search.py --iters 2 > gpurun_out/$2.log 2>&1
tail -3 gpurun_out/$2.log
