#!/bin/bash
# ncu --set full of the exact-search stage-2 kernel of config $1 (k $2): report gpurun_out/$3.ncu-rep
# (launch 0 of stage2_tc_kernel is the build's assignment brute force, launch 1 the first search)
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:stage2_tc_kernel -s ${4:-2} -c 1 \
   -o gpurun_out/$3 -f python scripts/prof_search.py --config $1 --k $2 --iters 2 > gpurun_out/$3.log 2>&1
tail -3 gpurun_out/$3.log
python scripts/ncu_hot.py gpurun_out/$3.ncu-rep 25 > gpurun_out/$3_summary.txt 2>&1
head -40 gpurun_out/$3_summary.txt
