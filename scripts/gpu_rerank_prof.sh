#!/bin/bash
# cfg3 re-rank (k = 10): full ncu capture of the second rerank launch (the first search's retry)
O=gpurun_out/rr; mkdir -p $O /tmp/ncu_reps
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k regex:'rerank_kernel<.int.10' -s 1 -c 1 -o /tmp/ncu_reps/rr -f \
   python scripts/prof_search.py --config cfg3 --iters 2 > $O/ncu.log 2>&1
python scripts/ncu_hot.py /tmp/ncu_reps/rr.ncu-rep 40 > $O/ncu_cfg3_rerank_summary.txt 2>&1
ncu -i /tmp/ncu_reps/rr.ncu-rep --page raw --csv > $O/raw.csv 2>&1
