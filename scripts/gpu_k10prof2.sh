#!/bin/bash
# cfg3: launch list of 3 searches (direct, captured, replayed) + full capture of stage 1 and the fix-up
O=gpurun_out/k10b; mkdir -p $O /tmp/ncu_reps
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_cfg3.csv \
   python scripts/prof_search.py --config cfg3 --iters 3 > $O/launches_cfg3.log 2>&1
python scripts/launches.py $O/launches_cfg3.csv 40 > $O/launches_cfg3.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:'stage1_tc_kernel|stage1_fixup' -c 2 -o /tmp/ncu_reps/k10s1 -f \
   python scripts/prof_search.py --config cfg3 --iters 1 > $O/ncu.log 2>&1
python scripts/ncu_hot.py /tmp/ncu_reps/k10s1.ncu-rep 40 > $O/ncu_cfg3_stage1_summary.txt 2>&1
