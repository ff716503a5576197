#!/bin/bash
# ncu --set full of the SIMT filter scans of a one-shot search (config $1, report prefix $2):
# launch 0 = nearest representative (dense), launch 1 = the list scan (grouped)
mkdir -p gpurun_out
for l in 0 1; do
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:simt_ -s $l -c 1 \
   -o gpurun_out/$2_l$l -f python scripts/prof_search.py --config $1 --iters 1 > gpurun_out/$2_l$l.log 2>&1
python scripts/ncu_hot.py gpurun_out/$2_l$l.ncu-rep 30 > gpurun_out/$2_l${l}_summary.txt 2>&1
head -45 gpurun_out/$2_l${l}_summary.txt
done
