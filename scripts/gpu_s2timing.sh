#!/bin/bash
# stage-2 role wait cycles (timing builds in scratch_t/) on cfg2
export RBC_INDEX_CACHE=/tmp/rbc_cfg2.rbci; rm -f $RBC_INDEX_CACHE
python scripts/kernel_timeline.py 2>&1 | grep "stage2_tc" | head -1
for t in timing tnoepi; do
  echo "== $t"; RBC_DEBUG_S2=1 RBC_B200_LIB=$PWD/scratch_t/librbc_b200_$t.so python scripts/kernel_timeline.py 2>&1 | grep "\[s2\]\|stage2_tc" | grep -v "lists#=0" | tail -3
done
