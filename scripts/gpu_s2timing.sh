#!/bin/bash
# stage-2 role wait cycles (timing builds) on cfg2, normal and pipeline-only (noepi) variants
export RBC_INDEX_CACHE=/tmp/rbc_cfg2.rbci; rm -f $RBC_INDEX_CACHE
python scripts/kernel_timeline.py 2>&1 | grep "stage2_tc\|span" | head -3
for t in timing tnoepi noepi; do
  echo "== $t"; RBC_DEBUG_S2=1 RBC_B200_LIB=$PWD/scratch_so/librbc_b200_$t.so python scripts/kernel_timeline.py 2>&1 | grep "\[s2\]\|stage2_tc" | tail -2
done
