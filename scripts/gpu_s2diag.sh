#!/bin/bash
# stage-2 diagnostics on cfg2: role wait cycles (timing build), kernel time of diagnostic variants
true || RBC_DEBUG_S2=1 RBC_B200_LIB=$PWD/scratch_so/librbc_b200_timing.so python scripts/prof_search.py --iters 2 2>&1 | grep "\[s2\]" | tail -1
mkdir -p gpurun_out
export RBC_INDEX_CACHE=/tmp/rbc_cfg2.rbci; rm -f $RBC_INDEX_CACHE
python scripts/kernel_timeline.py > gpurun_out/tl_base.txt 2>&1
for t in noepi lvl1 lvl2; do
  RBC_B200_LIB=$PWD/scratch_so/librbc_b200_$t.so python scripts/kernel_timeline.py > gpurun_out/tl_$t.txt 2>&1
done
for f in gpurun_out/tl_*.txt; do echo "$f: $(grep stage2_tc $f | head -3)"; done
