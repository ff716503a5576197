#!/bin/bash
# per-kernel device times (cfg2 k=1 and cfg3 k=10) of the current library and of the libraries in scratch_so/
export RBC_INDEX_CACHE=/tmp/rbc_cfg2.rbci; rm -f $RBC_INDEX_CACHE
echo "== current"; python scripts/kernel_timeline.py 2>&1 | grep "rerank\|stage2_tc\|span"
for f in scratch_so/librbc_b200_*.so; do
  echo "== $f"; RBC_B200_LIB=$PWD/$f python scripts/kernel_timeline.py 2>&1 | grep "rerank\|stage2_tc\|span"
done
