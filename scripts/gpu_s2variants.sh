#!/bin/bash
# stage-2 kernel time (cfg2) of the default library and of diagnostic variants in scratch_so/
export RBC_INDEX_CACHE=/tmp/rbc_cfg2.rbci; rm -f $RBC_INDEX_CACHE
echo "base: $(python scripts/kernel_timeline.py 2>&1 | grep stage2_tc | head -1 | awk '{print $4}')"
for f in scratch_so/librbc_b200_*.so; do
  t=$(basename $f .so); echo "${t#librbc_b200_}: $(RBC_B200_LIB=$PWD/$f python scripts/kernel_timeline.py 2>&1 | grep stage2_tc | head -1 | awk '{print $4}')"
done
