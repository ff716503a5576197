#!/bin/bash
# A/B of the cfg4 SIMT kernels: current library vs scratch_so/librbc_b200_v5.so (same box, same run)
for lib in "" "$PWD/scratch_so/librbc_b200_v5k.so"; do
  for rep in 1; do
    RBC_B200_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ab.csv \
      python scripts/prof_search.py --config cfg4 --iters 3 > /dev/null 2>&1
    echo "== ${lib:-current} rep $rep"; python scripts/launches.py gpurun_out/ab.csv 2>/dev/null | grep simt_tile | head -3
  done
done
