#!/bin/bash
# ncu --set full of the small kernels around the two tcgen05 scans (cfg2 exact search)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:'rerank_kernel|stage1_fixup_kernel|tile_fill_kernel|tile_count_kernel' -s 4 -c 4 \
   -o gpurun_out/prof_small -f python scripts/prof_search.py --iters 3 > gpurun_out/ncu_small.log 2>&1
tail -5 gpurun_out/ncu_small.log
