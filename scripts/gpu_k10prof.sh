#!/bin/bash
# k > 1 front half: parity, quick bench lines, then ncu --set full of cfg3's stage 1, fix-up,
# tile fill and re-rank (second search), summaries into gpurun_out/k10/
O=gpurun_out/k10; mkdir -p $O /tmp/ncu_reps
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc_bf.py -m gpu -x -q 2>&1 | tail -1
bash scripts/quick_bench.sh 2>&1 | tee $O/bench.txt
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:'stage1_tc_kernel|stage1_fixup|tile_fill|rerank' -s 4 -c 4 -o /tmp/ncu_reps/k10 -f \
   python scripts/prof_search.py --config cfg3 --iters 2 > $O/ncu.log 2>&1
python scripts/ncu_hot.py /tmp/ncu_reps/k10.ncu-rep 40 > $O/ncu_cfg3_front_summary.txt 2>&1
tail -3 $O/ncu.log
