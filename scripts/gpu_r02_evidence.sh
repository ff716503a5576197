#!/bin/bash
# Round-2 evidence run: full GPU suite, bench lines for every config (+ reference arm), ncu launch
# lists and --set full captures of the dominant kernels.  Everything lands in gpurun_out/r02e/.
O=gpurun_out/${R02E:-r02e}; mkdir -p $O
# full ncu reports stay on the box (gpurun copies back at most 64 MiB); their summaries come back
NR=/tmp/ncu_reps; mkdir -p $NR
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_cfg2.json 2> $O/bench_cfg2.err; tail -c 300 $O/bench_cfg2.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
for c in cfg1 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --k 10 --steps 10 --warmup 3 > $O/bench_cfg2_k10.json 2> $O/bench_cfg2_k10.err
# launch lists (per-launch device time, serialised): cfg2 and cfg4 searches
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg2.csv \
   python scripts/prof_search.py --config cfg2 --iters 3 > $O/launches_cfg2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg4.csv \
   python scripts/prof_search.py --config cfg4 --iters 3 > $O/launches_cfg4.log 2>&1
# full captures: cfg2 stage 1/2 of the second search, cfg4 SIMT scans + build selection, cfg3 stage 2
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:'stage[12]_tc_kernel|stage1_fixup|rerank|tile_fill' -s 6 -c 5 -o $NR/ncu_cfg2 -f \
   python scripts/prof_search.py --config cfg2 --iters 2 > $O/ncu_cfg2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'simt_tile|collect_kernel' -c 4 \
   -o $NR/ncu_cfg4 -f python scripts/prof_search.py --config cfg4 --iters 1 > $O/ncu_cfg4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage2_tc_kernel -s 3 -c 1 \
   -o $NR/ncu_cfg3 -f python scripts/prof_search.py --config cfg3 --iters 2 > $O/ncu_cfg3.log 2>&1
timeout 800 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_cfg5.csv \
   python scripts/prof_search.py --config cfg5 --iters 2 > $O/launches_cfg5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'s1_filter|s1_count|s1_fill|stage2_tc_kernel' \
   -s 5 -c 4 -o $NR/ncu_cfg5 -f python scripts/prof_search.py --config cfg5 --iters 3 > $O/ncu_cfg5.log 2>&1
timeout 300 python scripts/kernel_timeline.py 10000 10 cfg5 > $O/timeline_cfg5.txt 2>&1
timeout 300 python scripts/kernel_timeline.py > $O/timeline_cfg2.txt 2>&1
timeout 300 python scripts/kernel_timeline.py 100000 10 cfg2 > $O/timeline_cfg2_k10.txt 2>&1
timeout 300 python scripts/kernel_timeline.py 100000 10 cfg3 > $O/timeline_cfg3.txt 2>&1
for r in ncu_cfg2 ncu_cfg4 ncu_cfg3 ncu_cfg5; do python scripts/ncu_hot.py $NR/$r.ncu-rep 25 > $O/${r}_summary.txt 2>&1; done
ls -la $O
