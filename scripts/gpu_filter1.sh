#!/bin/bash
# filtered stage 1 (filter_stage1.cu): parity tests, the sharded d=128 tests, then the cfg5 bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_filter_stage1.py -m gpu -x -q > gpurun_out/pytest_f1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f1.log
tail -15 gpurun_out/pytest_f1.log
timeout 900 python -m pytest tests -m gpu -x -q -k "shard or l1 or exact or d128 or large_k" > gpurun_out/pytest_f1rel.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_f1rel.log
tail -5 gpurun_out/pytest_f1rel.log
timeout 900 python bench.py --config cfg5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
python -c "import json;d=json.load(open('gpurun_out/bench_cfg5.json'));r=d['roofline'];print('cfg5', round(d['value']/1e6,3),'Mq/s', round(d['ms_per_step'],3),'ms e2e',round(d['e2e']['value']/1e6,3), 'frac',round(r['frac'],3), r['phase_ms_per_step'])"
timeout 800 ncu --set full --clock-control none --import-source on -k regex:'s1_filter|s1_count|s1_fill' -c 3 -o gpurun_out/ncu_f1 -f python scripts/prof_search.py --config cfg5 --iters 1 > gpurun_out/ncu_f1.log 2>&1
python scripts/ncu_hot.py gpurun_out/ncu_f1.ncu-rep 25 > gpurun_out/ncu_f1_summary.txt 2>&1; head -60 gpurun_out/ncu_f1_summary.txt
