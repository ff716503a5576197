#!/bin/bash
# SIMT filter engine: parity tests, then cfg4/cfg1 quick bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_simt.py -m gpu -x -q > gpurun_out/pytest_simt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_simt.log
tail -15 gpurun_out/pytest_simt.log
timeout 900 python -m pytest tests -m gpu -x -q -k "one_shot or l1 or cfg4 or cfg1 or bf" > gpurun_out/pytest_rel.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_rel.log
tail -5 gpurun_out/pytest_rel.log
for c in cfg4 cfg1; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));r=d['roofline'];print('$c', round(d['value']/1e6,3),'Mq/s', round(d['ms_per_step'],3),'ms e2e',round(d['e2e']['value']/1e6,3), 'frac',round(r['frac'],3), r['phase_ms_per_step'], 'build', d['config']['index_build_s'], 'bf', d.get('gpu_bruteforce'))"
done
