#!/bin/bash
# Re-entry check: full GPU suite + quick bench of cfg1..cfg4 on the current tree.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -25 gpurun_out/pytest_gpu.log
for c in cfg1 cfg2 cfg3 cfg4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));r=d['roofline'];print('$c', round(d['value']/1e6,3),'Mq/s', round(d['ms_per_step'],3),'ms e2e',round(d['e2e']['value']/1e6,3), 'frac',round(r['frac'],3), r['phase_ms_per_step'], 'bf', d.get('gpu_bruteforce'))"
done
