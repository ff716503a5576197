#!/bin/bash
# One gpurun call: GPU tests (or a subset via $1), bench line, launch list of one cfg2 search.
mkdir -p gpurun_out
SEL=${1:-tests}
timeout 900 python -m pytest $SEL -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'],'phases',d['roofline']['phase_ms_per_step'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 400 --csv \
   --log-file gpurun_out/launches.csv python scripts/prof_search.py --iters 4 > gpurun_out/launches.log 2>&1
python scripts/launches.py gpurun_out/launches.csv 14
