#!/bin/bash
# quick device-resident timings: cfg2 (k=1), cfg2 k=10, cfg3 (no CPU / BF baselines)
for a in "cfg2" "cfg2 --k 10" "cfg3" ${EXTRA}; do
  python bench.py --config $a --steps 10 --warmup 3 --no-cpu-baseline --no-bf 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline'];print('$a', round(d['value']/1e6,2), 'Mq/s', round(d['ms_per_step'],3), 'ms', {k:round(v,3) for k,v in r['phase_ms_per_step'].items() if v}, 'frac', round(r['frac'],3))"
done
