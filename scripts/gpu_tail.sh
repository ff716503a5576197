#!/bin/bash
# stage-2 load balance: active cycles of the busiest / average SM per launch (cfg3 k=10, cfg2 k=10, cfg2 k=1)
mkdir -p gpurun_out
for a in "cfg3 10" "cfg2 10" "cfg2 1"; do
  set -- $a
  timeout 600 ncu --metrics sm__cycles_active.avg,sm__cycles_active.max,gpu__time_duration.sum --clock-control none \
     -k regex:stage2_tc_kernel -c 6 --csv python scripts/prof_search.py --config $1 --k $2 --iters 3 2>/dev/null \
     | grep -v "^==" | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ii=h.index('ID')
by={}
for r in rows[1:]: by.setdefault(r[ii],{})[r[mi]]=r[vi]
for i,m in by.items():
    a=float(m['sm__cycles_active.avg'].replace(',','')); x=float(m['sm__cycles_active.max'].replace(',',''))
    print('$1 k=$2 launch',i,'us',m['gpu__time_duration.sum'],'max/avg',round(x/a,3))
"
done
