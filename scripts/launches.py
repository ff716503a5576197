"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV): mean us per launch by kernel."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, data = rows[h], rows[h + 1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = defaultdict(lambda: [0, 0.0])
for r in data:
    v = float(r[vi].replace(",", ""))
    v = {"nsecond": v / 1e3, "usecond": v, "msecond": v * 1e3, "second": v * 1e6}.get(r[ui], v)
    agg[r[ki][:80]][0] += 1
    agg[r[ki][:80]][1] += v
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{t / c:10.1f} us x{c:3d}  {k}")
