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
    v = {"ns": v / 1e3, "nsecond": v / 1e3, "us": v, "usecond": v, "ms": v * 1e3, "msecond": v * 1e3,
         "s": v * 1e6, "second": v * 1e6}.get(r[ui], v)
    agg[r[ki][:80]][0] += 1
    agg[r[ki][:80]][1] += v
tot = sum(t for _, t in agg.values()) or 1.0
print(f"{'us/launch':>10} {'launches':>8} {'share':>6}  kernel")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{t / c:10.1f} {c:8d} {100 * t / tot:5.1f}%  {k}")
