"""Summarise an ncu report: headline metrics + top source lines by stall samples (cuda,sass view)."""
import csv
import subprocess
import sys


def run(args):
    return subprocess.run(["ncu", "-i", sys.argv[1]] + args, capture_output=True, text=True).stdout


raw = list(csv.reader(run(["--page", "raw", "--csv"]).splitlines()))
h, u, v = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "utchmma_src_fp16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__inst_executed.sum.per_cycle_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread"]
for i, name in enumerate(h):
    if any(name == w or name.endswith(w) for w in want):
        print(f"{name} = {v[i]} {u[i]}")
for i, name in enumerate(h):
    if "average_warps_issue_stalled" in name and name.endswith("per_issue_active.ratio"):
        try:
            if float(v[i]) > 0.2:
                print(f"{name.split('stalled_')[1].split('_per')[0]:24s} {v[i]}")
        except ValueError:
            pass
rows = list(csv.reader(run(["--page", "source", "--csv", "--print-source=cuda,sass"]).splitlines()))
cur, agg = None, []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 7 and r[0] not in ("", "Line No") and r[4].isdigit():
        agg.append((int(r[4]), cur, r[0], r[1].strip()[:95], r[7]))
tot = sum(a[0] for a in agg) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for a in sorted(agg, key=lambda a: -a[0])[:n]:
    print(f"{a[0]:7d} {100 * a[0] / tot:5.1f}% {a[1]}:{a[2]:>4} ex={a[4]:>9} {a[3]}")
