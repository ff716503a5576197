"""Summarise an ncu --set full report: per kernel, the headline metrics and stall reasons, then the
hottest source lines by stall samples (cuda,sass view; all profiled kernels aggregated).

    python scripts/ncu_hot.py gpurun_out/prof.ncu-rep [n_lines]
"""
import csv
import subprocess
import sys


def run(args):
    return subprocess.run(["ncu", "-i", sys.argv[1]] + args, capture_output=True, text=True).stdout


WANT = [
    "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed.sum.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
]

raw = list(csv.reader(run(["--page", "raw", "--csv"]).splitlines()))
h, u = raw[0], raw[1]
ki = h.index("Kernel Name")
seen = set()
for v in raw[2:]:
    name = v[ki].split("(")[0]
    if name in seen:
        continue
    seen.add(name)
    print(f"== {name}")
    for w in WANT:
        if w in h:
            i = h.index(w)
            print(f"   {w} = {v[i]} {u[i]}")
    stalls = []
    for i, col in enumerate(h):
        if "average_warps_issue_stalled" in col and col.endswith("per_issue_active.ratio"):
            try:
                stalls.append((float(v[i]), col.split("stalled_")[1].split("_per")[0]))
            except ValueError:
                pass
    print("   stalls per issue: " + ", ".join(f"{n} {s:.2f}" for s, n in sorted(stalls, reverse=True) if s > 0.1))

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
print(f"== top {n} source lines by stall samples (all kernels)")
for a in sorted(agg, key=lambda a: -a[0])[:n]:
    print(f"{a[0]:7d} {100 * a[0] / tot:5.1f}% {a[1]}:{a[2]:>4} ex={a[4]:>9} {a[3]}")
