"""Static SASS instruction counts of the library's kernels (cuobjdump -sass): evidence that the
tensor-core paths issue tcgen05.mma (UTCHMMA), tcgen05.ld (LDTM) and bulk copies (UBLKCP), and that
the SIMT filter issues packed fp32 (FADD2/FFMA2).

    python scripts/sass_summary.py > profiles/r02_sass_summary.txt
"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_1103_2635_b200/librbc_b200.so"
WANT = ["UTCHMMA", "UTCBAR", "LDTM", "UBLKCP", "SYNCS", "FADD2", "FFMA2", "FMNMX3", "DADD", "LDGSTS", "REDUX", "USETMAXREG"]


def demangle(n):
    r = subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
    r = r.replace("(anonymous namespace)::", "").replace("rbc::", "")
    return r.split("(")[0].replace("void ", "")


out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
fn, counts = None, collections.defaultdict(collections.Counter)
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        fn = m.group(1)
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
    if fn and m:
        for w in WANT:
            if m.group(1) == w:
                counts[fn][w] += 1
print(f"# static SASS counts per kernel, {LIB} (sm_100a); UTCHMMA = tcgen05.mma, LDTM = tcgen05.ld,")
print("# UBLKCP = cp.async.bulk, FADD2/FFMA2 = packed fp32 (SIMT filter), FMNMX3 = 3-input max,")
print("# DADD = fp64 add (exact re-rank, reference arithmetic), LDGSTS = cp.async, USETMAXREG = setmaxnreg")
rows = [(demangle(f), c) for f, c in counts.items() if any(c[w] for w in ("UTCHMMA", "LDTM", "UBLKCP", "FADD2", "FFMA2"))]
for name, c in sorted(rows):
    print(f"{name:60s} " + " ".join(f"{w}={c[w]}" for w in WANT if c[w]))
