"""Diagnostic: exact search on huge-magnitude data (|q - x| ~ 1e18) per engine vs the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from oracle import oracle  # noqa: E402
from rbc_testutil import uniform  # noqa: E402

import paper_1103_2635_b200 as rbc  # noqa: E402
from paper_1103_2635_b200 import _lib  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 80
x = uniform(3000, d, 5, scale=4e18, shift=-2e18)
q = uniform(200, d, 6, scale=4e18, shift=-2e18)
idx = rbc.build_exact(rbc.DataMatrix(x), 300, rbc.MetricSpec("l2", d), seed=3)
li, off, ld, radii = oracle.build_exact(x, idx.reps.rep_ids, "l2")
want = oracle.exact_query(x, idx.reps.rep_ids, li, off, ld, radii, q, 2, "l2")
for eng in (0, 1, 2):
    _lib.lib.rbc_set_engine(eng)
    got = rbc.exact_query_arrays(idx, q, 2)
    bad = [n for n, g, w in zip(("ids", "dists", "gamma", "pr", "p3", "cand"), got, want)
           if not np.array_equal(np.asarray(g).astype(np.asarray(w).dtype), w)]
    print("engine", eng, "mismatch:", bad)
    if bad:
        rows = np.nonzero((got[0] != want[0]).any(1))[0][:4]
        for r in rows:
            print("  q", r, "got", got[0][r], got[1][r], "want", want[0][r], want[1][r])
_lib.lib.rbc_set_engine(0)
