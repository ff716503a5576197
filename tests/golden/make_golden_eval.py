"""Golden vectors for eval.py / report.py rank errors, written by the REFERENCE implementation (rbcover 0.1.0).

Run in the build container only (the reference is not present on GPU boxes):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_eval.py

Inputs are regenerated from seeds in tests/test_eval_gpu.py (``gen_synthetic`` is pinned bit-for-bit by
tests/test_oracle_golden.py); only the reference's outputs are stored in tests/golden/eval_golden.npz.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import rbcover as R  # noqa: E402
from rbcover import report as RR  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "eval_golden.npz")


def inputs():
    """Kept in sync with tests/test_eval_gpu.py::inputs."""
    data = R.gen_synthetic("clusters", 3000, 8, 21, n_clusters=6, cluster_sigma=0.05)
    queries = R.gen_synthetic("clusters", 3200, 8, 21, n_clusters=6, cluster_sigma=0.05).values[3000:]
    return data, np.ascontiguousarray(queries)


def main():
    data, queries = inputs()
    x = data.values
    G = {}
    for kind in ("l2", "l1"):
        spec = R.MetricSpec(kind, 8)
        radii = np.array([0.0, 0.01, 0.05, 0.1, 0.3, 1.0, 10.0])
        G[f"ball_{kind}"] = np.array([[R.ball_count(data, x[c], r, spec) for r in radii] for c in (0, 7, 1234, 2999)])
        ests = []
        for seed, ns, nr, qq in ((0, 20, 8, None), (5, 7, 200, None), (9, 12, 16, queries[:50])):
            e = R.estimate_expansion_rate(data, spec, ns, nr, seed, queries=qq)
            ests.append([e.c_max, e.c_median, e.samples, e.radii_per_sample, float(e.includes_queries)])
        G[f"expansion_{kind}"] = np.array(ests)
        G[f"rank_{kind}"] = np.array([R.rank_error(data, queries[i], rid, spec)
                                      for i, rid in ((0, 0), (1, 17), (2, 2999), (3, 1500), (4, 42))])
        G[f"claim1_box_{kind}"] = R.claim1_counts(data, 60, spec, 40, 3)
        G[f"claim1_q_{kind}"] = R.claim1_counts(data, 200, spec, 30, 4, queries=queries)
        base = RR.run_baseline(data, queries, spec, 1)
        G[f"baseline_top16_{kind}"] = base.top_dists[:16]
        G[f"baseline_sha_{kind}"] = np.array(hashlib.sha256(np.ascontiguousarray(base.top_dists).tobytes()).hexdigest())
        rng = np.random.default_rng(11)
        pick = rng.integers(3000, size=len(queries))
        ret = R.pairwise_distances(queries, x, spec)[np.arange(len(queries)), pick].astype(np.float32)
        ret[:20] = base.top_dists[:20, 0]
        G[f"rank_ret_{kind}"] = ret
        G[f"rank_errors_{kind}"] = RR.rank_errors(data, queries, ret, base, spec)
    np.savez_compressed(OUT, **G)
    print(OUT, os.path.getsize(OUT), {k: v.shape for k, v in G.items()})


if __name__ == "__main__":
    main()
