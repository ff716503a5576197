"""Generate on-disk format fixtures (RBCM, CSV, RBCI) with the REFERENCE implementation (rbcover 0.1.0).

Run in the build container only (the reference is not present on GPU boxes):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_files.py

Writes small files under tests/golden/files/: the reference's own ``save_matrix`` (binary and CSV) of a seeded
clusters draw, and ``save_index`` of an exact (L2, bernoulli) and a one-shot (L1, fixed-count) index built by the
reference on that matrix.  tests/test_index_files.py checks that this package reads them and writes them back
byte for byte, and (on a GPU) that its own builds serialise to the same bytes.
"""

from __future__ import annotations

import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
import rbcover as R  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "files")

# (name, generator args) -- kept in sync with tests/test_index_files.py
MATRIX = dict(kind="clusters", n=400, d=6, seed=5, n_clusters=4, cluster_sigma=0.05)
EXACT = dict(n_r=20, seed=0, mode="bernoulli", metric="l2")
ONE_SHOT = dict(n_r=15, s=15, seed=3, mode="fixed-count", metric="l1")


def main():
    os.makedirs(OUT, exist_ok=True)
    m = MATRIX
    data = R.gen_synthetic(m["kind"], m["n"], m["d"], m["seed"], n_clusters=m["n_clusters"],
                           cluster_sigma=m["cluster_sigma"])
    R.save_matrix(data, os.path.join(OUT, "clusters.rbcm"))
    R.save_matrix(data, os.path.join(OUT, "clusters.csv"), fmt="csv")
    ex = R.build_exact(data, EXACT["n_r"], R.MetricSpec(EXACT["metric"], data.d), EXACT["seed"], mode=EXACT["mode"])
    R.save_index(ex, os.path.join(OUT, "exact_l2.rbci"))
    os_ = R.build_one_shot(data, ONE_SHOT["n_r"], ONE_SHOT["s"], R.MetricSpec(ONE_SHOT["metric"], data.d),
                           ONE_SHOT["seed"], mode=ONE_SHOT["mode"])
    R.save_index(os_, os.path.join(OUT, "one_shot_l1.rbci"))
    R.save_matrix(R.random_project(data, 3, 8), os.path.join(OUT, "random_project_3_8.rbcm"))
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
