"""Generate golden vectors from the REFERENCE implementation (rbcover 0.1.0).

Run in the build container only (the reference is not present on GPU boxes):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports the reference from /root/reference/pkg/src, runs its public API on
seeded inputs (the reference tests' own known-answer cases plus random shapes)
and writes tests/golden/golden.npz.  Inputs are NOT stored when they can be
regenerated from a seed (the generator itself is pinned by the ``gen_*`` cases).
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import rbcover as R  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
G: dict[str, np.ndarray] = {}


def put(name, arr):
    G[name] = np.asarray(arr)


def uniform(n, d, seed, scale=1.0, shift=0.0):
    return (np.random.default_rng(seed).random((n, d), dtype=np.float32) * np.float32(scale) + np.float32(shift))


def flat_lists(idx):
    lengths = np.array([len(a) for a in idx.list_ids], np.int64)
    offsets = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    return np.concatenate(idx.list_ids).astype(np.int64), offsets, np.concatenate(idx.list_dists).astype(np.float32)


def main():
    # --- generators (dataset.py:111-151), pinned so inputs can be regenerated
    put("gen_clusters_100_5_3", R.gen_synthetic("clusters", 100, 5, 3, n_clusters=4, cluster_sigma=0.05).values)
    put("gen_uniform_50_3_9", R.gen_synthetic("uniform", 50, 3, 9).values)

    # --- metric (metric.py:36-76)
    for d in (1, 2, 6, 8, 16, 21, 54, 64, 128):
        a = uniform(16, d, 1000 + d, 4.0, -2.0)
        b = uniform(24, d, 2000 + d, 4.0, -2.0)
        for kind in ("l2", "l1"):
            put(f"pair_{kind}_{d}", R.pairwise_distances(a, b, R.MetricSpec(kind, d)))

    # --- brute force (brute_force.py:165-217)
    x = uniform(2000, 8, 101)
    q = uniform(40, 8, 29)
    for kind in ("l2", "l1"):
        for k in (1, 4, 10):
            res = R.bf_search(q, x, R.MetricSpec(kind, 8), k=k)
            put(f"bf_{kind}_k{k}_ids", np.stack([nl.ids for nl in res.neighbors]))
            put(f"bf_{kind}_k{k}_dists", np.stack([nl.dists for nl in res.neighbors]))
    # ties: a lattice with many equal distances
    lat = np.stack(np.meshgrid(*[np.arange(6, dtype=np.float32)] * 3, indexing="ij"), -1).reshape(-1, 3)
    ql = np.array([[2.5, 2.5, 2.5], [0, 0, 0], [5, 5, 5], [1.5, 2.0, 3.5]], np.float32)
    for kind in ("l2", "l1"):
        res = R.bf_search(ql, lat, R.MetricSpec(kind, 3), k=12)
        put(f"bftie_{kind}_ids", np.stack([nl.ids for nl in res.neighbors]))
        put(f"bftie_{kind}_dists", np.stack([nl.dists for nl in res.neighbors]))

    # --- sampling (rbc.py:57-84)
    for n, nr, seed in ((10, 3, 0), (1000, 40, 5), (100_000, 1000, 0), (1_000_000, 1000, 0), (581_012, 763, 0),
                        (2_000_000, 1415, 0)):
        put(f"bern_{n}_{nr}_{seed}", R.sample_representatives(n, nr, seed, R.BERNOULLI).rep_ids)
    put("fixed_1000_50_2", R.sample_representatives(1000, 50, 2, R.FIXED_COUNT).rep_ids)

    # --- build_exact (rbc.py:147-180) and exact search (search.py:150-208)
    cases = [
        ("u8s0", uniform(2000, 8, 101), 50, "l2", 0),
        ("u8s1l1", uniform(2000, 8, 101), 45, "l1", 1),
        ("u6s0", uniform(1500, 6, 100), 40, "l2", 0),
        ("u6s1l1", uniform(1500, 6, 101), 40, "l1", 1),
        ("cl8", R.gen_synthetic("clusters", 2500, 8, 13, n_clusters=6, cluster_sigma=0.02).values, 50, "l2", 15),
    ]
    for name, data, nr, kind, seed in cases:
        spec = R.MetricSpec(kind, data.shape[1])
        idx = R.build_exact(R.DataMatrix(data), nr, spec, seed=seed)
        li, off, ld = flat_lists(idx)
        put(f"bx_{name}_reps", idx.reps.rep_ids)
        put(f"bx_{name}_ids", li)
        put(f"bx_{name}_off", off)
        put(f"bx_{name}_dists", ld)
        put(f"bx_{name}_radii", idx.radii)
        queries = uniform(120, data.shape[1], 7 + seed) if name != "cl8" else (
            data[np.random.default_rng(14).integers(len(data), size=100)]
            + np.random.default_rng(15).normal(0, 0.02, (100, data.shape[1])).astype(np.float32))
        put(f"bx_{name}_queries", queries)
        for k in (1, 3, 7):
            res, stats = R.exact_query_batch(idx, queries, k)
            put(f"xq_{name}_k{k}_ids", np.stack([nl.ids for nl in res]))
            put(f"xq_{name}_k{k}_dists", np.stack([nl.dists for nl in res]))
            put(f"xq_{name}_k{k}_gamma", np.array([s.gamma for s in stats], np.float32))
            put(f"xq_{name}_k{k}_prr", np.array([s.reps_pruned_radius for s in stats], np.int64))
            put(f"xq_{name}_k{k}_p3", np.array([s.reps_pruned_3gamma for s in stats], np.int64))
            put(f"xq_{name}_k{k}_cand", np.array([s.candidates_examined for s in stats], np.int64))

    # line KAT (rbc tests: reps {1,3})
    line = np.array([[0.0], [2.0], [5.0], [6.0], [9.0]], np.float32)
    idx = R.build_exact(R.DataMatrix(line), 2, R.MetricSpec("l2", 1), seed=0, rep_ids=[1, 3])
    li, off, ld = flat_lists(idx)
    put("line_ids", li)
    put("line_off", off)
    put("line_dists", ld)
    put("line_radii", idx.radii)

    # --- cfg-shaped clustered case (d=64), held-out queries from the same draw
    full = R.gen_synthetic("clusters", 20_000 + 200, 64, 1, n_clusters=16, cluster_sigma=0.05).values
    data, queries = np.ascontiguousarray(full[:20_000]), np.ascontiguousarray(full[20_000:])
    spec = R.MetricSpec("l2", 64)
    idx = R.build_exact(R.DataMatrix(data), 141, spec, seed=0)
    li, off, ld = flat_lists(idx)
    put("c64_reps", idx.reps.rep_ids)
    put("c64_ids", li)
    put("c64_off", off)
    put("c64_dists", ld)
    put("c64_radii", idx.radii)
    for k in (1, 10):
        res, stats = R.exact_query_batch(idx, queries, k)
        put(f"c64_k{k}_ids", np.stack([nl.ids for nl in res]))
        put(f"c64_k{k}_dists", np.stack([nl.dists for nl in res]))
        put(f"c64_k{k}_cand", np.array([s.candidates_examined for s in stats], np.int64))
        put(f"c64_k{k}_gamma", np.array([s.gamma for s in stats], np.float32))

    # --- build_one_shot (rbc.py:183-200) and one-shot search (search.py:90-141)
    for name, data, nr, s, kind, seed in (("u8", uniform(2000, 8, 101), 25, 10, "l2", 1),
                                          ("u8l1", uniform(2000, 8, 101), 30, 17, "l1", 4),
                                          ("u4", uniform(4000, 4, 42), 120, 120, "l2", 5)):
        spec = R.MetricSpec(kind, data.shape[1])
        idx = R.build_one_shot(R.DataMatrix(data), nr, s, spec, seed=seed)
        put(f"os_{name}_reps", idx.reps.rep_ids)
        put(f"os_{name}_lists", idx.list_ids)
        put(f"os_{name}_radii", idx.radii)
        queries = uniform(80, data.shape[1], 77)
        put(f"os_{name}_queries", queries)
        for k in (1, 3):
            res, stats = R.one_shot_query_batch(idx, queries, k)
            put(f"oq_{name}_k{k}_ids", np.stack([nl.ids for nl in res]))
            put(f"oq_{name}_k{k}_dists", np.stack([nl.dists for nl in res]))
            put(f"oq_{name}_k{k}_gamma", np.array([st.gamma for st in stats], np.float32))

    # --- range query (search.py:217-238)
    data = uniform(2000, 8, 101)
    idx = R.build_exact(R.DataMatrix(data), 40, R.MetricSpec("l2", 8), seed=11)
    li, off, ld = flat_lists(idx)
    put("rq_reps", idx.reps.rep_ids)
    rng = np.random.default_rng(4)
    for i in range(6):
        q = rng.random(8).astype(np.float32)
        radius = float(rng.random() * 0.6)
        ids, dists = R.range_query(idx, q, radius)
        put(f"rq_{i}_q", q)
        put(f"rq_{i}_radius", np.float64(radius))
        put(f"rq_{i}_ids", ids)
        put(f"rq_{i}_dists", dists)

    np.savez_compressed(OUT, **G)
    print(f"wrote {OUT}: {len(G)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
