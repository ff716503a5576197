"""GPU parity for k beyond the register top-k widths (the reference accepts any
k <= |R| for exact search, search.py:167-170, and any k <= s for one-shot,
search.py:104-105): k in {17, 64} run the 64-wide warp top-k, k > 64 the
materialise-and-sort path (csrc/exact_kernels.cu topk_large)."""

import numpy as np
import pytest

from rbc_testutil import uniform

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rbc():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1103_2635_b200 as m

    return m


def _eq(got, want):
    for g, w in zip(got, want):
        assert np.array_equal(np.asarray(g).astype(np.asarray(w).dtype), w)


@pytest.mark.parametrize("kind", ["l2", "l1"])
@pytest.mark.parametrize("k", [17, 64, 100, 300])
def test_exact_large_k_vs_oracle(rbc, oracle, kind, k):
    full = oracle.gen_clusters(20_000 + 150, 12, 31, n_clusters=6, cluster_sigma=0.05)
    x, q = full[:20_000], full[20_000:]
    idx = rbc.build_exact(rbc.DataMatrix(x), 400, rbc.MetricSpec(kind, 12), seed=2)
    got = rbc.exact_query_arrays(idx, q, k)
    li, off, ld = idx.flat_lists()
    _eq(got, oracle.exact_query(x, idx.reps.rep_ids, li, off, ld, idx.radii, q, k, kind))


@pytest.mark.parametrize("k", [17, 64, 65, 150])
def test_one_shot_large_k_vs_oracle(rbc, oracle, k):
    full = oracle.gen_clusters(15_000 + 120, 10, 8, n_clusters=5, cluster_sigma=0.05)
    x, q = full[:15_000], full[15_000:]
    idx = rbc.build_one_shot(rbc.DataMatrix(x), 120, 150, rbc.MetricSpec("l2", 10), seed=1, mode="fixed-count")
    _eq(rbc.one_shot_query_arrays(idx, q, k), oracle.one_shot_query(x, idx.reps.rep_ids, idx.list_ids, q, k))


def test_bf_subset_large_k(rbc, oracle):
    u = rbc.DataMatrix(uniform(3000, 6, 44))
    sub = np.arange(0, 3000, 3)
    for k in (65, 200):
        res = rbc.bf_search_subset(u.values[7], u, sub, rbc.MetricSpec("l2", 6), k=k)
        oi, od = oracle.bf_topk(u.values[7][None, :], u.values[sub], k)
        assert np.array_equal(res.neighbors[0].ids, sub[oi[0]]) and np.array_equal(res.neighbors[0].dists, od[0])


def test_exact_k_equals_n_reps(rbc, oracle):
    x = uniform(3000, 5, 3)
    idx = rbc.build_exact(rbc.DataMatrix(x), 90, rbc.MetricSpec("l2", 5), seed=0)
    k = idx.reps.size
    q = uniform(20, 5, 4)
    li, off, ld = idx.flat_lists()
    _eq(rbc.exact_query_arrays(idx, q, k), oracle.exact_query(x, idx.reps.rep_ids, li, off, ld, idx.radii, q, k))
