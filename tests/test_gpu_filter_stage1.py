"""GPU parity of the filtered exact-search stage 1 (csrc/filter_stage1.cu).

Indexes the tensor-core stage 1 does not cover (d > 64, and every L1 index) run stage 1 +
pruning (search.py:178-198) as an fp32 SIMT bound for every (query, rep) plus the exact fp64
distance only where gamma_k, a pruning test, a survivor or its 4 gamma cutoff needs it.  Every
output -- ids, distances, gamma_k, both pruning counts, candidates_examined -- must equal the
pinned oracle bit for bit, and the filtered engine must actually have run (or, for inputs it
cannot bound, have handed the batch back to the exact path).
"""

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
    from paper_1103_2635_b200 import _lib

    _lib.lib.rbc_set_engine(0)
    return m


def _counts():
    from paper_1103_2635_b200 import _lib

    return _lib.lib.rbc_filter_stage1_calls(), _lib.lib.rbc_filter_stage1_fallbacks()


def _check(rbc, oracle, x, q, nr, metric, k, seed=3, expect_filtered=True):
    d = x.shape[1]
    idx = rbc.build_exact(rbc.DataMatrix(x), nr, rbc.MetricSpec(metric, d), seed=seed)
    li, off, ld, radii = oracle.build_exact(x, idx.reps.rep_ids, metric)
    c0, f0 = _counts()
    got = rbc.exact_query_arrays(idx, q, k)
    c1, f1 = _counts()
    assert c1 > c0, "the filtered stage 1 did not run"
    if expect_filtered:
        assert f1 == f0, "the filtered stage 1 fell back to the exact path"
    want = oracle.exact_query(x, idx.reps.rep_ids, li, off, ld, radii, q, k, metric)
    names = ("ids", "dists", "gamma", "pruned_radius", "pruned_3gamma", "candidates")
    for name, g, w in zip(names, got, want):
        g = np.asarray(g).astype(np.asarray(w).dtype)
        assert np.array_equal(g, w), f"{name} differs in {int((g != w).sum())} entries"
    return f1 - f0


@pytest.mark.parametrize("metric", ["l2", "l1"])
@pytest.mark.parametrize("d", [65, 128, 131])
@pytest.mark.parametrize("k", [1, 4, 10, 16])
def test_filter_stage1_clusters(rbc, oracle, metric, d, k):
    full = oracle.gen_clusters(8000 + 700, d, 11 + d + k, n_clusters=8, cluster_sigma=0.05)
    _check(rbc, oracle, full[:8000], full[8000:], 90, metric, k)


@pytest.mark.parametrize("d", [3, 21, 54])
@pytest.mark.parametrize("k", [1, 10])
def test_filter_stage1_l1_low_dim(rbc, oracle, d, k):
    # exact L1 at the cfg4 / cfg3 dimensions: no tensor-core stage 1 for L1
    full = oracle.gen_clusters(12_000 + 900, d, 5 + d, n_clusters=10, cluster_sigma=0.05)
    _check(rbc, oracle, full[:12_000], full[12_000:], 110, "l1", k)


@pytest.mark.parametrize("metric", ["l2", "l1"])
def test_filter_stage1_uniform_wide(rbc, oracle, metric):
    # uniform data at d = 200: distances concentrate, so many reps sit near the 3 gamma and
    # gamma + psi boundaries and need the exact distance
    x = uniform(6000, 200, 1)
    q = uniform(500, 200, 2)
    _check(rbc, oracle, x, q, 80, metric, 5)


@pytest.mark.parametrize("metric", ["l2", "l1"])
def test_filter_stage1_ties(rbc, oracle, metric):
    # integer coordinates in {0, 1, 2}: exact ties everywhere (gamma candidates with equal
    # distances, equal rep distances at the predicate boundaries); near-tie storms may exceed
    # the candidate buffer and hand the batch back -- the results must match either way
    rng = np.random.default_rng(4)
    x = rng.integers(0, 3, size=(5000, 70)).astype(np.float32)
    q = np.concatenate([x[:100], rng.integers(0, 3, size=(300, 70)).astype(np.float32)])
    _check(rbc, oracle, x, q, 70, metric, 3, expect_filtered=False)


@pytest.mark.parametrize("d", [40, 80])
def test_huge_magnitudes(rbc, oracle, d):
    # coordinates ~1e18: beyond the tensor-core engines' fp32 range (tc_scan.cuh kTcMaxAbs), so
    # the index gets no tensor-core operands and the filter's overflowing sums are undecided
    # (exact fp64 there); results still bit-exact
    x = uniform(3000, d, 5, scale=4e18, shift=-2e18)
    q = uniform(200, d, 6, scale=4e18, shift=-2e18)
    _check(rbc, oracle, x, q, 300, "l2", 2, expect_filtered=False)


@pytest.mark.parametrize("d", [40, 80])
def test_huge_queries_only(rbc, oracle, d):
    # an ordinary index (tensor-core operands prepared) queried with a batch holding a few
    # out-of-range rows: the range checks send the batch to the SIMT / exact engines
    full = oracle.gen_clusters(6000 + 300, d, 31, n_clusters=6, cluster_sigma=0.05)
    x, q = full[:6000], full[6000:].copy()
    q[::50] *= np.float32(3e17)
    _check(rbc, oracle, x, q, 80, "l2", 3, expect_filtered=False)


def test_filter_stage1_small_rep_count(rbc, oracle):
    # |R| smaller than a warp, k = |R|
    full = oracle.gen_clusters(600 + 50, 96, 9, n_clusters=4, cluster_sigma=0.1)
    _check(rbc, oracle, full[:600], full[600:], 6, "l2", 6)


def test_filter_stage1_multi_chunk(rbc, oracle):
    # a batch over many 64-query filter tiles with a ragged last tile
    full = oracle.gen_clusters(20_000 + 4099, 72, 21, n_clusters=12, cluster_sigma=0.05)
    _check(rbc, oracle, full[:20_000], full[20_000:], 150, "l2", 7)


@pytest.mark.parametrize("huge", ["points", "queries"])
def test_huge_magnitudes_bf_and_one_shot(rbc, oracle, huge):
    # the brute-force scan (tensor-core sized: 2000 x 20000 pairs, engine 2 forces the filtered
    # engines) and the one-shot search with out-of-range points or queries: range-checked off
    # the tensor cores, bit-exact
    from paper_1103_2635_b200 import _lib

    d = 48
    x = oracle.gen_clusters(20_000, d, 41, n_clusters=6, cluster_sigma=0.05)
    q = oracle.gen_clusters(2000, d, 42, n_clusters=6, cluster_sigma=0.05)
    if huge == "points":
        x[::97] *= np.float32(5e16)
    else:
        q[::37] *= np.float32(5e16)
    _lib.lib.rbc_set_engine(2)
    try:
        spec = rbc.MetricSpec("l2", d)
        from paper_1103_2635_b200.brute_force import bf_search_arrays

        ids, dists = bf_search_arrays(q, x, spec, 4)
        wi, wd = oracle.bf_topk(q, x, 4, "l2")
        assert np.array_equal(ids, wi) and np.array_equal(dists, wd)
        idx = rbc.build_one_shot(rbc.DataMatrix(x), 140, 300, spec, seed=2)
        lists, radii = oracle.build_one_shot(x, idx.reps.rep_ids, 300, "l2")
        assert np.array_equal(np.asarray(idx.list_ids), lists) and np.array_equal(idx.radii, radii)
        got = rbc.one_shot_query_arrays(idx, q, 3)
        want = oracle.one_shot_query(x, idx.reps.rep_ids, lists, q, 3, "l2")
        for g, w in zip(got, want):
            assert np.array_equal(g, w)
    finally:
        _lib.lib.rbc_set_engine(0)
