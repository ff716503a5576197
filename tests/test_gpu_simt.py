"""GPU parity of the fp32 SIMT filter engine with exact fp64 re-rank (csrc/simt_scan.cu).

The L1 paths (north star: "L1 is an all-SIMT path") -- bf_search, the one-shot search's
nearest representative and list scan (search.py:90-141), the exact build's assignment
(rbc.py:164) and the one-shot build's s-lists (rbc.py:196-200) -- and the small L2 scans
run the fp32 filter; every answer must equal the pinned oracle bit for bit, and the
engine must actually have run (rbc_simt_scan_calls).
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

    # engine 3: the SIMT filter for every brute-force-shaped scan, at any size (auto mode keeps
    # small scans on the exact kernels and L2 on the tensor cores)
    _lib.lib.rbc_set_engine(3)
    yield m
    _lib.lib.rbc_set_engine(0)


def _calls():
    from paper_1103_2635_b200 import _lib

    return _lib.lib.rbc_simt_scan_calls()


@pytest.mark.parametrize("metric", ["l1", "l2"])
@pytest.mark.parametrize("d", [1, 3, 21, 32, 33, 64, 100, 128])
@pytest.mark.parametrize("k", [1, 3, 16, 32])
def test_simt_bf_vs_oracle(rbc, oracle, metric, d, k):
    x = oracle.gen_clusters(3000, d, 7 + d, n_clusters=6, cluster_sigma=0.08)
    q = np.concatenate([uniform(70, d, 3 * d), x[::150] + np.float32(0.001)]).astype(np.float32)
    c0 = _calls()
    ids, dists = rbc.brute_force.bf_search_arrays(q, x, rbc.MetricSpec(metric, d), k)
    assert _calls() > c0, "the SIMT filter did not run"
    oi, od = oracle.bf_topk(q, x, k, metric)
    assert np.array_equal(ids, oi) and np.array_equal(dists, od)


@pytest.mark.parametrize("metric", ["l1", "l2"])
def test_simt_bf_point_splits_and_slices(rbc, oracle, metric):
    # few queries over many points: point splits merged by merge_parts, and thread slices
    # (R > 1) merged inside the CTA
    d = 21
    x = oracle.gen_clusters(120_000, d, 5, n_clusters=8, cluster_sigma=0.05)
    for nq in (1, 3, 37, 300):
        q = uniform(nq, d, 100 + nq)
        for k in (1, 5):
            c0 = _calls()
            ids, dists = rbc.brute_force.bf_search_arrays(q, x, rbc.MetricSpec(metric, d), k)
            assert _calls() > c0
            oi, od = oracle.bf_topk(q, x, k, metric)
            assert np.array_equal(ids, oi) and np.array_equal(dists, od)


@pytest.mark.parametrize("metric", ["l1", "l2"])
def test_simt_ties_duplicates_and_zero_distances(rbc, oracle, metric):
    base = uniform(40, 6, 3)
    x = np.repeat(base, 30, axis=0)  # every distance appears 30 times: ties broken by lowest id
    q = np.concatenate([base[:15], uniform(20, 6, 4)]).astype(np.float32)
    for k in (1, 7, 32):
        ids, dists = rbc.brute_force.bf_search_arrays(q, x, rbc.MetricSpec(metric, 6), k)
        oi, od = oracle.bf_topk(q, x, k, metric)
        assert np.array_equal(ids, oi) and np.array_equal(dists, od)
    # integer lattice: many exactly equal L1 distances
    lat = np.stack(np.meshgrid(*[np.arange(20, dtype=np.float32)] * 3, indexing="ij"), -1).reshape(-1, 3)
    ql = np.round(uniform(50, 3, 9) * 19).astype(np.float32) + np.float32(0.5)
    ids, dists = rbc.brute_force.bf_search_arrays(ql, lat, rbc.MetricSpec(metric, 3), 12)
    oi, od = oracle.bf_topk(ql, lat, 12, metric)
    assert np.array_equal(ids, oi) and np.array_equal(dists, od)


def test_simt_tiny_and_huge_magnitudes(rbc, oracle):
    # distances near the fp32 underflow and large coordinates: the filter's absolute slack
    # and relative bound must keep every possible winner
    rng = np.random.default_rng(3)
    x = (rng.standard_normal((4000, 8)) * 1e-20).astype(np.float32)
    q = (rng.standard_normal((50, 8)) * 1e-20).astype(np.float32)
    for metric in ("l1", "l2"):
        ids, dists = rbc.brute_force.bf_search_arrays(q, x, rbc.MetricSpec(metric, 8), 4)
        oi, od = oracle.bf_topk(q, x, 4, metric)
        assert np.array_equal(ids, oi) and np.array_equal(dists, od)
    xb = (rng.standard_normal((4000, 8)) * 1e15).astype(np.float32)
    qb = (rng.standard_normal((50, 8)) * 1e15).astype(np.float32)
    for metric in ("l1", "l2"):
        ids, dists = rbc.brute_force.bf_search_arrays(qb, xb, rbc.MetricSpec(metric, 8), 4)
        oi, od = oracle.bf_topk(qb, xb, 4, metric)
        assert np.array_equal(ids, oi) and np.array_equal(dists, od)


@pytest.mark.parametrize("d", [2, 21, 40, 128])
@pytest.mark.parametrize("k", [1, 4, 17])
def test_simt_one_shot_l1_vs_oracle(rbc, oracle, d, k):
    x = oracle.gen_clusters(20_000, d, 30 + d, n_clusters=8, cluster_sigma=0.05)
    q = oracle.gen_clusters(3_000, d, 31 + d, n_clusters=8, cluster_sigma=0.05)
    s = 150
    idx = rbc.build_one_shot(rbc.DataMatrix(x), 141, s, rbc.MetricSpec("l1", d), seed=4)
    lists, radii = oracle.build_one_shot(x, idx.reps.rep_ids, s, "l1")
    assert np.array_equal(np.asarray(idx.list_ids), lists) and np.array_equal(idx.radii, radii)
    c0 = _calls()
    got = rbc.one_shot_query_arrays(idx, q, k)
    assert _calls() > c0, "the SIMT filter did not run"
    want = oracle.one_shot_query(x, idx.reps.rep_ids, lists, q, k, "l1")
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


def test_simt_one_shot_skewed_groups(rbc, oracle):
    # most queries share one representative (items of 256 queries plus a ragged tail), a few
    # representatives get one query each (thread slices)
    d = 21
    x = oracle.gen_clusters(30_000, d, 77, n_clusters=4, cluster_sigma=0.05)
    q = np.concatenate([np.repeat(x[:1], 1500, axis=0) + uniform(1500, d, 9) * np.float32(1e-3),
                        uniform(200, d, 10)]).astype(np.float32)
    idx = rbc.build_one_shot(rbc.DataMatrix(x), 100, 64, rbc.MetricSpec("l1", d), seed=1)
    lists, _ = oracle.build_one_shot(x, idx.reps.rep_ids, 64, "l1")
    for k in (1, 8):
        got = rbc.one_shot_query_arrays(idx, q, k)
        want = oracle.one_shot_query(x, idx.reps.rep_ids, lists, q, k, "l1")
        for g, w in zip(got, want):
            assert np.array_equal(g, w)


def test_simt_exact_build_assignment_l1(rbc, oracle):
    d = 21
    x = oracle.gen_clusters(50_000, d, 12, n_clusters=8, cluster_sigma=0.05)
    c0 = _calls()
    idx = rbc.build_exact(rbc.DataMatrix(x), 220, rbc.MetricSpec("l1", d), seed=3)
    assert _calls() > c0
    list_ids, offsets, list_dists, radii = oracle.build_exact(x, idx.reps.rep_ids, "l1")
    assert np.array_equal(np.concatenate(idx.list_ids), list_ids)
    assert np.array_equal(np.concatenate(idx.list_dists), list_dists)
    assert np.array_equal(idx.radii, radii)


def _select_calls():
    from paper_1103_2635_b200 import _lib

    return _lib.lib.rbc_select_calls(), _lib.lib.rbc_select_fallbacks()


@pytest.mark.parametrize("metric", ["l1", "l2"])
@pytest.mark.parametrize("s", [33, 150, 600])
def test_select_one_shot_build_vs_oracle(rbc, oracle, metric, s):
    # the one-shot build's s-lists for s > 32 go through the sampled-threshold selection
    d = 21 if metric == "l1" else 16
    x = oracle.gen_clusters(40_000, d, 50 + s, n_clusters=8, cluster_sigma=0.05)
    c0, _ = _select_calls()
    idx = rbc.build_one_shot(rbc.DataMatrix(x), 120, s, rbc.MetricSpec(metric, d), seed=2)
    assert _select_calls()[0] > c0, "the large-k selection did not run"
    lists, radii = oracle.build_one_shot(x, idx.reps.rep_ids, s, metric)
    assert np.array_equal(np.asarray(idx.list_ids), lists) and np.array_equal(idx.radii, radii)


@pytest.mark.parametrize("metric", ["l1", "l2"])
@pytest.mark.parametrize("k", [40, 100, 512])
def test_select_bf_large_k_vs_oracle(rbc, oracle, metric, k):
    d = 12
    x = oracle.gen_clusters(30_000, d, 9, n_clusters=5, cluster_sigma=0.06)
    x = np.concatenate([x, x[:500]])  # exact duplicates: ties broken by the lowest id
    q = np.concatenate([uniform(40, d, 11), x[::997] + np.float32(0.002)]).astype(np.float32)
    ids, dists = rbc.brute_force.bf_search_arrays(q, x, rbc.MetricSpec(metric, d), k)
    oi, od = oracle.bf_topk(q, x, k, metric)
    assert np.array_equal(ids, oi) and np.array_equal(dists, od)


def test_select_unrepresentative_sample_falls_back(rbc, oracle):
    # every sampled row (ids divisible by the stride) is far away and the rest sits next to
    # the queries: the sampled threshold is far too loose, the collection overflows and the
    # exact full sort takes over -- the keys must still be the reference's
    k, d = 160, 4
    stride = k // 8
    rng = np.random.default_rng(5)
    x = (rng.standard_normal((20_000, d)) * 0.01).astype(np.float32)
    x[::stride] += np.float32(50.0)
    q = (rng.standard_normal((6, d)) * 0.01).astype(np.float32)
    _, f0 = _select_calls()
    for metric in ("l1", "l2"):
        ids, dists = rbc.brute_force.bf_search_arrays(q, x, rbc.MetricSpec(metric, d), k)
        oi, od = oracle.bf_topk(q, x, k, metric)
        assert np.array_equal(ids, oi) and np.array_equal(dists, od)
    assert _select_calls()[1] > f0, "expected the exact fallback"


@pytest.mark.parametrize("metric", ["l1", "l2"])
@pytest.mark.parametrize("k", [1, 3])
def test_simt_one_shot_large_groups(rbc, oracle, metric, k):
    # about 100 queries per representative: three (d <= 24, k <= 4) or two queries per lane,
    # groups of more than one chunk
    d = 21
    x = oracle.gen_clusters(20_000, d, 61, n_clusters=8, cluster_sigma=0.05)
    q = oracle.gen_clusters(4_000, d, 62, n_clusters=8, cluster_sigma=0.05)
    idx = rbc.build_one_shot(rbc.DataMatrix(x), 40, 200, rbc.MetricSpec(metric, d), seed=5)
    lists, _ = oracle.build_one_shot(x, idx.reps.rep_ids, 200, metric)
    got = rbc.one_shot_query_arrays(idx, q, k)
    want = oracle.one_shot_query(x, idx.reps.rep_ids, lists, q, k, metric)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


@pytest.mark.parametrize("d", [3, 21, 64, 100])
@pytest.mark.parametrize("k", [1, 4, 10, 32])
def test_simt_exact_l1_search_vs_oracle(rbc, oracle, d, k):
    # exact L1 search: stage 2 (the surviving segments, search.py:183-186) regrouped by list on the
    # SIMT filter, per-segment rows merged per query; results and every stats field equal the oracle
    full = oracle.gen_clusters(20_000 + 1500, d, 70 + d, n_clusters=10, cluster_sigma=0.05)
    x, q = full[:20_000], full[20_000:]
    idx = rbc.build_exact(rbc.DataMatrix(x), 150, rbc.MetricSpec("l1", d), seed=6)
    li, off, ld, radii = oracle.build_exact(x, idx.reps.rep_ids, "l1")
    c0 = _calls()
    got = rbc.exact_query_arrays(idx, q, k)
    assert _calls() > c0, "the SIMT filter did not run"
    want = oracle.exact_query(x, idx.reps.rep_ids, li, off, ld, radii, q, k, "l1")
    for g, w in zip(got, want):
        assert np.array_equal(np.asarray(g).astype(np.asarray(w).dtype), w)
