"""GPU parity of the tcgen05 brute-force engine (survey kernel K1).

bf_search (brute_force.py:165-186), the exact build's nearest-representative
assignment (rbc.py:164) and the one-shot search's nearest representative
(search.py:114-115) run the tensor-core distance tile with the filter epilogue
and the exact fp64 re-rank.  Every test checks bit-exact equality with the
pinned oracle (or the exact SIMT engine at sizes the oracle is slow for) and
that the tensor-core path actually ran (rbc_tc_bf_calls).
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

    # engine 2: the tensor-core scans at every size (auto mode keeps small brute-force-shaped
    # scans on the exact SIMT kernels, where they are faster)
    _lib.lib.rbc_set_engine(2)
    yield m
    _lib.lib.rbc_set_engine(0)


def _calls():
    from paper_1103_2635_b200 import _lib

    return _lib.lib.rbc_tc_bf_calls()


def _exact_engine(rbc, fn):
    from paper_1103_2635_b200 import _lib

    _lib.lib.rbc_set_engine(1)
    try:
        return fn()
    finally:
        _lib.lib.rbc_set_engine(2)


@pytest.mark.parametrize("d", [1, 5, 16, 21, 54, 62, 63, 64])
@pytest.mark.parametrize("k", [1, 4, 10, 16, 32])
def test_tc_bf_vs_oracle(rbc, oracle, d, k):
    x = oracle.gen_clusters(6000, d, 11 + d, n_clusters=7, cluster_sigma=0.08)
    q = np.concatenate([uniform(90, d, 5 * d), x[::200] + np.float32(0.001)]).astype(np.float32)
    c0 = _calls()
    ids, dists = rbc.brute_force.bf_search_arrays(q, x, rbc.MetricSpec("l2", d), k)
    assert _calls() > c0, "the tensor-core brute force did not run"
    oi, od = oracle.bf_topk(q, x, k, "l2")
    assert np.array_equal(ids, oi) and np.array_equal(dists, od)


def test_tc_bf_ties_and_duplicates(rbc, oracle):
    # many exact duplicates (ties broken by lowest id) and a lattice with equal distances
    base = uniform(50, 8, 3)
    x = np.repeat(base, 40, axis=0)
    q = np.concatenate([base[:20], uniform(30, 8, 4)]).astype(np.float32)
    for k in (1, 7, 16):
        c0 = _calls()
        ids, dists = rbc.brute_force.bf_search_arrays(q, x, rbc.MetricSpec("l2", 8), k)
        assert _calls() > c0
        oi, od = oracle.bf_topk(q, x, k, "l2")
        assert np.array_equal(ids, oi) and np.array_equal(dists, od)
    lat = np.stack(np.meshgrid(*[np.arange(24, dtype=np.float32)] * 3, indexing="ij"), -1).reshape(-1, 3)
    ql = (uniform(40, 3, 9) * 23).astype(np.float32)
    ql[:10] = np.round(ql[:10]) + 0.5
    ids, dists = rbc.brute_force.bf_search_arrays(ql, lat, rbc.MetricSpec("l2", 3), 12)
    oi, od = oracle.bf_topk(ql, lat, 12, "l2")
    assert np.array_equal(ids, oi) and np.array_equal(dists, od)


@pytest.mark.parametrize("d", [3, 40, 64])
def test_tc_bf_scales_and_offsets(rbc, oracle, d):
    # far-off centre and mixed scales stress the centred f16 operands and the error bound
    rng = np.random.default_rng(d)
    x = (rng.standard_normal((8000, d)) * rng.choice([0.001, 1.0, 300.0], size=(8000, 1)) + 1000.0).astype(np.float32)
    q = (x[rng.integers(0, 8000, 300)] + rng.standard_normal((300, d)).astype(np.float32) * 0.01).astype(np.float32)
    for k in (1, 5):
        ids, dists = rbc.brute_force.bf_search_arrays(q, x, rbc.MetricSpec("l2", d), k)
        oi, od = oracle.bf_topk(q, x, k, "l2")
        assert np.array_equal(ids, oi) and np.array_equal(dists, od)


@pytest.mark.parametrize("k", [1, 10])
def test_tc_bf_large_matches_exact_engine(rbc, oracle, k):
    full = oracle.gen_clusters(200_000 + 4_000, 64, 1, n_clusters=64, cluster_sigma=0.05)
    x, q = full[:200_000], full[200_000:]
    spec = rbc.MetricSpec("l2", 64)
    c0 = _calls()
    fast = rbc.brute_force.bf_search_arrays(q, x, spec, k)
    assert _calls() > c0
    exact = _exact_engine(rbc, lambda: rbc.brute_force.bf_search_arrays(q, x, spec, k))
    assert np.array_equal(fast[0], exact[0]) and np.array_equal(fast[1], exact[1])
    oi, od = oracle.bf_topk(q[:256], x, k, "l2")
    assert np.array_equal(fast[0][:256], oi) and np.array_equal(fast[1][:256], od)


@pytest.mark.parametrize("d", [16, 54, 64])
def test_tc_build_assignment_vs_oracle(rbc, oracle, d):
    # the build's X x R assignment is a k = 1 brute force of every point over the reps
    x = oracle.gen_clusters(60_000, d, 3 + d, n_clusters=16, cluster_sigma=0.05)
    spec = rbc.MetricSpec("l2", d)
    c0 = _calls()
    idx = rbc.build_exact(rbc.DataMatrix(x), 245, spec, seed=4)
    assert _calls() > c0, "the build assignment did not use the tensor-core brute force"
    li, off, ld, radii = oracle.build_exact(x, idx.reps.rep_ids)
    ids, offsets, dists = idx.flat_lists()
    assert np.array_equal(ids, li) and np.array_equal(offsets, off) and np.array_equal(dists, ld)
    assert np.array_equal(idx.radii, radii)


def test_tc_one_shot_nearest_rep_vs_oracle(rbc, oracle):
    full = oracle.gen_clusters(50_000 + 3_000, 16, 7, n_clusters=8, cluster_sigma=0.05)
    x, q = full[:50_000], full[50_000:]
    spec = rbc.MetricSpec("l2", 16)
    idx = rbc.build_one_shot(rbc.DataMatrix(x), 224, 224, spec, seed=0, mode="fixed-count")
    c0 = _calls()
    got = rbc.one_shot_query_arrays(idx, q, 1)
    assert _calls() > c0
    want = oracle.one_shot_query(x, idx.reps.rep_ids, idx.list_ids, q, 1)
    for g, w in zip(got, want):
        assert np.array_equal(np.asarray(g).astype(np.asarray(w).dtype), w)


def _prepared_search(rbc, x, q, kind, k):
    import ctypes

    import torch
    from paper_1103_2635_b200 import _lib

    x_dev, q_dev = _lib.to_device(x), _lib.to_device(q)
    h = ctypes.c_void_p()
    sp = _lib.stream_ptr()
    _lib.check(_lib.lib.rbc_bf_prepare(_lib.ptr(x_dev), x.shape[0], x.shape[1], 0 if kind == "l2" else 1,
                                       ctypes.byref(h), sp), "prepare")
    try:
        ids = torch.empty((q.shape[0], k), dtype=torch.int64, device="cuda")
        ds = torch.empty((q.shape[0], k), dtype=torch.float32, device="cuda")
        c0 = _calls()
        _lib.check(_lib.lib.rbc_bf_search_prepared(h, _lib.ptr(q_dev), q.shape[0], k, _lib.ptr(ids), _lib.ptr(ds), sp),
                   "search")
        return ids.cpu().numpy(), ds.cpu().numpy(), _calls() > c0
    finally:
        _lib.lib.rbc_index_destroy(h)


@pytest.mark.parametrize("d,kind,k", [(64, "l2", 1), (64, "l2", 16), (21, "l2", 5), (7, "l2", 3), (21, "l1", 4),
                                      (100, "l2", 2), (64, "l2", 40), (160, "l2", 3)])
def test_tc_bf_prepared_vs_oracle(rbc, oracle, d, kind, k):
    # the prepared operand: partitioned tcgen05 scan for L2 d <= 128 k <= 16, else the exact SIMT scan
    full = oracle.gen_clusters(70_000 + 700, d, 17 + d, n_clusters=12, cluster_sigma=0.05)
    x, q = full[:70_000], full[70_000:]
    ids, dists, tc_ran = _prepared_search(rbc, x, q, kind, k)
    assert tc_ran == (kind == "l2" and d <= 128 and k <= 32)
    oi, od = oracle.bf_topk(q, x, k, kind)
    assert np.array_equal(ids, oi) and np.array_equal(dists, od)


def test_tc_bf_prepared_rejects_wrong_handle(rbc):
    import ctypes

    from paper_1103_2635_b200 import _lib

    assert _lib.lib.rbc_bf_search_prepared(None, None, 1, 1, None, None, None) != 0


def _scans():
    from paper_1103_2635_b200 import _lib

    return _lib.lib.rbc_tc_scan_calls()


@pytest.mark.parametrize("d", [65, 96, 126, 127, 128])
@pytest.mark.parametrize("k", [1, 10])
def test_tc_stage2_wide_d_vs_oracle(rbc, oracle, d, k):
    # d in (64, 128]: two K planes (and the separate aug plane for d > 126) on the tensor cores
    full = oracle.gen_clusters(30_000 + 500, d, 5 + d, n_clusters=8, cluster_sigma=0.05)
    x, q = full[:30_000], full[30_000:]
    idx = rbc.build_exact(rbc.DataMatrix(x), 173, rbc.MetricSpec("l2", d), seed=3)
    s0 = _scans()
    got = rbc.exact_query_arrays(idx, q, k)
    assert _scans() > s0, "stage 2 did not run on the tensor cores"
    li, off, ld = idx.flat_lists()
    want = oracle.exact_query(x, idx.reps.rep_ids, li, off, ld, idx.radii, q, k)
    for g, w in zip(got, want):
        assert np.array_equal(np.asarray(g).astype(np.asarray(w).dtype), w)


@pytest.mark.parametrize("d", [100, 128])
def test_tc_bf_wide_d_vs_oracle(rbc, oracle, d):
    x = oracle.gen_clusters(80_000, d, 9 + d, n_clusters=8, cluster_sigma=0.05)
    q = np.concatenate([uniform(500, d, d), x[::400] + np.float32(0.001)]).astype(np.float32)
    for k in (1, 5, 16):
        c0 = _calls()
        ids, dists = rbc.brute_force.bf_search_arrays(q, x, rbc.MetricSpec("l2", d), k)
        assert _calls() > c0
        oi, od = oracle.bf_topk(q, x, k, "l2")
        assert np.array_equal(ids, oi) and np.array_equal(dists, od)


@pytest.mark.parametrize("k", [17, 24, 32])
@pytest.mark.parametrize("d", [20, 64, 100])
def test_tc_stage2_k_up_to_32_vs_oracle(rbc, oracle, k, d):
    full = oracle.gen_clusters(30_000 + 400, d, 2 + d, n_clusters=10, cluster_sigma=0.05)
    x, q = full[:30_000], full[30_000:]
    idx = rbc.build_exact(rbc.DataMatrix(x), 173, rbc.MetricSpec("l2", d), seed=5)
    s0 = _scans()
    got = rbc.exact_query_arrays(idx, q, k)
    assert _scans() > s0, "stage 2 did not run on the tensor cores"
    li, off, ld = idx.flat_lists()
    want = oracle.exact_query(x, idx.reps.rep_ids, li, off, ld, idx.radii, q, k)
    for g, w in zip(got, want):
        assert np.array_equal(np.asarray(g).astype(np.asarray(w).dtype), w)


@pytest.mark.parametrize("d", [16, 64, 100])
@pytest.mark.parametrize("k", [1, 5, 32])
def test_tc_one_shot_scan_vs_oracle(rbc, oracle, d, k):
    # the one-shot list scan on the tensor cores: exactly the nearest rep's s-list per query
    full = oracle.gen_clusters(40_000 + 2_000, d, 21 + d, n_clusters=8, cluster_sigma=0.05)
    x, q = full[:40_000], full[40_000:]
    idx = rbc.build_one_shot(rbc.DataMatrix(x), 200, 300, rbc.MetricSpec("l2", d), seed=2)
    s0 = _scans()
    got = rbc.one_shot_query_arrays(idx, q, k)
    assert _scans() > s0, "the one-shot scan did not run on the tensor cores"
    want = oracle.one_shot_query(x, idx.reps.rep_ids, idx.list_ids, q, k)
    for g, w in zip(got, want):
        assert np.array_equal(np.asarray(g).astype(np.asarray(w).dtype), w)
    exact = _exact_engine(rbc, lambda: rbc.one_shot_query_arrays(idx, q, k))
    for g, w in zip(got, exact):
        assert np.array_equal(g, w)


def test_auto_engine_size_threshold(rbc, oracle):
    # auto mode: a small brute force stays on the exact scan, a large one takes the tensor cores
    from paper_1103_2635_b200 import _lib

    x = oracle.gen_clusters(20_000, 16, 3, n_clusters=4, cluster_sigma=0.05)
    _lib.lib.rbc_set_engine(0)
    try:
        c0 = _calls()
        rbc.brute_force.bf_search_arrays(x[:50], x, rbc.MetricSpec("l2", 16), 1)
        assert _calls() == c0
        big = oracle.gen_clusters(100_000, 16, 4, n_clusters=4, cluster_sigma=0.05)
        ids, dists = rbc.brute_force.bf_search_arrays(big[:1000], big, rbc.MetricSpec("l2", 16), 3)
        assert _calls() > c0
        oi, od = oracle.bf_topk(big[:1000], big, 3, "l2")
        assert np.array_equal(ids, oi) and np.array_equal(dists, od)
    finally:
        _lib.lib.rbc_set_engine(2)
