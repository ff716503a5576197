"""Full-size parity at the BASELINE.json configs that fit one GPU.

Every config is built and searched at its real shape and compared with the oracle (the C restatement of the
reference, OpenMP on the host cores) on ALL queries: representative sets, ownership lists, list distances and
radii bit for bit, then ids, distances and every SearchStats field bit for bit.

    cfg1  one-shot L2, clusters n=10k d=16 C=8, n_r=s=100 fixed-count, 1k queries
    cfg2  exact 1-NN L2, clusters n=1M d=64 C=64, n_r=1000 (|R|=1016), 100k queries
    cfg3  exact 10-NN L2, clusters n=581,012 d=54 C=8, n_r=763, 100k queries
    cfg4  one-shot 1-NN L1, clusters n=2M d=21 C=8, n_r=s=1415, 100k queries
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rbc():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1103_2635_b200 as rbc

    return rbc


def _held_out(rbc, n, nq, d, seed, c):
    full = rbc.gen_synthetic("clusters", n + nq, d, seed, n_clusters=c, cluster_sigma=0.05).values
    return np.ascontiguousarray(full[:n]), np.ascontiguousarray(full[n:])


def _check_exact(rbc, oracle, x, q, n_r, k, metric="l2"):
    d = x.shape[1]
    idx = rbc.build_exact(rbc.DataMatrix(x), n_r, rbc.MetricSpec(metric, d), seed=0)
    reps = oracle.bernoulli(x.shape[0], n_r / x.shape[0], 0)
    assert np.array_equal(idx.reps.rep_ids, reps), "representative set differs"
    li, off, ld, radii = oracle.build_exact(x, reps, metric=metric)
    ids, offsets, dists = idx.flat_lists()
    assert np.array_equal(offsets, off), "list lengths differ"
    assert np.array_equal(ids, li), "list ids differ"
    assert np.array_equal(dists, ld), "list distances differ"
    assert np.array_equal(idx.radii, radii), "radii differ"
    got = rbc.exact_query_arrays(idx, q, k)
    want = oracle.exact_query(x, reps, li, off, ld, radii, q, k, metric=metric)
    for g, w, name in zip(got, want, ("ids", "dists", "gamma", "pruned_radius", "pruned_3gamma", "candidates")):
        g = np.asarray(g).astype(np.asarray(w).dtype)
        bad = np.flatnonzero(~(g == w).reshape(len(q), -1).all(axis=1))
        assert bad.size == 0, f"{name} differ on {bad.size} of {len(q)} queries (first {bad[:5]})"
    return idx


def _check_one_shot(rbc, oracle, x, q, n_r, s, k, metric, mode):
    d = x.shape[1]
    idx = rbc.build_one_shot(rbc.DataMatrix(x), n_r, s, rbc.MetricSpec(metric, d), seed=0, mode=mode)
    if mode == "fixed-count":
        reps = np.sort(np.random.default_rng(0).choice(x.shape[0], size=n_r, replace=False)).astype(np.int64)
    else:
        reps = oracle.bernoulli(x.shape[0], n_r / x.shape[0], 0)
    assert np.array_equal(idx.reps.rep_ids, reps), "representative set differs"
    lists, radii = oracle.build_one_shot(x, reps, s, metric=metric)
    assert np.array_equal(np.asarray(idx.list_ids), lists), "one-shot lists differ"
    assert np.array_equal(idx.radii, radii), "one-shot radii differ"
    got = rbc.one_shot_query_arrays(idx, q, k)
    want = oracle.one_shot_query(x, reps, lists, q, k, metric=metric)
    for g, w, name in zip(got, want, ("ids", "dists", "gamma")):
        g = np.asarray(g).astype(np.asarray(w).dtype)
        bad = np.flatnonzero(~(g == w).reshape(len(q), -1).all(axis=1))
        assert bad.size == 0, f"{name} differ on {bad.size} of {len(q)} queries (first {bad[:5]})"
    return idx


def test_cfg1_full_size(rbc, oracle):
    x, q = _held_out(rbc, 10_000, 1_000, 16, 7, 8)
    for k in (1, 5):
        _check_one_shot(rbc, oracle, x, q, 100, 100, k, "l2", "fixed-count")


def test_cfg2_full_size_vs_oracle(rbc, oracle):
    """All 100k cfg2 queries and the whole 1M-point build against the oracle (not just engine vs engine)."""
    x, q = _held_out(rbc, 1_000_000, 100_000, 64, 1, 64)
    idx = _check_exact(rbc, oracle, x, q, 1000, 1)
    assert idx.reps.size == 1016


def test_cfg3_full_size_vs_oracle(rbc, oracle):
    x, q = _held_out(rbc, 581_012, 100_000, 54, 3, 8)
    _check_exact(rbc, oracle, x, q, 763, 10)


def test_cfg4_full_size_vs_oracle(rbc, oracle):
    """One-shot L1 at n=2M, d=21, s=1415: lists, radii and all 100k queries."""
    x, q = _held_out(rbc, 2_000_000, 100_000, 21, 4, 8)
    _check_one_shot(rbc, oracle, x, q, 1415, 1415, 1, "l1", "bernoulli")


@pytest.mark.parametrize("n_r", [9000, 20000])
def test_many_representatives_vs_oracle(rbc, oracle, n_r):
    """|R| above the tensor-core stage-1 limit (6144: SIMT stage 1 feeding tensor-core stage 2) and above the
    stage-2 tile-fill shared-memory limit (~17k: both stages on the exact path) -- the reference takes any |R|."""
    x, q = _held_out(rbc, 200_000, 1_000, 8, 11, 64)
    for k in (1, 4):
        _check_exact(rbc, oracle, x, q, n_r, k)


def test_hand_made_index_is_validated(rbc):
    """A hand-made exact index whose lists do not partition the points, or hold out-of-range ids, raises
    ValueError at upload instead of reading out of bounds on the device."""
    x, q = _held_out(rbc, 5_000, 10, 8, 12, 4)
    idx = rbc.build_exact(rbc.DataMatrix(x), 50, rbc.MetricSpec("l2", 8), seed=0)
    short = rbc.RbcExactIndex(idx.data, idx.metric, idx.reps, [a.copy() for a in idx.list_ids],
                              [a.copy() for a in idx.list_dists], idx.radii.copy())
    short.list_ids[0] = short.list_ids[0][:-1]
    short.list_dists[0] = short.list_dists[0][:-1]
    with pytest.raises(ValueError):
        rbc.exact_query_batch(short, q, 1)
    bad = rbc.RbcExactIndex(idx.data, idx.metric, idx.reps, [a.copy() for a in idx.list_ids],
                            [a.copy() for a in idx.list_dists], idx.radii.copy())
    bad.list_ids[1][0] = x.shape[0] + 5
    with pytest.raises(ValueError):
        rbc.exact_query_batch(bad, q, 1)
    # a reassigned field invalidates the device copy (searches read the current fields)
    ok = rbc.exact_query_arrays(idx, q, 1)
    idx.radii = idx.radii.copy()
    again = rbc.exact_query_arrays(idx, q, 1)
    assert np.array_equal(ok[0], again[0])
    assert idx._dev_fp is not None
