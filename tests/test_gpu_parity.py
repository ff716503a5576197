"""GPU parity: the B200 path vs reference golden vectors and the pinned oracle.

Every comparison is bit-exact (ids, float32 distances, representative sets,
ownership lists, radii and SearchStats), which is stronger than the north
star's 1e-5 relative tolerance.
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

    return m


def _ne(a, b):
    return not np.array_equal(np.asarray(a), np.asarray(b))


# ---- metric -------------------------------------------------------------------
@pytest.mark.parametrize("d", [1, 2, 6, 8, 16, 21, 54, 64, 128])
@pytest.mark.parametrize("kind", ["l2", "l1"])
def test_pairwise_golden(rbc, golden, d, kind):
    a = uniform(16, d, 1000 + d, 4.0, -2.0)
    b = uniform(24, d, 2000 + d, 4.0, -2.0)
    assert np.array_equal(rbc.pairwise_distances(a, b, rbc.MetricSpec(kind, d)), golden[f"pair_{kind}_{d}"])


def test_metric_kats(rbc):
    assert rbc.distance(np.array([0.0, 0.0]), np.array([3.0, 4.0]), rbc.MetricSpec("l2", 2)) == 5.0
    assert rbc.distance(np.array([1.0, 2.0, 3.0]), np.array([4.0, 0.0, 3.0]), rbc.MetricSpec("l1", 3)) == 5.0
    assert rbc.distance(np.array([3.0, 4.0]), np.array([3.0, 4.0]), rbc.MetricSpec("l2", 2)) == 0.0


@pytest.mark.parametrize("kind", ["l2", "l1"])
def test_pairwise_symmetry_and_zero_diagonal(rbc, kind):
    spec = rbc.MetricSpec(kind, 6)
    rng = np.random.default_rng(7)
    a = rng.random((40, 6), dtype=np.float32)
    b = rng.random((60, 6), dtype=np.float32)
    assert np.array_equal(rbc.pairwise_distances(a, b, spec), rbc.pairwise_distances(b, a, spec).T)
    x = (rng.random((100, 5), dtype=np.float32) - 0.5) * 1000
    assert np.all(np.diagonal(rbc.pairwise_distances(x, x, rbc.MetricSpec(kind, 5))) == 0.0)


@pytest.mark.parametrize("d", [3, 64, 200])
def test_pairwise_large_vs_oracle(rbc, oracle, d):
    a = uniform(300, d, 5, 10.0, -5.0)
    b = uniform(517, d, 6, 10.0, -5.0)
    for kind in ("l2", "l1"):
        assert np.array_equal(rbc.pairwise_distances(a, b, rbc.MetricSpec(kind, d)), oracle.pairwise(a, b, kind))


# ---- brute force ------------------------------------------------------------------
@pytest.mark.parametrize("kind", ["l2", "l1"])
@pytest.mark.parametrize("k", [1, 4, 10])
def test_bf_golden(rbc, golden, kind, k):
    res = rbc.bf_search(uniform(40, 8, 29), uniform(2000, 8, 101), rbc.MetricSpec(kind, 8), k=k)
    assert np.array_equal(np.stack([nl.ids for nl in res.neighbors]), golden[f"bf_{kind}_k{k}_ids"])
    assert np.array_equal(np.stack([nl.dists for nl in res.neighbors]), golden[f"bf_{kind}_k{k}_dists"])
    assert res.distance_evals == 40 * 2000


@pytest.mark.parametrize("kind", ["l2", "l1"])
def test_bf_ties_golden(rbc, golden, kind):
    lat = np.stack(np.meshgrid(*[np.arange(6, dtype=np.float32)] * 3, indexing="ij"), -1).reshape(-1, 3)
    ql = np.array([[2.5, 2.5, 2.5], [0, 0, 0], [5, 5, 5], [1.5, 2.0, 3.5]], np.float32)
    res = rbc.bf_search(ql, lat, rbc.MetricSpec(kind, 3), k=12)
    assert np.array_equal(np.stack([nl.ids for nl in res.neighbors]), golden[f"bftie_{kind}_ids"])
    assert np.array_equal(np.stack([nl.dists for nl in res.neighbors]), golden[f"bftie_{kind}_dists"])


@pytest.mark.parametrize("d", [1, 6, 16, 21, 54, 64, 128])
@pytest.mark.parametrize("k", [1, 3, 7, 10, 33])
def test_bf_vs_oracle(rbc, oracle, d, k):
    x = oracle.gen_clusters(3000, d, d, n_clusters=5, cluster_sigma=0.1)
    q = uniform(70, d, 3 * d)
    for kind in ("l2", "l1"):
        ids, dists = rbc.brute_force.bf_search_arrays(q, x, rbc.MetricSpec(kind, d), k)
        oi, od = oracle.bf_topk(q, x, k, kind)
        assert np.array_equal(ids, oi) and np.array_equal(dists, od)


def test_bf_large_k_sort_path(rbc, oracle):
    x = uniform(5000, 12, 1)
    q = uniform(9, 12, 2)
    ids, dists = rbc.brute_force.bf_search_arrays(q, x, rbc.MetricSpec("l2", 12), 512)
    oi, od = oracle.bf_topk(q, x, 512)
    assert np.array_equal(ids, oi) and np.array_equal(dists, od)


def test_bf_subset_kats(rbc):
    line = rbc.DataMatrix(np.array([[0.0], [2.0], [5.0], [6.0], [9.0]], dtype=np.float32))
    spec1 = rbc.MetricSpec("l2", 1)
    res = rbc.bf_search_subset(np.array([8.0], np.float32), line, [2, 3, 4], spec1, k=1)
    assert res.neighbors[0].ids.tolist() == [4] and res.distance_evals == 3
    with pytest.raises(ValueError):
        rbc.bf_search_subset(np.array([1.0], np.float32), line, [1, 1, 2], spec1, k=1)
    u = rbc.DataMatrix(uniform(2000, 8, 101))
    res = rbc.bf_search_subset(u.values[50], u, np.array([900, 50, 1500]), rbc.MetricSpec("l2", 8), k=1)
    assert res.neighbors[0].ids[0] == 50
    full = rbc.bf_search(u.values[3][None, :], u, rbc.MetricSpec("l2", 8), k=100)
    sub = rbc.bf_search_subset(u.values[3], u, np.arange(u.n), rbc.MetricSpec("l2", 8), k=100)
    assert np.array_equal(full.neighbors[0].ids, sub.neighbors[0].ids)
    assert np.array_equal(full.neighbors[0].dists, sub.neighbors[0].dists)


def test_merge_neighbor_lists(rbc):
    NL = rbc.NeighborList
    a = NL(0, np.array([3, 1]), np.array([0.5, 1.5], np.float32))
    b = NL(0, np.array([2, 9]), np.array([0.5, 0.7], np.float32))
    ab = rbc.merge_neighbor_lists(a, b, 3)
    ba = rbc.merge_neighbor_lists(b, a, 3)
    assert ab.ids.tolist() == [2, 3, 9] and np.array_equal(ab.ids, ba.ids) and np.array_equal(ab.dists, ba.dists)


# ---- sampling -------------------------------------------------------------------------
@pytest.mark.parametrize("n,nr,seed", [(10, 3, 0), (1000, 40, 5), (100_000, 1000, 0), (1_000_000, 1000, 0),
                                       (581_012, 763, 0), (2_000_000, 1415, 0)])
def test_bernoulli_golden(rbc, golden, n, nr, seed):
    assert np.array_equal(rbc.sample_representatives(n, nr, seed).rep_ids, golden[f"bern_{n}_{nr}_{seed}"])


def test_fixed_count_golden(rbc, golden):
    assert np.array_equal(rbc.sample_representatives(1000, 50, 2, rbc.FIXED_COUNT).rep_ids, golden["fixed_1000_50_2"])


def test_bernoulli_large_vs_oracle(rbc, oracle):
    for n, nr, seed in ((16_000_000, 4000, 0), (3_333_333, 17, 9)):
        assert np.array_equal(rbc.sample_representatives(n, nr, seed).rep_ids, oracle.bernoulli(n, nr / n, seed))


def test_empty_draw_retry(rbc, monkeypatch):
    import paper_1103_2635_b200.rbc as rbc_mod

    calls = []

    def always_empty(n, p, seed):
        calls.append(seed)
        return np.array([], dtype=np.int64)

    monkeypatch.setattr(rbc_mod, "_bernoulli_draw", always_empty)
    with pytest.raises(ValueError):
        rbc.sample_representatives(10, 1, seed=5)
    assert calls == [5, 6]


# ---- build + exact search -----------------------------------------------------------
def _case_data(oracle, name):
    if name == "cl8":
        return oracle.gen_clusters(2500, 8, 13, n_clusters=6, cluster_sigma=0.02), "l2"
    return {"u8s0": (uniform(2000, 8, 101), "l2"), "u8s1l1": (uniform(2000, 8, 101), "l1"),
            "u6s0": (uniform(1500, 6, 100), "l2"), "u6s1l1": (uniform(1500, 6, 101), "l1")}[name]


@pytest.mark.parametrize("name,nr,seed", [("u8s0", 50, 0), ("u8s1l1", 45, 1), ("u6s0", 40, 0), ("u6s1l1", 40, 1),
                                          ("cl8", 50, 15)])
def test_build_and_exact_search_golden(rbc, golden, oracle, name, nr, seed):
    data, kind = _case_data(oracle, name)
    idx = rbc.build_exact(rbc.DataMatrix(data), nr, rbc.MetricSpec(kind, data.shape[1]), seed=seed)
    assert np.array_equal(idx.reps.rep_ids, golden[f"bx_{name}_reps"])
    ids, off, dists = idx.flat_lists()
    assert np.array_equal(ids, golden[f"bx_{name}_ids"]) and np.array_equal(off, golden[f"bx_{name}_off"])
    assert np.array_equal(dists, golden[f"bx_{name}_dists"]) and np.array_equal(idx.radii, golden[f"bx_{name}_radii"])
    q = golden[f"bx_{name}_queries"]
    for k in (1, 3, 7):
        res, stats = rbc.exact_query_batch(idx, q, k)
        assert np.array_equal(np.stack([r.ids for r in res]), golden[f"xq_{name}_k{k}_ids"])
        assert np.array_equal(np.stack([r.dists for r in res]), golden[f"xq_{name}_k{k}_dists"])
        assert np.array_equal(np.array([s.gamma for s in stats], np.float32), golden[f"xq_{name}_k{k}_gamma"])
        assert [s.reps_pruned_radius for s in stats] == golden[f"xq_{name}_k{k}_prr"].tolist()
        assert [s.reps_pruned_3gamma for s in stats] == golden[f"xq_{name}_k{k}_p3"].tolist()
        assert [s.candidates_examined for s in stats] == golden[f"xq_{name}_k{k}_cand"].tolist()
        assert all(s.reps_total == s.dists_step1 == idx.reps.size for s in stats)


def test_line_kats(rbc):
    line = rbc.DataMatrix(np.array([[0.0], [2.0], [5.0], [6.0], [9.0]], dtype=np.float32))
    spec1 = rbc.MetricSpec("l2", 1)
    idx = rbc.build_exact(line, 2, spec1, seed=0, rep_ids=[1, 3])
    assert idx.list_ids[0].tolist() == [1, 0] and idx.list_ids[1].tolist() == [3, 2, 4]
    assert idx.list_dists[1].tolist() == [0.0, 1.0, 3.0] and idx.radii.tolist() == [2.0, 3.0]
    nl, st = rbc.exact_query(idx, np.array([4.9], np.float32), 1)
    assert nl.ids.tolist() == [2] and st.candidates_examined == 5
    assert st.gamma == pytest.approx(1.1, abs=1e-6)
    nl, st = rbc.exact_query(idx, np.array([0.1], np.float32), 1)
    assert nl.ids.tolist() == [0] and st.candidates_examined == 2
    assert st.reps_pruned_radius == 1 and st.reps_pruned_3gamma == 1
    os_idx = rbc.build_one_shot(line, 2, 3, spec1, seed=0, rep_ids=[1, 3])
    assert os_idx.list_ids.tolist() == [[1, 0, 2], [3, 2, 4]]
    assert rbc.one_shot_query(os_idx, np.array([8.0], np.float32), 1).ids.tolist() == [4]


def test_cfg_shaped_golden(rbc, golden, oracle):
    full = oracle.gen_clusters(20_200, 64, 1, n_clusters=16, cluster_sigma=0.05)
    data, q = full[:20_000], full[20_000:]
    idx = rbc.build_exact(rbc.DataMatrix(data), 141, rbc.MetricSpec("l2", 64), seed=0)
    assert np.array_equal(idx.reps.rep_ids, golden["c64_reps"])
    ids, off, dists = idx.flat_lists()
    assert np.array_equal(ids, golden["c64_ids"]) and np.array_equal(dists, golden["c64_dists"])
    for k in (1, 10):
        gi, gd, gg, _, _, gc = rbc.exact_query_arrays(idx, q, k)
        assert np.array_equal(gi, golden[f"c64_k{k}_ids"]) and np.array_equal(gd, golden[f"c64_k{k}_dists"])
        assert np.array_equal(gc, golden[f"c64_k{k}_cand"]) and np.array_equal(gg, golden[f"c64_k{k}_gamma"])


@pytest.mark.parametrize("d,kind,k", [(1, "l2", 3), (6, "l1", 7), (16, "l2", 10), (21, "l1", 1), (54, "l2", 10),
                                      (64, "l2", 1), (64, "l2", 5), (128, "l2", 10), (128, "l1", 3)])
def test_exact_search_vs_oracle(rbc, oracle, d, kind, k):
    n = 30_000
    full = oracle.gen_clusters(n + 500, d, 40 + d, n_clusters=12, cluster_sigma=0.05)
    x, q = full[:n], full[n:]
    nr = int(np.ceil(np.sqrt(n)))
    idx = rbc.build_exact(rbc.DataMatrix(x), nr, rbc.MetricSpec(kind, d), seed=3)
    reps = idx.reps.rep_ids
    li, off, ld, radii = oracle.build_exact(x, reps, kind)
    ids, offsets, dists = idx.flat_lists()
    assert np.array_equal(ids, li) and np.array_equal(offsets, off) and np.array_equal(dists, ld)
    got = rbc.exact_query_arrays(idx, q, k)
    want = oracle.exact_query(x, reps, li, off, ld, radii, q, k, kind)
    for g, w in zip(got, want):
        assert np.array_equal(np.asarray(g).astype(w.dtype), w)
    # exactness: equals brute force
    bi, bd = oracle.bf_topk(q, x, k, kind)
    assert np.array_equal(got[0], bi) and np.array_equal(got[1], bd)


def test_exact_search_duplicates_and_ties(rbc, oracle):
    # heavy duplication: many identical points and reps at equal distances
    base = np.repeat(uniform(50, 4, 11), 40, axis=0)
    q = np.concatenate([base[:30], uniform(30, 4, 12)])
    idx = rbc.build_exact(rbc.DataMatrix(base), 60, rbc.MetricSpec("l2", 4), seed=2)
    reps = idx.reps.rep_ids
    li, off, ld, radii = oracle.build_exact(base, reps)
    ids, offsets, dists = idx.flat_lists()
    assert np.array_equal(ids, li) and np.array_equal(dists, ld)
    for k in (1, 5, 16):
        got = rbc.exact_query_arrays(idx, q, k)
        want = oracle.exact_query(base, reps, li, off, ld, radii, q, k)
        for g, w in zip(got, want):
            assert np.array_equal(np.asarray(g).astype(w.dtype), w)


def test_k_validation(rbc):
    u = rbc.DataMatrix(uniform(2000, 8, 101))
    idx = rbc.build_exact(u, 10, rbc.MetricSpec("l2", 8), seed=6)
    with pytest.raises(ValueError):
        rbc.exact_query(idx, u.values[0], idx.reps.size + 1)
    nl, st = rbc.exact_query(idx, u.values[123], 1)
    assert nl.ids[0] == 123 and nl.dists[0] == 0.0


# ---- one-shot ---------------------------------------------------------------------------------
@pytest.mark.parametrize("name,nr,s,kind,seed", [("u8", 25, 10, "l2", 1), ("u8l1", 30, 17, "l1", 4),
                                                 ("u4", 120, 120, "l2", 5)])
def test_one_shot_golden(rbc, golden, name, nr, s, kind, seed):
    data = uniform(4000, 4, 42) if name == "u4" else uniform(2000, 8, 101)
    idx = rbc.build_one_shot(rbc.DataMatrix(data), nr, s, rbc.MetricSpec(kind, data.shape[1]), seed=seed)
    assert np.array_equal(idx.reps.rep_ids, golden[f"os_{name}_reps"])
    assert np.array_equal(idx.list_ids, golden[f"os_{name}_lists"]) and np.array_equal(idx.radii, golden[f"os_{name}_radii"])
    q = golden[f"os_{name}_queries"]
    for k in (1, 3):
        res, stats = rbc.one_shot_query_batch(idx, q, k)
        assert np.array_equal(np.stack([r.ids for r in res]), golden[f"oq_{name}_k{k}_ids"])
        assert np.array_equal(np.stack([r.dists for r in res]), golden[f"oq_{name}_k{k}_dists"])
        assert np.array_equal(np.array([st.gamma for st in stats], np.float32), golden[f"oq_{name}_k{k}_gamma"])
        assert all(st.candidates_examined == s for st in stats)


@pytest.mark.parametrize("d,kind,s", [(21, "l1", 141), (16, "l2", 40), (8, "l2", 300)])
def test_one_shot_vs_oracle(rbc, oracle, d, kind, s):
    n = 20_000
    full = oracle.gen_clusters(n + 300, d, 90 + d, n_clusters=8, cluster_sigma=0.05)
    x, q = full[:n], full[n:]
    idx = rbc.build_one_shot(rbc.DataMatrix(x), 141, s, rbc.MetricSpec(kind, d), seed=4)
    lists, radii = oracle.build_one_shot(x, idx.reps.rep_ids, s, kind)
    assert np.array_equal(idx.list_ids, lists) and np.array_equal(idx.radii, radii)
    for k in (1, 4):
        got = rbc.one_shot_query_arrays(idx, q, k)
        want = oracle.one_shot_query(x, idx.reps.rep_ids, lists, q, k, kind)
        for g, w in zip(got, want):
            assert np.array_equal(g, w)


def test_one_shot_s_equals_n_is_brute_force(rbc):
    u = rbc.DataMatrix(uniform(2000, 8, 101))
    spec = rbc.MetricSpec("l2", 8)
    idx = rbc.build_one_shot(u, 12, u.n, spec, seed=2)
    queries = np.random.default_rng(0).random((20, 8), dtype=np.float32)
    bf = rbc.bf_search(queries, u, spec, k=3)
    res, _ = rbc.one_shot_query_batch(idx, queries, 3)
    for a, b in zip(res, bf.neighbors):
        assert np.array_equal(a.ids, b.ids) and np.array_equal(a.dists, b.dists)


# ---- range query, pruning primitives --------------------------------------------------------
def test_range_query_golden(rbc, golden):
    u = rbc.DataMatrix(uniform(2000, 8, 101))
    idx = rbc.build_exact(u, 40, rbc.MetricSpec("l2", 8), seed=11)
    assert np.array_equal(idx.reps.rep_ids, golden["rq_reps"])
    for i in range(6):
        ids, dists = rbc.range_query(idx, golden[f"rq_{i}_q"], float(golden[f"rq_{i}_radius"]))
        assert np.array_equal(ids, golden[f"rq_{i}_ids"]) and np.array_equal(dists, golden[f"rq_{i}_dists"])
    ids, dists = rbc.range_query(idx, u.values[77], 0.0)
    assert ids.tolist() == [77] and dists.tolist() == [0.0]


def test_prune_and_cutoff_kats(rbc):
    assert rbc.prune_representatives(np.array([1.1, 2.9]), np.array([3.0, 2.0]), 1.1).tolist() == [0, 1]
    assert rbc.prune_representatives(np.array([1.9, 5.9]), np.array([2.0, 3.0]), 1.9).tolist() == [0]
    assert rbc.prune_representatives(np.array([0.0, 0.5, 2.0]), np.array([1.0, 1.0, 1.0]), 0.0).tolist() == [0]
    assert rbc.prune_representatives(np.array([2.0, 2.0]), np.array([1.0, 0.0]), 2.0).tolist() == [0, 1]
    assert rbc.list_cutoff(np.array([0.0, 1.0, 2.0, 5.0, 7.0]), 4.0) == 3
    assert rbc.list_cutoff(np.array([0.0, 1.0, 1.0, 2.0]), 1.0) == 3
    assert rbc.list_cutoff(np.array([0.1], np.float32), 0.1) == 0


# ---- tcgen05 building block --------------------------------------------------------------
@pytest.mark.parametrize("n", [16, 48, 128, 256])
def test_tc_selftest_tile(rbc, n):
    import torch

    from paper_1103_2635_b200 import _lib

    g = torch.Generator(device="cuda").manual_seed(n)
    a = torch.randn(128, 64, device="cuda", generator=g).half()
    b = torch.randn(n, 64, device="cuda", generator=g).half()
    c = torch.empty(128, n, device="cuda", dtype=torch.float32)
    _lib.check(_lib.lib.rbc_tc_selftest(_lib.ptr(a), _lib.ptr(b), _lib.ptr(c), n, _lib.stream_ptr()))
    ref = a.double() @ b.double().T
    err = (c.double() - ref).abs().max().item()
    assert err <= 1e-3 * ref.abs().max().item(), err


def _both_engines(rbc, idx, q, k):
    from paper_1103_2635_b200 import _lib

    try:
        _lib.lib.rbc_set_engine(1)
        exact = rbc.exact_query_arrays(idx, q, k)
    finally:
        _lib.lib.rbc_set_engine(0)
    fast = rbc.exact_query_arrays(idx, q, k)
    return fast, exact


@pytest.mark.parametrize("k", [1, 2, 10, 16])
def test_tc_engine_matches_exact_engine(rbc, oracle, k):
    full = oracle.gen_clusters(100_000 + 2_000, 64, 1, n_clusters=32, cluster_sigma=0.05)
    x, q = full[:100_000], full[100_000:]
    idx = rbc.build_exact(rbc.DataMatrix(x), 316, rbc.MetricSpec("l2", 64), seed=0)
    fast, exact = _both_engines(rbc, idx, q, k)
    for a, b in zip(fast, exact):
        assert np.array_equal(a, b)
    li, off, ld = idx.flat_lists()
    want = oracle.exact_query(x, idx.reps.rep_ids, li, off, ld, idx.radii, q[:300], k)
    assert np.array_equal(fast[0][:300], want[0]) and np.array_equal(fast[1][:300], want[1])


@pytest.mark.parametrize("d", [3, 17, 40, 64])
def test_tc_engine_scales_and_offsets(rbc, oracle, d):
    # large coordinate offsets and mixed scales stress the centred f16 operands and the error bound
    rng = np.random.default_rng(d)
    x = (rng.standard_normal((30_000, d)) * rng.choice([0.001, 1.0, 300.0], size=(30_000, 1)) + 1000.0).astype(np.float32)
    q = (x[rng.integers(0, 30_000, 400)] + rng.standard_normal((400, d)).astype(np.float32) * 0.01).astype(np.float32)
    idx = rbc.build_exact(rbc.DataMatrix(x), 173, rbc.MetricSpec("l2", d), seed=1)
    for k in (1, 5):
        fast, exact = _both_engines(rbc, idx, q, k)
        for a, b in zip(fast, exact):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("k", [1, 10])
def test_tc_engine_wide_tile_unions(rbc, oracle, k):
    # few clusters, many representatives: every tile's surviving-list union is large,
    # which exercises the stage-2 work-capacity re-run path on the first search
    full = oracle.gen_clusters(40_000 + 600, 32, 5, n_clusters=2, cluster_sigma=0.05)
    x, q = full[:40_000], full[40_000:]
    idx = rbc.build_exact(rbc.DataMatrix(x), 400, rbc.MetricSpec("l2", 32), seed=2)
    fast, exact = _both_engines(rbc, idx, q, k)
    for a, b in zip(fast, exact):
        assert np.array_equal(a, b)
    again = rbc.exact_query_arrays(idx, q, k)
    for a, b in zip(again, exact):
        assert np.array_equal(a, b)


def test_tc_engine_overflow_fallback(rbc):
    from paper_1103_2635_b200 import _lib

    base = np.repeat(uniform(20, 8, 3), 2000, axis=0)  # 2000 exact copies of each point: ties overflow the buffer
    idx = rbc.build_exact(rbc.DataMatrix(base), 30, rbc.MetricSpec("l2", 8), seed=0)
    q = base[::997][:12]
    fast, exact = _both_engines(rbc, idx, q, 1)
    for a, b in zip(fast, exact):
        assert np.array_equal(a, b)
    rbc.exact_query_arrays(idx, q, 1)
    assert _lib.lib.rbc_stage2_overflows() > 0


@pytest.mark.parametrize("k", [1, 10])
def test_graph_replay_matches_direct(rbc, oracle, monkeypatch, k):
    # repeating the same keys-level call captures the fused search into a CUDA graph
    # (1st call direct + arena measurement, 2nd capture + replay, then replay); every
    # replay must equal the direct launch path bit for bit, stats included
    import torch

    from paper_1103_2635_b200 import _lib

    full = oracle.gen_clusters(60_000 + 3_000, 64, 3, n_clusters=16, cluster_sigma=0.05)
    x, q = full[:60_000], full[60_000:]
    idx = rbc.build_exact(rbc.DataMatrix(x), 245, rbc.MetricSpec("l2", 64), seed=0)
    dev = idx._dev
    nq = q.shape[0]
    q_dev = _lib.to_device(q)

    def run(no_graph):
        if no_graph:
            monkeypatch.setenv("RBC_NO_GRAPH", "1")
        else:
            monkeypatch.delenv("RBC_NO_GRAPH", raising=False)
        outs = []
        keys = torch.empty((nq, k), dtype=torch.int64, device="cuda")
        gamma = torch.empty(nq, dtype=torch.float32, device="cuda")
        prr = torch.empty(nq, dtype=torch.int32, device="cuda")
        p3 = torch.empty(nq, dtype=torch.int32, device="cuda")
        cand = torch.empty(nq, dtype=torch.int64, device="cuda")
        stats = _lib.SearchStatsC(gamma.data_ptr(), prr.data_ptr(), p3.data_ptr(), cand.data_ptr())
        for _ in range(4):
            for t in (keys, gamma, prr, p3, cand):
                t.fill_(-7)
            _lib.check(_lib.lib.rbc_exact_search_keys(dev.handle, _lib.ptr(q_dev), nq, k, _lib.ptr(keys), stats,
                                                      _lib.stream_ptr()), "exact search")
            torch.cuda.synchronize()
            outs.append([t.cpu().numpy().copy() for t in (keys, gamma, prr, p3, cand)])
        return outs

    direct = run(True)[0]
    for rep in run(False):
        for a, b in zip(rep, direct):
            assert np.array_equal(a, b)


@pytest.fixture(scope="module")
def cfg2_full(rbc):
    """BASELINE cfg2 at full size: clusters(n = 1.1M, d = 64, seed 1, C = 64, sigma = 0.05) -> X 1M, Q 100k."""
    full = rbc.gen_synthetic("clusters", 1_100_000, 64, 1, n_clusters=64, cluster_sigma=0.05).values
    x, q = np.ascontiguousarray(full[:1_000_000]), np.ascontiguousarray(full[1_000_000:])
    idx = rbc.build_exact(rbc.DataMatrix(x), 1000, rbc.MetricSpec("l2", 64), seed=0)
    return x, q, idx


@pytest.mark.parametrize("k", [1, 10])
def test_cfg2_full_size_tc_matches_exact_engine(rbc, oracle, cfg2_full, k):
    """Full-size property: the tensor-core path (direct launch, graph capture, graph replay) equals the exact SIMT
    engine on all 100k cfg2 queries (ids, distances and every stats field), and the oracle on a sample."""
    x, q, idx = cfg2_full
    assert idx.reps.size == 1016
    fast, exact = _both_engines(rbc, idx, q, k)
    for _ in range(2):  # second and third calls: graph capture, then replay
        again = rbc.exact_query_arrays(idx, q, k)
        for a, b in zip(again, fast):
            assert np.array_equal(a, b)
    for a, b in zip(fast, exact):
        assert np.array_equal(a, b)
    li, off, ld = idx.flat_lists()
    sample = np.ascontiguousarray(q[::500])
    want = oracle.exact_query(x, idx.reps.rep_ids, li, off, ld, idx.radii, sample, k)
    assert np.array_equal(fast[0][::500], want[0]) and np.array_equal(fast[1][::500], want[1])
