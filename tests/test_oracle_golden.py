"""Pin the CPU oracle against golden vectors produced by the reference itself.

The oracle (oracle/rbc_oracle.c) is the parity checker for the GPU path, so it
must first reproduce the reference bit for bit (tests/golden/make_golden.py).
"""

import numpy as np
import pytest

from rbc_testutil import uniform


def test_generators_match_reference(golden, oracle):
    assert np.array_equal(oracle.gen_clusters(100, 5, 3, n_clusters=4, cluster_sigma=0.05),
                          golden["gen_clusters_100_5_3"])


@pytest.mark.parametrize("d", [1, 2, 6, 8, 16, 21, 54, 64, 128])
@pytest.mark.parametrize("kind", ["l2", "l1"])
def test_pairwise_bit_exact(golden, oracle, d, kind):
    a = uniform(16, d, 1000 + d, 4.0, -2.0)
    b = uniform(24, d, 2000 + d, 4.0, -2.0)
    assert np.array_equal(oracle.pairwise(a, b, kind), golden[f"pair_{kind}_{d}"])


@pytest.mark.parametrize("kind", ["l2", "l1"])
@pytest.mark.parametrize("k", [1, 4, 10])
def test_bf_topk(golden, oracle, kind, k):
    ids, dists = oracle.bf_topk(uniform(40, 8, 29), uniform(2000, 8, 101), k, kind)
    assert np.array_equal(ids, golden[f"bf_{kind}_k{k}_ids"])
    assert np.array_equal(dists, golden[f"bf_{kind}_k{k}_dists"])


@pytest.mark.parametrize("kind", ["l2", "l1"])
def test_bf_ties_lowest_id(golden, oracle, kind):
    lat = np.stack(np.meshgrid(*[np.arange(6, dtype=np.float32)] * 3, indexing="ij"), -1).reshape(-1, 3)
    ql = np.array([[2.5, 2.5, 2.5], [0, 0, 0], [5, 5, 5], [1.5, 2.0, 3.5]], np.float32)
    ids, dists = oracle.bf_topk(ql, lat, 12, kind)
    assert np.array_equal(ids, golden[f"bftie_{kind}_ids"])
    assert np.array_equal(dists, golden[f"bftie_{kind}_dists"])


@pytest.mark.parametrize("n,nr,seed", [(10, 3, 0), (1000, 40, 5), (100_000, 1000, 0), (1_000_000, 1000, 0),
                                       (581_012, 763, 0), (2_000_000, 1415, 0)])
def test_bernoulli_pcg64(golden, oracle, n, nr, seed):
    assert np.array_equal(oracle.bernoulli(n, nr / n, seed), golden[f"bern_{n}_{nr}_{seed}"])


CASES = {
    "u8s0": (lambda: uniform(2000, 8, 101), "l2"),
    "u8s1l1": (lambda: uniform(2000, 8, 101), "l1"),
    "u6s0": (lambda: uniform(1500, 6, 100), "l2"),
    "u6s1l1": (lambda: uniform(1500, 6, 101), "l1"),
}


def _cl8(oracle):
    return oracle.gen_clusters(2500, 8, 13, n_clusters=6, cluster_sigma=0.02)


@pytest.mark.parametrize("name", ["u8s0", "u8s1l1", "u6s0", "u6s1l1", "cl8"])
def test_build_exact_and_query(golden, oracle, name):
    if name == "cl8":
        data, kind = _cl8(oracle), "l2"
    else:
        mk, kind = CASES[name]
        data = mk()
    reps = golden[f"bx_{name}_reps"]
    li, off, ld, radii = oracle.build_exact(data, reps, kind)
    assert np.array_equal(li, golden[f"bx_{name}_ids"])
    assert np.array_equal(off, golden[f"bx_{name}_off"])
    assert np.array_equal(ld, golden[f"bx_{name}_dists"])
    assert np.array_equal(radii, golden[f"bx_{name}_radii"])
    q = golden[f"bx_{name}_queries"]
    for k in (1, 3, 7):
        ids, dists, gamma, prr, p3, cand = oracle.exact_query(data, reps, li, off, ld, radii, q, k, kind)
        assert np.array_equal(ids, golden[f"xq_{name}_k{k}_ids"])
        assert np.array_equal(dists, golden[f"xq_{name}_k{k}_dists"])
        assert np.array_equal(gamma, golden[f"xq_{name}_k{k}_gamma"])
        assert np.array_equal(prr, golden[f"xq_{name}_k{k}_prr"])
        assert np.array_equal(p3, golden[f"xq_{name}_k{k}_p3"])
        assert np.array_equal(cand, golden[f"xq_{name}_k{k}_cand"])


def test_line_kat(golden, oracle):
    line = np.array([[0.0], [2.0], [5.0], [6.0], [9.0]], np.float32)
    li, off, ld, radii = oracle.build_exact(line, np.array([1, 3]), "l2")
    assert li.tolist() == [1, 0, 3, 2, 4] == golden["line_ids"].tolist()
    assert ld.tolist() == [0.0, 2.0, 0.0, 1.0, 3.0]
    assert radii.tolist() == [2.0, 3.0]
    ids, dists, gamma, prr, p3, cand = oracle.exact_query(line, np.array([1, 3]), li, off, ld, radii,
                                                          np.array([[4.9], [0.1]], np.float32), 1)
    assert ids[:, 0].tolist() == [2, 0]
    assert cand.tolist() == [5, 2] and prr.tolist() == [0, 1] and p3.tolist() == [0, 1]


def test_cfg_shaped_d64(golden, oracle):
    full = oracle.gen_clusters(20_200, 64, 1, n_clusters=16, cluster_sigma=0.05)
    data, q = full[:20_000], full[20_000:]
    reps = oracle.bernoulli(20_000, 141 / 20_000, 0)
    assert np.array_equal(reps, golden["c64_reps"])
    li, off, ld, radii = oracle.build_exact(data, reps)
    assert np.array_equal(li, golden["c64_ids"]) and np.array_equal(ld, golden["c64_dists"])
    for k in (1, 10):
        ids, dists, gamma, _, _, cand = oracle.exact_query(data, reps, li, off, ld, radii, q, k)
        assert np.array_equal(ids, golden[f"c64_k{k}_ids"])
        assert np.array_equal(dists, golden[f"c64_k{k}_dists"])
        assert np.array_equal(cand, golden[f"c64_k{k}_cand"])
        assert np.array_equal(gamma, golden[f"c64_k{k}_gamma"])


@pytest.mark.parametrize("name,nr,s,kind", [("u8", 25, 10, "l2"), ("u8l1", 30, 17, "l1"), ("u4", 120, 120, "l2")])
def test_one_shot(golden, oracle, name, nr, s, kind):
    data = uniform(4000, 4, 42) if name == "u4" else uniform(2000, 8, 101)
    reps = golden[f"os_{name}_reps"]
    lists, radii = oracle.build_one_shot(data, reps, s, kind)
    assert np.array_equal(lists, golden[f"os_{name}_lists"])
    assert np.array_equal(radii, golden[f"os_{name}_radii"])
    q = golden[f"os_{name}_queries"]
    for k in (1, 3):
        ids, dists, gamma = oracle.one_shot_query(data, reps, lists, q, k, kind)
        assert np.array_equal(ids, golden[f"oq_{name}_k{k}_ids"])
        assert np.array_equal(dists, golden[f"oq_{name}_k{k}_dists"])
        assert np.array_equal(gamma, golden[f"oq_{name}_k{k}_gamma"])


def test_range_query(golden, oracle):
    data = uniform(2000, 8, 101)
    reps = golden["rq_reps"]
    li, off, ld, radii = oracle.build_exact(data, reps)
    for i in range(6):
        ids, dists = oracle.range_query(data, reps, li, off, ld, radii, golden[f"rq_{i}_q"], golden[f"rq_{i}_radius"])
        assert np.array_equal(ids, golden[f"rq_{i}_ids"])
        assert np.array_equal(dists, golden[f"rq_{i}_dists"])


def test_list_cutoff_kats(oracle):
    assert oracle.list_cutoff(np.array([0.0, 1.0, 2.0, 5.0, 7.0]), 4.0) == 3
    assert oracle.list_cutoff(np.array([1.0, 2.0]), 0.5) == 0
    assert oracle.list_cutoff(np.array([0.0, 1.0, 1.0, 2.0]), 1.0) == 3
    # f32 0.1 vs f64 0.1: numpy compares in f64 (search.py:82)
    assert oracle.list_cutoff(np.array([0.1], np.float32), 0.1) == 0
