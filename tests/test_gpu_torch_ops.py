"""torch.ops.rbc_b200.* (torch_ext/rbc_torch_ops.cpp over the C-ABI): CUDA tensors in and out on
the current stream, the same bit-exact results as the numpy-level API and the oracle."""

import numpy as np
import pytest

from rbc_testutil import uniform

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1103_2635_b200 as rbc
    from paper_1103_2635_b200 import torch_ops

    torch_ops.load()
    return torch, rbc, torch_ops


@pytest.mark.parametrize("metric", ["l2", "l1"])
@pytest.mark.parametrize("k", [1, 7, 40])
def test_torch_bf_search(env, oracle, metric, k):
    torch, rbc, ops = env
    x = oracle.gen_clusters(5000, 24, 3, n_clusters=6, cluster_sigma=0.06)
    q = uniform(77, 24, 4)
    ids, dists = ops.bf_search(torch.from_numpy(q).cuda(), torch.from_numpy(x).cuda(), rbc.MetricSpec(metric, 24), k)
    assert ids.is_cuda and ids.dtype == torch.int64 and dists.dtype == torch.float32
    oi, od = oracle.bf_topk(q, x, k, metric)
    assert np.array_equal(ids.cpu().numpy(), oi) and np.array_equal(dists.cpu().numpy(), od)


def test_torch_pairwise(env, oracle):
    torch, rbc, ops = env
    a, b = uniform(33, 10, 1), uniform(57, 10, 2)
    for metric in ("l2", "l1"):
        out = ops.pairwise_distances(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), rbc.MetricSpec(metric, 10))
        assert np.array_equal(out.cpu().numpy(), oracle.pairwise(a, b, metric))


@pytest.mark.parametrize("k", [1, 10])
def test_torch_exact_search_matches_api(env, oracle, k):
    torch, rbc, ops = env
    full = oracle.gen_clusters(40_000 + 2000, 32, 8, n_clusters=16, cluster_sigma=0.05)
    x, q = full[:40_000], full[40_000:]
    idx = rbc.build_exact(rbc.DataMatrix(x), 200, rbc.MetricSpec("l2", 32), seed=1)
    got = ops.exact_search(idx, torch.from_numpy(q).cuda(), k)
    want = rbc.exact_query_arrays(idx, q, k)
    for g, w in zip(got, want):
        assert np.array_equal(g.cpu().numpy().astype(np.asarray(w).dtype), np.asarray(w))
    li, off, ld, radii = oracle.build_exact(x, idx.reps.rep_ids)
    oi, od = oracle.exact_query(x, idx.reps.rep_ids, li, off, ld, radii, q, k)[:2]
    assert np.array_equal(got[0].cpu().numpy(), oi) and np.array_equal(got[1].cpu().numpy(), od)


def test_torch_one_shot_search_matches_api(env, oracle):
    torch, rbc, ops = env
    x = oracle.gen_clusters(30_000, 21, 9, n_clusters=8, cluster_sigma=0.05)
    q = oracle.gen_clusters(3_000, 21, 10, n_clusters=8, cluster_sigma=0.05)
    idx = rbc.build_one_shot(rbc.DataMatrix(x), 150, 150, rbc.MetricSpec("l1", 21), seed=3)
    got = ops.one_shot_search(idx, torch.from_numpy(q).cuda(), 3)
    want = rbc.one_shot_query_arrays(idx, q, 3)
    for g, w in zip(got, want):
        assert np.array_equal(g.cpu().numpy(), np.asarray(w))


def test_torch_ops_errors(env):
    torch, rbc, ops = env
    q = torch.zeros((4, 3), device="cuda")
    with pytest.raises(RuntimeError, match="same d"):
        ops.bf_search(q, torch.zeros((9, 4), device="cuda"), 0, 1)
    with pytest.raises(RuntimeError, match="float32"):
        ops.bf_search(q.double(), torch.zeros((9, 3), device="cuda", dtype=torch.float64), 0, 1)
    with pytest.raises(RuntimeError):
        ops.bf_search(q, torch.zeros((9, 3), device="cuda"), 0, 10)  # k > n (C-ABI EINVAL)
