"""GPU parity of the representative-sharded exact search (distributed.py), on one device.

P shard indices (rbc_index_exact_create_shard with the LPT plan) are searched
one after another on cuda:0 and their local key rows merged by the on-device
P-way merge, which is exactly what the ranks of a P-GPU job do around their
all_gather.  The result must equal the unsharded search and the oracle, and
the per-shard candidate counts must sum to the unsharded counts.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rbc():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1103_2635_b200 as m

    return m


@pytest.mark.parametrize("d,kind,k,world", [(64, "l2", 1, 2), (64, "l2", 10, 8), (54, "l2", 10, 4),
                                            (21, "l1", 3, 3), (128, "l2", 5, 8)])
def test_rep_sharded_search_equals_unsharded(rbc, oracle, d, kind, k, world):
    import torch

    from paper_1103_2635_b200 import _lib
    from paper_1103_2635_b200 import distributed as D

    n = 40_000
    full = oracle.gen_clusters(n + 700, d, 70 + d, n_clusters=16, cluster_sigma=0.05)
    x, q = full[:n], full[n:]
    idx = rbc.build_exact(rbc.DataMatrix(x), 200, rbc.MetricSpec(kind, d), seed=1)
    want = rbc.exact_query_arrays(idx, q, k)
    q_dev = _lib.to_device(q)
    parts, cands = [], []
    for r in range(world):
        sh = D.shard_exact_index(idx, r, world)
        assert sh.dev.nbytes < idx._dev.nbytes, "a shard must hold less than the full index"
        keys, (gamma, prr, p3, cand) = D.local_shard_keys(sh, q_dev, len(q), k)
        parts.append(keys)
        cands.append(_lib.to_host(cand))
        # stage 1 and pruning use every rep: identical on every shard
        assert np.array_equal(_lib.to_host(gamma), want[2])
        assert np.array_equal(_lib.to_host(prr), want[3]) and np.array_equal(_lib.to_host(p3), want[4])
    merged = D.device_merge_keys(torch.stack(parts), k) if world > 1 else parts[0]
    ids, dists = D.unpack_keys_host(_lib.to_host(merged))
    assert np.array_equal(ids, want[0]) and np.array_equal(dists, want[1])
    assert np.array_equal(np.sum(cands, axis=0), want[5])
    bi, bd = oracle.bf_topk(q, x, k, kind)
    assert np.array_equal(ids, bi) and np.array_equal(dists, bd)


def test_sharded_query_single_rank_api(rbc, oracle):
    """exact_query_sharded at world size 1 (no process group needed) equals exact_query_arrays."""
    import torch.distributed as dist

    from paper_1103_2635_b200 import distributed as D

    if dist.is_initialized():
        pytest.skip("process group already initialised")
    full = oracle.gen_clusters(20_000 + 300, 32, 5, n_clusters=8, cluster_sigma=0.05)
    x, q = full[:20_000], full[20_000:]
    import os

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        sh = D.build_exact_sharded(rbc.DataMatrix(x), 150, rbc.MetricSpec("l2", 32), 0, rank=0, world=1)
        got = D.exact_query_sharded(sh, q, 4)
        idx = rbc.build_exact(rbc.DataMatrix(x), 150, rbc.MetricSpec("l2", 32), seed=0)
        want = rbc.exact_query_arrays(idx, q, 4)
        for g, w in zip(got, want):
            assert np.array_equal(g, w)
    finally:
        dist.destroy_process_group()
