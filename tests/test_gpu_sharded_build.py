"""GPU parity of the sharded build.

build_exact_distributed at world size 1, and a P-shard simulation on one GPU: every
"rank" assigns its id slice with the tensor-core brute force, the entries are routed to
the owner shard as the all-to-all would deliver them (ascending ids, rank order), each
shard becomes an index through rbc_index_exact_create_local, and the per-shard top-k
rows merged with rbc_merge_topk must equal the unsharded search and the oracle.
(The collective exchange itself is tested with gloo at world size 2 in
tests/test_distributed_cpu.py.)
"""

import ctypes

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


def test_build_exact_distributed_world1(rbc, oracle):
    from paper_1103_2635_b200 import distributed as D

    full = oracle.gen_clusters(120_000 + 1_000, 64, 9, n_clusters=16, cluster_sigma=0.05)
    x, q = full[:120_000], full[120_000:]
    spec = rbc.MetricSpec("l2", 64)
    sh = D.build_exact_distributed(x, 0, x.shape[0], 346, spec, 0, 0, 1)
    idx = rbc.build_exact(rbc.DataMatrix(x), 346, spec, seed=0)
    assert np.array_equal(sh.rep_ids, idx.reps.rep_ids)
    assert np.array_equal(sh.radii, idx.radii)
    assert np.array_equal(sh.list_sizes, [len(a) for a in idx.list_ids])
    for k in (1, 10):
        got = D.exact_query_sharded(sh, q, k)
        want = rbc.exact_query_arrays(idx, q, k)
        for g, w in zip(got, want):
            assert np.array_equal(g, w)


def _shard_index(rbc, lib, rows_dev, rid_dev, nr, radii_dev, n, d, ent):
    import torch

    ids, owner, dist, xr = ent
    h = ctypes.c_void_p()
    t = [torch.from_numpy(a).cuda() for a in (ids, owner, dist, xr)]
    lib.check(lib.lib.rbc_index_exact_create_local(lib.ptr(rows_dev), lib.ptr(rid_dev), nr, lib.ptr(radii_dev), n, d,
                                                   0, lib.ptr(t[3]), lib.ptr(t[0]), lib.ptr(t[1]), lib.ptr(t[2]),
                                                   len(ids), ctypes.byref(h), lib.stream_ptr()), "create_local")
    from paper_1103_2635_b200.rbc import DeviceIndex

    return DeviceIndex(h, torch.cuda.current_device())


@pytest.mark.parametrize("P", [2, 4])
def test_sharded_build_simulation_cfg5_shape(rbc, oracle, P):
    import torch
    from paper_1103_2635_b200 import _lib
    from paper_1103_2635_b200 import distributed as D

    n, d, nq, k = 4_000_000, 128, 2_000, 10
    rng = np.random.default_rng(5)
    centers = rng.random((64, d))
    full = (centers[rng.integers(64, size=n + nq)] + 0.05 * rng.standard_normal((n + nq, d))).astype(np.float32)
    x, q = full[:n], full[n:]
    del full
    spec = rbc.MetricSpec("l2", d)
    idx = rbc.build_exact(rbc.DataMatrix(x), 2000, spec, seed=0)
    rid = idx.reps.rep_ids
    nr = rid.size
    rows = np.ascontiguousarray(x[rid])
    rows_dev, rid_dev = _lib.to_device(rows), _lib.to_device(rid)
    # every "rank" assigns its slice on the tensor cores
    parts = []
    for lo, hi in D.query_slices(n, P):
        o, dd = rbc.brute_force.bf_search_arrays(x[lo:hi], rows, spec, 1)
        parts.append((np.arange(lo, hi, dtype=np.int64), o.reshape(-1), dd.reshape(-1)))
    sizes = sum(np.bincount(p[1], minlength=nr) for p in parts)
    assert np.array_equal(sizes, [len(a) for a in idx.list_ids])
    plan = D.rep_shard_plan(sizes, P)
    radii = np.zeros(nr, np.float32)
    keys = []
    for r in range(P):
        # what the all-to-all delivers to rank r: each source's entries for r, sources in rank order
        sel = [(p[0][plan[p[1]] == r], p[1][plan[p[1]] == r], p[2][plan[p[1]] == r]) for p in parts]
        ids = np.concatenate([s[0] for s in sel])
        own = np.concatenate([s[1] for s in sel])
        dist = np.concatenate([s[2] for s in sel]).astype(np.float32)
        np.maximum.at(radii, own, dist)
        keys.append((ids, own, dist, np.ascontiguousarray(x[ids])))
    assert np.array_equal(radii, idx.radii)
    radii_dev = _lib.to_device(radii)
    q_dev = _lib.to_device(q)
    shard_keys = []
    for r in range(P):
        dev = _shard_index(rbc, _lib, rows_dev, rid_dev, nr, radii_dev, n, d, keys[r])
        kk = torch.empty((nq, k), dtype=torch.int64, device="cuda")
        _lib.check(_lib.lib.rbc_exact_search_keys(dev.handle, _lib.ptr(q_dev), nq, k, _lib.ptr(kk),
                                                  _lib.SearchStatsC(None, None, None, None), _lib.stream_ptr()),
                   "shard search")
        shard_keys.append(kk)
        del dev
    merged = D.device_merge_keys(torch.stack(shard_keys), k)
    ids, dists = D.unpack_keys_host(_lib.to_host(merged))
    want = rbc.exact_query_arrays(idx, q, k)
    assert np.array_equal(ids, want[0]) and np.array_equal(dists, want[1])
    oi, od = oracle.bf_topk(q[:48], x, k)
    assert np.array_equal(ids[:48], oi) and np.array_equal(dists[:48], od)
