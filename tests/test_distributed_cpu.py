"""Multi-rank host logic of paper_1103_2635_b200.distributed on CPU (gloo, world size 2).

The per-shard top-k rows are produced by the oracle (the checker) over each
rank's owned lists; the code under test is the plan (LPT rep sharding, query
slices) and the collective merge (all_reduce MIN for k = 1, all_gather + P-way
merge for k > 1, SUM of candidate counts, row all-gather of query shards).
The merged result must equal the oracle's brute force over all of X, i.e. the
unsharded exact search (exact RBC == brute force, SPEC acceptance criterion 1).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1103_2635_b200 import distributed as D


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _np_merge(stacked, k):
    """Checker-side P-way merge: the k smallest uint64 keys per row (empty = UINT64_MAX sorts last)."""
    a = stacked.numpy().view(np.uint64)
    rows = np.sort(np.concatenate(list(a), axis=1), axis=1)[:, :k]
    return torch.from_numpy(rows.view(np.int64).copy())


def _pack(ids, dists):
    bits = np.ascontiguousarray(dists, np.float32).view(np.uint32).astype(np.uint64)
    keys = (bits << np.uint64(32)) | ids.astype(np.uint64)
    keys[ids < 0] = np.uint64(0xFFFFFFFFFFFFFFFF)
    return keys.view(np.int64)


def _worker(rank, world, port, k, result_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as orc

        full = orc.gen_clusters(2_000 + 64, 8, 11, n_clusters=6, cluster_sigma=0.05)
        x, q = full[:2_000], full[2_000:]
        reps = orc.bernoulli(2_000, 40 / 2_000, 0)
        li, off, _, _ = orc.build_exact(x, reps)
        sizes = np.diff(off)
        plan = D.rep_shard_plan(sizes, world)
        owned = np.concatenate([li[off[p]: off[p + 1]] for p in range(len(sizes)) if plan[p] == rank])
        kk = min(k, len(owned))
        ids, dists = orc.bf_subsets(q, x, np.tile(owned, len(q)), np.arange(len(q) + 1) * len(owned), kk)
        ids = np.asarray(ids).reshape(len(q), kk)
        dists = np.asarray(dists).reshape(len(q), kk)
        if kk < k:  # shard with fewer than k points: pad with empty entries
            ids = np.concatenate([ids, -np.ones((len(q), k - kk), np.int64)], axis=1)
            dists = np.concatenate([dists, np.full((len(q), k - kk), np.inf, np.float32)], axis=1)
        local = torch.from_numpy(_pack(ids, dists))
        merged = D.merge_shard_keys(local, k, merge_fn=_np_merge)
        cand = torch.tensor([len(owned)], dtype=torch.int64)
        D.sum_over_ranks(cand)
        lo, hi = D.query_slices(len(q), world)[rank]
        rows = torch.arange(lo, hi, dtype=torch.int64)[:, None] * 10
        gathered = D.gather_query_shards(rows, len(q))
        np.savez(os.path.join(result_dir, f"r{rank}.npz"), keys=merged.numpy(), cand=cand.numpy(),
                 rows=gathered.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("k", [1, 5])
def test_rep_sharded_merge_equals_unsharded(tmp_path, k, oracle):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), k, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    full = oracle.gen_clusters(2_000 + 64, 8, 11, n_clusters=6, cluster_sigma=0.05)
    x, q = full[:2_000], full[2_000:]
    want_ids, want_d = oracle.bf_topk(q, x, k)
    want = _pack(np.asarray(want_ids).reshape(len(q), k), np.asarray(want_d).reshape(len(q), k))
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        assert np.array_equal(z["keys"], want), f"rank {r}: merged keys differ from brute force"
        assert int(z["cand"][0]) == 2_000, "candidate counts must sum to the union of the shards"
        assert np.array_equal(z["rows"][:, 0], np.arange(len(q)) * 10), "query-shard all-gather out of order"
        ids, dists = D.unpack_keys_host(z["keys"])
        assert np.array_equal(ids, np.asarray(want_ids).reshape(len(q), k))
        assert np.array_equal(dists, np.asarray(want_d).reshape(len(q), k))


def test_query_slices_cover_and_balance():
    for nq in (0, 1, 7, 100_000, 100_003):
        for world in (1, 2, 3, 8):
            sl = D.query_slices(nq, world)
            assert sl[0][0] == 0 and sl[-1][1] == nq
            assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
            sizes = [hi - lo for lo, hi in sl]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        D.query_slices(10, 0)


def test_rep_shard_plan_lpt():
    rng = np.random.default_rng(3)
    sizes = rng.integers(0, 8_000, size=1016)
    for world in (1, 2, 4, 8):
        plan = D.rep_shard_plan(sizes, world)
        assert plan.shape == sizes.shape and set(np.unique(plan)) <= set(range(world))
        load = np.bincount(plan, weights=sizes, minlength=world)
        # LPT bound: max load <= mean + largest item
        assert load.max() <= sizes.sum() / world + sizes.max()
        assert np.array_equal(plan, D.rep_shard_plan(sizes, world)), "plan must be deterministic"
        masks = sum(D.owned_mask(plan, r).astype(int) for r in range(world))
        assert np.all(masks == 1), "every list is owned by exactly one shard"


def test_unpack_keys_host_roundtrip():
    ids = np.array([[0, 5, -1]], np.int64)
    dists = np.array([[0.0, 1.5, np.inf]], np.float32)
    got_ids, got_d = D.unpack_keys_host(_pack(ids, dists))
    assert np.array_equal(got_ids, ids) and np.array_equal(got_d, dists)


def _build_worker(rank, world, port, result_dir):
    """Sharded-build host logic: slice assignment (oracle), size all-reduce, LPT plan, all-to-all of
    (id, owner, dist, row) to the owner shard, radii all-reduce(MAX)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as orc

        x = orc.gen_clusters(3_001, 6, 17, n_clusters=5, cluster_sigma=0.05)
        reps = orc.bernoulli(3_001, 60 / 3_001, 1)
        lo, hi = D.query_slices(x.shape[0], world)[rank]
        xl = x[lo:hi]
        rows = torch.zeros((len(reps), 6), dtype=torch.float32)
        mine = np.flatnonzero((reps >= lo) & (reps < hi))
        rows[torch.as_tensor(mine)] = torch.from_numpy(xl[reps[mine] - lo])
        dist.all_reduce(rows, op=dist.ReduceOp.SUM)
        own, dd = orc.bf_topk(xl, rows.numpy(), 1)
        owner = torch.from_numpy(np.asarray(own).reshape(-1).astype(np.int64))
        dists = torch.from_numpy(np.asarray(dd).reshape(-1).astype(np.float32))
        sizes = torch.bincount(owner, minlength=len(reps)).to(torch.int64)
        dist.all_reduce(sizes, op=dist.ReduceOp.SUM)
        plan = D.rep_shard_plan(sizes.numpy(), world)
        ids = torch.arange(lo, hi, dtype=torch.int64)
        r_ids, r_owner, r_dist, r_rows = D.exchange_to_owners(ids, owner, dists, torch.from_numpy(xl), plan)
        radii = torch.zeros(len(reps), dtype=torch.float32)
        radii.scatter_reduce_(0, r_owner, r_dist, reduce="amax")
        dist.all_reduce(radii, op=dist.ReduceOp.MAX)
        np.savez(os.path.join(result_dir, f"b{rank}.npz"), ids=r_ids.numpy(), owner=r_owner.numpy(),
                 dist=r_dist.numpy(), rows=r_rows.numpy(), radii=radii.numpy(), plan=plan, sizes=sizes.numpy())
    finally:
        dist.destroy_process_group()


def test_sharded_build_exchange_equals_single_build(tmp_path, oracle):
    world = 2
    mp.start_processes(_build_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    x = oracle.gen_clusters(3_001, 6, 17, n_clusters=5, cluster_sigma=0.05)
    reps = oracle.bernoulli(3_001, 60 / 3_001, 1)
    li, off, ld, radii = oracle.build_exact(x, reps)
    seen = np.zeros(x.shape[0], np.int64)
    for r in range(world):
        z = np.load(tmp_path / f"b{r}.npz")
        assert np.array_equal(z["sizes"], np.diff(off)), "global list sizes"
        assert np.array_equal(z["radii"], radii), "all-reduced radii equal the single build's"
        assert np.all(np.diff(z["ids"]) > 0), "entries must arrive in increasing id order"
        assert np.array_equal(z["rows"], x[z["ids"]]), "rows travel with their ids"
        assert np.all(z["plan"][z["owner"]] == r), "every received entry belongs to this shard"
        # the local stable sort (rbc_index_exact_create_local) = lexsort((id, dist, owner))
        o = np.lexsort((z["ids"], z["dist"], z["owner"]))
        for p in np.flatnonzero(z["plan"] == r):
            sel = z["owner"][o] == p
            assert np.array_equal(z["ids"][o][sel], li[off[p]: off[p + 1]]), f"list {p} ids"
            assert np.array_equal(z["dist"][o][sel], ld[off[p]: off[p + 1]]), f"list {p} dists"
        seen[z["ids"]] += 1
    assert np.all(seen == 1), "every point lands on exactly one shard"
