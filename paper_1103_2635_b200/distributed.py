"""Multi-GPU RBC search: query sharding and representative sharding.

One process per GPU (torch.distributed, backend "nccl" on B200s, "gloo" in the
CPU tests).  Two layouts, both results-identical to the single-GPU search:

* **Query sharding** (cfg2/cfg3).  Every rank holds the whole index (the build
  is deterministic, so each rank builds it redundantly -- no broadcast) and
  searches a contiguous slice of the queries.  The query loop has no
  collective; ``gather_query_shards`` exists only for callers that want every
  rank to see the full result.
* **Representative sharding** (cfg5; the paper's proposed distribution,
  PAPER.md:909-916).  Every rank keeps all representatives and radii, so
  stage 1, gamma_k and the pruning are identical everywhere, but only the
  ownership lists of its shard (a longest-processing-time assignment of reps
  by list length).  Each rank scans its surviving local lists and produces a
  local top-k of key64 = (f32 bits(dist) << 32) | id; the exact global top-k
  is the k smallest keys over the ranks:
    - k = 1: one ``all_reduce(MIN)`` on the int64 keys (key64 order is the
      reference's (distance, id) order, so MIN is the exact merge);
    - k > 1: ``all_gather`` of the [nq, k] key rows and an on-device P-way
      merge (``rbc_merge_topk``).
  ``candidates_examined`` is summed with ``all_reduce(SUM)``; gamma and the
  pruned counts are computed from all reps on every rank, so they are equal.

The collective steps take plain torch tensors so the same code runs on NCCL
(CUDA tensors) and on gloo (CPU tensors, tests/test_distributed_cpu.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib

EMPTY_KEY = -1                      # UINT64_MAX reinterpreted as int64 (library "no entry")
MAX_KEY = np.iinfo(np.int64).max    # its stand-in for MIN reductions


# ---- plans (host logic) ------------------------------------------------------
def query_slices(nq: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, balanced [lo, hi) query slices, one per rank (sizes differ by at most 1)."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    if nq < 0:
        raise ValueError("nq must be >= 0")
    base, extra = divmod(nq, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def rep_shard_plan(list_sizes, world: int) -> np.ndarray:
    """Shard of every representative: LPT on ownership-list length (SURVEY §7 hard part 7).

    Lists are taken longest first (ties: lower rep position first) and each goes
    to the currently lightest shard (ties: lower rank).  Deterministic, so every
    rank computes the same plan without communication.
    """
    sizes = np.asarray(list_sizes, dtype=np.int64).reshape(-1)
    if world < 1:
        raise ValueError("world size must be >= 1")
    order = np.lexsort((np.arange(sizes.size), -sizes))
    load = np.zeros(world, dtype=np.int64)
    owner = np.empty(sizes.size, dtype=np.int32)
    for p in order:
        r = int(np.argmin(load))  # argmin returns the lowest rank on ties
        owner[p] = r
        load[r] += sizes[p]
    return owner


def owned_mask(plan: np.ndarray, rank: int) -> np.ndarray:
    return (np.asarray(plan) == rank).astype(np.uint8)


def unpack_keys_host(keys: np.ndarray):
    """key64 rows -> (ids int64, dists float32); empty entries -> (-1, +inf) (brute_force.py:71-74)."""
    k = np.ascontiguousarray(keys).view(np.uint64)
    ids = (k & np.uint64(0xFFFFFFFF)).astype(np.int64)
    dists = (k >> np.uint64(32)).astype(np.uint32).view(np.float32)
    empty = k == np.uint64(0xFFFFFFFFFFFFFFFF)
    ids[empty] = -1
    dists = dists.copy()
    dists[empty] = np.inf
    return ids, dists


# ---- collectives -------------------------------------------------------------
def _dist():
    import torch.distributed as dist

    return dist


def _world(group=None) -> int:
    """World size of the group, 1 when no process group is initialised (single process)."""
    dist = _dist()
    return dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1


def merge_shard_keys(local_keys, k: int, group=None, merge_fn=None):
    """Exact global top-k from every rank's local top-k key rows.

    ``local_keys``: int64 tensor [nq, k] (EMPTY_KEY = no entry), on the rank's
    device.  Returns the merged int64 key tensor [nq, k] on every rank.
    ``merge_fn(stacked [P, nq, k] int64 tensor, k) -> [nq, k]`` performs the
    P-way merge for k > 1 (default: the on-device ``rbc_merge_topk``).
    """
    dist = _dist()
    world = _world(group)
    if world == 1:
        return local_keys
    if k == 1:
        keys = local_keys.clone()
        keys[keys == EMPTY_KEY] = MAX_KEY
        dist.all_reduce(keys, op=dist.ReduceOp.MIN, group=group)
        keys[keys == MAX_KEY] = EMPTY_KEY
        return keys
    gathered = [local_keys.new_empty(local_keys.shape) for _ in range(world)]
    dist.all_gather(gathered, local_keys.contiguous(), group=group)
    import torch

    stacked = torch.stack(gathered)
    return (merge_fn or device_merge_keys)(stacked, k)


def device_merge_keys(stacked, k: int):
    """P-way merge of key rows on the GPU (rbc_merge_topk), returned as packed keys."""
    t = _lib.require_cuda()
    parts, nq, k_in = stacked.shape
    ids = _lib.empty((nq, k), t.int64)
    dists = _lib.empty((nq, k), t.float32)
    _lib.check(_lib.lib.rbc_merge_topk(_lib.ptr(stacked.contiguous()), parts, nq, k_in, k, _lib.ptr(ids),
                                       _lib.ptr(dists), _lib.stream_ptr()), "merge_topk")
    bits = dists.view(t.int32).to(t.int64) & 0xFFFFFFFF
    keys = (bits << 32) | (ids & 0xFFFFFFFF)
    keys[ids < 0] = EMPTY_KEY
    return keys


def sum_over_ranks(tensor, group=None):
    dist = _dist()
    if _world(group) > 1:
        dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=group)
    return tensor


def gather_query_shards(local, nq: int, group=None):
    """All-gather per-rank query-slice results (rows) into the full [nq, ...] tensor on every rank."""
    dist = _dist()
    world = _world(group)
    if world == 1:
        return local
    sl = query_slices(nq, world)
    width = max(hi - lo for lo, hi in sl)
    pad = local.new_zeros((width,) + tuple(local.shape[1:]))
    pad[: local.shape[0]] = local
    parts = [pad.new_empty(pad.shape) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    import torch

    return torch.cat([p[: hi - lo] for p, (lo, hi) in zip(parts, sl)])


# ---- sharded exact index -----------------------------------------------------
@dataclass
class ShardedExactIndex:
    """One rank's representative shard of an exact index (all reps, the owned lists)."""

    index: object          # the full RbcExactIndex (host arrays), or None after a sharded build
    plan: np.ndarray       # shard of every rep position
    rank: int
    world: int
    dev: object = None     # DeviceIndex of the shard
    list_sizes: np.ndarray = None  # global list length of every rep
    rep_ids: np.ndarray = None
    radii: np.ndarray = None
    metric: object = None

    def __post_init__(self):
        if self.index is not None:
            if self.list_sizes is None:
                self.list_sizes = np.array([len(a) for a in self.index.list_ids], np.int64)
            if self.rep_ids is None:
                self.rep_ids = self.index.reps.rep_ids
            if self.radii is None:
                self.radii = np.asarray(self.index.radii, np.float32)
            if self.metric is None:
                self.metric = self.index.metric

    @property
    def n_reps(self) -> int:
        return int(len(self.rep_ids))

    @property
    def owned_points(self) -> int:
        return int(np.asarray(self.list_sizes)[self.plan == self.rank].sum())


def shard_exact_index(index, rank: int, world: int) -> ShardedExactIndex:
    """Device shard of a built exact index: rbc_index_exact_create_shard with this rank's lists."""
    from .rbc import _create_exact_device

    sizes = [len(a) for a in index.list_ids]
    plan = rep_shard_plan(sizes, world)
    spec = index.metric
    ids, offsets, dists = index.flat_lists()
    dev = _create_exact_device(_lib.to_device(index.data.values), index.data.n, spec,
                               _lib.to_device(index.reps.rep_ids), index.reps.size, _lib.to_device(ids),
                               _lib.to_device(offsets), _lib.to_device(dists),
                               _lib.to_device(np.asarray(index.radii, np.float32)), owned=owned_mask(plan, rank))
    return ShardedExactIndex(index, plan, rank, world, dev)


def build_exact_sharded(data, n_r, spec, seed, rank: int, world: int, **kw) -> ShardedExactIndex:
    """Build the exact index (deterministic, so every rank builds the same one) and keep this rank's shard."""
    from .rbc import build_exact

    index = build_exact(data, n_r, spec, seed, **kw)
    sh = shard_exact_index(index, rank, world)
    index._dev = None  # drop the full device copy; the shard is what this rank searches
    return sh


def exchange_to_owners(ids, owner, dist, rows, plan, group=None):
    """All-to-all of assignment entries to the rank that owns their representative.

    ``ids`` int64 [m], ``owner`` int64 [m] (rep positions), ``dist`` float32 [m], ``rows``
    float32 [m, d]: torch tensors on the collective's device (CUDA for NCCL, CPU for gloo).
    Each source sends its entries for a destination in their local order (a stable
    partition), and the received blocks are concatenated in source-rank order -- so with
    contiguous ascending id slices per rank the received entries are in increasing id
    order, which the local stable sort relies on (rbc_index_exact_create_local).
    Returns the received (ids, owner, dist, rows).
    """
    import torch

    dist_ = _dist()
    world = dist_.get_world_size(group)
    plan_t = torch.as_tensor(np.asarray(plan, np.int64), device=owner.device)
    dest = plan_t[owner]
    order = torch.sort(dest, stable=True).indices
    send = torch.bincount(dest, minlength=world).to(torch.int64)
    recv = torch.empty_like(send)
    dist_.all_to_all_single(recv, send, group=group)
    sc, rc = send.tolist(), recv.tolist()

    def a2a(t):
        out = t.new_empty((sum(rc),) + tuple(t.shape[1:]))
        dist_.all_to_all_single(out, t[order].contiguous(), rc, sc, group=group)
        return out

    return a2a(ids), a2a(owner), a2a(dist), a2a(rows)


def build_exact_distributed(x_local, id_lo: int, n_total: int, n_r: int, spec, seed: int, rank: int, world: int,
                            group=None, mode: str = "bernoulli", rep_ids=None) -> ShardedExactIndex:
    """Sharded exact build: each rank holds only its id slice
    x_local = X[id_lo : id_lo + m] and ends with the ownership lists of its rep shard.

    1. every rank draws the same representatives (rbc.py:62-84) and all-reduces their rows;
    2. each rank assigns its slice to the nearest representative (the tcgen05 brute force of
       every point over the reps: rbc.py:164);
    3. list sizes all-reduce(SUM) -> the same LPT rep-shard plan on every rank;
    4. all-to-all of (id, owner, dist, row) to the owning rank;
    5. list radii: local max, all-reduce(MAX) (rbc.py:172-175);
    6. the received entries become the shard's lists (stable radix sort on (owner, dist)).
    Per-rank device memory holds the slice and the shard, about 2/P of the points.
    The concatenated shard lists equal the single-GPU build's lists, bit for bit.
    """
    import torch

    from .rbc import _resolve_reps, DeviceIndex

    dist_ = _dist()
    t = _lib.require_cuda()
    xl = _lib.to_device(np.ascontiguousarray(x_local, np.float32))
    m, d = int(xl.shape[0]), int(xl.shape[1])
    if d != spec.dim:
        raise ValueError(f"dimension mismatch: data d={d}, metric dim={spec.dim}")
    reps = _resolve_reps(n_total, n_r, seed, mode, rep_ids)
    rid = np.asarray(reps.rep_ids, np.int64)
    nr = int(rid.size)
    rid_dev = _lib.to_device(rid)
    # 1. representative rows: each rep row is contributed by the one rank whose slice holds it
    rows = torch.zeros((nr, d), dtype=torch.float32, device="cuda")
    mine = np.flatnonzero((rid >= id_lo) & (rid < id_lo + m))
    if mine.size:
        rows[torch.as_tensor(mine, device="cuda")] = xl[torch.as_tensor(rid[mine] - id_lo, device="cuda")]
    if world > 1:
        dist_.all_reduce(rows, op=dist_.ReduceOp.SUM, group=group)
    # 2. nearest representative of every local point (key64 argmin: lowest position on ties)
    owner = torch.empty((m, 1), dtype=torch.int64, device="cuda")
    dists = torch.empty((m, 1), dtype=torch.float32, device="cuda")
    if m:
        _lib.check(_lib.lib.rbc_bf_search(_lib.ptr(xl), m, _lib.ptr(rows), nr, d, spec.code, 1, _lib.ptr(owner),
                                          _lib.ptr(dists), _lib.stream_ptr()), "shard assignment")
    owner, dists = owner.view(-1), dists.view(-1)
    # 3. global list sizes -> plan
    sizes = torch.bincount(owner, minlength=nr).to(torch.int64)
    if world > 1:
        dist_.all_reduce(sizes, op=dist_.ReduceOp.SUM, group=group)
    sizes_h = _lib.to_host(sizes)
    plan = rep_shard_plan(sizes_h, world)
    # 4. entries to their owner shard
    ids = torch.arange(id_lo, id_lo + m, dtype=torch.int64, device="cuda")
    if world > 1:
        ids, owner, dists, xl = exchange_to_owners(ids, owner, dists, xl, plan, group)
    # 5. radii
    radii = torch.empty(nr, dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib.rbc_local_list_radii(_lib.ptr(owner), _lib.ptr(dists), int(owner.numel()), nr,
                                             _lib.ptr(radii), _lib.stream_ptr()), "list radii")
    if world > 1:
        dist_.all_reduce(radii, op=dist_.ReduceOp.MAX, group=group)
    # 6. the shard index
    handle = ctypes.c_void_p()
    _lib.check(_lib.lib.rbc_index_exact_create_local(_lib.ptr(rows), _lib.ptr(rid_dev), nr, _lib.ptr(radii), n_total, d,
                                                     spec.code, _lib.ptr(xl), _lib.ptr(ids), _lib.ptr(owner),
                                                     _lib.ptr(dists), int(owner.numel()), ctypes.byref(handle),
                                                     _lib.stream_ptr()), "shard index create")
    dev = DeviceIndex(handle, t.cuda.current_device())
    return ShardedExactIndex(None, plan, rank, world, dev, list_sizes=sizes_h, rep_ids=rid,
                             radii=_lib.to_host(radii), metric=spec)


def local_shard_keys(sh: ShardedExactIndex, q_dev, nq: int, k: int):
    """This rank's local top-k key rows [nq, k] (int64, EMPTY_KEY = none) and search stats tensors."""
    t = _lib.require_cuda()
    keys = _lib.empty((nq, k), t.int64)
    gamma = _lib.empty((nq,), t.float32)
    prr = _lib.empty((nq,), t.int32)
    p3 = _lib.empty((nq,), t.int32)
    cand = _lib.empty((nq,), t.int64)
    stats = _lib.SearchStatsC(gamma.data_ptr(), prr.data_ptr(), p3.data_ptr(), cand.data_ptr())
    _lib.check(_lib.lib.rbc_exact_search_keys(sh.dev.handle, _lib.ptr(q_dev), nq, k, _lib.ptr(keys), stats,
                                              _lib.stream_ptr()), "sharded exact search")
    return keys, (gamma, prr, p3, cand)


def exact_query_sharded(sh: ShardedExactIndex, queries, k: int = 1, group=None):
    """Exact k-NN over the rep-sharded index: local scan + key merge (same outputs as exact_query_arrays)."""
    from .search import _queries

    qv = _queries(queries)
    n_reps = sh.n_reps
    if not 1 <= k <= n_reps:
        raise ValueError(f"k must be in [1, |R|={n_reps}], got {k}")
    if qv.shape[1] != sh.metric.dim:
        raise ValueError(f"dimension mismatch: queries d={qv.shape[1]}, metric dim={sh.metric.dim}")
    nq = qv.shape[0]
    keys, (gamma, prr, p3, cand) = local_shard_keys(sh, _lib.to_device(qv), nq, k)
    merged = merge_shard_keys(keys, k, group)
    sum_over_ranks(cand, group)
    ids, dists = unpack_keys_host(_lib.to_host(merged))
    if nq and (ids < 0).any():
        bad = int(np.flatnonzero((ids < 0).any(axis=1))[0])
        raise ValueError(f"k must be in [1, {int(_lib.to_host(cand)[bad])}], got {k}")
    return ids, dists, _lib.to_host(gamma), _lib.to_host(prr), _lib.to_host(p3), _lib.to_host(cand)


def exact_query_qsharded(index, queries, k: int = 1, rank: int = 0, world: int = 1, group=None, gather=True):
    """Query-sharded exact search: this rank searches its slice; optionally all-gather the rows."""
    from .search import exact_query_arrays, _queries

    qv = _queries(queries)
    lo, hi = query_slices(qv.shape[0], world)[rank]
    out = exact_query_arrays(index, qv[lo:hi], k)
    if not gather or world == 1:
        return out
    t = _lib.torch()
    dev = "cuda" if t.cuda.is_available() else "cpu"
    full = []
    for a in out:
        ten = t.from_numpy(np.ascontiguousarray(a)).to(dev)
        full.append(_lib.to_host(gather_query_shards(ten, qv.shape[0], group)))
    return tuple(full)


__all__ = [
    "ShardedExactIndex", "build_exact_distributed", "build_exact_sharded", "exchange_to_owners", "exact_query_qsharded", "exact_query_sharded",
    "gather_query_shards", "merge_shard_keys", "owned_mask", "query_slices", "rep_shard_plan",
    "shard_exact_index", "unpack_keys_host",
]
