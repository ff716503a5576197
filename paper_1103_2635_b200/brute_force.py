"""The brute-force primitive BF(Q, X) on the GPU (reference brute_force.py).

``bf_search`` / ``bf_search_subset`` / ``distance_rows`` /
``merge_neighbor_lists`` keep the reference signatures, validation and return
types; the work runs in the sm_100a kernels behind the C-ABI.  ``workers`` and
the tile sizes are accepted for compatibility and do not change results (the
reference guarantees the same, brute_force.py:8-12).
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .dataset import _as_values
from .metric import MetricSpec, _pairwise_device

DEFAULT_TILE_QUERIES = 256
DEFAULT_TILE_POINTS = 1024
MAX_WARP_K = 64


def resolve_workers(workers: int | None) -> int:
    if workers is None:
        return os.cpu_count() or 1
    if workers < 1:
        raise ValueError("workers must be >= 1")
    return workers


@dataclass
class NeighborList:
    """k nearest points for one query: ids ascending by (distance, id)."""

    query_id: int
    ids: np.ndarray
    dists: np.ndarray

    @property
    def k(self) -> int:
        return len(self.ids)


@dataclass
class BruteForceResult:
    """Search output plus the exact number of distance evaluations spent."""

    neighbors: list[NeighborList] = field(default_factory=list)
    distance_evals: int = 0


def _pack_keys(dists: np.ndarray, ids: np.ndarray) -> np.ndarray:
    bits = np.ascontiguousarray(dists, dtype=np.float32).view(np.uint32).astype(np.uint64)
    return (bits << np.uint64(32)) | np.asarray(ids).astype(np.uint64)


def _check_dims(qv: np.ndarray, xv: np.ndarray, spec: MetricSpec) -> None:
    if qv.ndim != 2 or xv.ndim != 2:
        raise ValueError("expected 2-D query and database arrays")
    if qv.shape[1] != spec.dim or xv.shape[1] != spec.dim:
        raise ValueError(
            f"dimension mismatch: queries d={qv.shape[1]}, database d={xv.shape[1]}, metric dim={spec.dim}"
        )


def _rows(ids: np.ndarray, dists: np.ndarray, base: int = 0) -> list[NeighborList]:
    return [NeighborList(base + q, ids[q], dists[q]) for q in range(ids.shape[0])]


def bf_search_arrays(qv: np.ndarray, xv: np.ndarray, spec: MetricSpec, k: int, x_dev=None):
    """(ids[nq,k] int64, dists[nq,k] float32) of the exhaustive scan."""
    t = _lib.require_cuda()
    nq, n = qv.shape[0], xv.shape[0]
    q_dev = _lib.to_device(qv)
    x_dev = _lib.to_device(xv) if x_dev is None else x_dev
    ids = _lib.empty((nq, k), t.int64)
    dists = _lib.empty((nq, k), t.float32)
    _lib.check(_lib.lib.rbc_bf_search(_lib.ptr(q_dev), nq, _lib.ptr(x_dev), n, spec.dim, spec.code, k,
                                      _lib.ptr(ids), _lib.ptr(dists), _lib.stream_ptr()), "bf_search")
    return _lib.to_host(ids), _lib.to_host(dists)


def bf_search(
    queries,
    data,
    spec: MetricSpec,
    k: int,
    workers: int | None = None,
    tile_queries: int = DEFAULT_TILE_QUERIES,
    tile_points: int = DEFAULT_TILE_POINTS,
) -> BruteForceResult:
    """Exact k nearest neighbours of every query by exhaustive scan (brute_force.py:165-186)."""
    qv = _as_values(queries)
    xv = _as_values(data)
    _check_dims(qv, xv, spec)
    if not 1 <= k <= xv.shape[0]:
        raise ValueError(f"k must be in [1, {xv.shape[0]}], got {k}")
    if workers is not None:
        resolve_workers(workers)
    if qv.shape[0] == 0:
        return BruteForceResult([], 0)
    ids, dists = bf_search_arrays(qv, xv, spec, k)
    return BruteForceResult(_rows(ids, dists), qv.shape[0] * xv.shape[0])


def bf_search_subset(q, data, subset_ids, spec: MetricSpec, k: int) -> BruteForceResult:
    """Exact k-NN of one query restricted to the listed rows (brute_force.py:189-217)."""
    qv = np.asarray(q, dtype=np.float32).reshape(1, -1)
    xv = _as_values(data)
    _check_dims(qv, xv, spec)
    ids = np.asarray(subset_ids, dtype=np.int64).reshape(-1)
    if ids.size == 0:
        raise ValueError("subset id list is empty")
    if ids.min() < 0 or ids.max() >= xv.shape[0]:
        raise ValueError("subset id out of range")
    if np.unique(ids).size != ids.size:
        raise ValueError("duplicate id in subset list")
    if not 1 <= k <= ids.size:
        raise ValueError(f"k must be in [1, {ids.size}], got {k}")
    t = _lib.require_cuda()
    q_dev = _lib.to_device(qv)
    if k <= MAX_WARP_K:
        x_dev = _lib.to_device(xv)
        sid = _lib.to_device(ids)
        off = _lib.to_device(np.array([0, ids.size], np.int64))
        out_ids = _lib.empty((1, k), t.int64)
        out_d = _lib.empty((1, k), t.float32)
        _lib.check(_lib.lib.rbc_bf_search_subsets(_lib.ptr(q_dev), 1, _lib.ptr(x_dev), xv.shape[0], spec.dim,
                                                  spec.code, k, _lib.ptr(sid), _lib.ptr(off), _lib.ptr(out_ids),
                                                  _lib.ptr(out_d), _lib.stream_ptr()), "bf_search_subset")
        r_ids, r_d = _lib.to_host(out_ids)[0], _lib.to_host(out_d)[0]
    else:
        # large k: scan the gathered rows, then map local positions to global ids
        sub = np.ascontiguousarray(xv[ids])
        loc, r_d = bf_search_arrays(qv, sub, spec, k)
        r_ids, r_d = ids[loc[0]], r_d[0]
    return BruteForceResult([NeighborList(0, r_ids, r_d)], ids.size)


def distance_rows(
    queries,
    data,
    spec: MetricSpec,
    workers: int | None = None,
    tile_queries: int = DEFAULT_TILE_QUERIES,
    tile_points: int = DEFAULT_TILE_POINTS,
) -> np.ndarray:
    """Full |queries| x |data| float32 distance matrix (brute_force.py:220-251)."""
    qv = _as_values(queries)
    xv = _as_values(data)
    _check_dims(qv, xv, spec)
    if qv.shape[0] == 0 or xv.shape[0] == 0:
        return np.empty((qv.shape[0], xv.shape[0]), np.float32)
    out = _pairwise_device(_lib.to_device(qv), qv.shape[0], _lib.to_device(xv), xv.shape[0], spec)
    return _lib.to_host(out)


def merge_neighbor_lists(a: NeighborList, b: NeighborList, k: int) -> NeighborList:
    """Merge two partial results over disjoint id sets into the best k (brute_force.py:97-106)."""
    t = _lib.require_cuda()
    keys = np.concatenate((_pack_keys(a.dists, a.ids), _pack_keys(b.dists, b.ids)))
    width = len(keys)
    kk = min(k, width)
    if kk == 0:
        return NeighborList(a.query_id, np.empty(0, np.int64), np.empty(0, np.float32))
    keys_dev = _lib.to_device(keys.view(np.int64))
    ids = _lib.empty((1, kk), t.int64)
    dists = _lib.empty((1, kk), t.float32)
    _lib.check(_lib.lib.rbc_merge_topk(_lib.ptr(keys_dev), 1, 1, width, kk, _lib.ptr(ids), _lib.ptr(dists),
                                       _lib.stream_ptr()), "merge_neighbor_lists")
    return NeighborList(a.query_id, _lib.to_host(ids)[0], _lib.to_host(dists)[0])
