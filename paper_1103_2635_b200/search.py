"""Query algorithms over a random ball cover index (reference search.py).

Both algorithms run end to end on the GPU: stage 1 (query x representative
distances), the float64 triangle-inequality pruning with the 4*gamma_k list
cutoff, and stage 2 (the k-NN scan of the surviving list prefixes).  Results
and every ``SearchStats`` field equal the reference's (the candidate set is
computed with the reference's exact comparisons).

``exact_query_arrays`` / ``one_shot_query_arrays`` return plain arrays; the
``*_batch`` functions wrap them in the reference's NeighborList / SearchStats
objects.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .brute_force import NeighborList, resolve_workers
from .rbc import RbcExactIndex, RbcOneShotIndex, device_index

MAX_K = None  # no cap: k > 64 runs the exact materialise-and-sort top-k (csrc/exact_kernels.cu topk_large)


@dataclass
class SearchStats:
    """Per-query instrumentation (search.py:43-59)."""

    gamma: float
    reps_total: int
    reps_pruned_radius: int
    reps_pruned_3gamma: int
    candidates_examined: int
    dists_step1: int


def prune_representatives(rep_dists: np.ndarray, radii: np.ndarray, gamma_k: float) -> np.ndarray:
    """Positions of representatives surviving both tests, in float64 (search.py:62-74)."""
    d = np.ascontiguousarray(rep_dists, dtype=np.float64).reshape(-1)
    r = np.ascontiguousarray(radii, dtype=np.float64).reshape(-1)
    if d.shape != r.shape:
        raise ValueError("rep_dists and radii must have the same length")
    if d.size == 0:
        return np.empty(0, np.int64)
    t = _lib.require_cuda()
    mask = _lib.empty((d.size,), t.uint8)
    d_dev, r_dev = _lib.to_device(d), _lib.to_device(r)  # keep alive until the kernel has run
    _lib.check(_lib.lib.rbc_prune_representatives(_lib.ptr(d_dev), _lib.ptr(r_dev), d.size, float(gamma_k),
                                                  _lib.ptr(mask), _lib.stream_ptr()), "prune")
    return np.flatnonzero(_lib.to_host(mask))


def list_cutoff(sorted_rep_dists: np.ndarray, threshold: float) -> int:
    """Leading entries of an ascending list that are <= threshold, f64 compare (search.py:77-82)."""
    a = np.ascontiguousarray(sorted_rep_dists, dtype=np.float64).reshape(-1)
    if a.size == 0:
        return 0
    t = _lib.require_cuda()
    out = _lib.empty((1,), t.int64)
    thr = _lib.to_device(np.array([np.float64(threshold)]))
    a_dev = _lib.to_device(a)
    _lib.check(_lib.lib.rbc_list_cutoff(_lib.ptr(a_dev), a.size, _lib.ptr(thr), 1, _lib.ptr(out),
                                        _lib.stream_ptr()), "list_cutoff")
    return int(_lib.to_host(out)[0])


def _queries(queries) -> np.ndarray:
    qv = np.asarray(getattr(queries, "values", queries), dtype=np.float32)
    if qv.ndim == 1:
        qv = qv[None, :]
    return np.ascontiguousarray(qv)


def exact_query_arrays(index: RbcExactIndex, queries, k: int = 1, q_dev=None):
    """ids[nq,k], dists[nq,k], gamma[nq], pruned_radius[nq], pruned_3gamma[nq], candidates[nq]."""
    qv = _queries(queries)
    n_reps = index.reps.size
    if not 1 <= k <= n_reps:
        raise ValueError(f"k must be in [1, |R|={n_reps}] so the stage-1 bound exists, got {k}")
    if k > index.data.n:
        raise ValueError(f"k={k} exceeds database size {index.data.n}")
    if qv.shape[1] != index.metric.dim:
        raise ValueError(f"dimension mismatch: queries d={qv.shape[1]}, metric dim={index.metric.dim}")
    t = _lib.require_cuda()
    dev = device_index(index)
    nq = qv.shape[0]
    if q_dev is None:
        q_dev = _lib.to_device(qv)
    ids = _lib.empty((nq, k), t.int64)
    dists = _lib.empty((nq, k), t.float32)
    gamma = _lib.empty((nq,), t.float32)
    prr = _lib.empty((nq,), t.int32)
    p3 = _lib.empty((nq,), t.int32)
    cand = _lib.empty((nq,), t.int64)
    stats = _lib.SearchStatsC(gamma.data_ptr(), prr.data_ptr(), p3.data_ptr(), cand.data_ptr())
    _lib.check(_lib.lib.rbc_exact_search(dev.handle, _lib.ptr(q_dev), nq, k, _lib.ptr(ids), _lib.ptr(dists), stats,
                                         _lib.stream_ptr()), "exact search")
    out = tuple(_lib.to_host(a) for a in (ids, dists, gamma, prr, p3, cand))
    if nq and out[0].min() < 0:
        bad = int(np.flatnonzero((out[0] < 0).any(axis=1))[0])
        raise ValueError(f"k must be in [1, {int(out[5][bad])}], got {k}")
    return out


def exact_query_batch(index: RbcExactIndex, queries, k: int = 1, workers: int | None = None):
    """Exact k-NN for a batch of queries (search.py:150-208)."""
    if workers is not None:
        resolve_workers(workers)
    ids, dists, gamma, prr, p3, cand = exact_query_arrays(index, queries, k)
    n_reps = index.reps.size
    # per-query objects from bulk conversions (tolist, row iteration): the same values as
    # float(gamma[i]) / int(...) per element, at a fraction of the per-query cost
    results = [NeighborList(i, r_ids, r_d) for i, (r_ids, r_d) in enumerate(zip(ids, dists))]
    stats = [
        SearchStats(g, n_reps, a, b, c, n_reps)
        for g, a, b, c in zip(gamma.tolist(), prr.tolist(), p3.tolist(), cand.tolist())
    ]
    return results, stats


def exact_query(index: RbcExactIndex, q, k: int = 1):
    """Exact k-NN search for a single query point (search.py:211-214)."""
    results, stats = exact_query_batch(index, np.asarray(q, dtype=np.float32)[None, :], k, workers=1)
    return results[0], stats[0]


def one_shot_query_arrays(index: RbcOneShotIndex, queries, k: int = 1, q_dev=None):
    """ids[nq,k], dists[nq,k], gamma[nq] (gamma = distance to the nearest rep)."""
    qv = _queries(queries)
    if not 1 <= k <= index.s:
        raise ValueError(f"k must be in [1, s={index.s}], got {k}")
    if qv.shape[1] != index.metric.dim:
        raise ValueError(f"dimension mismatch: queries d={qv.shape[1]}, metric dim={index.metric.dim}")
    t = _lib.require_cuda()
    dev = device_index(index)
    nq = qv.shape[0]
    if q_dev is None:
        q_dev = _lib.to_device(qv)
    ids = _lib.empty((nq, k), t.int64)
    dists = _lib.empty((nq, k), t.float32)
    gamma = _lib.empty((nq,), t.float32)
    _lib.check(_lib.lib.rbc_one_shot_search(dev.handle, _lib.ptr(q_dev), nq, k, _lib.ptr(ids), _lib.ptr(dists),
                                            _lib.ptr(gamma), _lib.stream_ptr()), "one-shot search")
    return _lib.to_host(ids), _lib.to_host(dists), _lib.to_host(gamma)


def one_shot_query_batch(index: RbcOneShotIndex, queries, k: int = 1, workers: int | None = None):
    """One-shot search for a batch of queries (search.py:90-141)."""
    if workers is not None:
        resolve_workers(workers)
    ids, dists, gamma = one_shot_query_arrays(index, queries, k)
    n_reps = index.reps.size
    results = [NeighborList(i, r_ids, r_d) for i, (r_ids, r_d) in enumerate(zip(ids, dists))]
    stats = [SearchStats(g, n_reps, 0, 0, index.s, n_reps) for g in gamma.tolist()]
    return results, stats


def one_shot_query(index: RbcOneShotIndex, q, k: int = 1) -> NeighborList:
    """One-shot search for a single query point (search.py:144-147)."""
    results, _ = one_shot_query_batch(index, np.asarray(q, dtype=np.float32)[None, :], k, workers=1)
    return results[0]


def range_query(index: RbcExactIndex, q, radius: float):
    """All points within ``radius`` of q, sorted by (distance, id) (search.py:217-238)."""
    import ctypes

    if radius < 0:
        raise ValueError("radius must be >= 0")
    qv = np.ascontiguousarray(np.asarray(q, dtype=np.float32).reshape(-1))
    if qv.shape[0] != index.metric.dim:
        raise ValueError(f"dimension mismatch: query d={qv.shape[0]}, metric dim={index.metric.dim}")
    dev = device_index(index)
    cap = index.data.n
    ids = np.empty(cap, np.int64)
    dists = np.empty(cap, np.float32)
    count = ctypes.c_int64(0)
    _lib.check(_lib.lib.rbc_range_query_host(dev.handle, qv.ctypes.data_as(ctypes.c_void_p), float(radius), cap,
                                             ids.ctypes.data_as(ctypes.c_void_p),
                                             dists.ctypes.data_as(ctypes.c_void_p), ctypes.byref(count),
                                             _lib.stream_ptr()), "range_query")
    c = count.value
    return ids[:c].copy(), dists[:c].copy()
