"""Ground-truth counts on the GPU: ball counts, expansion-rate estimate, rank error, Claim-1 counts.

Mirrors reference eval.py:21-170 and the rank-error half of report.py:62-95 (``Baseline``, ``run_baseline``,
``rank_errors``).  The reference materialises a full distance row per probe and counts in numpy; here every count
is one ``rbc_count_within`` launch (warp per query over all of X, the reference's fp32 distances, numpy's
f64 comparison), so no n-length row leaves the device.  Results are identical to the reference's
(tests/test_eval_gpu.py against tests/golden/eval_golden.npz, written by the reference).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .brute_force import _check_dims, bf_search_arrays
from .dataset import DataMatrix, _as_values
from .metric import MetricSpec, pairwise_distances
from .rbc import sample_representatives

RANK_BASELINE_K = 512  # report.py:26


def _max_thresholds(d: int) -> int:
    return max(1, (46 * 1024 - 16 - 4 * d) // 140)  # rbc_count_within's per-query shared state


def count_within(qv: np.ndarray, xv: np.ndarray, spec: MetricSpec, thresholds: np.ndarray, strict: bool,
                 x_dev=None, want_max: bool = False):
    """counts[i, t] = #{j : f64(dist(q_i, x_j)) < thr[i, t]} (strict) or <= (closed); optionally row maxima."""
    t = _lib.require_cuda()
    qv = np.ascontiguousarray(qv, np.float32)
    thr = np.ascontiguousarray(np.asarray(thresholds, np.float64).reshape(qv.shape[0], -1))
    nq, nt = thr.shape
    n = xv.shape[0]
    x_dev = _lib.to_device(xv) if x_dev is None else x_dev
    q_dev = _lib.to_device(qv)
    counts = np.empty((nq, nt), np.int64)
    dmax = _lib.empty((nq,), t.float32) if want_max else None
    step = _max_thresholds(spec.dim)
    lo = 0
    while True:
        hi = min(nt, lo + step)
        c_dev = _lib.empty((nq, hi - lo), t.int64)
        t_dev = _lib.to_device(np.ascontiguousarray(thr[:, lo:hi]))
        _lib.check(_lib.lib.rbc_count_within(_lib.ptr(q_dev), nq, _lib.ptr(x_dev), n, spec.dim, spec.code,
                                             _lib.ptr(t_dev), hi - lo, int(strict), _lib.ptr(c_dev),
                                             _lib.ptr(dmax if lo == 0 else None), _lib.stream_ptr()), "count_within")
        counts[:, lo:hi] = _lib.to_host(c_dev)
        lo = hi
        if lo >= nt:
            break
    return (counts, _lib.to_host(dmax)) if want_max else counts


def ball_count(data, center, radius: float, spec: MetricSpec) -> int:
    """Points of ``data`` in the closed ball B(center, radius) (eval.py:21-27)."""
    if radius < 0:
        raise ValueError("radius must be >= 0")
    xv = _as_values(data)
    cv = np.asarray(center, dtype=np.float32).reshape(1, -1)
    _check_dims(cv, xv, spec)
    return int(count_within(cv, xv, spec, np.array([[radius]], np.float64), strict=False)[0, 0])


@dataclass
class ExpansionEstimate:
    """Observed doubling ratios |B(x,2r)| / |B(x,r)| over sampled centers and radii (eval.py:30-39)."""

    c_max: float
    c_median: float
    samples: int
    radii_per_sample: int
    includes_queries: bool = False


def estimate_expansion_rate(data, spec: MetricSpec, n_samples: int, n_radii: int, seed: int,
                            queries=None) -> ExpansionEstimate:
    """Doubling-ratio estimate of the expansion rate (eval.py:42-107).

    Same centers (``default_rng(seed).integers``), same radii and the same ratio filter (|B(x,r)| >= 10) as the
    reference.  The diameter pass is one count launch with row maxima; a center's nearest-neighbour distance is
    the second entry of its exact top-2 (the reference's ``sort(row)[1]``); each center's 2*n_radii ball sizes
    are one count row with the radii and their doubles as thresholds.
    """
    if n_samples < 1 or n_radii < 1:
        raise ValueError("n_samples and n_radii must be >= 1")
    xv = _as_values(data)
    includes_queries = queries is not None
    if includes_queries:
        xv = np.ascontiguousarray(np.vstack((xv, _as_values(queries))))
    n = xv.shape[0]
    _check_dims(xv[:1], xv, spec)
    rng = np.random.default_rng(seed)
    centers = rng.integers(n, size=min(n_samples, n))
    cv = np.ascontiguousarray(xv[centers])
    x_dev = _lib.to_device(xv)

    _, row_max = count_within(cv, xv, spec, np.empty((len(centers), 0)), strict=False, x_dev=x_dev, want_max=True)
    r_hi = float(row_max.max()) / 2.0
    if n > 1:
        _, top2 = bf_search_arrays(cv, xv, spec, 2, x_dev=x_dev)
        nn = top2[:, 1].astype(np.float64)
    else:
        nn = np.zeros(len(centers))

    exponents = np.linspace(0.0, 1.0, n_radii)
    keep = [i for i in range(len(centers)) if 0.0 < nn[i] < r_hi]
    ratios: list[float] = []
    if keep:
        radii = np.stack([nn[i] * (r_hi / nn[i]) ** exponents for i in keep])
        counts = count_within(cv[keep], xv, spec, np.hstack((radii, 2.0 * radii)), strict=False, x_dev=x_dev)
        inner, outer = counts[:, :n_radii], counts[:, n_radii:]
        for row in range(len(keep)):
            ok = inner[row] >= 10
            ratios.extend((outer[row][ok] / inner[row][ok]).tolist())
    if not ratios:
        return ExpansionEstimate(1.0, 1.0, len(centers), n_radii, includes_queries)
    arr = np.asarray(ratios)
    return ExpansionEstimate(float(arr.max()), float(np.median(arr)), len(centers), n_radii, includes_queries)


def rank_error(data, q, returned_id: int, spec: MetricSpec) -> int:
    """Database points strictly closer to q than the returned one (eval.py:110-123)."""
    xv = _as_values(data)
    if not 0 <= returned_id < xv.shape[0]:
        raise ValueError(f"returned_id {returned_id} out of range")
    qv = np.asarray(q, dtype=np.float32).reshape(1, -1)
    _check_dims(qv, xv, spec)
    ret = pairwise_distances(qv, xv[returned_id:returned_id + 1], spec)[0, 0]
    return int(count_within(qv, xv, spec, np.array([[ret]], np.float64), strict=True)[0, 0])


def claim1_counts(data, n_r: int, spec: MetricSpec, n_queries: int, seed: int, queries=None) -> np.ndarray:
    """Strictly-closer counts behind the expected-ball-size argument (eval.py:126-164).

    Query i draws its own Bernoulli representative set with seed ``rng.integers(2**63)`` (same stream as the
    reference), gamma_i = its nearest representative's distance (one batched exact subset scan, k=1), and the
    count is one strict count launch over all queries.
    """
    xv = _as_values(data)
    n = xv.shape[0]
    rng = np.random.default_rng(seed)
    if queries is None:
        lo = xv.min(axis=0).astype(np.float64)
        hi = xv.max(axis=0).astype(np.float64)
        qv = (lo + rng.random((n_queries, xv.shape[1])) * (hi - lo)).astype(np.float32)
    else:
        qv = _as_values(queries)
        if qv.shape[0] < n_queries:
            raise ValueError(f"need {n_queries} queries, got {qv.shape[0]}")
        qv = np.ascontiguousarray(qv[:n_queries])
    _check_dims(qv, xv, spec)
    if n_queries == 0:
        return np.empty(0, np.int64)
    t = _lib.require_cuda()
    rep_lists = [sample_representatives(n, n_r, int(rng.integers(2**63)), mode="bernoulli").rep_ids
                 for _ in range(n_queries)]
    offsets = np.zeros(n_queries + 1, np.int64)
    np.cumsum([len(r) for r in rep_lists], out=offsets[1:])
    x_dev = _lib.to_device(xv)
    q_dev = _lib.to_device(qv)
    # named, so the buffers outlive the launch (a freed temporary can be handed to the next upload)
    sub_ids = _lib.to_device(np.concatenate(rep_lists))
    sub_off = _lib.to_device(offsets)
    ids = _lib.empty((n_queries, 1), t.int64)
    gamma = _lib.empty((n_queries, 1), t.float32)
    _lib.check(_lib.lib.rbc_bf_search_subsets(_lib.ptr(q_dev), n_queries, _lib.ptr(x_dev), n, spec.dim, spec.code, 1,
                                              _lib.ptr(sub_ids), _lib.ptr(sub_off), _lib.ptr(ids), _lib.ptr(gamma),
                                              _lib.stream_ptr()), "claim1 gamma")
    thr = _lib.to_host(gamma).astype(np.float64)
    return count_within(qv, xv, spec, thr, strict=True, x_dev=x_dev)[:, 0]


def claim1_trial(data, n_r: int, spec: MetricSpec, n_queries: int, seed: int, queries=None) -> float:
    """Mean strictly-closer count over fresh representative samples (eval.py:167-170)."""
    return float(claim1_counts(data, n_r, spec, n_queries, seed, queries).mean())


# ---- brute-force baseline and rank errors (report.py:53-95) ---------------------------------------------------

@dataclass
class Baseline:
    """Brute-force reference: per-query eval cost, timing, and top distances (report.py:53-59)."""

    top_dists: np.ndarray  # (n_queries, K) ascending
    evals_per_query: int
    query_wall_s: float


def run_baseline(data: DataMatrix, queries: np.ndarray, spec: MetricSpec, k: int, workers=None) -> Baseline:
    """Exact top-max(k, 512) distances of every query (report.py:62-68), one GPU scan."""
    xv, qv = _as_values(data), _as_values(queries)
    _check_dims(qv, xv, spec)
    top_k = min(xv.shape[0], max(k, RANK_BASELINE_K))
    t0 = time.perf_counter()
    _, top = bf_search_arrays(qv, xv, spec, top_k)
    return Baseline(top, xv.shape[0], time.perf_counter() - t0)


def rank_errors(data: DataMatrix, queries: np.ndarray, returned_dists: np.ndarray, baseline: Baseline,
                spec: MetricSpec) -> np.ndarray:
    """Exact rank (strictly-closer count) of each returned top-1 distance (report.py:71-95).

    Ranks inside the baseline depth are read off it; deeper ones are one batched strict count launch.
    """
    xv = _as_values(data)
    top = baseline.top_dists
    # the caller's values as given (float64 returned distances compare in float64, as in the
    # reference); float32 only for the searchsorted branch (report.py:88)
    ret = np.asarray(returned_dists)
    ranks = np.empty(len(ret), dtype=np.int64)
    escaped = []
    for i, r in enumerate(ret):
        if r <= top[i, -1] or top.shape[1] >= xv.shape[0]:
            ranks[i] = np.searchsorted(top[i], np.float32(r), side="left")
        else:
            escaped.append(i)
    if escaped:
        qv = np.ascontiguousarray(_as_values(queries)[escaped])
        ranks[escaped] = count_within(qv, xv, spec, ret[escaped].astype(np.float64), strict=True)[:, 0]
    return ranks
