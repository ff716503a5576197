"""ctypes front-end of the CPU oracle (TEST INFRASTRUCTURE ONLY).

The oracle is a plain-C restatement of the reference rbcover 0.1.0 algorithm
(``oracle/rbc_oracle.c``; each C function cites the reference file:line it
follows).  It is the parity checker for the B200 path and the timed CPU arm of
``bench.py`` (``cpu_baseline`` / ``--impl reference``).  Nothing in the product
package imports this module.

Pinned: tests/test_oracle_golden.py checks every function here against golden
vectors produced by the reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "librbc_oracle.so")
_lib = None

L2, L1 = 0, 1
_METRIC = {"l2": L2, "l1": L1}

_f32p = ctypes.POINTER(ctypes.c_float)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i64 = ctypes.c_int64
_int = ctypes.c_int


def build() -> str:
    """Compile the oracle with its Makefile (gcc, OpenMP, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_threads.restype = _int
        L.orc_pairwise.argtypes = [_f32p, _i64, _f32p, _i64, _int, _int, _f32p]
        L.orc_bf_topk.argtypes = [_f32p, _i64, _f32p, _i64, _int, _int, _int, _i64p, _f32p]
        L.orc_bf_subsets.argtypes = [_f32p, _i64, _f32p, _int, _int, _int, _i64p, _i64p, _i64p, _f32p]
        L.orc_bernoulli.argtypes = [_i64, ctypes.c_double] + [ctypes.c_uint64] * 4 + [_i64p]
        L.orc_bernoulli.restype = _i64
        L.orc_build_exact.argtypes = [_f32p, _i64, _int, _int, _i64p, _i64, _i64p, _i64p, _f32p, _f32p]
        L.orc_build_one_shot.argtypes = [_f32p, _i64, _int, _int, _i64p, _i64, _int, _i64p, _f32p]
        L.orc_list_cutoff.argtypes = [_f32p, _i64, ctypes.c_double]
        L.orc_list_cutoff.restype = _i64
        L.orc_exact_query.argtypes = [_f32p, _int, _int, _i64p, _i64, _i64p, _i64p, _f32p, _f32p, _f32p, _i64,
                                      _int, _i64p, _f32p, _f32p, _i64p, _i64p, _i64p]
        L.orc_exact_query.restype = _i64
        L.orc_one_shot_query.argtypes = [_f32p, _int, _int, _i64p, _i64, _i64p, _int, _f32p, _i64, _int, _i64p,
                                         _f32p, _f32p]
        L.orc_range_query.argtypes = [_f32p, _int, _int, _i64p, _i64, _i64p, _i64p, _f32p, _f32p, _f32p,
                                      ctypes.c_double, _i64, _i64p, _f32p]
        L.orc_range_query.restype = _i64
        _lib = L
    return _lib


def _f(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a, a.ctypes.data_as(_f32p)


def _i(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(_i64p)


def threads() -> int:
    return int(lib().orc_threads())


def pairwise(a, b, metric="l2"):
    a, pa = _f(a)
    b, pb = _f(b)
    out = np.empty((a.shape[0], b.shape[0]), np.float32)
    lib().orc_pairwise(pa, a.shape[0], pb, b.shape[0], a.shape[1], _METRIC[metric], out.ctypes.data_as(_f32p))
    return out


def bf_topk(q, x, k, metric="l2"):
    q, pq = _f(q)
    x, px = _f(x)
    ids = np.empty((q.shape[0], k), np.int64)
    dists = np.empty((q.shape[0], k), np.float32)
    lib().orc_bf_topk(pq, q.shape[0], px, x.shape[0], q.shape[1], _METRIC[metric], k, ids.ctypes.data_as(_i64p),
                      dists.ctypes.data_as(_f32p))
    return ids, dists


def bf_subsets(q, x, cand, offsets, k, metric="l2"):
    q, pq = _f(q)
    x, px = _f(x)
    cand, pc = _i(cand)
    offsets, po = _i(offsets)
    ids = np.empty((q.shape[0], k), np.int64)
    dists = np.empty((q.shape[0], k), np.float32)
    lib().orc_bf_subsets(pq, q.shape[0], px, q.shape[1], _METRIC[metric], k, pc, po, ids.ctypes.data_as(_i64p),
                         dists.ctypes.data_as(_f32p))
    return ids, dists


def pcg64_state(seed: int):
    """(state_hi, state_lo, inc_hi, inc_lo) of numpy's default_rng(seed)."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m = (1 << 64) - 1
    return s >> 64, s & m, inc >> 64, inc & m


def bernoulli(n, p, seed):
    out = np.empty(n, np.int64)
    cnt = lib().orc_bernoulli(n, float(p), *pcg64_state(seed), out.ctypes.data_as(_i64p))
    return out[:cnt].copy()


def build_exact(x, rep_ids, metric="l2"):
    x, px = _f(x)
    rep_ids, pr = _i(rep_ids)
    n, nr = x.shape[0], rep_ids.shape[0]
    list_ids = np.empty(n, np.int64)
    offsets = np.empty(nr + 1, np.int64)
    list_dists = np.empty(n, np.float32)
    radii = np.empty(nr, np.float32)
    lib().orc_build_exact(px, n, x.shape[1], _METRIC[metric], pr, nr, list_ids.ctypes.data_as(_i64p),
                          offsets.ctypes.data_as(_i64p), list_dists.ctypes.data_as(_f32p),
                          radii.ctypes.data_as(_f32p))
    return list_ids, offsets, list_dists, radii


def build_one_shot(x, rep_ids, s, metric="l2"):
    x, px = _f(x)
    rep_ids, pr = _i(rep_ids)
    nr = rep_ids.shape[0]
    lists = np.empty((nr, s), np.int64)
    radii = np.empty(nr, np.float32)
    lib().orc_build_one_shot(px, x.shape[0], x.shape[1], _METRIC[metric], pr, nr, s, lists.ctypes.data_as(_i64p),
                             radii.ctypes.data_as(_f32p))
    return lists, radii


def list_cutoff(sorted_dists, thr):
    a, pa = _f(sorted_dists)
    return int(lib().orc_list_cutoff(pa, a.shape[0], float(thr)))


def exact_query(x, rep_ids, list_ids, offsets, list_dists, radii, q, k, metric="l2"):
    """Returns ids[nq,k], dists[nq,k], gamma[nq], pruned_radius, pruned_3gamma, candidates."""
    x, px = _f(x)
    rep_ids, pr = _i(rep_ids)
    list_ids, pl = _i(list_ids)
    offsets, po = _i(offsets)
    list_dists, pd = _f(list_dists)
    radii, prr = _f(radii)
    q, pq = _f(q)
    nq = q.shape[0]
    ids = np.empty((nq, k), np.int64)
    dists = np.empty((nq, k), np.float32)
    gamma = np.empty(nq, np.float32)
    prc = np.empty(nq, np.int64)
    p3 = np.empty(nq, np.int64)
    cand = np.empty(nq, np.int64)
    bad = lib().orc_exact_query(px, x.shape[1], _METRIC[metric], pr, rep_ids.shape[0], pl, po, pd, prr, pq, nq, k,
                                ids.ctypes.data_as(_i64p), dists.ctypes.data_as(_f32p), gamma.ctypes.data_as(_f32p),
                                prc.ctypes.data_as(_i64p), p3.ctypes.data_as(_i64p), cand.ctypes.data_as(_i64p))
    if bad:
        raise ValueError(f"query {-bad - 1}: fewer candidates than k={k}")
    return ids, dists, gamma, prc, p3, cand


def one_shot_query(x, rep_ids, lists, q, k, metric="l2"):
    x, px = _f(x)
    rep_ids, pr = _i(rep_ids)
    lists, pl = _i(lists)
    q, pq = _f(q)
    nq = q.shape[0]
    ids = np.empty((nq, k), np.int64)
    dists = np.empty((nq, k), np.float32)
    gamma = np.empty(nq, np.float32)
    lib().orc_one_shot_query(px, x.shape[1], _METRIC[metric], pr, rep_ids.shape[0], pl, lists.shape[1], pq, nq, k,
                             ids.ctypes.data_as(_i64p), dists.ctypes.data_as(_f32p), gamma.ctypes.data_as(_f32p))
    return ids, dists, gamma


def range_query(x, rep_ids, list_ids, offsets, list_dists, radii, q, eps, metric="l2"):
    x, px = _f(x)
    rep_ids, pr = _i(rep_ids)
    list_ids, pl = _i(list_ids)
    offsets, po = _i(offsets)
    list_dists, pd = _f(list_dists)
    radii, prr = _f(radii)
    q, pq = _f(np.asarray(q, np.float32).reshape(-1))
    cap = x.shape[0]
    ids = np.empty(cap, np.int64)
    dists = np.empty(cap, np.float32)
    cnt = lib().orc_range_query(px, x.shape[1], _METRIC[metric], pr, rep_ids.shape[0], pl, po, pd, prr, pq,
                                float(eps), cap, ids.ctypes.data_as(_i64p), dists.ctypes.data_as(_f32p))
    return ids[:cnt].copy(), dists[:cnt].copy()


def gen_clusters(n, d, seed, n_clusters=8, cluster_sigma=0.05):
    """Input generator restated from reference dataset.py:142-148 (numpy)."""
    rng = np.random.default_rng(seed)
    centers = rng.random((n_clusters, d))
    assignment = rng.integers(n_clusters, size=n)
    return np.ascontiguousarray((centers[assignment] + cluster_sigma * rng.standard_normal((n, d))).astype(np.float32))
