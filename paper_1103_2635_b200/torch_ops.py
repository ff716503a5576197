"""The hot path as registered PyTorch operators: ``torch.ops.rbc_b200.*``.

A thin C++ layer (``torch_ext/rbc_torch_ops.cpp`` -> ``librbc_torch_ops.so``) over the C-ABI
(``include/rbc_b200.h``): CUDA tensors in and out, on the caller's current stream, so the
search composes with other torch code (CUDA graphs, ``torch.compile`` graphs calling the op)
without a host round trip.  Each op is one call into the sm_100a library; results are the
same bit-exact keys as the numpy-level API.

    bf_search(queries, data, metric, k) -> (ids, dists)        brute_force.py:165-186
    pairwise_distances(a, b, metric) -> dists                    metric.py:57-76
    exact_search(index, queries, k) -> (ids, dists, gamma, pruned_radius, pruned_3gamma, candidates)
                                                                 search.py:150-208
    one_shot_search(index, queries, k) -> (ids, dists, gamma)   search.py:90-141

``index`` is a built index (``RbcExactIndex`` / ``RbcOneShotIndex``; its device copy is
uploaded on first use) and ``metric`` a ``MetricSpec`` or its code (0 = l2, 1 = l1).
"""

from __future__ import annotations

import os

from . import _lib

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librbc_torch_ops.so")
_loaded = False


def load():
    """Register the operators (loads librbc_torch_ops.so once); returns ``torch.ops.rbc_b200``."""
    global _loaded
    t = _lib.torch()
    if not _loaded:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run python -m paper_1103_2635_b200._build")
        _lib.lib  # the C-ABI library first (the operator library links against it)
        t.ops.load_library(LIB_PATH)
        _loaded = True
    return t.ops.rbc_b200


def _code(metric) -> int:
    return metric if isinstance(metric, int) else metric.code


def _handle(index) -> int:
    from .rbc import device_index

    return int(device_index(index).handle.value)


def bf_search(queries, data, metric, k: int):
    return load().bf_search(queries, data, _code(metric), k)


def pairwise_distances(a, b, metric):
    return load().pairwise_distances(a, b, _code(metric))


def exact_search(index, queries, k: int = 1):
    return load().exact_search(_handle(index), queries, k)


def one_shot_search(index, queries, k: int = 1):
    return load().one_shot_search(_handle(index), queries, k)
