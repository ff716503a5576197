"""CPU-side checks: the C-ABI library loads and exports every declared symbol,
and the Python boundary rejects bad arguments exactly like the reference
(ValueError before any device work)."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "rbc_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rbc_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import ctypes

    from paper_1103_2635_b200 import _lib

    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, f"missing exports: {missing}"
    assert set(syms) == set(_lib.EXPORTS), "ctypes binding and header disagree"


def test_library_is_sm100a():
    from paper_1103_2635_b200 import _lib

    blob = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in blob


def test_abi_version_and_error_channel():
    from paper_1103_2635_b200 import _lib

    assert _lib.lib.rbc_abi_version() == 1
    rc = _lib.lib.rbc_build_exact(None, 10, 4, 7, None, 3, None, None, None, None, None)
    assert rc == _lib.RBC_EINVAL and "metric" in _lib.last_error()


def test_metric_spec_validation():
    import paper_1103_2635_b200 as rbc

    with pytest.raises(ValueError):
        rbc.MetricSpec("cosine", 4)
    with pytest.raises(ValueError):
        rbc.MetricSpec("l2", 0)


def test_argument_validation_matches_reference():
    import paper_1103_2635_b200 as rbc

    u = rbc.DataMatrix(np.random.default_rng(101).random((200, 8), dtype=np.float32))
    spec = rbc.MetricSpec("l2", 8)
    with pytest.raises(ValueError):
        rbc.bf_search(u.values[:2], u, spec, k=0)
    with pytest.raises(ValueError):
        rbc.bf_search(u.values[:2], u, spec, k=u.n + 1)
    with pytest.raises(ValueError):
        rbc.bf_search(np.zeros((2, 5), np.float32), u, spec, k=1)
    q = np.array([1.0], np.float32)
    line = rbc.DataMatrix(np.array([[0.0], [2.0], [5.0]], np.float32))
    with pytest.raises(ValueError):
        rbc.bf_search_subset(q, line, [], rbc.MetricSpec("l2", 1), k=1)
    with pytest.raises(ValueError):
        rbc.bf_search_subset(q, line, [1, 1, 2], rbc.MetricSpec("l2", 1), k=1)
    with pytest.raises(ValueError):
        rbc.bf_search_subset(q, line, [0, 7], rbc.MetricSpec("l2", 1), k=1)
    for args in ((10, 0, 0), (10, 11, 0), (10, 5, -1)):
        with pytest.raises(ValueError):
            rbc.sample_representatives(*args)
    with pytest.raises(ValueError):
        rbc.sample_representatives(10, 5, 0, mode="poisson")
    with pytest.raises(ValueError):
        rbc.build_one_shot(u, 20, u.n + 1, spec, seed=0)
    with pytest.raises(rbc.DataError):
        rbc.DataMatrix(np.array([[np.nan, 1.0]], np.float32))


def test_param_formulas():
    import paper_1103_2635_b200 as rbc

    assert rbc.standard_params_exact(10_000, 1.0) == 100
    assert rbc.standard_params_exact(100, 4.0) == 80
    assert rbc.one_shot_params(10_000, 1.0, np.exp(-1.0)) == (100, 100)
    with pytest.raises(ValueError):
        rbc.one_shot_params(100, 1.0, 1.5)


def test_no_cpu_fallback_without_device():
    import torch

    import paper_1103_2635_b200 as rbc

    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(RuntimeError, match="CUDA device"):
        rbc.pairwise_distances(np.zeros((2, 3), np.float32), np.zeros((2, 3), np.float32), rbc.MetricSpec("l2", 3))


def test_torch_ops_registered():
    # torch.ops.rbc_b200.* (torch_ext/rbc_torch_ops.cpp) load and carry the hot-path schemas;
    # no compute without a GPU
    from paper_1103_2635_b200 import torch_ops

    ops = torch_ops.load()
    for name, args in (("bf_search", "queries, Tensor data, int metric, int k"),
                       ("pairwise_distances", "a, Tensor b, int metric"),
                       ("exact_search", "index, Tensor queries, int k"),
                       ("one_shot_search", "index, Tensor queries, int k")):
        schema = str(getattr(ops, name).default._schema)
        assert schema.startswith(f"rbc_b200::{name}("), schema
        assert args in schema, schema
