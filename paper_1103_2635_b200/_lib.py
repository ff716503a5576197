"""ctypes binding of the C-ABI (include/rbc_b200.h) and device plumbing.

The product path always runs through librbc_b200.so (hand-written sm_100a
CUDA).  There is no CPU fallback: if the library is missing, importing this
module raises, and any search without a CUDA device raises RuntimeError.
PyTorch is used only for device memory, streams and host<->device copies.
"""

from __future__ import annotations

import ctypes
import os
import warnings

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RBC_B200_LIB") or os.path.join(_HERE, "librbc_b200.so")

_LIB = None


def _load():
    """Load librbc_b200.so once (first use).  A missing library raises ImportError then:
    there is no CPU fallback.  Loading lazily lets ``python -m paper_1103_2635_b200._build``
    import the package on a clean checkout before the library exists."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA library first "
                "(python -m paper_1103_2635_b200._build, or __graft_entry__.build())"
            )
        L = ctypes.CDLL(LIB_PATH)
        for _name, (_args, _res) in EXPORTS.items():
            f = getattr(L, _name)
            f.argtypes = _args
            f.restype = _res
        _LIB = L
    return _LIB


def __getattr__(name):  # PEP 562: ``_lib.lib`` loads the library on first access
    if name == "lib":
        return _load()
    raise AttributeError(name)

RBC_OK, RBC_EINVAL, RBC_ECUDA, RBC_ENOMEM, RBC_EFEWCAND = 0, 1, 2, 3, 4
METRIC_CODE = {"l2": 0, "l1": 1}

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_u64 = ctypes.c_uint64


class SearchStatsC(ctypes.Structure):
    _fields_ = [("gamma", _p), ("reps_pruned_radius", _p), ("reps_pruned_3gamma", _p), ("candidates", _p)]


EXPORTS = {
    "rbc_last_error": ([], ctypes.c_char_p),
    "rbc_abi_version": ([], ctypes.c_int),
    "rbc_launch_count": ([], _i64),
    "rbc_profile_enable": ([ctypes.c_int], ctypes.c_int),
    "rbc_profile_read": ([_p, _p, _i32], ctypes.c_int),
    "rbc_pairwise_distances": ([_p, _i64, _p, _i64, _i32, _i32, _p, _p], ctypes.c_int),
    "rbc_bf_search": ([_p, _i64, _p, _i64, _i32, _i32, _i32, _p, _p, _p], ctypes.c_int),
    "rbc_bf_prepare": ([_p, _i64, _i32, _i32, ctypes.POINTER(_p), _p], ctypes.c_int),
    "rbc_bf_search_prepared": ([_p, _p, _i64, _i32, _p, _p, _p], ctypes.c_int),
    "rbc_bf_search_subsets": ([_p, _i64, _p, _i64, _i32, _i32, _i32, _p, _p, _p, _p, _p], ctypes.c_int),
    "rbc_count_within": ([_p, _i64, _p, _i64, _i32, _i32, _p, _i32, _i32, _p, _p, _p], ctypes.c_int),
    "rbc_merge_topk": ([_p, _i32, _i64, _i32, _i32, _p, _p, _p], ctypes.c_int),
    "rbc_bernoulli_draw": ([_i64, ctypes.c_double, _u64, _u64, _u64, _u64, _p, ctypes.POINTER(_i64), _p],
                           ctypes.c_int),
    "rbc_build_exact": ([_p, _i64, _i32, _i32, _p, _i64, _p, _p, _p, _p, _p], ctypes.c_int),
    "rbc_build_one_shot": ([_p, _i64, _i32, _i32, _p, _i64, _i32, _p, _p, _p], ctypes.c_int),
    "rbc_index_exact_create": ([_p, _i64, _i32, _i32, _p, _i64, _p, _p, _p, _p, ctypes.POINTER(_p), _p],
                               ctypes.c_int),
    "rbc_index_exact_create_shard": ([_p, _i64, _i32, _i32, _p, _i64, _p, _p, _p, _p, _p, ctypes.POINTER(_p), _p],
                                     ctypes.c_int),
    "rbc_index_one_shot_create": ([_p, _i64, _i32, _i32, _p, _i64, _p, _i32, _p, ctypes.POINTER(_p), _p],
                                  ctypes.c_int),
    "rbc_index_destroy": ([_p], ctypes.c_int),
    "rbc_index_device_bytes": ([_p], _i64),
    "rbc_exact_search": ([_p, _p, _i64, _i32, _p, _p, SearchStatsC, _p], ctypes.c_int),
    "rbc_exact_search_keys": ([_p, _p, _i64, _i32, _p, SearchStatsC, _p], ctypes.c_int),
    "rbc_one_shot_search": ([_p, _p, _i64, _i32, _p, _p, _p, _p], ctypes.c_int),
    "rbc_exact_search_host": ([_p, _p, _i64, _i32, _p, _p, SearchStatsC, _p], ctypes.c_int),
    "rbc_one_shot_search_host": ([_p, _p, _i64, _i32, _p, _p, _p, _p], ctypes.c_int),
    "rbc_range_query_host": ([_p, _p, ctypes.c_double, _i64, _p, _p, ctypes.POINTER(_i64), _p], ctypes.c_int),
    "rbc_prune_representatives": ([_p, _p, _i64, ctypes.c_double, _p, _p], ctypes.c_int),
    "rbc_list_cutoff": ([_p, _i64, _p, _i64, _p, _p], ctypes.c_int),
    "rbc_tc_selftest": ([_p, _p, _p, _i32, _p], ctypes.c_int),
    "rbc_set_engine": ([ctypes.c_int], ctypes.c_int),
    "rbc_stage2_overflows": ([], _i64),
    "rbc_tc_bf_calls": ([], _i64),
    "rbc_simt_scan_calls": ([], _i64),
    "rbc_select_calls": ([], _i64),
    "rbc_select_fallbacks": ([], _i64),
    "rbc_filter_stage1_calls": ([], _i64),
    "rbc_filter_stage1_fallbacks": ([], _i64),
    "rbc_index_exact_create_local": ([_p, _p, _i64, _p, _i64, _i32, _i32, _p, _p, _p, _p, _i64, ctypes.POINTER(_p), _p],
                                     ctypes.c_int),
    "rbc_local_list_radii": ([_p, _p, _i64, _i64, _p, _p], ctypes.c_int),
    "rbc_tc_scan_calls": ([], _i64),
}
def last_error() -> str:
    msg = _load().rbc_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    if rc == RBC_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc in (RBC_EINVAL, RBC_EFEWCAND):
        raise ValueError(msg)
    if rc == RBC_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


# ---- device plumbing (torch only allocates / copies / provides streams) -----
_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as _t

        _torch = _t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("paper_1103_2635_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback")
    return t


def stream_ptr():
    t = require_cuda()
    return ctypes.c_void_p(t.cuda.current_stream().cuda_stream)


def to_device(a: np.ndarray, dtype=None):
    """Upload a host array through pinned memory."""
    t = require_cuda()
    a = np.ascontiguousarray(a, dtype=dtype)
    with warnings.catch_warnings():  # read-only DataMatrix values: the tensor is only read
        warnings.simplefilter("ignore")
        host = t.from_numpy(a)
    if a.nbytes >= (1 << 20):
        host = host.pin_memory()
    return host.to("cuda", non_blocking=True)


def empty(shape, dtype):
    t = require_cuda()
    return t.empty(shape, dtype=dtype, device="cuda")


def ptr(tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(tensor.data_ptr()) if tensor is not None else ctypes.c_void_p(0)


def to_host(tensor) -> np.ndarray:
    return tensor.cpu().numpy()


def launch_count() -> int:
    return int(_load().rbc_launch_count())


PHASES = ("stage1", "prune", "stage2", "build", "scan")


def profile_enable(on: bool = True) -> None:
    _load().rbc_profile_enable(1 if on else 0)


def profile_read() -> dict:
    """{phase: (total_ms, intervals)} of the CUDA-event phase timers."""
    ms = (ctypes.c_double * 8)()
    cnt = (ctypes.c_int64 * 8)()
    check(_load().rbc_profile_read(ms, cnt, 8), "profile_read")
    return {name: (ms[i], cnt[i]) for i, name in enumerate(PHASES)}
