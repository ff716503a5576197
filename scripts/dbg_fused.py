"""Debug driver: time the cfg2 exact search with/without stats and profiling."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def main():
    import torch

    import paper_1103_2635_b200 as rbc
    from paper_1103_2635_b200 import _lib

    x, q = bench.gen_inputs(0)
    index = rbc.build_exact(rbc.DataMatrix(x), bench.NR, rbc.MetricSpec("l2", bench.D), seed=bench.REP_SEED)
    q_dev = _lib.to_device(q)
    keys = torch.empty((bench.NQ, 1), dtype=torch.int64, device="cuda")
    gamma = torch.empty(bench.NQ, dtype=torch.float32, device="cuda")
    prr = torch.empty(bench.NQ, dtype=torch.int32, device="cuda")
    p3 = torch.empty(bench.NQ, dtype=torch.int32, device="cuda")
    cand = torch.empty(bench.NQ, dtype=torch.int64, device="cuda")
    full = _lib.SearchStatsC(gamma.data_ptr(), prr.data_ptr(), p3.data_ptr(), cand.data_ptr())
    none = _lib.SearchStatsC(None, None, None, None)
    sptr = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for name, stats, prof in (("none", none, False), ("full", full, False), ("none+prof", none, True),
                              ("full+prof", full, True)):
        for _ in range(3):
            _lib.check(_lib.lib.rbc_exact_search_keys(index._dev.handle, _lib.ptr(q_dev), bench.NQ, 1,
                                                      _lib.ptr(keys), stats, sptr))
        torch.cuda.synchronize()
        _lib.profile_enable(prof)
        l0 = _lib.launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            _lib.check(_lib.lib.rbc_exact_search_keys(index._dev.handle, _lib.ptr(q_dev), bench.NQ, 1,
                                                      _lib.ptr(keys), stats, sptr))
        e1.record()
        torch.cuda.synchronize()
        ph = _lib.profile_read() if prof else None
        _lib.profile_enable(False)
        print(name, "ms/step", e0.elapsed_time(e1) / 5, "launches/step", (_lib.launch_count() - l0) / 5,
              "ovf", _lib.lib.rbc_stage2_overflows(), ph, flush=True)


if __name__ == "__main__":
    main()
