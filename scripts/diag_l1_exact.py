"""Diagnostic: exact L1 search on cfg4-shaped data (n=2M, d=21, C=8, n_r=1415, 100k queries, k=1 and 10):
the SIMT filter stage 2 (auto engine) against the exact fp64 engine (engine 1); identical keys."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    import torch

    import paper_1103_2635_b200 as rbc
    from paper_1103_2635_b200 import _lib

    bench.select_config("cfg4")
    x, q = bench.gen_inputs(0)
    idx = rbc.build_exact(rbc.DataMatrix(x), bench.NR, rbc.MetricSpec("l1", bench.D), seed=bench.REP_SEED)
    dev = idx._dev
    sptr = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    q_dev = _lib.to_device(q)
    stats = _lib.SearchStatsC(None, None, None, None)
    for k in (1, 10):
        out = {}
        for eng in (0, 1):
            _lib.lib.rbc_set_engine(eng)
            keys = torch.empty((bench.NQ, k), dtype=torch.int64, device="cuda")
            times = []
            for it in range(3):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                _lib.check(_lib.lib.rbc_exact_search_keys(dev.handle, _lib.ptr(q_dev), bench.NQ, k, _lib.ptr(keys),
                                                          stats, sptr))
                e1.record()
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
            out[eng] = keys.clone()
            print(f"k={k} engine {eng}: {min(times):.2f} ms per {bench.NQ} queries", flush=True)
        assert torch.equal(out[0], out[1]), "engines differ"
    _lib.lib.rbc_set_engine(0)
    print("identical keys")


if __name__ == "__main__":
    main()
