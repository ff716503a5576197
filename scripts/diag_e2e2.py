"""Diagnostic: per-call wall times of the host-buffer search and its H2D copy alone (cfg2)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def main():
    import torch

    import paper_1103_2635_b200 as rbc
    from paper_1103_2635_b200 import _lib

    x, q = bench.gen_inputs(0)
    index = rbc.build_exact(rbc.DataMatrix(x), bench.NR, rbc.MetricSpec("l2", bench.D), seed=bench.REP_SEED)
    dev = index._dev
    sptr = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    q_pin = torch.from_numpy(q).pin_memory()
    ids_h = torch.empty((bench.NQ, 1), dtype=torch.int64).pin_memory()
    dists_h = torch.empty((bench.NQ, 1), dtype=torch.float32).pin_memory()
    ts = []
    for i in range(40):
        t0 = time.perf_counter()
        _lib.check(_lib.lib.rbc_exact_search_host(dev.handle, ctypes.c_void_p(q_pin.data_ptr()), bench.NQ, 1,
                                                  ctypes.c_void_p(ids_h.data_ptr()), ctypes.c_void_p(dists_h.data_ptr()),
                                                  _lib.SearchStatsC(None, None, None, None), sptr))
        ts.append((time.perf_counter() - t0) * 1e3)
    print("host-call ms:", " ".join(f"{t:.2f}" for t in ts), flush=True)
    qd = torch.empty_like(q_pin, device="cuda")
    hs = []
    for i in range(20):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        qd.copy_(q_pin, non_blocking=True)
        torch.cuda.synchronize()
        hs.append((time.perf_counter() - t0) * 1e3)
    print("H2D ms:", " ".join(f"{t:.2f}" for t in hs), flush=True)


if __name__ == "__main__":
    main()
