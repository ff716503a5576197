"""Diagnostic: device search time vs batch size, H2D/D2H copy times, host-buffer e2e call (cfg2)."""
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
    st = torch.cuda.current_stream()
    sptr = ctypes.c_void_p(st.cuda_stream)
    q_dev = _lib.to_device(q)
    keys = torch.empty((bench.NQ, 1), dtype=torch.int64, device="cuda")
    stats = _lib.SearchStatsC(None, None, None, None)

    def dev_time(m, reps=10):
        for _ in range(3):
            _lib.check(_lib.lib.rbc_exact_search_keys(dev.handle, _lib.ptr(q_dev), m, 1, _lib.ptr(keys), stats, sptr))
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            _lib.check(_lib.lib.rbc_exact_search_keys(dev.handle, _lib.ptr(q_dev), m, 1, _lib.ptr(keys), stats, sptr))
            e1.record(st)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        return ts[len(ts) // 2]

    for m in (25000, 50000, 100000):
        t = dev_time(m)
        print(f"device nq={m}: {t:.3f} ms  {m / t / 1e3:.2f} Mq/s", flush=True)
    q_pin = torch.from_numpy(q).pin_memory()
    qd = torch.empty_like(q_pin, device="cuda")
    for _ in range(3):
        qd.copy_(q_pin, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(10):
        qd.copy_(q_pin, non_blocking=True)
    e1.record(st)
    e1.synchronize()
    t = e0.elapsed_time(e1) / 10
    print(f"H2D {q.nbytes / 1e6:.1f} MB: {t:.3f} ms  {q.nbytes / t / 1e6:.1f} GB/s", flush=True)
    # the same bytes as 4 concurrent copies on side streams
    ss = [torch.cuda.Stream() for _ in range(4)]
    n4 = q_pin.shape[0] // 4
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(10):
        for j, s2 in enumerate(ss):
            s2.wait_stream(st)
            with torch.cuda.stream(s2):
                qd[j * n4:(j + 1) * n4].copy_(q_pin[j * n4:(j + 1) * n4], non_blocking=True)
        for s2 in ss:
            st.wait_stream(s2)
    e1.record(st)
    e1.synchronize()
    t = e0.elapsed_time(e1) / 10
    print(f"H2D x4 streams: {t:.3f} ms  {q.nbytes / t / 1e6:.1f} GB/s", flush=True)
    ids_h = torch.empty((bench.NQ, 1), dtype=torch.int64).pin_memory()
    dists_h = torch.empty((bench.NQ, 1), dtype=torch.float32).pin_memory()
    for label, fn in (("rbc_exact_search_host", _lib.lib.rbc_exact_search_host),):
        ts = []
        for i in range(13):
            t0 = time.perf_counter()
            _lib.check(fn(dev.handle, ctypes.c_void_p(q_pin.data_ptr()), bench.NQ, 1, ctypes.c_void_p(ids_h.data_ptr()),
                          ctypes.c_void_p(dists_h.data_ptr()), _lib.SearchStatsC(None, None, None, None), sptr))
            if i >= 3:
                ts.append(time.perf_counter() - t0)
        ts.sort()
        print(f"{label}: median {ts[len(ts) // 2] * 1e3:.3f} ms  {bench.NQ / ts[len(ts) // 2] / 1e6:.2f} Mq/s", flush=True)


if __name__ == "__main__":
    main()
