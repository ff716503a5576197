"""Time one cfg2 exact search (median of 10) with the library named by RBC_B200_LIB; prints phase times."""
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
    st = torch.cuda.current_stream()
    sptr = ctypes.c_void_p(st.cuda_stream)
    q_dev = _lib.to_device(q)
    keys = torch.empty((bench.NQ, 1), dtype=torch.int64, device="cuda")
    stats = _lib.SearchStatsC(None, None, None, None)

    def run():
        _lib.check(_lib.lib.rbc_exact_search_keys(index._dev.handle, _lib.ptr(q_dev), bench.NQ, 1, _lib.ptr(keys),
                                                  stats, sptr))

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    _lib.profile_enable(True)
    ts = []
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        run()
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ph = _lib.profile_read()
    _lib.profile_enable(False)
    ts.sort()
    tag = os.path.basename(os.environ.get("RBC_B200_LIB", "default"))
    print(f"{tag}: step {ts[5]:.3f} ms  " + "  ".join(f"{k}={v[0] / v[1]:.3f}" for k, v in ph.items() if v[1]),
          flush=True)


if __name__ == "__main__":
    main()
