"""Per-kernel device timeline of exact searches (cfg2 by default; args: nq k config) via torch.profiler (CUPTI), no replay/serialisation:
kernel durations, start offsets and the idle gaps between kernels inside one search."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_1103_2635_b200 as rbc
    from paper_1103_2635_b200 import _lib
    from paper_1103_2635_b200.rbc import device_index

    if len(sys.argv) > 3:  # optional config name (default cfg2)
        bench.select_config(sys.argv[3], int(sys.argv[2]) if len(sys.argv) > 2 else None)
    nq = int(sys.argv[1]) if len(sys.argv) > 1 else bench.NQ
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    x, q = bench.gen_inputs(0)
    cache = os.environ.get("RBC_INDEX_CACHE")  # diagnostic library variants load the normal build's index
    if cache and os.path.exists(cache):
        index = rbc.load_index(cache)
    else:
        index = rbc.build_exact(rbc.DataMatrix(x), bench.NR, rbc.MetricSpec("l2", bench.D), seed=bench.REP_SEED)
        if cache:
            rbc.save_index(index, cache)
    device_index(index)  # upload (a loaded index uploads on first use)
    sptr = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    q_dev = _lib.to_device(q)
    keys = torch.empty((bench.NQ, k), dtype=torch.int64, device="cuda")
    stats = _lib.SearchStatsC(None, None, None, None)

    def run():
        _lib.check(_lib.lib.rbc_exact_search_keys(device_index(index).handle, _lib.ptr(q_dev), nq, k, _lib.ptr(keys), stats,
                                                  sptr))

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            run()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    ev.sort(key=lambda e: e.time_range.start)
    # split into searches at the pilot kernel
    runs, cur = [], []
    for e in ev:
        if ("pilot_key" in e.name or "s1_filter" in e.name or "pairwise_kernel" in e.name) and cur:
            runs.append(cur)
            cur = []
        cur.append(e)
    runs.append(cur)
    r = runs[-1]
    t0 = r[0].time_range.start
    prev_end = t0
    print(f"nq={nq} k={k}: one search, {len(r)} device ops, span {(r[-1].time_range.end - t0) / 1e3:.3f} ms")
    for e in r:
        s, d = e.time_range.start, e.time_range.end - e.time_range.start
        gap = s - prev_end
        print(f"  +{(s - t0) / 1e3:8.3f} ms  {d / 1e3:8.3f} ms  gap {gap / 1e3:7.3f}  {e.name[:90]}")
        prev_end = max(prev_end, e.time_range.end)


if __name__ == "__main__":
    main()
