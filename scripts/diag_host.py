"""Diagnostic: host enqueue timeline of one exact search (RBC_DEBUG_HOST) at a few batch sizes."""
import ctypes
import os
import sys

os.environ["RBC_DEBUG_HOST"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def main():
    import torch

    import paper_1103_2635_b200 as rbc
    from paper_1103_2635_b200 import _lib

    x, q = bench.gen_inputs(0)
    index = rbc.build_exact(rbc.DataMatrix(x), bench.NR, rbc.MetricSpec("l2", bench.D), seed=bench.REP_SEED)
    sptr = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    q_dev = _lib.to_device(q)
    keys = torch.empty((bench.NQ, 1), dtype=torch.int64, device="cuda")
    stats = _lib.SearchStatsC(None, None, None, None)
    for m in (6250, 100000):
        for rep in range(4):
            print(f"--- nq={m} rep={rep}", file=sys.stderr, flush=True)
            _lib.check(_lib.lib.rbc_exact_search_keys(index._dev.handle, _lib.ptr(q_dev), m, 1, _lib.ptr(keys), stats,
                                                      sptr))
            torch.cuda.synchronize()


if __name__ == "__main__":
    main()
