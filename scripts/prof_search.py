"""Profiling driver: build a config's index (default cfg2), run `--iters` searches (for ncu / launch lists)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--config", default="cfg2")
    args = ap.parse_args()
    bench.select_config(args.config, args.k)
    args.k = bench.K
    import ctypes

    import torch

    import paper_1103_2635_b200 as rbc
    from paper_1103_2635_b200 import _lib

    x, q = bench.gen_inputs(0)
    cfg = bench.CFG
    spec = rbc.MetricSpec(cfg["metric"], bench.D)
    if cfg["kind"] == "exact":
        index = rbc.build_exact(rbc.DataMatrix(x), bench.NR, spec, seed=bench.REP_SEED)
    else:
        index = rbc.build_one_shot(rbc.DataMatrix(x), bench.NR, cfg["s"], spec, seed=bench.REP_SEED, mode=cfg["mode"])
    torch.cuda.synchronize()
    print("built", file=sys.stderr)
    q_dev = _lib.to_device(q)
    keys = torch.empty((bench.NQ, args.k), dtype=torch.int64, device="cuda")
    stats = _lib.SearchStatsC(None, None, None, None)
    sptr = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    ids = torch.empty((bench.NQ, args.k), dtype=torch.int64, device="cuda")
    dists = torch.empty((bench.NQ, args.k), dtype=torch.float32, device="cuda")
    for _ in range(args.iters):
        if cfg["kind"] == "exact":
            _lib.check(_lib.lib.rbc_exact_search_keys(index._dev.handle, _lib.ptr(q_dev), bench.NQ, args.k,
                                                      _lib.ptr(keys), stats, sptr))
        else:
            _lib.check(_lib.lib.rbc_one_shot_search(index._dev.handle, _lib.ptr(q_dev), bench.NQ, args.k,
                                                    _lib.ptr(ids), _lib.ptr(dists), None, sptr))
    torch.cuda.synchronize()
    print("overflows", _lib.lib.rbc_stage2_overflows(), file=sys.stderr)


if __name__ == "__main__":
    main()
