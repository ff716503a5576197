"""Diagnostic: exact search at a bench config, timed, with stage-2 work statistics (RBC_DEBUG_CAND=1)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
import paper_1103_2635_b200 as rbc

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
k = int(sys.argv[2]) if len(sys.argv) > 2 else None
bench.select_config(cfg, k)
x, q = bench.gen_inputs(0)
spec = rbc.MetricSpec(bench.CFG["metric"], bench.D)
idx = rbc.build_exact(rbc.DataMatrix(x), bench.NR, spec, seed=0)
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ids, dists, gamma, pr, p3, cand = rbc.exact_query_arrays(idx, q, bench.K)
    torch.cuda.synchronize()
    print(f"{cfg} k={bench.K}: {1e3*(time.perf_counter()-t0):.2f} ms (host API); mean cand {cand.mean():.0f}, "
          f"algorithmic pairs {cand.sum():.4g}", flush=True)
