"""Diagnostic: tensor-core brute force (prepared operand) timing and overflow count on cfg2-shaped data."""
import ctypes, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1103_2635_b200 as rbc
from paper_1103_2635_b200 import _lib
from oracle import oracle as orc

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
d = 64
full = orc.gen_clusters(n + 18944, d, 1, n_clusters=64, cluster_sigma=0.05)
x, q = full[:n], full[n:]
x_dev = _lib.to_device(x)
s = torch.cuda.current_stream()
sp = ctypes.c_void_p(s.cuda_stream)
h = ctypes.c_void_p()
torch.cuda.synchronize(); t0 = time.perf_counter()
_lib.check(_lib.lib.rbc_bf_prepare(_lib.ptr(x_dev), n, d, 0, ctypes.byref(h), sp), "prep")
torch.cuda.synchronize(); print(f"prepare {1e3*(time.perf_counter()-t0):.1f} ms", flush=True)
for m in (1024, 18944):
    for k in (1, 10):
        qd = _lib.to_device(q[:m])
        ids = torch.empty((m, k), dtype=torch.int64, device="cuda")
        ds = torch.empty((m, k), dtype=torch.float32, device="cuda")
        for it in range(3):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            _lib.check(_lib.lib.rbc_bf_search_prepared(h, _lib.ptr(qd), m, k, _lib.ptr(ids), _lib.ptr(ds), sp), "bf")
            e1.record(s); e1.synchronize()
            dt = e0.elapsed_time(e1) / 1e3
        print(f"m={m} k={k}: {dt*1e3:.2f} ms  overflows={_lib.lib.rbc_stage2_overflows()}  "
              f"TF/s={2*d*m*n/dt/1e12:.1f}", flush=True)
        if m == 1024:
            oi, od = orc.bf_topk(q[:64], x, k, "l2")
            assert np.array_equal(ids[:64].cpu().numpy(), oi) and np.array_equal(ds[:64].cpu().numpy(), od), "mismatch"
_lib.lib.rbc_index_destroy(h)
