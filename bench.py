"""Benchmark: exact RBC 1-NN queries/sec at n=1M, d=64 (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

One step = one exact_query_batch of the rank's 100k queries (k=1) against the
device-resident index (X 1M x 64 float32, |R| = 1016 from n_r = 1000, seed 0).
Inputs: reference generator ``clusters`` (C=64, sigma=0.05, seed 1), n + nq
points, first n = X, last nq = Q (held out from the same draw).  Rank r > 0
draws its own held-out queries from the same cluster centres (seed 1000 + r).
Scaling is weak (query sharding, no data-path collective; the index is built
redundantly per rank, deterministically).

The JSON line carries value (device-resident q/s), e2e (the C-ABI host-buffer
call, H2D of queries + D2H of results inside the timed region), the roofline
of the dominant kernel, the CPU baseline (the oracle restatement on the host's
cores, bounded sample) and the clocks seen during the timed region.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N, D, NQ, C, SIGMA, DATA_SEED, NR, REP_SEED, K = 1_000_000, 64, 100_000, 64, 0.05, 1, 1000, 0, 1
METRIC = "RBC queries/sec (exact 1-NN, n=1M d=64)"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def gen_inputs(rank: int):
    rng = np.random.default_rng(DATA_SEED)
    centers = rng.random((C, D))
    assignment = rng.integers(C, size=N + NQ)
    full = (centers[assignment] + SIGMA * rng.standard_normal((N + NQ, D))).astype(np.float32)
    x, q = np.ascontiguousarray(full[:N]), np.ascontiguousarray(full[N:])
    if rank > 0:
        r2 = np.random.default_rng(1000 + rank)
        q = np.ascontiguousarray((centers[r2.integers(C, size=NQ)] + SIGMA * r2.standard_normal((NQ, D))).astype(np.float32))
    return x, q


def ncu_traffic(kernel="stage2_tc_kernel"):
    """dram__bytes_read + dram__bytes_write per launch of `kernel` from the newest committed
    ncu --set full summary under profiles/ (bytes), or None."""
    import glob
    import re
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_v*_kernels.txt")),
                   key=lambda f: int(re.search(r"_v(\d+)_", f).group(1)))
    for path in reversed(files):
        block, total = None, 0.0
        for line in open(path):
            if line.startswith("== "):
                block = kernel in line
            elif block and "dram__bytes_" in line:
                m = re.search(r"= ([\d.]+) (\w+)", line)
                if m:
                    total += float(m.group(1)) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(m.group(2), 1)
        if total > 0:
            return {"bytes_per_launch": total, "source": os.path.relpath(path, ROOT)}
    return None


def gpu_local_cpus(device: int):
    """CPUs on the GPU's NUMA node (sysfs local_cpulist of its PCI function), or None."""
    try:
        import torch

        pr = torch.cuda.get_device_properties(device)
        bdf = f"{pr.pci_domain_id:04x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bdf}/local_cpulist") as f:
            spec = f.read().strip()
        cpus = set()
        for part in spec.split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        cpus &= os.sched_getaffinity(0)
        return cpus or None
    except Exception:
        return None


def peaks():
    try:
        with open(PEAKS) as f:
            p = json.load(f)
        return {"hbm": p["hbm_gbs"], "tensor": p["bf16_tflops"], "src": "measured"}
    except Exception:
        return {"hbm": 6650.0, "tensor": 1590.0, "src": "fallback"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return
        # NVML start-up takes driver locks that stall CUDA calls (a ~1 s hiccup was
        # seen inside a timed step): keep it out of the timed region by waiting for
        # several samples before returning
        t0 = time.time()
        while time.time() - t0 < 8.0:
            with open(self.path) as f:
                if sum(1 for _ in f) >= 3:
                    break
            time.sleep(0.05)
        time.sleep(0.2)

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                rows.append(f)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        load = [s for s in sm if s > 0.5 * (max(sm) if sm else 1)]
        return {"sm_mhz": statistics.median(load or sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows)}


def cpu_baseline(x, q, index, budget_s=12.0):
    """The oracle (C restatement of the reference, OpenMP) on the host cores, bounded query sample."""
    from oracle import oracle as orc

    orc.build()
    reps = index.reps.rep_ids
    li, off, ld = index.flat_lists()
    radii = index.radii
    m = 256
    t0 = time.perf_counter()
    orc.exact_query(x, reps, li, off, ld, radii, q[:m], K)
    dt = time.perf_counter() - t0
    m2 = int(min(len(q), max(m, m * budget_s / max(dt, 1e-3))))
    t0 = time.perf_counter()
    orc.exact_query(x, reps, li, off, ld, radii, q[:m2], K)
    dt = time.perf_counter() - t0
    return {"value": m2 / dt, "unit": "queries/s", "cores": orc.threads(), "kind": "port",
            "sample": f"{m2} of the {len(q)} cfg2 queries, exact 1-NN via oracle/rbc_oracle.c (OpenMP)"}


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm's CPU restatement (oracle) on this host's cores."""
    if rank != 0:
        return
    from oracle import oracle as orc

    orc.build()
    x, q = gen_inputs(0)
    t0 = time.perf_counter()
    reps = orc.bernoulli(N, NR / N, REP_SEED)
    li, off, ld, radii = orc.build_exact(x, reps)
    build_s = time.perf_counter() - t0
    per_step = 1024
    times = []
    for step in range(args.warmup + args.steps):
        lo = (step * per_step) % (NQ - per_step)
        t0 = time.perf_counter()
        orc.exact_query(x, reps, li, off, ld, radii, q[lo: lo + per_step], K)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
    value = per_step * len(times) / sum(times)
    line = {"metric": METRIC, "value": value, "unit": "queries/s", "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg2: exact RBC 1-NN L2, clusters n=1M d=64 C=64 sigma=0.05, |R|=1016",
                       "queries_per_step": per_step, "index_build_s": build_s},
            "cpu_baseline": {"value": value, "unit": "queries/s", "cores": orc.threads(), "kind": "port",
                             "sample": f"{per_step} queries per step (oracle/rbc_oracle.c, OpenMP)"},
            "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    global K, METRIC
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-bf", action="store_true")
    ap.add_argument("--k", type=int, default=K, help="neighbours per query (the headline line is k=1)")
    args = ap.parse_args()
    if args.k != K:
        K = args.k
        METRIC = METRIC.replace("exact 1-NN", f"exact {K}-NN")

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_1103_2635_b200 as rbc
    from paper_1103_2635_b200 import _lib

    x, q = gen_inputs(rank)
    data = rbc.DataMatrix(x)
    spec = rbc.MetricSpec("l2", D)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    index = rbc.build_exact(data, NR, spec, seed=REP_SEED)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    dev = index._dev
    n_reps = index.reps.size

    stream = torch.cuda.current_stream()
    sptr = ctypes.c_void_p(stream.cuda_stream)
    q_dev = _lib.to_device(q)
    keys = torch.empty((NQ, K), dtype=torch.int64, device="cuda")
    gamma = torch.empty(NQ, dtype=torch.float32, device="cuda")
    prr = torch.empty(NQ, dtype=torch.int32, device="cuda")
    p3 = torch.empty(NQ, dtype=torch.int32, device="cuda")
    cand = torch.empty(NQ, dtype=torch.int64, device="cuda")
    stats = _lib.SearchStatsC(gamma.data_ptr(), prr.data_ptr(), p3.data_ptr(), cand.data_ptr())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def step():
        _lib.check(_lib.lib.rbc_exact_search_keys(dev.handle, _lib.ptr(q_dev), NQ, K, _lib.ptr(keys), stats, sptr),
                   "exact search")

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- e2e: C-ABI host-buffer call, pinned queries in, results out --------
    # (measured before the clock sampler starts: nvidia-smi's NVML polling stalls host calls)
    # host buffers and the calling thread on the GPU's NUMA node (the DMA then never
    # crosses the socket link); the previous affinity is restored afterwards
    old_aff = os.sched_getaffinity(0)
    local_cpus = gpu_local_cpus(local)
    if local_cpus:
        os.sched_setaffinity(0, local_cpus)
    q_pin = torch.from_numpy(q.copy()).pin_memory()
    ids_h = torch.empty((NQ, K), dtype=torch.int64).pin_memory()
    dists_h = torch.empty((NQ, K), dtype=torch.float32).pin_memory()
    e2e_times = []
    for i in range(args.warmup + max(3, args.steps // 2)):
        t0 = time.perf_counter()
        _lib.check(_lib.lib.rbc_exact_search_host(dev.handle, ctypes.c_void_p(q_pin.data_ptr()), NQ, K,
                                                  ctypes.c_void_p(ids_h.data_ptr()),
                                                  ctypes.c_void_p(dists_h.data_ptr()),
                                                  _lib.SearchStatsC(None, None, None, None), sptr), "e2e")
        if i >= args.warmup:
            e2e_times.append(time.perf_counter() - t0)
    os.sched_setaffinity(0, old_aff)
    # median: the host call's wall time carries OS scheduling noise; min/median/max go to stderr
    e2e_s = statistics.median(e2e_times)
    log(f"e2e host cpus: {len(local_cpus) if local_cpus else 'unrestricted'}; per-call ms: "
        + " ".join(f"{1e3 * t:.2f}" for t in e2e_times))
    log(f"e2e ms: min {1e3 * min(e2e_times):.3f} median {1e3 * e2e_s:.3f} max {1e3 * max(e2e_times):.3f} "
        f"(n={len(e2e_times)})")
    if dist:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_block = {"value": world * NQ / e2e_s, "unit": "queries/s", "h2d_bytes_per_step": int(q.nbytes),
           "d2h_bytes_per_step": int(ids_h.numel() * 8 + dists_h.numel() * 4)}

    for _ in range(args.warmup):  # back to the device-resident call (re-captures its graph)
        step()
    torch.cuda.synchronize()

    # ---- timed region: device-resident inputs --------------------------------
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = _lib.launch_count()
    times = []
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        flush.zero_()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        step()
        ev1.record(stream)
        ev1.synchronize()
        times.append(ev0.elapsed_time(ev1))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches = _lib.launch_count() - launches0
    # phase split (stage 1 / stage 2 / scan) from a separate pass with the CUDA-event phase
    # timers on; the timers force direct launches (no graph replay), so they stay out of
    # the timed loop above
    _lib.profile_enable(True)
    for _ in range(3):  # direct-launch warm-up (scratch pool regrowth after the graph arena)
        step()
    torch.cuda.synchronize()
    per_step = []
    for _ in range(11):  # per-step phase times, median per phase
        _lib.profile_enable(True)  # clears the records
        flush.zero_()
        step()
        torch.cuda.synchronize()
        per_step.append(_lib.profile_read())
    phases = {name: (statistics.median(p[name][0] for p in per_step), 1 if per_step[0][name][1] else 0)
              for name in per_step[0]}
    _lib.profile_enable(False)
    clk = clocks.stop()

    srt = sorted(times)
    log(f"step ms: min {srt[0]:.3f} median {srt[len(srt) // 2]:.3f} max {srt[-1]:.3f}; slowest {['%.3f' % t for t in srt[-5:]]}")
    total_ms = sum(times)
    if dist:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = world * NQ * args.steps / (total_ms / 1e3)

    # ---- algorithmic work (reference-rule counts) ---------------
    cand_h = cand.cpu().numpy()
    flops_per_step = 2.0 * D * (n_reps * NQ + float(cand_h.sum()))
    stage2_ms, stage2_n = phases["stage2"]
    stage2_flops = 2.0 * D * float(cand_h.sum())
    pk = peaks()
    traffic = ncu_traffic()
    achieved_tf = stage2_flops * stage2_n / (stage2_ms / 1e3) / 1e12 if stage2_ms > 0 else None
    roofline = {"bound": "tensor", "achieved": achieved_tf, "peak": pk["tensor"], "unit": "TFLOP/s",
                "frac": (achieved_tf / pk["tensor"]) if achieved_tf else None,
                "traffic": (traffic or {}).get("bytes_per_launch"), "traffic_unit": "bytes/launch",
                "traffic_src": (traffic or {}).get("source"),
                "kernel": "stage-2 scan (exact search)", "peak_src": pk["src"],
                "phase_ms_per_step": {k2: (v[0] / v[1] if v[1] else None) for k2, v in phases.items()},
                "step_share": (stage2_ms / stage2_n) / ms_per_step if stage2_n else None}

    # ---- GPU brute-force baseline (paper Table 3 framing) -------------------
    bf = None
    if not args.no_bf and rank == 0:
        m = 2048
        qb = q_dev[:m]
        ids_b = torch.empty((m, 1), dtype=torch.int64, device="cuda")
        d_b = torch.empty((m, 1), dtype=torch.float32, device="cuda")
        x_dev = _lib.to_device(x)
        for it in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _lib.check(_lib.lib.rbc_bf_search(_lib.ptr(qb), m, _lib.ptr(x_dev), N, D, 0, 1, _lib.ptr(ids_b),
                                              _lib.ptr(d_b), sptr), "bf")
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        bf = {"value": m / dt, "unit": "queries/s", "sample": f"{m} queries x 1M points, k=1, exact SIMT scan (rbc_bf_search)",
              "rbc_speedup": (value / world) / (m / dt)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(x, q, index)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"cfg2: exact RBC {K}-NN L2, clusters n=1M d=64 C=64 sigma=0.05, |R|=1016",
                           "queries_per_rank": NQ, "k": K, "n_reps": n_reps, "parallelism": f"query-shard x{world}",
                           "l2_flush": "256 MiB write between timed steps", "index_build_s": build_s,
                           "mean_candidates": float(cand_h.mean()), "flops_per_step": flops_per_step,
                           "step_ms_min": min(times), "step_ms_median": sorted(times)[len(times) // 2],
                           "arith": "f32 inputs; f16 tcgen05 filter; exact re-rank in f64 (reference rule)"},
                "e2e": e2e_block, "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu,
                "gpu_bruteforce": bf, "clocks": clk}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
