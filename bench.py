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

# BASELINE.json configs: the headline (default) is cfg2; the others are
# bench lines of their own (``--config cfgN``), committed under profiles/.
CONFIGS = {
    "cfg1": dict(kind="oneshot", n=10_000, d=16, nq=1_000, C=8, seed=7, n_r=100, s=100, mode="fixed-count",
                 metric="l2", k=1, workload="cfg1: one-shot RBC 1-NN L2, clusters n=10k d=16 C=8, n_r=s=100 "
                                           "(fixed-count), 1k queries"),
    "cfg2": dict(kind="exact", n=1_000_000, d=64, nq=100_000, C=64, seed=1, n_r=1000, metric="l2", k=1,
                 workload="cfg2: exact RBC 1-NN L2, clusters n=1M d=64 C=64 sigma=0.05, |R|=1016"),
    "cfg3": dict(kind="exact", n=581_012, d=54, nq=100_000, C=8, seed=3, n_r=763, metric="l2", k=10,
                 workload="cfg3: exact RBC 10-NN L2, Covertype-shaped clusters n=581,012 d=54 C=8, "
                          "n_r=763 (|R|~777), 100k queries per rank"),
    "cfg4": dict(kind="oneshot", n=2_000_000, d=21, nq=100_000, C=8, seed=4, n_r=1415, s=1415, mode="bernoulli",
                 metric="l1", k=1, workload="cfg4: one-shot RBC 1-NN L1, Robot-shaped clusters n=2M d=21 C=8, "
                                            "n_r=s=1415 (|R|~1455), 100k queries"),
    "cfg5": dict(kind="exact", n=16_000_000, d=128, nq=10_000, C=64, seed=5, n_r=4000, metric="l2", k=10,
                 rep_shard=True,
                 workload="cfg5: exact RBC 10-NN L2, clusters n=16M d=128 C=64 sigma=0.05, n_r=4000 (|R|~4000), "
                          "X sharded by representative over the GPUs (sharded build + per-query key merge), "
                          "10k queries per step served by all ranks"),
}
SIGMA, REP_SEED = 0.05, 0
CFG = CONFIGS["cfg2"]
N, D, NQ, C, DATA_SEED, NR, K = (CFG[x] for x in ("n", "d", "nq", "C", "seed", "n_r", "k"))
METRIC = "RBC queries/sec (exact 1-NN, n=1M d=64)"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def select_config(name: str, k=None):
    """Point the module-level workload constants at config `name` (k overrides its k)."""
    global CFG, N, D, NQ, C, DATA_SEED, NR, K, METRIC
    CFG = dict(CONFIGS[name])
    if k is not None:
        CFG["k"] = k
    N, D, NQ, C, DATA_SEED, NR, K = (CFG[x] for x in ("n", "d", "nq", "C", "seed", "n_r", "k"))
    kind = "exact" if CFG["kind"] == "exact" else "one-shot"
    nn = f"{N / 1e6:g}M" if N >= 1_000_000 else f"{N / 1e3:g}k"
    METRIC = f"RBC queries/sec ({kind} {K}-NN{' L1' if CFG['metric'] == 'l1' else ''}, n={nn} d={D})"
    if name == "cfg2" and K == 1:
        METRIC = "RBC queries/sec (exact 1-NN, n=1M d=64)"  # BASELINE.json's metric string


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def gen_inputs(rank: int):
    """Reference generator ``clusters`` (dataset.py:142-148): n + nq rows, X = first n, Q = the rest."""
    rng = np.random.default_rng(DATA_SEED)
    centers = rng.random((C, D))
    assignment = rng.integers(C, size=N + NQ)
    full = (centers[assignment] + SIGMA * rng.standard_normal((N + NQ, D))).astype(np.float32)
    x, q = np.ascontiguousarray(full[:N]), np.ascontiguousarray(full[N:])
    if rank > 0:
        r2 = np.random.default_rng(1000 + rank)
        q = np.ascontiguousarray((centers[r2.integers(C, size=NQ)] + SIGMA * r2.standard_normal((NQ, D))).astype(np.float32))
    return x, q


def gen_inputs_chunked(rows_per_chunk: int = 1 << 20):
    """gen_inputs for large n: the same random stream (centres, assignment, then the normals
    row-major), drawn in row chunks straight into float32 so the float64 temporaries stay small."""
    rng = np.random.default_rng(DATA_SEED)
    centers = rng.random((C, D))
    assignment = rng.integers(C, size=N + NQ)
    full = np.empty((N + NQ, D), np.float32)
    for r0 in range(0, N + NQ, rows_per_chunk):
        r1 = min(N + NQ, r0 + rows_per_chunk)
        full[r0:r1] = centers[assignment[r0:r1]] + SIGMA * rng.standard_normal((r1 - r0, D))
    return full[:N], full[N:]


def run_rep_shard(args, rank, world, local):
    """cfg5: the database sharded by representative over the ranks.  The
    build is the sharded build (each rank assigns its id slice, all-to-all to the owner
    shard); every rank searches ALL queries over its shard and the per-query top-k keys are
    merged over NCCL (all_gather + rbc_merge_topk).  value = queries / max-over-ranks time
    (strong scaling: the work per query is split over the ranks)."""
    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1103_2635_b200 as rbc
    from paper_1103_2635_b200 import _lib
    from paper_1103_2635_b200 import distributed as Dm

    x, q = gen_inputs_chunked()
    lo, hi = Dm.query_slices(N, world)[rank]
    spec = rbc.MetricSpec("l2", D)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sh = Dm.build_exact_distributed(x[lo:hi], lo, N, NR, spec, REP_SEED, rank, world)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    stream = torch.cuda.current_stream()
    sptr = ctypes.c_void_p(stream.cuda_stream)
    q_dev = _lib.to_device(q)
    keys = torch.empty((NQ, K), dtype=torch.int64, device="cuda")
    cand = torch.empty(NQ, dtype=torch.int64, device="cuda")
    stats = _lib.SearchStatsC(None, None, None, cand.data_ptr())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step():
        _lib.check(_lib.lib.rbc_exact_search_keys(sh.dev.handle, _lib.ptr(q_dev), NQ, K, _lib.ptr(keys), stats,
                                                  sptr), "shard search")
        return Dm.merge_shard_keys(keys, K)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # e2e: the Python API (numpy queries in, numpy ids/dists/stats out, merge included)
    e2e_times = []
    for i in range(1 + max(2, min(args.steps, 5))):
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        Dm.exact_query_sharded(sh, q, K)
        if i >= 1:
            e2e_times.append(time.perf_counter() - t0)
    e2e_s = statistics.median(e2e_times)
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
    # phase split of this rank's search (stage-2 scan alone = the dominant kernel)
    _lib.profile_enable(True)
    _lib.check(_lib.lib.rbc_exact_search_keys(sh.dev.handle, _lib.ptr(q_dev), NQ, K, _lib.ptr(keys), stats, sptr), "p")
    torch.cuda.synchronize()
    _lib.profile_enable(True)
    _lib.check(_lib.lib.rbc_exact_search_keys(sh.dev.handle, _lib.ptr(q_dev), NQ, K, _lib.ptr(keys), stats, sptr), "p")
    torch.cuda.synchronize()
    phases = _lib.profile_read()
    _lib.profile_enable(False)
    clk = clocks.stop()
    total_ms = sum(times)
    cand_local = float(cand.sum().item())
    if dist:
        t = torch.tensor([total_ms, e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, e2e_s = (float(v) for v in t.tolist())
        c = torch.tensor([cand_local], dtype=torch.float64, device="cuda")
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        cand_total = float(c.item())
    else:
        cand_total = cand_local
    value = NQ * args.steps / (total_ms / 1e3)
    pk = peaks()
    scan_ms = phases["scan"][0]
    scan_work = 2.0 * D * cand_local
    achieved = scan_work / (scan_ms / 1e3) / 1e12 if scan_ms > 0 else None
    roofline = {"bound": "tensor", "achieved": achieved, "peak": pk["tensor"], "unit": "TFLOP/s",
                "frac": achieved / pk["tensor"] if achieved else None, "peak_src": pk["src"], "traffic": None,
                "traffic_unit": "bytes/launch", "traffic_src": None, "kernel": f"stage2_tc_kernel<{kt_of(K)}, 2>",
                "work_per_launch": scan_work, "work_rule": "2*d*candidates on this rank (reference-rule counts)",
                "phase_ms_per_step": {k2: v[0] for k2, v in phases.items()}}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # exact RBC returns the brute-force k-NN (SPEC acceptance 1): the oracle's brute force
        # over all 16M points on the host cores, a small query sample
        from oracle import oracle as orc

        orc.build()
        m = 8
        t0 = time.perf_counter()
        orc.bf_topk(q[:m], x, K)
        dt = time.perf_counter() - t0
        cpu = {"value": m / dt, "unit": "queries/s", "cores": orc.threads(), "kind": "port",
               "sample": f"{m} of the {NQ} cfg5 queries, brute-force {K}-NN over all {N} points via "
                         "oracle/rbc_oracle.c (OpenMP) -- the oracle's RBC build of 16M x 128 takes ~10 min"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": CFG["workload"], "queries_per_step": NQ, "k": K, "n_reps": sh.n_reps,
                           "parallelism": f"rep-shard x{world}", "l2_flush": "256 MiB write between timed steps",
                           "index_build_s": build_s, "mean_candidates": cand_total / NQ,
                           "shard_points": sh.owned_points,
                           "arith": "f32 inputs; f16 tcgen05 filter (two K planes); exact re-rank in f64"},
                "e2e": {"value": NQ / e2e_s, "unit": "queries/s", "h2d_bytes_per_step": int(q.nbytes),
                        "d2h_bytes_per_step": int(NQ * K * 12 + NQ * 24),
                        "call": "distributed.exact_query_sharded (numpy in/out, NCCL merge)"},
                "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu, "gpu_bruteforce": None,
                "clocks": clk}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def kt_of(k: int) -> int:
    """Template width of the stage-2 / re-rank kernels serving k (tc_stage2.cu launch dispatch)."""
    return 1 if k == 1 else 4 if k <= 4 else 8 if k <= 8 else 10 if k == 10 else 16 if k <= 16 else 32


def ncu_traffic(kernel: str, cfg: str):
    """dram__bytes_read + dram__bytes_write per launch of exactly `kernel` (e.g. "stage2_tc_kernel<1>")
    from the newest committed ncu --set full summary for config `cfg` under profiles/, or None.
    Summary files: r<round>_ncu_[<cfg>_]v<ver>_kernels.txt (no cfg tag = cfg2)."""
    import glob
    import re
    found = []
    for path in glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_*kernels.txt")):
        m = re.match(r"r(\d+)_ncu_(?:(cfg\d)_)?v(\d+)_kernels\.txt$", os.path.basename(path))
        if m and (m.group(2) or "cfg2") == cfg:
            found.append(((int(m.group(1)), int(m.group(3))), path))
    for _, path in sorted(found, reverse=True):
        block, total = None, 0.0
        for line in open(path):
            if line.startswith("== "):
                name = line[3:].strip().split("::")[-1]
                block = name == kernel
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


def _nn_label():
    return f"{'exact' if CFG['kind'] == 'exact' else 'one-shot'} {K}-NN {CFG['metric'].upper()}"


def oracle_index(x, index):
    """The oracle's view of a built index (rep ids + lists)."""
    reps = index.reps.rep_ids
    if CFG["kind"] == "exact":
        li, off, ld = index.flat_lists()
        return (reps, li, off, ld, index.radii)
    return (reps, np.asarray(index.list_ids, np.int64))


def oracle_search(orc, x, oidx, q):
    if CFG["kind"] == "exact":
        reps, li, off, ld, radii = oidx
        return orc.exact_query(x, reps, li, off, ld, radii, q, K, metric=CFG["metric"])
    reps, lists = oidx
    return orc.one_shot_query(x, reps, lists, q, K, metric=CFG["metric"])


def cpu_baseline(x, q, index, cfg_name, budget_s=12.0):
    """The oracle (C restatement of the reference, OpenMP) on the host cores, bounded query sample."""
    from oracle import oracle as orc

    orc.build()
    oidx = oracle_index(x, index)
    m = min(256, len(q))
    t0 = time.perf_counter()
    oracle_search(orc, x, oidx, q[:m])
    dt = time.perf_counter() - t0
    m2 = int(min(len(q), max(m, m * budget_s / max(dt, 1e-3))))
    t0 = time.perf_counter()
    oracle_search(orc, x, oidx, q[:m2])
    dt = time.perf_counter() - t0
    return {"value": m2 / dt, "unit": "queries/s", "cores": orc.threads(), "kind": "port",
            "sample": f"{m2} of the {len(q)} {cfg_name} queries, {_nn_label()} via oracle/rbc_oracle.c (OpenMP)"}


def oracle_build(orc, x):
    """The reference's build on the oracle (rbc.py:147-200), timed by the caller."""
    if CFG["kind"] == "exact":
        reps = orc.bernoulli(N, NR / N, REP_SEED)
        li, off, ld, radii = orc.build_exact(x, reps, metric=CFG["metric"])
        return (reps, li, off, ld, radii)
    if CFG.get("mode") == "fixed-count":
        reps = np.sort(np.random.default_rng(REP_SEED).choice(N, size=NR, replace=False)).astype(np.int64)
    else:
        reps = orc.bernoulli(N, NR / N, REP_SEED)
    lists, _ = orc.build_one_shot(x, reps, CFG["s"], metric=CFG["metric"])
    return (reps, lists)


def run_reference(args, rank, world, cfg_name):
    """--impl reference: the reference algorithm's CPU restatement (oracle) on this host's cores."""
    if rank != 0:
        return
    from oracle import oracle as orc

    orc.build()
    x, q = gen_inputs(0)
    t0 = time.perf_counter()
    oidx = oracle_build(orc, x)
    build_s = time.perf_counter() - t0
    per_step = min(1024, NQ)
    times = []
    for step in range(args.warmup + args.steps):
        lo = (step * per_step) % max(1, NQ - per_step)
        t0 = time.perf_counter()
        oracle_search(orc, x, oidx, q[lo: lo + per_step])
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
    value = per_step * len(times) / sum(times)
    line = {"metric": METRIC, "value": value, "unit": "queries/s", "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CFG["workload"], "queries_per_step": per_step, "k": K, "index_build_s": build_s},
            "cpu_baseline": {"value": value, "unit": "queries/s", "cores": orc.threads(), "kind": "port",
                             "sample": f"{per_step} queries per step, {_nn_label()} (oracle/rbc_oracle.c, OpenMP); "
                                       "the Python reference itself measured 233.9 q/s on 8 cores for cfg2 "
                                       "(SURVEY.md §6.3)"},
            "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def simt_peak_gops(sm_mhz):
    """fp32 SIMT lane-op peak: 148 SMs x 128 lanes x clock (SURVEY.md §8d, L1 roofline)."""
    return 148 * 128 * (sm_mhz or 1965.0) * 1e6 / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS), help="BASELINE.json config (default cfg2)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-bf", action="store_true")
    ap.add_argument("--k", type=int, default=None, help="neighbours per query (default: the config's k)")
    args = ap.parse_args()
    select_config(args.config, args.k)
    exact = CFG["kind"] == "exact"

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world, args.config)
    if CFG.get("rep_shard"):
        return run_rep_shard(args, rank, world, local)

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
    spec = rbc.MetricSpec(CFG["metric"], D)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if exact:
        index = rbc.build_exact(data, NR, spec, seed=REP_SEED)
    else:
        index = rbc.build_one_shot(data, NR, CFG["s"], spec, seed=REP_SEED, mode=CFG["mode"])
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    dev = index._dev
    n_reps = index.reps.size

    stream = torch.cuda.current_stream()
    sptr = ctypes.c_void_p(stream.cuda_stream)
    q_dev = _lib.to_device(q)
    keys = torch.empty((NQ, K), dtype=torch.int64, device="cuda")
    ids_d = torch.empty((NQ, K), dtype=torch.int64, device="cuda")
    dists_d = torch.empty((NQ, K), dtype=torch.float32, device="cuda")
    gamma = torch.empty(NQ, dtype=torch.float32, device="cuda")
    prr = torch.empty(NQ, dtype=torch.int32, device="cuda")
    p3 = torch.empty(NQ, dtype=torch.int32, device="cuda")
    cand = torch.empty(NQ, dtype=torch.int64, device="cuda")
    stats = _lib.SearchStatsC(gamma.data_ptr(), prr.data_ptr(), p3.data_ptr(), cand.data_ptr())
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def step():
        if exact:
            _lib.check(_lib.lib.rbc_exact_search_keys(dev.handle, _lib.ptr(q_dev), NQ, K, _lib.ptr(keys), stats,
                                                      sptr), "exact search")
        else:
            _lib.check(_lib.lib.rbc_one_shot_search(dev.handle, _lib.ptr(q_dev), NQ, K, _lib.ptr(ids_d),
                                                    _lib.ptr(dists_d), _lib.ptr(gamma), sptr), "one-shot search")

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

    def host_call():
        if exact:
            _lib.check(_lib.lib.rbc_exact_search_host(dev.handle, ctypes.c_void_p(q_pin.data_ptr()), NQ, K,
                                                      ctypes.c_void_p(ids_h.data_ptr()),
                                                      ctypes.c_void_p(dists_h.data_ptr()),
                                                      _lib.SearchStatsC(None, None, None, None), sptr), "e2e")
        else:
            _lib.check(_lib.lib.rbc_one_shot_search_host(dev.handle, ctypes.c_void_p(q_pin.data_ptr()), NQ, K,
                                                         ctypes.c_void_p(ids_h.data_ptr()),
                                                         ctypes.c_void_p(dists_h.data_ptr()), None, sptr), "e2e")

    e2e_times = []
    for i in range(args.warmup + max(3, args.steps // 2)):
        t0 = time.perf_counter()
        host_call()
        if i >= args.warmup:
            e2e_times.append(time.perf_counter() - t0)
    # the drop-in Python API itself (numpy queries in, numpy ids/dists/stats out)
    api_times = []
    for i in range(2 + 5):
        t0 = time.perf_counter()
        if exact:
            rbc.exact_query_arrays(index, q, K)
        else:
            rbc.one_shot_query_arrays(index, q, K)
        if i >= 2:
            api_times.append(time.perf_counter() - t0)
    # the reference-shaped call (list[NeighborList], list[SearchStats]: one dataclass pair per query)
    nb = min(NQ, 10_000)
    batch_times = []
    for i in range(1 + 3):
        t0 = time.perf_counter()
        if exact:
            rbc.exact_query_batch(index, q[:nb], K)
        else:
            rbc.one_shot_query_batch(index, q[:nb], K)
        if i >= 1:
            batch_times.append(time.perf_counter() - t0)
    os.sched_setaffinity(0, old_aff)
    # median: the host call's wall time carries OS scheduling noise; min/median/max go to stderr
    e2e_s = statistics.median(e2e_times)
    api_s = statistics.median(api_times)
    log(f"e2e host cpus: {len(local_cpus) if local_cpus else 'unrestricted'}; per-call ms: "
        + " ".join(f"{1e3 * t:.2f}" for t in e2e_times))
    log(f"e2e ms: min {1e3 * min(e2e_times):.3f} median {1e3 * e2e_s:.3f} max {1e3 * max(e2e_times):.3f} "
        f"(n={len(e2e_times)}); python API ms: " + " ".join(f"{1e3 * t:.2f}" for t in api_times))
    if dist:
        t = torch.tensor([e2e_s, api_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s, api_s = (float(v) for v in t.tolist())
    e2e_block = {"value": world * NQ / e2e_s, "unit": "queries/s", "h2d_bytes_per_step": int(q.nbytes),
                 "d2h_bytes_per_step": int(ids_h.numel() * 8 + dists_h.numel() * 4),
                 "api": {"value": world * NQ / api_s, "unit": "queries/s",
                         "call": ("exact_query_arrays" if exact else "one_shot_query_arrays")
                         + " (numpy in, numpy ids/dists/stats out; pageable host memory)"},
                 "api_batch": {"value": nb / statistics.median(batch_times), "unit": "queries/s",
                               "sample": f"{nb} queries per call",
                               "call": ("exact_query_batch" if exact else "one_shot_query_batch")
                               + " (the reference's return types: a NeighborList and SearchStats per query)"}}

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
    # phase split from a separate pass with the CUDA-event phase timers on (recorded on the
    # launching stream around each kernel group; "scan" brackets the dominant kernel alone:
    # stage2_tc_kernel for the exact search, the list scan for one-shot).  The timers force
    # direct launches (no graph replay), so they stay out of the timed loop above
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
    pk = peaks()
    scan_ms, scan_n = phases["scan"]
    if exact:
        cand_h = cand.cpu().numpy().astype(np.float64)
        mean_cand = float(cand_h.mean())
    else:
        mean_cand = float(CFG["s"])
    evals = NQ * (n_reps + mean_cand)
    flops_per_step = 2.0 * D * evals
    scan_work = 2.0 * D * NQ * mean_cand  # the dominant kernel's algorithmic work per launch
    if CFG["metric"] == "l2":
        kname = f"stage2_tc_kernel<{kt_of(K)}, {1 if D <= 64 else 2}>" if exact else f"oneshot scan (k={K})"
        traffic = ncu_traffic(kname, args.config)
        achieved = scan_work * scan_n / (scan_ms / 1e3) / 1e12 if scan_ms > 0 else None
        roofline = {"bound": "tensor", "achieved": achieved, "peak": pk["tensor"], "unit": "TFLOP/s",
                    "frac": (achieved / pk["tensor"]) if achieved else None, "peak_src": pk["src"]}
    else:
        # the one-shot list scan on the fp32 SIMT filter engine (simt_scan.cu simt_tile_kernel<metric,
        # DMAX, KT, QPT>; grouped items use one query per lane when the mean group is below 96)
        dmax = 24 if D <= 24 else 64 if D <= 64 else 128
        kt = 1 if K <= 1 else 4 if K <= 4 else 16 if K <= 16 else 32
        qpt = 2 if (D <= 64 and K <= 16 and NQ >= 96 * n_reps) else 1
        kname = f"simt_tile_kernel<1, {dmax}, {kt}, {qpt}>"
        traffic = ncu_traffic(kname, args.config)
        achieved = scan_work * scan_n / (scan_ms / 1e3) / 1e9 if scan_ms > 0 else None
        peak = simt_peak_gops((clk or {}).get("sm_mhz"))
        roofline = {"bound": "simt", "achieved": achieved, "peak": peak, "unit": "Glane-op/s",
                    "frac": (achieved / peak) if achieved else None,
                    "peak_src": "148 SMs x 128 fp32 lanes x measured SM clock"}
    roofline.update({
        "traffic": (traffic or {}).get("bytes_per_launch"), "traffic_unit": "bytes/launch",
        "traffic_src": (traffic or {}).get("source"), "kernel": kname,
        "work_per_launch": scan_work, "work_rule": "2*d*candidates (reference-rule counts from SearchStats)",
        "phase_ms_per_step": {k2: (v[0] / v[1] if v[1] else None) for k2, v in phases.items()},
        "step_share": (scan_ms / scan_n) / ms_per_step if scan_n else None})

    # ---- GPU brute-force baseline (paper Table 3 framing) -------------------
    bf = None
    if not args.no_bf and rank == 0:
        # one full wave of 128-query tiles (148 SMs); the operand is prepared once (rbc_bf_prepare:
        # the points partitioned into f16 residual lists) and every search scans all of it
        m = min(NQ, 148 * 128)
        qb = q_dev[:m]
        ids_b = torch.empty((m, K), dtype=torch.int64, device="cuda")
        d_b = torch.empty((m, K), dtype=torch.float32, device="cuda")
        x_dev = _lib.to_device(x)
        metric_code = 0 if CFG["metric"] == "l2" else 1
        bfh = ctypes.c_void_p()
        torch.cuda.synchronize()
        t_prep = time.perf_counter()
        _lib.check(_lib.lib.rbc_bf_prepare(_lib.ptr(x_dev), N, D, metric_code, ctypes.byref(bfh), sptr), "bf prepare")
        torch.cuda.synchronize()
        t_prep = time.perf_counter() - t_prep
        launches0, simt0 = _lib.lib.rbc_tc_bf_calls(), _lib.lib.rbc_simt_scan_calls()
        bf_times = []
        for it in range(3):
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            _lib.check(_lib.lib.rbc_bf_search_prepared(bfh, _lib.ptr(qb), m, K, _lib.ptr(ids_b), _lib.ptr(d_b), sptr),
                       "bf")
            ev1.record(stream)
            ev1.synchronize()
            bf_times.append(ev0.elapsed_time(ev1) / 1e3)
        dt = statistics.median(bf_times[1:])
        tc_used = _lib.lib.rbc_tc_bf_calls() > launches0
        simt_used = _lib.lib.rbc_simt_scan_calls() > simt0
        _lib.lib.rbc_index_destroy(bfh)
        bf_flops = 2.0 * D * m * N  # algorithmic: every (query, point) pair, 2 d flops
        bf = {"value": m / dt, "unit": "queries/s",
              "sample": f"{m} queries x {N} points, k={K}, rbc_bf_search_prepared (bf_search over a prepared "
                        f"operand), device-resident",
              "engine": ("tcgen05 f16 filter + exact fp64 re-rank" if tc_used else
                         "fp32 SIMT filter + exact fp64 re-rank" if simt_used else "exact fp64 SIMT"),
              "prepare_s": t_prep, "ms": dt * 1e3, "achieved_tflops": bf_flops / dt / 1e12,
              "frac_of_peak": (bf_flops / dt / 1e12 / pk["tensor"] if CFG["metric"] == "l2" else
                               bf_flops / dt / 1e9 / simt_peak_gops((clk or {}).get("sm_mhz"))),
              "rbc_speedup": (value / world) / (m / dt)}
        del x_dev

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(x, q, index, args.config)

    if rank == 0:
        cfg = {"workload": CFG["workload"], "queries_per_rank": NQ, "k": K, "n_reps": n_reps,
               "parallelism": f"query-shard x{world}", "l2_flush": "256 MiB write between timed steps",
               "index_build_s": build_s, "mean_candidates": mean_cand, "flops_per_step": flops_per_step,
               "step_ms_min": min(times), "step_ms_median": sorted(times)[len(times) // 2],
               "arith": ("f32 inputs; f16 tcgen05 filter; exact re-rank in f64 (reference rule)"
                         if CFG["metric"] == "l2" else
                         "f32 inputs; fp32 SIMT filter; exact re-rank in f64 (reference rule)")}
        if not exact:
            cfg["s"] = CFG["s"]
        line = {"metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
                "e2e": e2e_block, "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu,
                "gpu_bruteforce": bf, "clocks": clk}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
