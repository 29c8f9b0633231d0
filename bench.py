#!/usr/bin/env python3
"""Benchmark of the B200 RESCAL MU hot path (contract: see DESIGN.md §Measurement).

A "step" is one MU iteration (rescal.py:114-146 + the tracked relative error of
rescal.py:218-222) over the whole synthetic tensor. Workloads (BASELINE.json
configs):
  cfg3 (default): dense m=16, n=32768, k=32 -- the north_star target; at N>1
                  the same tensor on the 1x2 / 2x2 / 2x4 grid ("scaling":
                  "strong").
  cfg2          : dense m=16, n=8192, k=16 per GPU. At N>1 the global tensor
                  grows to n = 8192*sqrt(N) on the p_r x p_c grid so every GPU
                  holds one cfg2-sized block (the paper's weak-scaling setup,
                  PAPER.md:1027-1030); value counts block-iterations
                  (= N per global iteration) -> "scaling": "weak".
  cfg4          : sparse m=32, n=2^20, density 1e-5, k=16 (CSR/CSC engine), untracked.
  cfg5          : RESCALk (rescalk()) dense m=8, n=16384, r=10 members per k, 200
                  iterations each, k in [--k-min, --k-max] (default 15..16 of the
                  full 2..16 sweep); members spread over the N GPUs as replicas.
                  A step = one member MU iteration; value = member-iterations/s.
  cfg1          : dense m=8, n=256, k=4 (latency-bound).

Launch: python bench.py [--gpus N --steps K --warmup W]. For N>1 either under
        torchrun (one rank per GPU) or plainly: bench.py then starts its own N
        rank processes (RANK / LOCAL_RANK / WORLD_SIZE, rendezvous on
        127.0.0.1) and rank 0 prints the line.
        python bench.py --impl reference ...  (CPU reference arm; rank 0 only)
At N=1 the default run also times cfg1, cfg2 and cfg4 on the device
(`secondary`, short runs; --no-secondary skips them).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "cfg1": dict(m=8, n=256, k=4),
    "cfg2": dict(m=16, n=8192, k=16),
    "cfg3": dict(m=16, n=32768, k=32),
    "cfg4": dict(m=32, n=1 << 20, k=16, density=1e-5),
    "cfg5": dict(m=8, n=16384, k=16, k_min=15, k_max=16, r=10, iters=200),
}
METRIC = "MU iters/sec + effective TFLOP/s (dense) / HBM GB/s (sparse) at 1/2/4/8 B200"
SEED = 20220218


# measured random 64-B-row gather ceiling of one B200 (LDG.128, 4 lanes/row, 2^27 rows
# from a 67 MB table; profiles/r01s3_gather_ceiling.log)
GATHER_CEILING_GROWS = 145.2


def ncu_traffic(config, world):
    """dram read+write bytes per launch of the dominant kernel from the committed
    ncu --set full capture (profiles/ncu_traffic.json; single-GPU captures)."""
    if world != 1:
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            e = json.load(f).get(config)
        return None if e is None else float(e["dram_read_bytes"] + e["dram_write_bytes"])
    except Exception:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.lines = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        # wait for the first sample so the sampler is live before the timed region
        t0 = time.perf_counter()
        while self.proc and not self.lines and time.perf_counter() - t0 < 5.0:
            time.sleep(0.02)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# distributed plumbing


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend="gloo")
        return dist, dist.get_rank(), world, int(os.environ.get("LOCAL_RANK", "0"))
    return None, 0, 1, 0


def spawn_ranks(n):
    """`python bench.py --gpus N` without torchrun: start N rank processes of
    this same command (one per GPU, rendezvous on 127.0.0.1) and wait for them.
    Rank 0 prints the JSON line; the exit code is the worst of the ranks'."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env))
    rc = 0
    for pr in procs:
        rc = max(rc, pr.wait())
    return rc


def max_over_ranks(dist, v):
    if dist is None:
        return v
    import torch

    t = torch.tensor([float(v)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


def workload(name, world):
    c = dict(CONFIGS[name])
    if name == "cfg2" and world > 1:
        c["n"] = int(round(8192 * math.sqrt(world)))
    return c


def grid_of(world):
    pr = int(math.isqrt(world))
    while world % pr:
        pr -= 1
    return pr, world // pr


def units_per_iteration(name, world):
    """cfg2 at N>1 is weak scaling: one global iteration = N block-iterations."""
    return world if (name == "cfg2" and world > 1) else 1


def config_dict(name, world):
    """The `config` object of the JSON line; identical for both arms."""
    c = workload(name, world)
    m, n, k = c["m"], c["n"], c["k"]
    pr, pc = grid_of(world)
    sparse = "density" in c
    if sparse:
        wl = f"{name}: sparse m={m} n={n} density={c['density']} k={k}"
    else:
        wl = f"{name}: dense m={m} n={n} k={k}"
    if world > 1:
        wl += f", {pr}x{pc} grid, per-GPU block {n // pr}x{n // pc} (+padding)"
    return {
        "workload": wl,
        "per_step": "one MU iteration (rescal.py:114-146), untracked; tracked rate in `tracked`",
        "l2": ("inputs larger than L2: CSR+CSC streams >> 0.126 GB" if sparse else
               f"inputs larger than L2 ({4.0 * m * n * n / world / 1e9:.1f} GB of X per GPU vs 0.126 GB)"),
        "grid": f"{pr}x{pc}", "parallelism": f"p_r x p_c = {pr}x{pc}",
        "engine": "csr-gather" if sparse else ("tcgen05" if k <= 32 else "simt"),
    }


# ---------------------------------------------------------------------------
# CPU side (oracle = reference algorithm restated; the only place bench runs it)


def host_tensor(m, n, pinned=False):
    """The exact fp32 values the device generator (rk_fill_uniform) produces."""
    from paper_2202_09512_b200 import _lib

    total = m * n * n
    if pinned:
        import torch

        buf = torch.empty(total, dtype=torch.float32, pin_memory=True).numpy()
    else:
        buf = np.empty(total, dtype=np.float32)
    step = 1 << 28
    for off in range(0, total, step):
        cnt = min(step, total - off)
        buf[off:off + cnt] = _lib.uniform_values(SEED, off, cnt)
    return buf.reshape(m, n, n)


def cpu_reference(x32, k, m, budget_s=12.0, max_slices=None):
    """Time oracle.mu_iteration (fp64, numpy/OpenBLAS on all host cores) on a
    bounded sample of the first slices of the workload (x32 holds them);
    returns (it/s scaled to all m slices, cores, sample, step seconds)."""
    import oracle

    n = x32.shape[1]
    cores = len(os.sched_getaffinity(0))
    # slices per step: aim for ~budget/4 seconds per step from a 1-slice probe
    a, r = oracle.random_init(n, k, m, 0)
    probe = [x32[0].astype(np.float64)]
    t0 = time.perf_counter()
    oracle.mu_iteration(probe, a.copy(), r[:1].copy(), 1e-16)
    per_slice = max(time.perf_counter() - t0, 1e-6)
    ms = max(1, min(x32.shape[0], int((budget_s / 4) / per_slice)))
    if max_slices:
        ms = min(ms, max_slices)
    xs = [x32[t].astype(np.float64) for t in range(ms)]
    times = []
    t_start = time.perf_counter()
    while len(times) < 2 or (time.perf_counter() - t_start < budget_s and len(times) < 20):
        rr = r[:ms].copy()
        t0 = time.perf_counter()
        oracle.mu_iteration(xs, a.copy(), rr, 1e-16)
        times.append(time.perf_counter() - t0)
    t_step = statistics.median(times)
    it_s = 1.0 / (t_step * m / ms)
    sample = (f"oracle.mu_iteration fp64 (untracked, rescal.py:114-146 restated), {ms} of {m} slices "
              f"n={n} k={k}, median of {len(times)} reps, scaled x{m / ms:.2f} to all slices")
    return it_s, cores, sample, t_step


def cpu_reference_sparse(n, m, k, density, budget_s=12.0):
    """oracle.mu_iteration (scipy CSR, fp64) on a bounded sample of slices of
    the same synthetic sparse tensor; scaled to all m slices."""
    import oracle
    import scipy.sparse as sps
    from paper_2202_09512_b200 import _lib

    cores = len(os.sched_getaffinity(0))
    e = _lib.Engine(n, min(m, 2), k, sparse=True)
    e.fill_sparse_uniform(SEED, int(round(density * n * n)))
    ptr, idx, val = e.csr_arrays()
    e.close()
    xs = [sps.csr_matrix((val[ptr[t, 0]:ptr[t, -1]].astype(np.float64), idx[ptr[t, 0]:ptr[t, -1]],
                          ptr[t] - ptr[t, 0]), shape=(n, n)) for t in range(ptr.shape[0])]
    a, r = oracle.random_init(n, k, len(xs), 0)
    times = []
    t_start = time.perf_counter()
    while len(times) < 1 or (time.perf_counter() - t_start < budget_s and len(times) < 5):
        t0 = time.perf_counter()
        oracle.mu_iteration(xs, a.copy(), r.copy(), 1e-16)
        times.append(time.perf_counter() - t0)
    t_step = statistics.median(times)
    it_s = 1.0 / (t_step * m / len(xs))
    sample = (f"oracle.mu_iteration fp64 on {len(xs)} of {m} CSR slices (n={n}, nnz/slice~{idx.size // len(xs)}, "
              f"k={k}; scipy sparsetools), median of {len(times)} reps, scaled x{m / len(xs):.0f}")
    return it_s, cores, sample


# ---------------------------------------------------------------------------


def run_reference(args, world):
    """CPU reference arm: the oracle's restatement of _mu_iteration (fp64
    numpy/OpenBLAS on every host core), rank 0 only, each step a bounded sample
    of the workload's slices scaled to the full tensor."""
    c = workload(args.config, world)
    m, n, k = c["m"], c["n"], c["k"]
    threads = len(os.sched_getaffinity(0))
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ.setdefault(var, str(threads))
    import oracle

    units = units_per_iteration(args.config, world)
    line = {"impl": "reference", "metric": METRIC, "unit": "it/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True,
            "scaling": "weak" if units > 1 else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic uniform [0,1) (fp32-representable)", "config": config_dict(args.config, world)}
    per_step = max(2.0, 120.0 / max(1, args.steps + args.warmup))
    rng = np.random.default_rng(SEED)
    if "density" in c:
        it_s, cores, sample = cpu_reference_sparse(n, m, k, c["density"], budget_s=min(30.0, per_step * 4))
        t_full = 1.0 / it_s
    else:
        a, r = oracle.random_init(n, k, m, 0)
        # a bounded sample of the workload: ms slices of the full n x n tensor
        probe = rng.random((1, n, n), dtype=np.float32).astype(np.float64)
        t0 = time.perf_counter()
        oracle.mu_iteration([probe[0]], a.copy(), r[:1].copy(), 1e-16)
        per_slice = time.perf_counter() - t0
        del probe
        cap = max(1, int(24e9 // (8 * n * n)))  # host memory: <= 24 GB of fp64 slices
        ms = max(1, min(m, cap, int(per_step / max(per_slice, 1e-6))))
        x = [rng.random((n, n), dtype=np.float32).astype(np.float64) for _ in range(ms)]
        for _ in range(args.warmup):
            oracle.mu_iteration(x, a.copy(), r[:ms].copy(), 1e-16)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            oracle.mu_iteration(x, a.copy(), r[:ms].copy(), 1e-16)
        dt = time.perf_counter() - t0
        t_full = dt / args.steps * (m / ms)
        cores = threads
        sample = (f"each step: oracle.mu_iteration fp64 untracked on {ms} of {m} slices "
                  f"(n={n}, k={k}); time scaled x{m / ms:.2f} to the full tensor")
    value = units / t_full
    line.update({"value": value, "ms_per_step": t_full * 1e3,
                 "tflops_effective": 4.0 * m * n * n * k * value / units / 1e12 if "density" not in c else None,
                 "cpu_baseline": {"value": value, "unit": "it/s", "cores": cores, "kind": "port", "sample": sample},
                 "e2e": {"value": value, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
    print(json.dumps(line), flush=True)


def measure_device(name, world, steps, warmup, local_rank, dist, tracked=True, clocks=True):
    """Device-resident timing of `steps` MU iterations of workload `name`
    (X generated on the device; CUDA events on the engine stream, max over
    ranks). Returns a dict of the measured quantities."""
    import paper_2202_09512_b200 as rk
    from paper_2202_09512_b200 import _lib
    from paper_2202_09512_b200.multigpu import make_grid_engine

    c = workload(name, world)
    m, n, k = c["m"], c["n"], c["k"]
    sparse = "density" in c
    cfg = rk.SolverConfig(max_iters=steps, device=local_rank)
    f0 = rk.random_init(n, k, m, 0)
    eps = float(cfg.epsilon)
    if world > 1:
        eng, info = make_grid_engine(n, m, k, cfg=cfg, sparse=sparse)
    else:
        eng, info = _lib.Engine(n, m, k, device=local_rank, sparse=sparse), None
    out = {"nnz": 0}
    try:
        if sparse:
            eng.fill_sparse_uniform(SEED, int(round(c["density"] * n * n)))
            out["nnz"] = eng.nnz
        else:
            eng.fill_uniform(SEED)
        eng.set_factors(f0.A, f0.R)
        t_w = time.perf_counter()
        eng.run(warmup, eps, track_error=False)
        per_it = (time.perf_counter() - t_w) / max(1, warmup)
        # a short timed region falls between two 100 ms clock samples: the
        # sampler then also covers an untimed soak of the same iteration
        soak = 0 if per_it * steps >= 0.5 else min(20000, int(0.4 / max(per_it, 1e-6)) + 1)
        soak = int(max_over_ranks(dist, soak))  # grid ranks must run the same iteration count
        sampler = ClockSampler(local_rank) if clocks else None
        if sampler:
            sampler.__enter__()
        try:
            if soak:
                eng.set_factors(f0.A, f0.R)
                eng.run(soak, eps, track_error=False)
            # the timed run: graph-replayed production path, untracked
            eng.set_factors(f0.A, f0.R)
            barrier(dist)
            t_wall = time.perf_counter()
            eng.run(steps, eps, track_error=False)
            out["wall_s"] = time.perf_counter() - t_wall
            out["run_ms"] = max_over_ranks(dist, eng.timing()["run_ms"])
            out["launches"] = eng.timing()["launches"]
        finally:
            if sampler:
                sampler.__exit__(None, None, None)
        out["clocks"] = sampler.summary() if sampler else None
        out["soak"] = soak
        # per-launch CUDA events around the dominant kernel (separate run:
        # the events split the graph into per-iteration launches)
        eng.set_factors(f0.A, f0.R)
        eng.set_option(1, 1)
        barrier(dist)
        eng.run(steps, eps, track_error=False)
        tm = eng.timing()
        out["profiled_run_ms"] = max_over_ranks(dist, tm["run_ms"])
        out["k1_ms"] = max_over_ranks(dist, tm["k1_ms"])
        eng.set_option(1, 0)
        out["info"] = eng.info()
        if tracked and not sparse:
            eng.set_factors(f0.A, f0.R)
            barrier(dist)
            _, tr_t = eng.run(steps, eps, track_error=True)
            out["tracked_ms"] = max_over_ranks(dist, eng.timing()["run_ms"])
            out["trace_last"] = float(tr_t[-1]) if len(tr_t) else None
    finally:
        eng.close()
    if info is not None and not sparse:
        out["elems"] = m * info["rows"] * info["cols"]
        out["block"] = (info["rows"], info["cols"])
    else:
        out["elems"] = m * n * n
    return out


def roofline_of(name, world, d, hbm_peak, peak_kind):
    c = workload(name, world)
    m, n, k = c["m"], c["n"], c["k"]
    sparse = "density" in c
    if sparse:
        # CSR pass: stream indices + values (8 B/nnz) + int64 row pointers, write P
        k_pad = 16 if k <= 16 else 32
        bytes_k1 = 8.0 * d["nnz"] + 8.0 * m * (n + 1) + 4.0 * m * n * k_pad
    else:
        # the local block's X planes read once (hi+lo bf16 = 4 B per element)
        bytes_k1 = 4.0 * d["elems"]
    achieved = bytes_k1 / (d["k1_ms"] / 1e3) / 1e9
    return {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
            "traffic": ncu_traffic(name, world),
            "kernel": ("sp_csr_pass (P = X A, CSR, A rows gathered from L2)" if sparse else
                       "k1_tc_kernel (P = X A, Q = X^T A, 3xBF16 tcgen05)"), "peak_kind": peak_kind,
            "bytes_per_launch": bytes_k1, "k1_ms": d["k1_ms"],
            "k1_share_of_step": d["k1_ms"] / (d["profiled_run_ms"] / max(1, d.get("steps", 1)))
            if d.get("profiled_run_ms") else None}


def run_ours(args, dist, rank, world, local_rank):
    import paper_2202_09512_b200 as rk
    from paper_2202_09512_b200 import _lib

    name = args.config
    c = workload(name, world)
    m, n, k = c["m"], c["n"], c["k"]
    hbm_peak, bf16_peak, peak_kind = peaks()
    sparse = "density" in c
    units = units_per_iteration(name, world)

    # ---------------- device-resident timed region --------------------------
    d = measure_device(name, world, args.steps, args.warmup, local_rank, dist)
    d["steps"] = args.steps
    value = units * args.steps / (d["run_ms"] / 1e3)
    flops_iter = 4.0 * m * n * n * k if not sparse else 4.0 * d["nnz"] * k
    line = {
        "metric": METRIC, "value": value, "unit": "it/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": d["run_ms"] / args.steps, "higher_is_better": True,
        "scaling": "weak" if units > 1 else "strong",
        "vs_baseline": None, "dtype": "f32" if sparse else "3xbf16-split",
        "precision": ("CSR/CSC values and A in fp32, fp32 accumulate per nonzero row; k x k updates fp64"
                      if sparse else
                      "3xBF16 split (north_star's fp32-accurate split precision): X = Xh + Xl and "
                      "A = Ah + Al as bf16 pairs, products Xh*Ah + Xh*Al + Xl*Ah on tcgen05 with fp32 "
                      "TMEM accumulation; every k x k step in fp64"),
        "data": ("synthetic uniform-random (i,j) pattern, values U(0,1], device-generated, canonical CSR"
                 if sparse else "synthetic uniform [0,1) fp32-representable, device-generated"),
        "config": config_dict(name, world),
        "tflops_effective": flops_iter * args.steps / (d["run_ms"] / 1e3) / 1e12,
        "roofline": roofline_of(name, world, d, hbm_peak, peak_kind),
        "gpu_launches": int(d["launches"]),
        "gather_ceiling": ({
            "note": "the sparse pass gathers one A row (64 B, its own 128 B line) per stored entry; the "
                    "LSU/L1TEX path retires ~2.0 cycles per random line per SM whatever the load width "
                    "or the table size (8-67 MB); TMA gather4 / cp.async.bulk are ~10x slower "
                    "(tools/tma_gather_bench.cu, profiles/r01s3_gather_ceiling.log)",
            "rows_per_launch": float(d["nnz"]), "achieved_grows_s": d["nnz"] / (d["k1_ms"] / 1e3) / 1e9,
            "ceiling_grows_s": GATHER_CEILING_GROWS,
            "frac": d["nnz"] / (d["k1_ms"] / 1e3) / 1e9 / GATHER_CEILING_GROWS} if sparse else None),
        "tracked": ({"value": units * args.steps / (d["tracked_ms"] / 1e3), "unit": "it/s", "ms_total": d["tracked_ms"],
                     "note": "track_error=True: per-iteration rel. error + 1 trace-only tail pass per solve",
                     "trace_last": d["trace_last"]} if "tracked_ms" in d else None),
        "clocks": {**(d["clocks"] or {}), "window": (f"untimed soak of {d['soak']} iterations + the timed region"
                                                    if d["soak"] else "the timed region")},
        "device_ms": {"timed_run": d["run_ms"], "profiled_run": d["profiled_run_ms"], "wall_s": d["wall_s"],
                      "note": "value = the timed (graph-replayed) run; k1_ms from the profiled run "
                              "(per-launch CUDA events around K1)"},
    }
    if world > 1:
        line["exchange"] = ("peer-memory (NVLink IPC, fused into the numerator / A-update kernels)"
                            if d["info"].get("peer_exchange") else "nccl")

    # ---------------- end to end through the public API (host buffers) ------
    if not args.no_e2e:
        try:
            line["e2e"] = e2e_leg(args, dist, rank, world, local_rank, units)
        except Exception as exc:  # report, never hide
            line["e2e"] = {"value": None, "unit": "it/s", "error": repr(exc)[:300],
                           "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}

    # ---------------- secondary configs (device-timed, N=1 default run) ------
    if world == 1 and not args.no_secondary and name == "cfg3":
        sec = {}
        for nm, st in (("cfg1", 2000), ("cfg2", 100), ("cfg4", 20)):
            try:
                dd = measure_device(nm, 1, st, 5, local_rank, None, tracked=False, clocks=True)
                dd["steps"] = st
                cc = workload(nm, 1)
                sec[nm] = {"workload": config_dict(nm, 1)["workload"], "value": st / (dd["run_ms"] / 1e3),
                           "unit": "it/s", "steps": st, "ms_per_step": dd["run_ms"] / st,
                           "roofline": roofline_of(nm, 1, dd, hbm_peak, peak_kind),
                           "clocks": dd["clocks"], "gpu_launches": int(dd["launches"]),
                           "nnz": dd["nnz"] if "density" in cc else None}
            except Exception as exc:
                sec[nm] = {"error": repr(exc)[:300]}
        try:  # cfg5: the public rescalk() on k = 15..16 of the sweep (20 members x 200 iterations)
            import paper_2202_09512_b200 as rk

            c5 = CONFIGS["cfg5"]
            xh = host_tensor(c5["m"], c5["n"], pinned=True)
            x5 = rk.RelTensor(xh)
            t0 = time.perf_counter()
            rep = rk.rescalk(x5, c5["k_min"], c5["k_max"], c5["r"], cfg=rk.SolverConfig(max_iters=c5["iters"],
                                                                                        device=local_rank),
                             pcfg=rk.PerturbConfig(delta=0.02, base_seed=0))
            secs = time.perf_counter() - t0
            units5 = (c5["k_max"] - c5["k_min"] + 1) * c5["r"] * c5["iters"]
            sec["cfg5"] = {"workload": f"cfg5: rescalk dense m={c5['m']} n={c5['n']} k={c5['k_min']}..{c5['k_max']} "
                                       f"r={c5['r']} iters={c5['iters']} (public API, host tensor, incl. upload, "
                                       "resampling, clustering, refit)",
                           "value": units5 / secs, "unit": "member-it/s", "seconds": secs, "k_opt": rep.k_opt}
            del x5, xh
        except Exception as exc:
            sec["cfg5"] = {"error": repr(exc)[:300]}
        line["secondary"] = sec

    # ---------------- CPU baseline (rank 0, N=1 only) -----------------------
    if world == 1 and rank == 0 and not args.no_cpu:
        threads = len(os.sched_getaffinity(0))
        try:
            if sparse:
                it_s, cores, sample = cpu_reference_sparse(n, m, k, c["density"], budget_s=args.cpu_budget)
            else:
                xs = host_tensor(min(m, 2), n, pinned=False)
                it_s, cores, sample, t_step = cpu_reference(xs, k, m, budget_s=args.cpu_budget)
            line["cpu_baseline"] = {"value": it_s, "unit": "it/s", "cores": cores, "kind": "port",
                                    "sample": sample}
        except Exception as exc:
            line["cpu_baseline"] = {"value": None, "unit": "it/s", "cores": threads, "kind": "port",
                                    "sample": f"failed: {exc!r}"[:300]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    barrier(dist)


def gpu_local_cpus(dev):
    """The host CPUs NVML reports as local to CUDA device ``dev`` (its NUMA
    node), within this process's affinity; None when unknown."""
    try:
        import pynvml
        import torch

        p = torch.cuda.get_device_properties(dev)
        bus = "%08x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, ((os.cpu_count() or 64) + 63) // 64)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1}
        cpus &= os.sched_getaffinity(0)
        return cpus or None
    except Exception:
        return None


def e2e_leg(args, dist, rank, world, local_rank, units):
    """e2e with the process bound to the GPU's local CPUs while the pinned
    host input is allocated (first touch places its pages on the GPU's NUMA
    node) and the timed call runs -- as a NUMA-aware caller would; a far-node
    buffer cost the H2D copy ~15 % on some boxes. Affinity restored after."""
    old = os.sched_getaffinity(0)
    local = gpu_local_cpus(local_rank)
    if local:
        os.sched_setaffinity(0, local)
    try:
        out = e2e_leg_body(args, dist, rank, world, local_rank, units)
    finally:
        os.sched_setaffinity(0, old)
    if out is not None and isinstance(out, dict):
        out.setdefault("phases", {})["gpu_local_cpus"] = len(local) if local else None
    return out


def e2e_leg_body(args, dist, rank, world, local_rank, units):
    """The same metric through the public API with host buffers: the host->
    device copy of X (pinned), the solve and the factor download are inside
    the timed region. N=1: rescal_solve(RelTensor / SparseRelTensor);
    N>1: solve_on_grid(BlockSource) -- every rank uploads its own block."""
    import paper_2202_09512_b200 as rk
    from paper_2202_09512_b200 import _lib

    c = workload(args.config, world)
    m, n, k = c["m"], c["n"], c["k"]
    sparse = "density" in c
    f0 = rk.random_init(n, k, m, 0)
    cfg = lambda iters: rk.SolverConfig(max_iters=iters, track_error=False, device=local_rank)  # noqa: E731
    phases = {}
    if sparse:
        if world > 1:
            raise RuntimeError("sparse e2e at N>1 not measured (device-generated blocks only)")
        import scipy.sparse as sps

        e4 = _lib.Engine(n, m, k, device=local_rank, sparse=True)
        e4.fill_sparse_uniform(SEED, int(round(c["density"] * n * n)))
        ptr, idx, val = e4.csr_arrays()
        e4.close()
        slices = [sps.csr_matrix((val[ptr[t, 0]:ptr[t, -1]], idx[ptr[t, 0]:ptr[t, -1]], ptr[t] - ptr[t, 0]),
                                 shape=(n, n)) for t in range(m)]
        x = rk.SparseRelTensor(slices)  # canonical form checked outside the timed region
        rk.rescal_solve(x, k, cfg(max(1, args.warmup)), initial=f0)  # untimed warm-up call
        t0 = time.perf_counter()
        f, tr = rk.rescal_solve(x, k, cfg(args.steps), initial=f0)
        e2e_s = time.perf_counter() - t0
        h2d = int(ptr.nbytes + idx.nbytes + val.nbytes) + f0.A.nbytes + f0.R.nbytes
        d2h = f.A.nbytes + f.R.nbytes
        api = "rescal_solve(SparseRelTensor(host CSR), k, SolverConfig(max_iters=steps, track_error=False))"
    elif world == 1:
        xh = host_tensor(m, n, pinned=True)
        x = rk.RelTensor(xh)  # validation outside the timed region, as a caller would
        rk.rescal_solve(x, k, cfg(max(1, args.warmup)), initial=f0)  # untimed warm-up call
        from paper_2202_09512_b200 import solver as _solver

        phases["engine_reused"] = getattr(_solver._CACHE, "entry", None) is not None
        t0 = time.perf_counter()
        f, tr = rk.rescal_solve(x, k, cfg(args.steps), initial=f0)
        e2e_s = time.perf_counter() - t0
        h2d = xh.nbytes + f0.A.nbytes + f0.R.nbytes
        d2h = f.A.nbytes + f.R.nbytes + tr.nbytes
        api = "rescal_solve(RelTensor(pinned fp32 host X), k, SolverConfig(max_iters=steps, track_error=False))"
        del x, xh
    else:
        import torch
        from paper_2202_09512_b200.multigpu import BlockSource, make_grid_engine

        # this rank's block of the synthetic tensor in pinned host memory
        # (untimed: it is the input), generated by a throw-away grid engine
        eg, lay = make_grid_engine(n, m, k, cfg=cfg(1))
        blk0 = eg.block_uniform(SEED, lay["rows"], lay["cols"])
        eg.close()
        blk = torch.empty(blk0.shape, dtype=torch.float32, pin_memory=True).numpy()
        blk[...] = blk0
        del blk0
        src = BlockSource(n, m, lambda info: blk, dtype=np.float32)
        rk.solve_on_grid(src, k, cfg(max(1, args.warmup)), initial=f0)  # untimed warm-up call
        barrier(dist)
        t0 = time.perf_counter()
        f, tr, info = rk.solve_on_grid(src, k, cfg(args.steps), initial=f0)
        e2e_s = max_over_ranks(dist, time.perf_counter() - t0)
        phases = {kk: vv for kk, vv in info.timing.items() if kk.endswith("_s")}
        h2d = blk.nbytes + f0.A.nbytes + f0.R.nbytes
        d2h = f.A.nbytes + f.R.nbytes
        api = ("solve_on_grid(BlockSource(pinned fp32 host block of this rank), k, "
               "SolverConfig(max_iters=steps, track_error=False))")
    return {"value": units * args.steps / e2e_s, "unit": "it/s",
            "h2d_bytes_per_step": int(h2d / args.steps), "d2h_bytes_per_step": int(d2h / args.steps),
            "api": api, "seconds": e2e_s, "phases": phases,
            "protocol": "one untimed warm-up call, then one timed call of `steps` iterations (upload of X + "
                        "solve + factor download inside the timed region)"}


def run_rescalk(args, dist, rank, world, local_rank):
    """cfg5: the public rescalk() driver end to end (device tensor upload,
    per-member PCG64 resampling on the device, MU solves, host clustering,
    device regress_r / rel_error)."""
    import paper_2202_09512_b200 as rk

    c = dict(CONFIGS["cfg5"])
    k_min = args.k_min or c["k_min"]
    k_max = args.k_max or c["k_max"]
    m, n, r, iters = c["m"], c["n"], c["r"], c["iters"]
    xh = host_tensor(m, n, pinned=True)
    x = rk.RelTensor(xh)

    def allgather(obj):
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    cfg = rk.SolverConfig(max_iters=iters, device=local_rank)
    pcfg = rk.PerturbConfig(delta=0.02, base_seed=0)
    claim = None
    if world > 1:  # dynamic member assignment through the rendezvous store
        from torch.distributed import distributed_c10d as _c10d

        store = _c10d._get_default_store()
        tag = f"rk_member_{time.time_ns() if rank == 0 else 0}"
        tag = allgather(tag)[0]
        claim = lambda: store.add(tag, 1)  # noqa: E731
    # untimed warm-up: one solve of `warmup` iterations on this rank's GPU
    # (context, module loading, allocator)
    rk.rescal_solve(x, k_min, rk.SolverConfig(max_iters=max(3, args.warmup), device=local_rank))
    barrier(dist)
    with ClockSampler(local_rank) as clocks:
        t0 = time.perf_counter()
        rep = rk.rescalk(x, k_min, k_max, r, cfg=cfg, pcfg=pcfg,
                         world=(rank, world) if world > 1 else None,
                         allgather=allgather if world > 1 else None, claim=claim)
        secs = max_over_ranks(dist, time.perf_counter() - t0)
    members = (k_max - k_min + 1) * r
    units = members * iters
    line = {
        "metric": METRIC, "value": units / secs, "unit": "member-it/s", "n_gpus": world,
        "steps": units, "warmup": max(3, args.warmup), "ms_per_step": secs * 1e3 / units,
        "higher_is_better": True, "clocks": clocks.summary(),
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic uniform [0,1) fp32-representable",
        "config": {"workload": f"cfg5: rescalk dense m={m} n={n} k={k_min}..{k_max} r={r} "
                               f"iters={iters} (full sweep is k=2..16)",
                   "per_step": "one member MU iteration inside rescalk() (tracked, default config)",
                   "parallelism": f"replicas x{world}" + (" (members claimed dynamically)" if world > 1 else "")},
        "k_opt": rep.k_opt, "seconds": secs, "members": members, "timing_rank0": rep.timing,
        "per_k": {str(e.k): {"s_min": e.s_min, "rel_error": e.rel_error} for e in rep.entries},
        "e2e": {"value": units / secs, "unit": "member-it/s",
                "h2d_bytes_per_step": int(xh.nbytes / units), "d2h_bytes_per_step": 0,
                "api": "rescalk(RelTensor(pinned host X), k_min, k_max, r)"},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    barrier(dist)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--k-min", type=int, default=0)
    ap.add_argument("--k-max", type=int, default=0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        # CPU reference arm: rank 0 alone runs it; other ranks exit without work
        world = int(os.environ.get("WORLD_SIZE", str(max(1, args.gpus))))
        if int(os.environ.get("RANK", "0")) != 0:
            return 0
        run_reference(args, world)
        return 0
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    dist, rank, world, local_rank = dist_setup()
    if args.config == "cfg5":
        run_rescalk(args, dist, rank, world, local_rank)
    else:
        run_ours(args, dist, rank, world, local_rank)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
