"""Dense e2e phases at cfg3 (one GPU): engine creation, upload of pinned fp32
X, solve, download -- where rescal_solve's end-to-end time goes."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import bench
import paper_2202_09512_b200 as rk
from paper_2202_09512_b200 import _lib

m, n, k, steps = 16, 32768, 32, 30
t0 = time.perf_counter()
xh = bench.host_tensor(m, n, pinned=True)
print(f"host tensor {time.perf_counter() - t0:.1f} s", flush=True)
f0 = rk.random_init(n, k, m, 0)
for rep in range(2):
    ts = {}
    t = time.perf_counter()
    e = _lib.Engine(n, m, k, device=0)
    ts["create"] = time.perf_counter() - t
    t = time.perf_counter()
    e.upload(xh)
    ts["upload"] = time.perf_counter() - t
    t = time.perf_counter()
    e.set_factors(f0.A, f0.R)
    ts["set_factors"] = time.perf_counter() - t
    t = time.perf_counter()
    e.run(steps, 1e-16, track_error=False)
    ts["run"] = time.perf_counter() - t
    t = time.perf_counter()
    a, r = e.get_factors()
    ts["get"] = time.perf_counter() - t
    t = time.perf_counter()
    e.close()
    ts["close"] = time.perf_counter() - t
    print(rep, {a: round(b, 4) for a, b in ts.items()}, f"upload {xh.nbytes / ts['upload'] / 1e9:.1f} GB/s", flush=True)
x = rk.RelTensor(xh)
for rep in range(2):
    t = time.perf_counter()
    rk.rescal_solve(x, k, rk.SolverConfig(max_iters=steps, track_error=False), initial=f0)
    print("rescal_solve", rep, round(time.perf_counter() - t, 4), flush=True)
import cProfile, pstats
pr = cProfile.Profile()
pr.enable()
rk.rescal_solve(x, k, rk.SolverConfig(max_iters=steps, track_error=False), initial=f0)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
