"""Iteration time at k_pad 48 / 64 (n = 8192, m = 16): tcgen05 K1 vs the SIMT
K1, and the K1 share (rk_time_k1). python tools/kwide_probe.py"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2202_09512_b200 as rk
from paper_2202_09512_b200 import _lib
n, m = 8192, 16
for k in (48, 64):
    for engine in ("tc", "simt"):
        e = _lib.Engine(n, m, k, device=0, engine=engine)
        e.fill_uniform(5)
        f0 = rk.random_init(n, k, m, 2)
        e.set_factors(f0.A, f0.R)
        e.run(3, 1e-16, track_error=False)
        import torch
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e.run(20, 1e-16, track_error=False)
        dt = (time.perf_counter() - t0) / 20
        k1 = e.time_k1(5) if hasattr(e, "time_k1") else float("nan")
        inf = e.info()
        print(f"k={k} engine={engine} ({inf['engine']}) strips={inf['strips']} tiles={inf['strip_tiles']} "
              f"{dt * 1e3:.3f} ms/it  K1 {k1:.3f} ms  X {4 * m * n * n / 1e9:.2f} GB -> {4 * m * n * n / k1 / 1e6:.0f} GB/s",
              flush=True)
        e.close()
