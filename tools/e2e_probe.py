"""Time the phases of one rescal_solve call through the public API (diagnostics)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2202_09512_b200 as rk  # noqa: E402
from paper_2202_09512_b200 import _lib  # noqa: E402

n, m, k, steps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
xh = torch.empty((m, n, n), dtype=torch.float32, pin_memory=True).numpy()
xh[...] = np.random.default_rng(0).random((m, n, n), dtype=np.float32)
f0 = rk.random_init(n, k, m, 0)
for rep in range(2):
    t = {}
    t0 = time.perf_counter()
    e = _lib.Engine(n, m, k)
    t["create"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    e.upload(xh)
    t["upload"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    e.set_factors(f0.A, f0.R)
    t["set_factors"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    e.run(steps, 1e-16, track_error=False)
    t["run"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    e.get_factors()
    t["get"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    e.close()
    t["close"] = time.perf_counter() - t0
    print(rep, {a: round(b * 1e3, 1) for a, b in t.items()}, "ms")
