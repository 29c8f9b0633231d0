"""rescal_solve end to end, repeated, with a phase split (diagnostics)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2202_09512_b200 as rk  # noqa: E402
from paper_2202_09512_b200 import solver  # noqa: E402

n, m, k, steps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
xh = torch.empty((m, n, n), dtype=torch.float32, pin_memory=True).numpy()
xh[...] = np.random.default_rng(0).random((m, n, n), dtype=np.float32)
x = rk.RelTensor(xh)
f0 = rk.random_init(n, k, m, 0)
orig = solver._engine_for


def timed_engine_for(*a, **kw):
    t0 = time.perf_counter()
    e = orig(*a, **kw)
    print(f"   engine_for {1e3 * (time.perf_counter() - t0):.1f} ms")
    return e


solver._engine_for = timed_engine_for
if len(sys.argv) > 5:  # mimic bench.py: a device-generated engine first
    from paper_2202_09512_b200 import _lib
    e = _lib.Engine(n, m, k)
    e.fill_uniform(1)
    e.set_factors(f0.A, f0.R)
    e.run(10, 1e-16, track_error=False)
    e.close()
    print("bench-like engine done")
for rep in range(3):
    t0 = time.perf_counter()
    f, tr = rk.rescal_solve(x, k, rk.SolverConfig(max_iters=steps, track_error=False), initial=f0)
    print(rep, f"rescal_solve {1e3 * (time.perf_counter() - t0):.1f} ms")
