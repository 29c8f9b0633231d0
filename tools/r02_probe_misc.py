"""cfg1 engine choice (tcgen05 vs SIMT K1 at tiny n) and pageable vs pinned
dense upload rate (parallel host staging copies)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_2202_09512_b200 as rk
from paper_2202_09512_b200 import _lib

out = {}
for n, m, k in ((256, 8, 4), (512, 8, 8), (1024, 8, 16)):
    for eng_name in ("tc", "simt"):
        e = _lib.Engine(n, m, k, device=0, engine=eng_name)
        e.fill_uniform(3)
        f0 = rk.random_init(n, k, m, 0)
        e.set_factors(f0.A, f0.R)
        e.run(200, 1e-16, track_error=False)
        e.set_factors(f0.A, f0.R)
        e.run(3000, 1e-16, track_error=False)
        out[f"n{n}_k{k}_{eng_name}_it_s"] = 3000 / (e.timing()["run_ms"] / 1e3)
        e.close()
n, m = 8192, 16
x = np.random.default_rng(0).random((m, n, n), dtype=np.float32)
xp = torch.empty((m, n, n), dtype=torch.float32, pin_memory=True).numpy()
xp[...] = x
e = _lib.Engine(n, m, 16, device=0)
for name, arr in (("pageable", x), ("pinned", xp), ("pageable2", x), ("pinned2", xp)):
    t0 = time.perf_counter()
    e.upload(arr)
    dt = time.perf_counter() - t0
    out[f"upload_{name}_GBs"] = arr.nbytes / dt / 1e9
e.close()
print(json.dumps(out))
