"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): the tcgen05 K1 (mbarrier / TMA / TMEM pipeline, merged and
unmerged Q), the fused k-wide chain and the separate k2 kernels, the tail and
direct residual, update_r / update_a, regress_r, rel_error, the resampling
kernels, and the sparse CSR/CSC engine. Sizes are tiny: the tools instrument
every access."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import scipy.sparse as sp

import paper_2202_09512_b200 as rk
from paper_2202_09512_b200 import _lib

rng = np.random.default_rng(0)
for n, m, k in ((256, 3, 16), (384, 2, 32), (1664, 2, 32)):
    x = rk.RelTensor(rng.random((m, n, n), dtype=np.float32))
    f, tr = rk.rescal_solve(x, k, rk.SolverConfig(max_iters=4, seed=1))
    eng = _lib.Engine(n, m, k)
    eng.upload(x.slices)
    eng.set_factors(f.A, f.R)
    eng.run(3, 1e-16, track_error=True)
    eng.update_r(1e-16)
    eng.update_a(1e-16)
    eng.regress_r(20, 1e-8, 1e-16)
    eng.residual()
    eng.perturb((0, 3, (k, 1)), 0.02)
    eng.run(2, 1e-16, track_error=True)
    eng.restore()
    eng.close()
    rk.regress_r(x, f.A, max_iters=30)
    rk.rel_error(x, f)
    print("dense", n, m, k, "ok", flush=True)
# sparse engine
n, m, k = 3000, 2, 16
s = [sp.random(n, n, density=0.002, random_state=t, format="csr", dtype=np.float32) for t in range(m)]
xs = rk.SparseRelTensor(s)
f, tr = rk.rescal_solve(xs, k, rk.SolverConfig(max_iters=3, seed=2))
rk.perturb(xs, rk.PerturbConfig(delta=0.02), 1)
rk.rel_error(xs, f)
print("sparse ok", flush=True)
