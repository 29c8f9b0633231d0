"""Sparse rescal_solve end to end, repeated (diagnostics; RK_UPLOAD_TIMING=1 for the upload split)."""
import sys
import time

import scipy.sparse as sps

sys.path.insert(0, ".")
import paper_2202_09512_b200 as rk  # noqa: E402
from paper_2202_09512_b200 import _lib  # noqa: E402

n, m, k, steps = 1 << 20, 32, 16, 10
e4 = _lib.Engine(n, m, k, sparse=True)
e4.fill_sparse_uniform(20220218, int(round(1e-5 * n * n)))
ptr, idx, val = e4.csr_arrays()
e4.close()
slices = [sps.csr_matrix((val[ptr[t, 0]:ptr[t, -1]], idx[ptr[t, 0]:ptr[t, -1]], ptr[t] - ptr[t, 0]), shape=(n, n))
          for t in range(m)]
t0 = time.perf_counter()
x = rk.SparseRelTensor(slices)
print(f"SparseRelTensor {time.perf_counter() - t0:.2f} s")
f0 = rk.random_init(n, k, m, 0)
for rep in range(4):
    t0 = time.perf_counter()
    f, tr = rk.rescal_solve(x, k, rk.SolverConfig(max_iters=steps, track_error=False), initial=f0)
    print(rep, f"rescal_solve {time.perf_counter() - t0:.3f} s", flush=True)
