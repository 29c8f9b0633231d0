"""Parity at the BASELINE.json sizes (GPU suite).

cfg2 (dense m=16, n=8192, k=16): the full oracle (numpy fp64, the reference's
operation order) is affordable for a few iterations on the box's host cores,
so the device factors are compared with it directly on the same synthetic
tensor (the device generator's exact fp32 values, read back with
rk_block_uniform) and the same initial A/R.

cfg4 (sparse m=32, n=2^20, density 1e-5, k=16, 3.5e8 stored entries): one MU
iteration from a known start, checked through properties the oracle can form
cheaply at that size — the core update of slice 0 (one scipy SpMM) and the A
update of a sample of rows (their CSR rows / CSC columns on the host), both
against the device's own R after the iteration (rescal.py:124-145).
"""

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from conftest import rel_fro

pytestmark = pytest.mark.gpu

rk = pytest.importorskip("paper_2202_09512_b200")
from paper_2202_09512_b200 import _lib  # noqa: E402


def test_cfg2_full_size_matches_oracle():
    n, m, k, iters, seed = 8192, 16, 16, 3, 11
    eng = _lib.Engine(n, m, k, device=0, engine="tc")
    try:
        eng.fill_uniform(seed)
        x = eng.block_uniform(seed, n, n)  # exact fp32 values of the device tensor
        f0 = rk.random_init(n, k, m, 5)
        eng.set_factors(f0.A, f0.R)
        done, trace = eng.run(iters, 1e-16, track_error=True)
        a_dev, r_dev = eng.get_factors()
    finally:
        eng.close()
    assert done == iters and len(trace) == iters
    assert np.all(np.diff(trace) <= 1e-9), trace  # MU never increases the error
    a, r = f0.A.copy(), f0.R.copy()
    xs = [x[t] for t in range(m)]
    for _ in range(iters):
        a = oracle.mu_iteration(xs, a, r, 1e-16)
    assert rel_fro(a_dev, a) <= 1e-4 and rel_fro(r_dev, r) <= 1e-4, (rel_fro(a_dev, a), rel_fro(r_dev, r))
    # the trace's last value against the oracle's residual of the same iterate
    err = np.sqrt(oracle.sq_residual(xs, a, r) / oracle.sq_norm(xs))
    assert abs(trace[-1] - err) <= 1e-5, (trace[-1], err)


def test_cfg4_full_size_one_iteration_properties():
    n, m, k, eps = 1 << 20, 32, 16, 1e-16
    nnz_target = int(round(1e-5 * n * n))
    eng = _lib.Engine(n, m, k, device=0, sparse=True)
    try:
        eng.fill_sparse_uniform(7, nnz_target)
        nnz = eng.nnz
        f0 = rk.random_init(n, k, m, 3)
        eng.set_factors(f0.A, f0.R)
        eng.run(1, eps, track_error=False)
        a1, r1 = eng.get_factors()
        indptr, indices, data = eng.csr_arrays()
        cptr, cidx, cval = eng.csc_arrays(nnz)
    finally:
        eng.close()
    assert nnz > 0.99 * m * nnz_target
    assert np.isfinite(a1).all() and np.isfinite(r1).all() and (a1 >= 0).all() and (r1 >= 0).all()
    a0, r0 = f0.A, f0.R
    g = a0.T @ a0
    # core update of slice 0 (rescal.py:128-132)
    x0 = sp.csr_matrix((data[indptr[0, 0]:indptr[0, -1]].astype(np.float64),
                        indices[indptr[0, 0]:indptr[0, -1]], indptr[0] - indptr[0, 0]), shape=(n, n))
    s0 = a0.T @ (x0 @ a0)
    r1_0 = r0[0] * s0 / (g @ (r0[0] @ g) + eps)
    assert rel_fro(r1[0], r1_0) <= 1e-5, rel_fro(r1[0], r1_0)
    # A update of sampled rows with the device's new cores (rescal.py:133-145)
    rows = np.random.default_rng(0).choice(n, 512, replace=False)
    mm = sum(r1[t].T @ g @ r1[t] + r1[t] @ g @ r1[t].T for t in range(m))
    num = np.zeros((len(rows), k))
    for t in range(m):
        for q, i in enumerate(rows):
            b, e = indptr[t, i], indptr[t, i + 1]
            p_ti = data[b:e].astype(np.float64) @ a0[indices[b:e]]
            b, e = cptr[t, i], cptr[t, i + 1]
            q_ti = cval[b:e].astype(np.float64) @ a0[cidx[b:e]]
            num[q] += p_ti @ r1[t].T + q_ti @ r1[t]
    a1_ref = a0[rows] * num / (a0[rows] @ mm + m * eps)
    assert rel_fro(a1[rows], a1_ref) <= 1e-5, rel_fro(a1[rows], a1_ref)
