"""Sparse-X path (CSR/CSC engine) parity on the B200 (pytest -m gpu)."""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from conftest import golden, rel_fro

pytestmark = pytest.mark.gpu
rk = pytest.importorskip("paper_2202_09512_b200")
from paper_2202_09512_b200 import _lib  # noqa: E402


def random_sparse(n, m, density, seed):
    rng = np.random.default_rng(seed)
    slices = []
    for _ in range(m):
        nnz = int(density * n * n)
        r = rng.integers(0, n, nnz)
        c = rng.integers(0, n, nnz)
        v = rng.random(nnz) + 0.01
        slices.append(sp.coo_matrix((v, (r, c)), shape=(n, n)))
    return rk.SparseRelTensor(slices)


def test_device_csc_construction_is_scipy_tocsc():
    x = random_sparse(700, 3, 0.004, 1)
    eng = _lib.Engine(700, 3, 8, sparse=True)
    eng.upload_csr(list(x.slices))
    ptr, idx, val = eng.csc_arrays(x.nnz)
    off = 0
    for t, s in enumerate(x.slices):
        c = s.tocsc()
        c.sort_indices()
        np.testing.assert_array_equal(ptr[t] - off, c.indptr)
        np.testing.assert_array_equal(idx[off:off + c.nnz], c.indices)
        np.testing.assert_array_equal(val[off:off + c.nnz], c.data.astype(np.float32))
        off += c.nnz
    eng.close()


def test_sparse_golden_matches_reference():
    g = golden("sparse12")
    xs = rk.SparseRelTensor([sp.csr_matrix(g["X"][t]) for t in range(2)])
    f, tr = rk.rescal_solve(xs, 2, rk.SolverConfig(max_iters=40, seed=3))
    assert rel_fro(f.A, g["A"]) <= 1e-4 and rel_fro(f.R, g["R"]) <= 1e-4
    assert np.max(np.abs(tr - g["trace"])) <= 1e-5


@pytest.mark.parametrize("n,m,k,density,iters", [(3000, 4, 16, 1e-3, 20), (2049, 3, 32, 2e-3, 10), (500, 2, 5, 0.02, 30)])
def test_sparse_engine_matches_oracle(n, m, k, density, iters):
    x = random_sparse(n, m, density, n)
    a0, r0 = oracle.random_init(n, k, m, 2)
    f, tr = rk.rescal_solve(x, k, rk.SolverConfig(max_iters=iters, track_error=False),
                            initial=rk.RescalFactors(a0, r0))
    ao, ro, _ = oracle.solve(list(x.slices), k, oracle.OracleConfig(max_iters=iters, track_error=False),
                             initial=(a0, r0))
    assert rel_fro(f.A, ao) <= 1e-4 and rel_fro(f.R, ro) <= 1e-4


def test_sparse_trace_and_rel_error():
    x = random_sparse(400, 2, 0.03, 7)
    a0, r0 = oracle.random_init(400, 4, 2, 3)
    f, tr = rk.rescal_solve(x, 4, rk.SolverConfig(max_iters=15), initial=rk.RescalFactors(a0, r0))
    ao, ro, tro = oracle.solve(list(x.slices), 4, oracle.OracleConfig(max_iters=15), initial=(a0, r0))
    assert np.max(np.abs(tr - tro)) <= 1e-5
    e = rk.rel_error(x, rk.RescalFactors(ao, ro))
    assert e == pytest.approx(oracle.rel_error(list(x.slices), ao, ro), abs=1e-5)


def test_sparse_split_api():
    x = random_sparse(300, 2, 0.05, 9)
    a0, r0 = oracle.random_init(300, 3, 2, 4)
    f0 = rk.RescalFactors(a0, r0)
    np.testing.assert_allclose(rk.update_r(x, f0).R, oracle.update_r(list(x.slices), a0, r0), rtol=1e-4)
    np.testing.assert_allclose(rk.update_a(x, f0).A, oracle.update_a(list(x.slices), a0, r0), rtol=1e-4)


def test_sparse_perturbation_matches_reference_field():
    x = random_sparse(60, 2, 0.1, 11)
    eng = _lib.Engine(60, 2, 4, sparse=True)
    eng.upload_csr(list(x.slices))
    eng.perturb((5, 3, (2, 3)), 0.02)
    ptr, idx, val = eng.csr_arrays()
    ref = oracle.perturb_sparse(list(x.slices), 0.02, 5, (2, 3))
    np.testing.assert_array_equal(idx, np.concatenate([s.indices for s in ref]))
    np.testing.assert_allclose(val, np.concatenate([s.data for s in ref]).astype(np.float32), rtol=2e-7)
    eng.close()


def test_device_sparse_generator_is_canonical():
    eng = _lib.Engine(5000, 2, 16, sparse=True)
    eng.fill_sparse_uniform(3, 20000)
    ptr, idx, val = eng.csr_arrays()
    for t in range(2):
        b, e = ptr[t, 0], ptr[t, -1]
        s = sp.csr_matrix((val[b:e], idx[b:e], ptr[t] - b), shape=(5000, 5000))
        c = s.copy()
        c.sum_duplicates()
        c.sort_indices()
        assert c.nnz == s.nnz and np.array_equal(c.indices, s.indices)
        assert (val[b:e] > 0).all() and (val[b:e] <= 1).all()
    eng.close()
