"""NNDSVD start on the device (rescal.py:327-372; pytest -m gpu).

The reference takes the leading singular triplets of the unfolding
M = [X_1 .. X_m | X_1^T .. X_m^T] from LAPACK (dense) or ARPACK svds
(sparse); the device runs a subspace iteration on M M^T with its own
products. The first four tests are the reference's TestNndsvdInit bodies
(test_rescal.py:180-212) through this package; the rest compare with the
reference's outputs on a planted tensor (tests/golden/nndsvd64.npz) within
the north_star tolerance (relative Frobenius 1e-4 on A and R, 1e-5 on the
error trace).
"""
import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden, rel_fro

pytestmark = pytest.mark.gpu
rk = pytest.importorskip("paper_2202_09512_b200")


def random_tensor(n, m, seed):
    return rk.RelTensor(np.random.default_rng(seed).random((m, n, n)))


def test_rank_one_matches_power_iteration():
    rng = np.random.default_rng(18)
    a_vec = rng.random(10)
    b_vec = rng.random(10)
    x = rk.RelTensor(np.stack([np.outer(a_vec, b_vec)]))
    f = rk.nndsvd_init(x, 1)
    m_mat = np.concatenate([x.slices[0], x.slices[0].T], axis=1)
    gram = m_mat @ m_mat.T
    v = np.ones(10)
    for _ in range(500):
        v = gram @ v
        v /= np.linalg.norm(v)
    cos = abs(v @ f.A[:, 0]) / np.linalg.norm(f.A[:, 0])
    assert cos >= 1 - 1e-8


def test_identity_slices_invariants():
    x = rk.RelTensor(np.stack([np.eye(6)]))
    f = rk.nndsvd_init(x, 1)
    assert np.all(f.A >= 0) and np.all(f.R >= 0)
    assert np.linalg.norm(f.A[:, 0]) > 0


def test_deficient_column_filled():
    rng = np.random.default_rng(19)
    v = rng.random(8)
    x = rk.RelTensor(np.stack([np.outer(v, v)]))  # rank-1, k=2 requested
    f = rk.nndsvd_init(x, 2)
    assert np.all(f.A >= 0)
    assert np.all(f.A[:, 1] > 0)


def test_deterministic():
    x = random_tensor(8, 2, seed=20)
    f1 = rk.nndsvd_init(x, 3)
    f2 = rk.nndsvd_init(x, 3)
    assert np.array_equal(f1.A, f2.A) and np.array_equal(f1.R, f2.R)


def test_dense_matches_reference_golden():
    g = golden("nndsvd64")
    f = rk.nndsvd_init(rk.RelTensor(g["X"]), 4)
    assert rel_fro(f.A, g["A"]) <= 1e-4
    assert rel_fro(f.R, g["R"]) <= 1e-4


def test_nndsvd_initialised_solve_matches_reference_golden():
    g = golden("nndsvd64")
    f, tr = rk.rescal_solve(rk.RelTensor(g["X"]), 4, rk.SolverConfig(max_iters=50, init="nndsvd"))
    assert rel_fro(f.A, g["A50"]) <= 1e-4
    assert rel_fro(f.R, g["R50"]) <= 1e-4
    assert len(tr) == len(g["trace50"])
    assert np.max(np.abs(tr - g["trace50"])) <= 1e-5


def test_sparse_matches_reference_golden():
    g = golden("nndsvd64")
    slices, off = [], 0
    for t in range(len(g["sp_nnz"])):
        nz = int(g["sp_nnz"][t])
        slices.append(sp.csr_matrix((g["sp_data"][off:off + nz], g["sp_indices"][off:off + nz],
                                     g["sp_indptr"][t]), shape=(64, 64)))
        off += nz
    f = rk.nndsvd_init(rk.SparseRelTensor(slices), 3)
    assert rel_fro(f.A, g["spA"]) <= 1e-4
    assert rel_fro(f.R, g["spR"]) <= 1e-4
