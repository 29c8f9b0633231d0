"""Pin the CPU oracle to the reference's own outputs (CPU suite).

The fixtures in tests/golden were produced by the unmodified reference
(tests/golden/make_golden.py). The oracle keeps the reference's fp64
operation order, so on this numpy/OpenBLAS build most cases agree exactly;
the assertion bound is 1e-12 relative to leave room for BLAS-kernel
differences on another host.
"""

import hashlib

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from conftest import golden, rel_fro, uniform_x

TIGHT = 1e-12


def _slices(x):
    return [x[t] for t in range(x.shape[0])]


def test_cfg1_uniform_trajectory():
    g = golden("cfg1_uniform")
    m, n, seed = (int(v) for v in g["x_recipe"])
    x32 = uniform_x(m, n, seed)
    assert hashlib.sha256(x32.tobytes()).hexdigest() == str(g["x_sha"])
    a0, r0 = oracle.random_init(n, 4, m, 0)
    np.testing.assert_array_equal(a0, g["A0"])
    np.testing.assert_array_equal(r0, g["R0"])
    a, r, tr = oracle.solve(_slices(x32.astype(np.float64)), 4, oracle.OracleConfig(max_iters=200),
                            initial=(a0, r0))
    assert rel_fro(a, g["A"]) <= TIGHT and rel_fro(r, g["R"]) <= TIGHT
    assert np.max(np.abs(tr - g["trace"])) <= TIGHT


def test_cfg1_untracked_matches():
    g = golden("cfg1_uniform")
    gu = golden("cfg1_untracked")
    x = uniform_x(8, 256, 0).astype(np.float64)
    a, r, tr = oracle.solve(_slices(x), 4, oracle.OracleConfig(max_iters=200, track_error=False),
                            initial=(g["A0"], g["R0"]))
    assert len(tr) == int(gu["trace_len"]) == 0
    assert rel_fro(a, gu["A"]) <= TIGHT and rel_fro(r, gu["R"]) <= TIGHT


@pytest.mark.parametrize("name,k,iters,tol", [("planted64", 4, 300, None), ("exact16_tol", 3, 2000, 1e-4)])
def test_planted_trajectories(name, k, iters, tol):
    g = golden(name)
    a, r, tr = oracle.solve(_slices(g["X"]), k, oracle.OracleConfig(max_iters=iters, tolerance=tol),
                            initial=(g["A0"], g["R0"]))
    assert len(tr) == len(g["trace"])
    assert rel_fro(a, g["A"]) <= TIGHT and rel_fro(r, g["R"]) <= TIGHT
    assert np.max(np.abs(tr - g["trace"])) <= TIGHT


def test_all_ones_known_answer():
    g = golden("all_ones")
    a, r, tr = oracle.solve(_slices(g["X"]), 1, oracle.OracleConfig(max_iters=2000, tolerance=1e-8, seed=3))
    assert len(tr) == len(g["trace"])
    an, rn = oracle.finalize_normalize(a, r)
    np.testing.assert_allclose(an[:, 0], [1 / np.sqrt(2)] * 2, rtol=1e-5)
    assert rn[0, 0, 0] == pytest.approx(2.0, rel=1e-5)
    assert rel_fro(an, g["An"]) <= TIGHT and rel_fro(rn, g["Rn"]) <= TIGHT


def test_split_api_and_rel_error():
    g = golden("split7")
    xs = _slices(g["X"])
    assert rel_fro(oracle.update_r(xs, g["A0"], g["R0"]), g["R_upd"]) <= TIGHT
    assert rel_fro(oracle.update_a(xs, g["A0"], g["R0"]), g["A_upd"]) <= TIGHT
    r1 = oracle.update_r(xs, g["A0"], g["R0"])
    a1 = oracle.update_a(xs, g["A0"], r1)
    assert rel_fro(a1, g["A_split"]) <= TIGHT
    # split == fused one iteration, bit-identical (test_rescal.py:294-301)
    af, rf, _ = oracle.solve(xs, 2, oracle.OracleConfig(max_iters=1, track_error=False), initial=(g["A0"], g["R0"]))
    np.testing.assert_array_equal(af, a1)
    np.testing.assert_array_equal(rf, r1)
    assert oracle.rel_error(xs, g["A0"], g["R0"]) == pytest.approx(float(g["rel_err"]), rel=TIGHT)


def test_fp32_path_dtype():
    g = golden("fp32_small")
    a, r, tr = oracle.solve(_slices(g["X"]), 2, oracle.OracleConfig(max_iters=20, seed=1), dtype=np.float32)
    assert a.dtype == np.float32 and r.dtype == np.float32
    assert rel_fro(a, g["A"]) <= 1e-6 and rel_fro(r, g["R"]) <= 1e-6


def test_regress_r_and_rel_error():
    g = golden("regress16")
    xs = _slices(g["X"])
    rf = oracle.regress_r(xs, g["A"])
    assert rel_fro(rf, g["R_fit"]) <= TIGHT
    assert oracle.rel_error(xs, g["A"], rf) == pytest.approx(float(g["err"]), rel=1e-9, abs=1e-15)


def test_finalize_normalize():
    g = golden("normalize")
    a, r = oracle.finalize_normalize(g["A0"], g["R0"])
    np.testing.assert_array_equal(a, g["A"])
    np.testing.assert_array_equal(r, g["R"])


def test_perturbation_field_and_perturb():
    g = golden("perturb9")
    fld = oracle.perturbation_field(9, 2, 0.02, 5, (3, 4))
    np.testing.assert_array_equal(fld, g["field"])
    np.testing.assert_array_equal(oracle.perturb_dense(g["X"], 0.02, 5, (3, 4)), g["Xp"])
    # sparse: stored values only, identical index arrays
    slices, off = [], 0
    for t, nnz in enumerate(g["sp_nnz"]):
        nnz = int(nnz)
        slices.append(sp.csr_matrix((g["sp_data"][off:off + nnz], g["sp_indices"][off:off + nnz], g["sp_indptr"][t]),
                                    shape=(9, 9)))
        off += nnz
    psp = oracle.perturb_sparse(slices, 0.02, 5, (3, 4))
    np.testing.assert_array_equal(np.concatenate([s.data for s in psp]), g["psp_data"])
    np.testing.assert_array_equal(np.concatenate([s.indices for s in psp]), g["psp_indices"])


def test_pcg64_restatement_matches_field():
    g = golden("perturb9")
    u = oracle.uniform_doubles((5, 3, (3, 4)), 2 * 81)
    np.testing.assert_array_equal(1.0 + 0.02 * (2.0 * u - 1.0), g["field"].ravel())
    u_tail = oracle.uniform_doubles((5, 3, (3, 4)), 7, offset=100)
    np.testing.assert_array_equal(u_tail, oracle.uniform_doubles((5, 3, (3, 4)), 107)[100:])


def test_csr_canonicalisation_bit_exact():
    g = golden("csr_canon")
    c = oracle.canonical_csr(sp.coo_matrix((np.abs(g["vals"]) * (g["vals"] >= 0), (g["rows"], g["cols"])), shape=(4, 4)))
    # the golden input contains a negative duplicate that cancels a positive one
    c2 = oracle.canonical_csr(sp.coo_matrix((g["vals"], (g["rows"], g["cols"])), shape=(4, 4)))
    np.testing.assert_array_equal(c2.indptr, g["indptr"])
    np.testing.assert_array_equal(c2.indices, g["indices"])
    np.testing.assert_array_equal(c2.data, g["data"])
    assert c.has_sorted_indices


def test_sparse_solve_matches_reference():
    g = golden("sparse12")
    xs = [oracle.canonical_csr(sp.csr_matrix(g["X"][t])) for t in range(2)]
    a, r, tr = oracle.solve(xs, 2, oracle.OracleConfig(max_iters=40), initial=(g["A0"], g["R0"]))
    assert rel_fro(a, g["A"]) <= 1e-10 and rel_fro(r, g["R"]) <= 1e-10
    assert np.max(np.abs(tr - g["trace"])) <= 1e-10


def test_grid_solution_matches_serial_oracle():
    g = golden("grid7_p4")
    a0, r0 = oracle.random_init(7, 2, 2, 4)
    a, r, tr = oracle.solve(_slices(g["X"]), 2, oracle.OracleConfig(max_iters=40), initial=(a0, r0))
    assert rel_fro(a, g["A"]) <= 1e-8 and np.max(np.abs(tr - g["trace"])) <= 1e-8


def test_rescalk_oracle_matches_reference():
    g = golden("rescalk16")
    rep = oracle.rescalk_oracle(g["X"], 2, 4, 4, oracle.OracleConfig(max_iters=120, seed=6), delta=0.02, base_seed=6)
    assert rep["k_opt"] == int(g["k_opt"])
    for (k, s_min, s_avg, err), k_ref, smr, sar, er in zip(rep["entries"], g["ks"], g["s_min"], g["s_avg"], g["rel_error"]):
        assert k == int(k_ref)
        assert abs(s_min - smr) <= 1e-10 and abs(s_avg - sar) <= 1e-10 and abs(err - er) <= 1e-10
        np.testing.assert_allclose(rep["medians"][k], g[f"medians_k{k}"], atol=1e-10)


def test_nndsvd_oracle_matches_reference():
    g = golden("nndsvd64")
    a, r = oracle.nndsvd_init(_slices(g["X"]), 4)
    assert rel_fro(a, g["A"]) <= TIGHT and rel_fro(r, g["R"]) <= TIGHT
    slices, off = [], 0
    for t in range(len(g["sp_nnz"])):
        nz = int(g["sp_nnz"][t])
        slices.append(sp.csr_matrix((g["sp_data"][off:off + nz], g["sp_indices"][off:off + nz],
                                     g["sp_indptr"][t]), shape=(64, 64)))
        off += nz
    a2, r2 = oracle.nndsvd_init(slices, 3)
    # ARPACK's start vector is random: agreement to the solver tolerance
    assert rel_fro(a2, g["spA"]) <= 1e-8 and rel_fro(r2, g["spR"]) <= 1e-8
