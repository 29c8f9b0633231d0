"""Parity of the CUDA path against the reference (golden fixtures) and the
oracle — GPU suite (run on a B200 via gpurun: pytest -m gpu).

Tolerances are the north_star's: relative Frobenius difference of A and R
<= 1e-4 after N iterations, reconstruction error within 1e-5 (absolute, on
the trace), selected k identical. The device computes X contractions in
3xBF16 split precision with fp32 accumulation and every k x k step in fp64.
"""

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from conftest import golden, rel_fro, uniform_x

pytestmark = pytest.mark.gpu

rk = pytest.importorskip("paper_2202_09512_b200")

TOL_F = 1e-4   # relA, relR
TOL_E = 1e-5   # |err_gpu - err_ref|


def _solve(x, k, iters, a0, r0, engine="auto", tol=None, track=True):
    cfg = rk.SolverConfig(max_iters=iters, tolerance=tol, track_error=track, engine=engine)
    return rk.rescal_solve(rk.RelTensor(x), k, cfg, initial=rk.RescalFactors(a0, r0))


@pytest.mark.parametrize("engine", ["tc", "simt"])
def test_cfg1_uniform_200_iterations(engine):
    g = golden("cfg1_uniform")
    x = uniform_x(8, 256, 0).astype(np.float64)
    f, tr = _solve(x, 4, 200, g["A0"], g["R0"], engine=engine)
    assert f.A.dtype == np.float64 and len(tr) == 200
    assert rel_fro(f.A, g["A"]) <= TOL_F
    assert rel_fro(f.R, g["R"]) <= TOL_F
    assert abs(tr[-1] - g["trace"][-1]) <= TOL_E
    assert np.max(np.abs(tr - g["trace"])) <= TOL_E


def test_cfg1_untracked():
    g = golden("cfg1_uniform")
    gu = golden("cfg1_untracked")
    x = uniform_x(8, 256, 0).astype(np.float64)
    f, tr = _solve(x, 4, 200, g["A0"], g["R0"], track=False)
    assert len(tr) == 0
    assert rel_fro(f.A, gu["A"]) <= TOL_F and rel_fro(f.R, gu["R"]) <= TOL_F


def test_planted64_300_iterations():
    g = golden("planted64")
    f, tr = _solve(g["X"], 4, 300, g["A0"], g["R0"])
    assert rel_fro(f.A, g["A"]) <= TOL_F and rel_fro(f.R, g["R"]) <= TOL_F
    assert np.max(np.abs(tr - g["trace"])) <= TOL_E


def test_exact_recovery_with_tolerance_stop():
    g = golden("exact16_tol")
    f, tr = _solve(g["X"], 3, 2000, g["A0"], g["R0"], tol=1e-4)
    n_ref = len(g["trace"])
    assert tr[-1] < 1e-4 and abs(len(tr) - n_ref) <= 2
    m = min(len(tr), n_ref)
    assert np.max(np.abs(tr[:m] - g["trace"][:m])) <= TOL_E
    assert rel_fro(f.A, g["A"]) <= 1e-3  # stop iteration may differ by one step


def test_all_ones_rank_one_known_answer():
    x = rk.RelTensor(np.ones((1, 2, 2)))
    f, tr = rk.rescal_solve(x, 1, rk.SolverConfig(max_iters=2000, tolerance=1e-8, seed=3))
    assert tr[-1] <= 1e-6
    nrm = rk.finalize_normalize(f)
    np.testing.assert_allclose(nrm.A[:, 0], [1 / np.sqrt(2)] * 2, rtol=1e-5)
    assert nrm.R[0, 0, 0] == pytest.approx(2.0, rel=1e-5)


def test_split_api_matches_reference_and_fused_iteration():
    g = golden("split7")
    x = rk.RelTensor(g["X"])
    f0 = rk.RescalFactors(g["A0"], g["R0"])
    fr = rk.update_r(x, f0)
    assert rel_fro(fr.R, g["R_upd"]) <= TOL_F
    fa = rk.update_a(x, f0)
    assert rel_fro(fa.A, g["A_upd"]) <= TOL_F
    fs = rk.update_a(x, fr)
    assert rel_fro(fs.A, g["A_split"]) <= TOL_F
    ff, _ = rk.rescal_solve(x, 2, rk.SolverConfig(max_iters=1, track_error=False), initial=f0)
    # split == fused, bit-identical on the device too (test_rescal.py:294-301)
    np.testing.assert_array_equal(ff.A, fs.A)
    np.testing.assert_array_equal(ff.R, fs.R)
    assert rk.rel_error(x, f0) == pytest.approx(float(g["rel_err"]), abs=1e-6)


def test_fp32_dtype_preserved():
    g = golden("fp32_small")
    f, tr = rk.rescal_solve(rk.RelTensor(g["X"]), 2, rk.SolverConfig(max_iters=20, seed=1))
    assert f.A.dtype == np.float32 and f.R.dtype == np.float32
    assert rel_fro(f.A, g["A"]) <= TOL_F and rel_fro(f.R, g["R"]) <= TOL_F
    assert np.max(np.abs(tr - g["trace"])) <= TOL_E


def test_regress_r_and_rel_error():
    g = golden("regress16")
    x = rk.RelTensor(g["X"])
    rf = rk.regress_r(x, g["A"])
    assert rel_fro(rf, g["R_fit"]) <= TOL_F
    assert rk.rel_error(x, rk.RescalFactors(g["A"], rf)) == pytest.approx(float(g["err"]), abs=TOL_E)


def test_sparse_input_matches_reference():
    g = golden("sparse12")
    xs = rk.SparseRelTensor([sp.csr_matrix(g["X"][t]) for t in range(2)])
    f, tr = rk.rescal_solve(xs, 2, rk.SolverConfig(max_iters=40, seed=3))
    assert rel_fro(f.A, g["A"]) <= TOL_F and np.max(np.abs(tr - g["trace"])) <= TOL_E


def test_device_pcg64_bit_exact():
    from paper_2202_09512_b200 import _lib

    ent = (5, 3, (3, 4))
    ref = np.random.default_rng(np.random.SeedSequence(ent)).random(5000)
    np.testing.assert_array_equal(_lib.pcg64_draws(ent, 0, 5000), ref)
    np.testing.assert_array_equal(_lib.pcg64_draws(ent, 4321, 300), ref[4321:4621])


def test_rescalk_selects_reference_k():
    g = golden("rescalk16")
    x = rk.RelTensor(g["X"])
    rep = rk.rescalk(x, 2, 4, r=4, cfg=rk.SolverConfig(max_iters=120, seed=6),
                     pcfg=rk.PerturbConfig(delta=0.02, base_seed=6))
    assert rep.k_opt == int(g["k_opt"])
    for e, smr, sar, er in zip(rep.entries, g["s_min"], g["s_avg"], g["rel_error"]):
        assert abs(e.s_min - smr) <= 1e-4 and abs(e.s_avg - sar) <= 1e-4
        assert abs(e.rel_error - er) <= TOL_E
        np.testing.assert_allclose(e.medians, g[f"medians_k{e.k}"], atol=1e-4)


@pytest.mark.parametrize("n,m,k,iters", [(1024, 4, 16, 20), (640, 3, 32, 15), (1100, 2, 27, 10), (200, 2, 5, 30),
                                         (300, 2, 40, 8), (1300, 3, 48, 6), (700, 2, 64, 8), (2200, 2, 57, 4),
                                         (400, 2, 130, 4)])
def test_engines_match_oracle_midsize(n, m, k, iters):
    """k_pad 48 / 64 (k = 33..64) run K1 on tensor cores too (K1<48> with 6,
    K1<64> with 4 column tiles per strip; several strips here); k = 130 is
    SIMT only."""
    x = uniform_x(m, n, 7).astype(np.float64)
    a0, r0 = oracle.random_init(n, k, m, 3)
    ao, ro, tro = oracle.solve([x[t] for t in range(m)], k, oracle.OracleConfig(max_iters=iters),
                               initial=(a0, r0))
    for engine in ("tc", "simt"):
        if engine == "tc" and k > 64:
            continue
        f, tr = _solve(x, k, iters, a0, r0, engine=engine)
        assert rel_fro(f.A, ao) <= TOL_F, engine
        assert rel_fro(f.R, ro) <= TOL_F, engine
        assert np.max(np.abs(tr - tro)) <= TOL_E, engine


def test_zero_locking_and_nonnegativity():
    x = uniform_x(2, 96, 25).astype(np.float64)
    f0 = rk.random_init(96, 3, 2, 26)
    a, r = f0.A.copy(), f0.R.copy()
    a[1, 2] = 0.0
    r[1, 0, 0] = 0.0
    f, _ = rk.rescal_solve(rk.RelTensor(x), 3, rk.SolverConfig(max_iters=10), initial=rk.RescalFactors(a, r))
    assert f.A[1, 2] == 0.0 and f.R[1, 0, 0] == 0.0
    assert f.A.min() >= 0 and f.R.min() >= 0


def test_errors():
    x = rk.RelTensor(uniform_x(1, 8, 1).astype(np.float64))
    with pytest.raises(rk.DataError):
        rk.rescal_solve(x, 9)
    with pytest.raises(rk.DataError):
        rk.rescal_solve(rk.RelTensor(np.zeros((1, 3, 3))), 1)
    bad = uniform_x(1, 8, 1).astype(np.float64)
    bad[0, 2, 3] = np.inf
    with pytest.raises(rk.NumericalError):
        rk.rescal_solve(rk.RelTensor(bad), 2, rk.SolverConfig(max_iters=5))


def test_trace_monotone_cfg1_planted():
    x, a_t, r_t = None, None, None
    g = golden("planted64")
    f, tr = rk.rescal_solve(rk.RelTensor(g["X"]), 4, rk.SolverConfig(max_iters=100, seed=10))
    assert np.all(np.diff(tr) <= 1e-6 * np.maximum(tr[:-1], 1e-30))


def test_engine_reuse_is_transparent():
    """A solve on the engine kept from the previous call (same shape) returns
    the same bytes as one on a freshly created engine."""
    n, m, k = 200, 3, 6
    x1 = np.random.default_rng(1).random((m, n, n))
    x2 = np.random.default_rng(2).random((m, n, n))
    f0 = rk.random_init(n, k, m, 4)
    cfg = rk.SolverConfig(max_iters=25)
    rk.rescal_solve(rk.RelTensor(x1), k, cfg, initial=f0)          # leaves an engine behind
    fa, ta = rk.rescal_solve(rk.RelTensor(x2), k, cfg, initial=f0)  # reuses it
    rk.release_cached_memory()
    fb, tb = rk.rescal_solve(rk.RelTensor(x2), k, cfg, initial=f0)  # fresh engine
    assert np.array_equal(fa.A, fb.A) and np.array_equal(fa.R, fb.R) and np.array_equal(ta, tb)
    assert rel_fro(rk.update_r(rk.RelTensor(x2), fa).R, rk.update_r(rk.RelTensor(x2), fb).R) == 0.0
