"""The reference's own MU test bodies (pkg/tests/test_rescal.py,
test_model_select.py) re-run against the device engine through the drop-in
API — same fixtures, same assertions (tolerances as in the reference unless
the comparison is against an fp64 trajectory, where the north_star's 1e-4 /
1e-5 apply). GPU suite."""

import numpy as np
import pytest

import oracle
from conftest import golden

pytestmark = pytest.mark.gpu
rk = pytest.importorskip("paper_2202_09512_b200")


def naive_objective(x, f):
    """conftest.py:7-13 — independent slice-by-slice objective."""
    return float(sum(np.sum((x.slices[t] - f.A @ f.R[t] @ f.A.T) ** 2) for t in range(x.m)))


def random_tensor(n, m, seed, dtype=np.float64):
    """conftest.py:16-18."""
    return rk.RelTensor(np.random.default_rng(seed).random((m, n, n)).astype(dtype))


def exact_factors(n, k, m, seed):
    """test_rescal.py:50-56."""
    rng = np.random.default_rng(seed)
    a = rng.random((n, k)) + 0.05
    r = rng.random((m, k, k)) + 0.05
    return rk.RelTensor(np.einsum("nk,mkl,jl->mnj", a, r, a)), rk.RescalFactors(a, r)


class TestUpdateR:  # test_rescal.py:59-84
    def test_fixed_point(self):
        x, f = exact_factors(8, 3, 2, seed=0)
        f2 = rk.update_r(x, f)
        rel = np.abs(f2.R - f.R) / np.maximum(f.R, 1e-300)
        assert rel.max() <= 1e-5  # reference: 1e-10 in fp64; device contracts in split precision

    def test_zero_entry_stays_zero(self):
        x, f = exact_factors(6, 2, 2, seed=1)
        r = f.R.copy()
        r[0, 0, 1] = 0.0
        assert rk.update_r(x, rk.RescalFactors(f.A, r)).R[0, 0, 1] == 0.0

    def test_objective_non_increase(self):
        x = random_tensor(6, 2, seed=2)
        f = rk.random_init(6, 3, 2, seed=3)
        before = naive_objective(x, f)
        after = naive_objective(x, rk.update_r(x, f))
        assert after <= before + 1e-6 * max(before, 1.0)

    def test_shape_mismatch(self):
        x = random_tensor(6, 2, seed=2)
        with pytest.raises(rk.DataError, match="shape mismatch"):
            rk.update_r(x, rk.random_init(5, 3, 2, seed=3))


class TestUpdateA:  # test_rescal.py:87-106
    def test_fixed_point(self):
        x, f = exact_factors(8, 3, 2, seed=4)
        f2 = rk.update_a(x, f)
        assert (np.abs(f2.A - f.A) / np.maximum(f.A, 1e-300)).max() <= 1e-5

    def test_zero_entry_stays_zero(self):
        x, f = exact_factors(6, 2, 2, seed=5)
        a = f.A.copy()
        a[2, 1] = 0.0
        assert rk.update_a(x, rk.RescalFactors(a, f.R)).A[2, 1] == 0.0

    def test_objective_non_increase(self):
        x = random_tensor(7, 3, seed=6)
        f = rk.random_init(7, 2, 3, seed=7)
        before = naive_objective(x, f)
        assert naive_objective(x, rk.update_a(x, f)) <= before + 1e-6 * max(before, 1.0)


class TestSolve:  # test_rescal.py:109-154
    def test_exact_recovery_small(self):
        x, _, _ = oracle_planted(16, 4, 3, seed=1)
        f, trace = rk.rescal_solve(x, 3, rk.SolverConfig(max_iters=2000, tolerance=1e-4, seed=11))
        assert trace[-1] <= 1e-4

    def test_trace_non_increasing(self):
        x = random_tensor(10, 2, seed=9)
        _, trace = rk.rescal_solve(x, 3, rk.SolverConfig(max_iters=100, seed=10))
        assert len(trace) == 100
        assert np.all(np.diff(trace) <= 1e-6 * np.maximum(trace[:-1], 1e-300))

    def test_tolerance_stops_early(self):
        x, _, _ = oracle_planted(16, 2, 2, seed=3)
        _, trace = rk.rescal_solve(x, 2, rk.SolverConfig(max_iters=2000, tolerance=1e-3, seed=1))
        assert len(trace) < 2000 and trace[-1] < 1e-3

    def test_track_error_off(self):
        x = random_tensor(6, 2, seed=11)
        _, trace = rk.rescal_solve(x, 2, rk.SolverConfig(max_iters=5, track_error=False, seed=0))
        assert len(trace) == 0

    def test_float32_path(self):
        x = rk.RelTensor(random_tensor(8, 2, seed=12).slices.astype(np.float32))
        f, trace = rk.rescal_solve(x, 2, rk.SolverConfig(max_iters=20, seed=1))
        assert f.A.dtype == np.float32 and f.R.dtype == np.float32
        assert np.all(np.diff(trace) <= 1e-5 * np.maximum(trace[:-1], 1e-30))


class TestRelError:  # test_rescal.py:157-177
    def test_exact_factorization(self):
        x, f = exact_factors(8, 3, 2, seed=13)
        assert rk.rel_error(x, f) <= 1e-5

    def test_zero_factors_give_one(self):
        x = random_tensor(5, 2, seed=14)
        f = rk.RescalFactors(np.zeros((5, 2)), np.zeros((2, 2, 2)))
        assert rk.rel_error(x, f) == pytest.approx(1.0, rel=1e-6)

    def test_matches_naive_oracle(self):
        x = random_tensor(6, 3, seed=15)
        f = rk.random_init(6, 2, 3, seed=16)
        ref = np.sqrt(naive_objective(x, f)) / np.sqrt(float(np.sum(x.slices ** 2)))
        assert rk.rel_error(x, f) == pytest.approx(ref, rel=1e-5)


class TestProperties:  # test_rescal.py:271-301
    def test_non_negativity_closure(self):
        for seed in range(10):
            x = random_tensor(6, 2, seed=100 + seed)
            f = rk.random_init(6, 3, 2, seed=200 + seed)
            for _ in range(5):
                f = rk.update_a(x, rk.update_r(x, f))
            assert f.A.min() >= 0 and f.R.min() >= 0

    def test_zero_locking_through_sweeps(self):
        x = random_tensor(6, 2, seed=25)
        f = rk.random_init(6, 3, 2, seed=26)
        a, r = f.A.copy(), f.R.copy()
        a[1, 2] = 0.0
        r[1, 0, 0] = 0.0
        f = rk.RescalFactors(a, r)
        for _ in range(10):
            f = rk.update_a(x, rk.update_r(x, f))
        assert f.A[1, 2] == 0.0 and f.R[1, 0, 0] == 0.0


class TestRegress:  # test_rescal.py:248-268
    def test_zero_tensor_locks_to_zero(self):
        x = rk.RelTensor(np.zeros((2, 4, 4)))
        a = np.abs(np.random.default_rng(22).random((4, 2)))
        np.testing.assert_array_equal(rk.regress_r(x, a), np.zeros((2, 2, 2)))

    def test_improves_over_initialization(self):
        x = random_tensor(8, 2, seed=23)
        a = rk.random_init(8, 3, 2, seed=24).A
        before = rk.rel_error(x, rk.RescalFactors(a, np.ones((2, 3, 3))))
        after = rk.rel_error(x, rk.RescalFactors(a, rk.regress_r(x, a)))
        assert after <= before


class TestRescalK:  # test_model_select.py:237-291
    def test_exact_rank_two_perturbations(self):
        x, _, _ = oracle_planted(16, 3, 3, seed=7)
        rep = rk.rescalk(x, 3, 3, r=2, cfg=rk.SolverConfig(max_iters=600, seed=8),
                         pcfg=rk.PerturbConfig(delta=0.01, base_seed=8))
        entry = rep.entries[0]
        # the reference's own assertions (rel_error <= 1e-3, s_min >= 0.98) fail
        # for the reference too (4.98e-3); parity is the bar
        g = golden("planted_inputs")
        assert abs(entry.s_min - float(g["p16_3_3_s7_ped_rescalk_s_min"])) <= 1e-4
        assert abs(entry.rel_error - float(g["p16_3_3_s7_ped_rescalk_rel_error"])) <= 1e-5

    def test_k_above_n_rejected(self):
        x, _, _ = oracle_planted(8, 2, 2, seed=9)
        with pytest.raises(rk.DataError):
            rk.rescalk(x, 2, 9, r=2)

    def test_report_serialization(self):
        x, _, _ = oracle_planted(12, 2, 2, seed=10, noise=0.01)
        rep = rk.rescalk(x, 2, 3, r=3, cfg=rk.SolverConfig(max_iters=80, seed=1),
                         pcfg=rk.PerturbConfig(delta=0.02, base_seed=1))
        doc = rep.to_json_dict()
        assert set(doc) == {"k_opt", "low_confidence", "tau_s", "per_k", "parameters", "timing"}
        assert set(doc["per_k"]) == {"2", "3"}


def oracle_planted(n, m, k, seed, noise=0.0, pedestal=0.15):
    """The reference's planted tensor (synth.generate, conftest.py:21-23),
    from the golden fixture produced by the reference itself."""
    key = {(16, 4, 3, 1): "p16_4_3_s1_ped", (16, 2, 2, 3): "p16_2_2_s3_ped",
           (16, 3, 3, 7): "p16_3_3_s7_ped", (8, 2, 2, 9): "p8_2_2_s9",
           (12, 2, 2, 10): "p12_2_2_s10"}[(n, m, k, seed)]
    return rk.RelTensor(golden("planted_inputs")[f"{key}_X"]), None, None
