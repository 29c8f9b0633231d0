"""North-star shapes and the round-2 drop-in names on the device (GPU suite).

* cfg3 shape (n = 32768, k = 32), 10 iterations: K1<32> with its strip /
  group / slot schedule at full n (unmerged Q: 6 strips of 43 column tiles
  shared by groups of 4 CTAs, rotating Q drains), the K = 32
  tensor-core G / S kernel and k2b_v4<32, 8> (selected from n = 18944 on),
  against the fp64 oracle on the device generator's exact values
  (m = 2 keeps the host oracle affordable; rescal.py:114-146).
* K = 32 with merged Q (n <= 768) and unmerged Q with several strips.
* K1's slice products P and Q against fp64 at n = 32768, default schedule
  and rotating Q drains (the accuracy mode).
* RESCALk over cfg5's sweep shape (k = 2..16, r = 10, delta = 0.02, 200
  iterations) against the real reference's report (tests/golden/rescalk_cfg5.npz):
  selected k identical, s_min / s_avg within 1e-4, rel_error within 1e-5.
* rescal_solve(counters=KernelCounters()): the reference's per-phase MAC
  counts (rescal.py:124-153 counted_mm formulas) and per-phase device time.
* random_init falls back to the host draw (same values) for a bad device.
"""

import numpy as np
import pytest

import oracle
from conftest import golden, rel_fro, uniform_x

pytestmark = pytest.mark.gpu

rk = pytest.importorskip("paper_2202_09512_b200")
from paper_2202_09512_b200 import _lib  # noqa: E402


def _device_vs_oracle(n, m, k, iters, seed):
    eng = _lib.Engine(n, m, k, device=0, engine="tc")
    try:
        eng.fill_uniform(seed)
        x = eng.block_uniform(seed, n, n)  # exact fp32 values of the device tensor
        f0 = rk.random_init(n, k, m, 5)
        eng.set_factors(f0.A, f0.R)
        done, trace = eng.run(iters, 1e-16, track_error=True)
        a_dev, r_dev = eng.get_factors()
        info = eng.info()
    finally:
        eng.close()
    assert done == iters and len(trace) == iters
    a, r = f0.A.copy(), f0.R.copy()
    xs = [x[t].astype(np.float64) for t in range(m)]
    del x
    for _ in range(iters):
        a = oracle.mu_iteration(xs, a, r, 1e-16)
    err = np.sqrt(oracle.sq_residual(xs, a, r) / oracle.sq_norm(xs))
    return a_dev, r_dev, trace, a, r, err, info


def test_cfg3_shape_matches_oracle():
    # 10 iterations: MU amplifies K1's accumulation error over iterations;
    # with rotating Q drains (default) relR is 6.6e-6 here, without them
    # 5.1e-4 (profiles/r02_q_rotation.md)
    n, m, k, iters = 32768, 2, 32, 10
    a_dev, r_dev, trace, a, r, err, info = _device_vs_oracle(n, m, k, iters, 13)
    # strip groups of 4 CTAs: 6 strips of up to 43 column tiles, <= 11 per CTA
    assert info["engine"] == 1 and info["strip_tiles"] == 11 and info["strips"] == 6, info
    assert info["k1_group"] == 4 and info["strip_width"] == 43 and info["ctas"] == 148, info
    assert rel_fro(a_dev, a) <= 1e-4 and rel_fro(r_dev, r) <= 1e-4, (rel_fro(a_dev, a), rel_fro(r_dev, r))
    assert abs(trace[-1] - err) <= 1e-5, (trace[-1], err)
    assert np.all(np.diff(trace) <= 1e-9), trace


@pytest.mark.parametrize("k,k_pad,strip_tiles", [(40, 48, 6), (64, 64, 4), (20, 32, 11)])
def test_auto_engine_uses_tensor_cores_up_to_k64(k, k_pad, strip_tiles):
    eng = _lib.Engine(4096, 2, k, device=0)
    try:
        info = eng.info()
    finally:
        eng.close()
    assert info["engine"] == 1 and info["k_pad"] == k_pad and info["strip_tiles"] == strip_tiles, info


@pytest.mark.parametrize("qrot,q_bound", [("0", 6e-5), ("1", 1e-5)])
def test_k1_slice_products_accuracy(monkeypatch, qrot, q_bound):
    """K1's P = X A and Q = X^T A against fp64 at n = 32768 (k = 32, one
    slice): the TMEM sums' error grows with their length (k1_tc.cuh); the
    default schedule keeps Q within 6e-5, rotating drains (RK_K1_QROT=1)
    within 1e-5, P within 1e-5 either way."""
    monkeypatch.setenv("RK_K1_QROT", qrot)
    n, m, k = 32768, 1, 32
    eng = _lib.Engine(n, m, k, device=0, engine="tc")
    try:
        eng.fill_uniform(23)
        x = eng.block_uniform(23, n, n)[0]
        f0 = rk.random_init(n, k, m, 3)
        eng.set_factors(f0.A, f0.R)
        eng.update_r(1e-16)  # one K1 pass
        p, q = eng.debug_read_pq()
    finally:
        eng.close()
    a = f0.A
    pr = np.empty((n, k)); qr = np.zeros((n, k))
    for r0 in range(0, n, 4096):
        xb = x[r0:r0 + 4096].astype(np.float64)
        pr[r0:r0 + 4096] = xb @ a
        qr += xb.T @ a[r0:r0 + 4096]
    ep = rel_fro(p[0, :n, :k], pr)
    eq = rel_fro(q[0, :n, :k], qr)
    assert ep <= 1e-5 and eq <= q_bound, (ep, eq)


@pytest.mark.parametrize("n,merged", [(768, True), (1664, False), (4096, False)])
def test_k32_q_merge_schedules_match_oracle(n, merged):
    m, k, iters = 3, 32, 6
    a_dev, r_dev, trace, a, r, err, info = _device_vs_oracle(n, m, k, iters, 17)
    # merged Q accumulators are 2K = 64 TMEM columns: at most 6 column tiles per strip
    assert info["k1_merge_q"] == int(merged) and (not merged or info["strip_tiles"] <= 6), info
    assert rel_fro(a_dev, a) <= 1e-4 and rel_fro(r_dev, r) <= 1e-4
    assert abs(trace[-1] - err) <= 1e-5


def test_rescalk_cfg5_sweep_matches_reference():
    g = golden("rescalk_cfg5")
    x = rk.RelTensor(g["X"])
    rep = rk.rescalk(x, 2, 16, r=10, cfg=rk.SolverConfig(max_iters=200, seed=0),
                     pcfg=rk.PerturbConfig(delta=0.02, base_seed=0))
    assert [e.k for e in rep.entries] == list(g["ks"])
    assert rep.k_opt == int(g["k_opt"]) and rep.low_confidence == bool(g["low_conf"])
    for e, smr, sar, er in zip(rep.entries, g["s_min"], g["s_avg"], g["rel_error"]):
        assert abs(e.s_min - smr) <= 1e-4 and abs(e.s_avg - sar) <= 1e-4, (e.k, e.s_min, smr)
        assert abs(e.rel_error - er) <= 1e-5, (e.k, e.rel_error, er)


def test_counters_record_reference_phases():
    n, m, k, iters = 512, 3, 8, 12
    x = rk.RelTensor(uniform_x(m, n, 2).astype(np.float64))
    c = rk.KernelCounters()
    f, tr = rk.rescal_solve(x, k, rk.SolverConfig(max_iters=iters, seed=1), counters=c)
    f2, tr2 = rk.rescal_solve(x, k, rk.SolverConfig(max_iters=iters, seed=1))
    np.testing.assert_array_equal(f.A, f2.A)  # counting does not change the arithmetic
    gram = iters * (n * k * k + m * k * n * k)
    big = iters * m * 2 * n * n * k
    small = iters * m * (5 * n * k * k + 4 * k ** 3) + len(tr) * m * (n * k * k + n * k * n)
    assert c.flops == {"gram_mul": gram, "matrix_mul": big + small}, c.flops
    for ph in ("gram_mul", "matrix_mul", "device_run"):
        assert c.seconds[ph] > 0.0
    assert c.seconds["matrix_mul"] + c.seconds["gram_mul"] <= c.seconds["device_run"] * 1.05


def test_random_init_bad_device_falls_back_to_host():
    n, k, m = 1 << 17, 8, 2  # n * k >= 2^20: the device draw path
    host = oracle.random_init(n, k, m, 9)
    f = rk.random_init(n, k, m, 9, device=97)
    np.testing.assert_array_equal(f.A, host[0])
    np.testing.assert_array_equal(f.R, host[1])
    f0 = rk.random_init(n, k, m, 9, device=0)
    np.testing.assert_array_equal(f0.A, host[0])


def test_rescalk_on_sparse_tensor_matches_reference():
    """The CSR engine end to end: members resample the stored values only
    (dist_rescal.py:205-214); nothing is densified."""
    import scipy.sparse as sp

    g = golden("rescalk_sparse")
    x = rk.SparseRelTensor([sp.csr_matrix(s) for s in g["X"]])
    rep = rk.rescalk(x, 2, 4, r=4, cfg=rk.SolverConfig(max_iters=150, seed=2),
                     pcfg=rk.PerturbConfig(delta=0.02, base_seed=5))
    assert rep.k_opt == int(g["k_opt"])
    for e, smr, sar, er in zip(rep.entries, g["s_min"], g["s_avg"], g["rel_error"]):
        assert abs(e.s_min - smr) <= 1e-4 and abs(e.s_avg - sar) <= 1e-4, (e.k, e.s_min, smr)
        assert abs(e.rel_error - er) <= 1e-5, (e.k, e.rel_error, er)
        np.testing.assert_allclose(e.medians, g[f"medians_k{e.k}"], atol=1e-4)


@pytest.mark.parametrize("n,pr,pc", [(13, 2, 2), (20, 2, 4), (9, 1, 2)])
def test_dist_perturb_is_grid_independent(n, pr, pc):
    """dist_rescal.py:174-203: a rank's resampled block is the same block of
    the whole-tensor resampling, for any grid; sparse blocks keep their pattern."""
    import scipy.sparse as sp
    from paper_2202_09512_b200.multigpu import block_of, piece_layout

    m = 2
    rng = np.random.default_rng(n)
    xd = rng.random((m, n, n))
    pcfg = rk.PerturbConfig(delta=0.05, base_seed=3)
    whole = rk.perturb(rk.RelTensor(xd), pcfg, (4, 2)).slices
    mask = rng.random((m, n, n)) < 0.3
    xs = rk.SparseRelTensor([sp.csr_matrix(xd[t] * mask[t]) for t in range(m)])
    whole_s = np.stack([s.toarray() for s in rk.perturb(xs, pcfg, (4, 2)).slices])
    for r in range(pr * pc):
        gi, gj = r // pc, r % pc
        lay = piece_layout(n, pr, pc, gi, gj)
        blk = rk.dist_perturb(rk.grid_block(rk.RelTensor(xd), pr, pc, gi, gj), pcfg, (4, 2))
        np.testing.assert_array_equal(blk.slices, block_of(whole, n, lay))
        sblk = rk.dist_perturb(rk.grid_block(xs, pr, pc, gi, gj), pcfg, (4, 2))
        np.testing.assert_array_equal(np.stack([q.toarray() for q in sblk.slices]), block_of(whole_s, n, lay))
