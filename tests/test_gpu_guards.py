"""Memory-safety and race evidence without compute-sanitizer (closed on the GPU
pool: profiles/r02_memcheck.log).

* Guard bands (rk_debug_guards): every device block allocated while guards
  are on is followed by 64 KB of a fixed pattern. A sweep over the engines and
  entry points at ragged shapes (n not a multiple of 128, k not a multiple of
  16, k > 32, sparse rows without entries) must leave every band intact.
* Determinism: the K1 mbarrier / TMA / TMEM pipeline, the deterministic
  partial reductions and the k x k kernels must give bit-identical factors on
  repeated runs from the same start (a race shows up as run-to-run noise).
* Concurrency: two engines on one GPU at once (strip-group K1 is launched
  cooperatively) finish with the factors of their serial runs.
"""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import uniform_x

pytestmark = pytest.mark.gpu

rk = pytest.importorskip("paper_2202_09512_b200")
from paper_2202_09512_b200 import _lib  # noqa: E402


def _sweep():
    rng = np.random.default_rng(0)
    for n, m, k in ((300, 3, 16), (200, 2, 5), (131, 2, 27), (700, 2, 32), (257, 2, 40), (1664, 2, 32)):
        x = rk.RelTensor(uniform_x(m, n, n + k))
        for engine in ("auto", "simt"):
            f, tr = rk.rescal_solve(x, k, rk.SolverConfig(max_iters=5, seed=1, engine=engine))
        fr = rk.update_r(x, f)
        rk.update_a(x, fr)
        rk.regress_r(x, f.A, max_iters=20)
        rk.rel_error(x, f)
        rk.perturb(x, rk.PerturbConfig(delta=0.02), (k, 1))
    # tolerance stop and the direct residual switch
    xe = rk.RelTensor(uniform_x(2, 96, 3))
    rk.rescal_solve(xe, 4, rk.SolverConfig(max_iters=50, tolerance=0.45))
    # sparse engine, with empty rows and columns
    n, m = 1500, 2
    sl = []
    for t in range(m):
        d = sp.random(n, n, density=0.003, random_state=t, format="csr", dtype=np.float64)
        d = d.tolil()
        d[:50, :] = 0
        d[:, -40:] = 0
        sl.append(sp.csr_matrix(d))
    xs = rk.SparseRelTensor(sl)
    for k in (8, 16, 27):
        f, tr = rk.rescal_solve(xs, k, rk.SolverConfig(max_iters=4, seed=2))
        rk.rel_error(xs, f)
    rk.nndsvd_init(rk.RelTensor(uniform_x(2, 64, 9)), 3)
    rk.rescalk(rk.RelTensor(uniform_x(2, 48, 5)), 2, 3, r=2, cfg=rk.SolverConfig(max_iters=10))
    rk.rescalk(xs, 2, 3, r=2, cfg=rk.SolverConfig(max_iters=5))


def test_no_write_past_any_device_buffer():
    rk.release_cached_memory()
    _lib.debug_guards(True)
    try:
        # positive control: a deliberate 3-byte overrun must be seen
        b0, _ = _lib.debug_check_guards()
        _lib.check(_lib.load().rk_debug_overrun(3))
        b1, _ = _lib.debug_check_guards()
        assert b1 - b0 == 3, (b0, b1)
        _sweep()
        rk.release_cached_memory()  # frees the kept engine: its bands are checked on free
        bad, live = _lib.debug_check_guards()
    finally:
        _lib.debug_guards(False)
    assert bad - b1 == 0, f"{bad - b1} guard bytes overwritten"


@pytest.mark.parametrize("n,m,k", [(1024, 4, 16), (1664, 3, 32), (20000, 2, 32)])
def test_repeated_runs_are_bit_identical(n, m, k):
    x = uniform_x(m, n, 11)
    f0 = rk.random_init(n, k, m, 2)
    eng = _lib.Engine(n, m, k, device=0)
    try:
        eng.upload(x)
        ref = None
        for rep in range(6):
            eng.set_factors(f0.A, f0.R)
            _, tr = eng.run(12, 1e-16, track_error=True)
            a, r = eng.get_factors()
            cur = (a.tobytes(), r.tobytes(), tr.tobytes())
            if ref is None:
                ref = cur
            assert cur == ref, f"run {rep} differs from run 0"
    finally:
        eng.close()


def test_concurrent_engines_with_strip_groups():
    """Two engines solving at once on one GPU (two host threads, two streams):
    K1 with strip groups (members wait for each other's P tiles) is launched
    cooperatively, so both solves finish and match their serial results."""
    import threading

    n, m, k, iters = 16384, 2, 32, 6
    starts = [rk.random_init(n, k, m, 40 + i) for i in range(2)]

    def solve(i, out):
        eng = _lib.Engine(n, m, k, device=0)
        try:
            eng.fill_uniform(50 + i)
            assert eng.info()["k1_group"] == 2
            eng.set_factors(starts[i].A, starts[i].R)
            eng.run(iters, 1e-16, track_error=False)
            out[i] = eng.get_factors()
        finally:
            eng.close()

    serial = {}
    for i in range(2):
        solve(i, serial)
    conc = {}
    th = [threading.Thread(target=solve, args=(i, conc)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in th), "concurrent solves did not finish"
    for i in range(2):
        assert np.array_equal(conc[i][0], serial[i][0]) and np.array_equal(conc[i][1], serial[i][1])
