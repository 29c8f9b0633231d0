"""Drop-in RESCAL MU solver API backed by the sm_100a engine.

Mirrors the public functions of the reference serial solver
(pkg/src/rescalkit/rescal.py) — same names, signatures, defaults, dtypes and
error classes — but every tensor contraction runs in ``librescal_b200.so``:

  rescal_solve      rescal.py:186-225   -> rk_set_factors + rk_run + rk_get_factors
  update_r          rescal.py:228-240   -> rk_update_r
  update_a          rescal.py:243-258   -> rk_update_a
  rel_error         rescal.py:269-276   -> rk_residual
  regress_r         rescal.py:293-324   -> rk_regress_r
  finalize_normalize, random_init       host k-sized math (identical to the reference)

Numerics: the tensor is held as bf16 hi+lo planes and contracted with 3xBF16
tcgen05 MMAs (fp32 accumulate); all k x k algebra and the factor masters are
fp64 on the device. Results are returned in x.dtype (rescal.py:205-209).
"""

from __future__ import annotations

import contextlib
import os
import threading
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .exceptions import DataError, NumericalError
from .containers import dense_slices, is_sparse, tensor_dtype

_SEED_TAG_A = 1
_SEED_TAG_R = 2
_DENSIFY_MAX = 1 << 28  # elements: a sparse tensor this small may run on the dense engine when k > 32


@dataclass
class SolverConfig:
    """Solver settings; defaults and validation as rescal.py:30-53.

    ``engine`` (extension): "auto" | "tc" (tcgen05) | "simt" (CUDA cores);
    ``device`` (extension): CUDA ordinal, default LOCAL_RANK or 0.
    """

    max_iters: int = 200
    epsilon: float = 1e-16
    tolerance: float | None = None
    init: str = "random"  # "random" | "nndsvd"
    seed: int = 0
    track_error: bool = True
    engine: str = "auto"
    device: int | None = None

    def __post_init__(self):
        if self.max_iters < 1:
            raise DataError(f"max_iters must be >= 1, got {self.max_iters}")
        if not self.epsilon > 0:
            raise DataError(f"epsilon must be > 0, got {self.epsilon}")
        if self.init not in ("random", "nndsvd"):
            raise DataError(f"unknown init {self.init!r}")
        if self.engine not in _lib.ENGINES:
            raise DataError(f"unknown engine {self.engine!r}")


@dataclass
class RescalFactors:
    """Entity matrix A (n x k) and core stack R (m x k x k); rescal.py:56-88."""

    A: np.ndarray
    R: np.ndarray

    def __post_init__(self):
        self.A = np.asarray(self.A)
        self.R = np.asarray(self.R)
        if self.A.ndim != 2 or self.R.ndim != 3:
            raise DataError(f"bad factor shapes {self.A.shape}, {self.R.shape}")
        if self.R.shape[1] != self.R.shape[2] or self.R.shape[1] != self.A.shape[1]:
            raise DataError(f"inconsistent latent dimension: A {self.A.shape}, R {self.R.shape}")
        if (self.A.size and self.A.min() < 0) or (self.R.size and self.R.min() < 0):
            raise DataError("factors must be non-negative")

    @property
    def n(self) -> int:
        return self.A.shape[0]

    @property
    def k(self) -> int:
        return self.A.shape[1]

    @property
    def m(self) -> int:
        return self.R.shape[0]

    def copy(self) -> "RescalFactors":
        return RescalFactors(self.A.copy(), self.R.copy())


def random_init(n: int, k: int, m: int, seed, dtype=np.float64, device: int | None = None) -> RescalFactors:
    """Seeded uniform start, partition independent (rescal.py:173-183):
    A from SeedSequence((seed, 1)), R from SeedSequence((seed, 2)), drawn in
    fp64 then cast. ``device`` (extension): the GPU that draws a large A
    (default: LOCAL_RANK); any device failure falls back to the host draw,
    which gives the same values."""
    gr = np.random.default_rng(np.random.SeedSequence((seed, _SEED_TAG_R)))
    a = _device_uniform(seed, _SEED_TAG_A, n * k, device)
    if a is None:
        ga = np.random.default_rng(np.random.SeedSequence((seed, _SEED_TAG_A)))
        a = ga.random((n, k), dtype=np.float64)
    return RescalFactors(a.reshape(n, k).astype(dtype),
                         gr.random((m, k, k), dtype=np.float64).astype(dtype))


# Large starts (n*k >= 2^20 doubles, e.g. 0.3 s of sequential host PCG64 at
# n = 2^20, k = 16) are drawn on the GPU: the same PCG64 stream, each thread
# jumping ahead to its element (rk_pcg64_draws_on), bit-identical to numpy.
_DEVICE_DRAW_MIN = 1 << 20


def _device_uniform(seed, tag, count, device=None):
    if count < _DEVICE_DRAW_MIN or not isinstance(seed, (int, np.integer)):
        return None
    try:
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", "0"))
        if not 0 <= device < _lib.device_count():
            return None
        return _lib.pcg64_random_on(int(device), (int(seed), tag), count)
    except Exception:  # noqa: BLE001 — no library / no GPU / OOM: the host generator gives the same values
        return None


def finalize_normalize(f: RescalFactors) -> RescalFactors:
    """Unit-norm columns of A with D R_t D compensation (rescal.py:279-290)."""
    norms = np.linalg.norm(f.A, axis=0)
    scale = np.where(norms > 0, norms, 1.0).astype(f.A.dtype)
    return RescalFactors(f.A / scale, f.R * scale[None, :, None] * scale[None, None, :])


# ---------------------------------------------------------------------------
# engine plumbing


# One idle engine per host thread is kept for the next call with the same
# (device, n, m, k, engine kind): repeated small solves (RESCALk members,
# update_r / update_a / rel_error loops) skip handle creation (stream, pinned
# control block, buffer set-up: ~5 ms at cfg1 against ~1 ms of iterations).
# Engines of any size are kept (a cfg3-sized call then skips handle and plan
# set-up and reuses its captured graphs); a kept engine that does not match
# the next call is closed BEFORE the new one is created, so at most one
# tensor's device storage is held per thread. The library's allocator keeps
# freed blocks cached either way; release_cached_memory() drops both. Every
# use re-uploads x and resets the factors, so a cached engine is
# indistinguishable from a fresh one.
_CACHE = threading.local()
_CACHE_MAX_BYTES = 1 << 40


def _engine_key(x, k, cfg: SolverConfig):
    device = cfg.device if cfg.device is not None else int(os.environ.get("LOCAL_RANK", "0"))
    sparse = is_sparse(x) and k <= 32
    return (device, x.n, x.m, k, "sparse" if sparse else cfg.engine)


def _engine_for(x, k, cfg: SolverConfig):
    """Device engine holding ``x``: the CSR/CSC engine for sparse tensors
    (k <= 32), the dense tcgen05/SIMT engine otherwise."""
    key = _engine_key(x, k, cfg)
    cached = getattr(_CACHE, "entry", None)
    _CACHE.entry = None
    if cached is not None and cached[0] == key and cached[1].k == k:
        eng = cached[1]
    else:
        eng = None
        if cached is not None:
            cached[1].close()  # free its device storage before the new engine allocates
    if key[4] != "sparse" and is_sparse(x) and x.m * x.n * x.n > _DENSIFY_MAX:
        if eng is not None:
            eng.close()
        raise DataError(f"the sparse (CSR) engine supports k <= 32 (k={k}); a dense copy of this "
                        f"tensor ({x.m}x{x.n}x{x.n}) is too large")
    if eng is None:
        eng = (_lib.Engine(x.n, x.m, k, device=key[0], sparse=True) if key[4] == "sparse"
               else _lib.Engine(x.n, x.m, k, device=key[0], engine=cfg.engine))
    try:
        if key[4] == "sparse":
            eng.upload_csr(list(x.slices))
        else:
            eng.upload(dense_slices(x))
    except BaseException:
        eng.close()  # a rejected upload must not leave the engine holding device memory
        raise
    eng._cache_key = key
    return eng


def drop_cached_engine() -> None:
    """Close this thread's kept engine (callers that create their own engine
    for a large tensor, e.g. rescalk, free its device storage first)."""
    old = getattr(_CACHE, "entry", None)
    _CACHE.entry = None
    if old is not None:
        old[1].close()


def _release_engine(eng) -> None:
    """Keep the engine for the next call (closing the one kept before)."""
    key = getattr(eng, "_cache_key", None)
    dense_bytes = 4 * eng.m * eng.n * eng.n
    if key is None or (not eng.sparse and dense_bytes > _CACHE_MAX_BYTES) or (
            eng.sparse and eng.nnz * 8 > _CACHE_MAX_BYTES):
        eng.close()
        return
    old = getattr(_CACHE, "entry", None)
    if old is not None and old[1] is not eng:
        old[1].close()
    _CACHE.entry = ((key[0], eng.n, eng.m, eng.k, key[4]), eng)


def release_cached_memory() -> None:
    """Close the kept engines (this thread's single-GPU engine, the process's
    grid engine) and return the device allocator's cached blocks."""
    old = getattr(_CACHE, "entry", None)
    _CACHE.entry = None
    if old is not None:
        old[1].close()
    from .multigpu import release_grid_cache

    release_grid_cache()
    _lib.release_cached_memory()


@contextlib.contextmanager
def _engine_ctx(x, k, cfg: SolverConfig):
    eng = _engine_for(x, k, cfg)
    try:
        yield eng
    finally:
        _release_engine(eng)


def _check_shapes(x, f: RescalFactors) -> None:
    if f.A.shape[0] != x.n or f.R.shape[0] != x.m:
        raise DataError(
            f"shape mismatch: tensor (n={x.n}, m={x.m}) vs factors A {f.A.shape}, R {f.R.shape}")


def _to_dtype(a, dt):
    return np.asarray(a).astype(dt, copy=False)


class KernelCounters:
    """Multiply-add and time accounting per kernel phase (grid.py:72-94).

    The reference counts the MACs of every ``counted_mm`` call under the
    phases ``gram_mul`` (A^T A, A^T X A), ``matrix_mul`` (dense products) and
    ``matrix_mul_sparse`` (sparse-left products) and times them on the host.
    Here ``rescal_solve(counters=...)`` records the same MAC counts (the
    reference's per-call formulas summed analytically, rescal.py:124-153) and
    the device time of the kernels behind each phase, measured with CUDA
    events between the phases of every iteration (the run is not graph-
    replayed while counting); ``device_run`` is the whole solve."""

    def __init__(self):
        self.flops = {}
        self.seconds = {}

    def add_flops(self, phase: str, n: int) -> None:
        self.flops[phase] = self.flops.get(phase, 0) + int(n)

    def add_time(self, phase: str, dt: float) -> None:
        self.seconds[phase] = self.seconds.get(phase, 0.0) + dt

    @contextlib.contextmanager
    def timed(self, phase: str):
        t0 = time.perf_counter()
        try:
            yield
        finally:
            self.add_time(phase, time.perf_counter() - t0)

    def total_flops(self) -> int:
        return sum(self.flops.values())


def _count_iteration(counters, x, k: int, iters: int, tracked: int) -> None:
    """MACs of `iters` MU iterations and `tracked` residual evaluations, with
    the reference's counted_mm formulas (x@y of (a,b)@(b,c) counts a*b*c; a
    sparse left operand counts nnz*c)."""
    n, m = x.n, x.m
    sparse = is_sparse(x)
    gram = n * k * k + m * k * n * k  # ata, atxa per slice
    small = m * (5 * n * k * k + 4 * k ** 3)  # xart ar art artatar aratart + rata deno_r atar atart
    counters.add_flops("gram_mul", iters * gram)
    counters.add_flops("matrix_mul", iters * small + tracked * m * (n * k * k + n * k * n))
    if sparse:
        counters.add_flops("matrix_mul_sparse", iters * 2 * k * sum(s.nnz for s in x.slices))
    else:
        counters.add_flops("matrix_mul", iters * m * 2 * n * n * k)


def _phase_times(counters, eng, iters: int) -> None:
    """Device time per phase of the last profiled run -> reference phase names."""
    ph = eng.phase_timing()  # ms per iteration: k1, k2a, allreduce, k2f, numer_rs, apply_gather
    big = "matrix_mul_sparse" if eng.sparse else "matrix_mul"
    counters.add_time(big, ph["k1"] * iters / 1e3)
    counters.add_time("gram_mul", ph["k2a"] * iters / 1e3)
    counters.add_time("matrix_mul", (ph["k2f"] + ph["numer_rs"] + ph["apply_gather"]) * iters / 1e3)
    if ph["allreduce"]:
        counters.add_time("all_reduce", ph["allreduce"] * iters / 1e3)


def rescal_solve(x, k: int, cfg: SolverConfig | None = None, initial=None, counters=None,
                 engine: "_lib.Engine | None" = None):
    """Factorize ``x`` at rank ``k``; returns (RescalFactors, error trace).

    Same contract as rescal.py:186-225: ``initial`` is copied, otherwise the
    seeded random start; the trace holds err_l after each iteration and the
    loop stops once err_l < tolerance. ``counters`` (a KernelCounters)
    receives the reference's per-phase MAC counts and the device time of
    each phase. ``engine`` (extension) reuses a device-resident tensor across
    calls.
    """
    cfg = cfg or SolverConfig()
    if not 1 <= k <= x.n:
        raise DataError(f"need 1 <= k <= n, got k={k}, n={x.n}")
    dt = tensor_dtype(x)
    if initial is not None:
        f = initial.copy()
        if f.A.shape != (x.n, k) or f.R.shape != (x.m, k, k):
            raise DataError("initial factors do not match tensor/k")
    else:
        f = None if cfg.init == "nndsvd" else random_init(x.n, k, x.m, cfg.seed, dtype=dt, device=cfg.device)
    own = engine is None
    eng = engine if engine is not None else _engine_for(x, k, cfg)
    try:
        if f is None:  # rescal.py:202-203
            f = nndsvd_init(x, k, eps=cfg.epsilon, cfg=cfg, engine=eng)
        # the reference casts the start to x.dtype (rescal.py:206-208)
        a0 = _to_dtype(f.A, dt).astype(np.float64)
        r0 = _to_dtype(f.R, dt).astype(np.float64)
        if eng.k != k:
            eng.set_rank(k)
        eng.set_factors(a0, r0)
        eps = float(dt.type(cfg.epsilon))
        if counters is not None:
            eng.set_option(1, 1)  # per-phase CUDA events (no graph replay while counting)
        try:
            done, trace = eng.run(cfg.max_iters, eps, track_error=cfg.track_error, tol=cfg.tolerance)
        finally:
            if counters is not None:
                eng.set_option(1, 0)
        a, r = eng.get_factors()
        if counters is not None:
            _count_iteration(counters, x, k, done, len(trace))
            _phase_times(counters, eng, done)
            counters.add_time("device_run", eng.timing()["run_ms"] / 1e3)
    finally:
        if own:
            _release_engine(eng)
    return RescalFactors(a.astype(dt), r.astype(dt)), np.asarray(trace)


def update_r(x, f: RescalFactors, cfg: SolverConfig | None = None) -> RescalFactors:
    """One multiplicative pass over all cores with A fixed (rescal.py:228-240)."""
    cfg = cfg or SolverConfig()
    _check_shapes(x, f)
    dt = f.A.dtype
    with _engine_ctx(x, f.k, cfg) as eng:
        eng.set_factors(f.A.astype(np.float64), f.R.astype(np.float64))
        eng.update_r(float(dt.type(cfg.epsilon)))
        _, r = eng.get_factors()
    return RescalFactors(f.A, r.astype(f.R.dtype))


def update_a(x, f: RescalFactors, cfg: SolverConfig | None = None) -> RescalFactors:
    """One accumulated multiplicative update of A, cores fixed (rescal.py:243-258)."""
    cfg = cfg or SolverConfig()
    _check_shapes(x, f)
    dt = f.A.dtype
    with _engine_ctx(x, f.k, cfg) as eng:
        eng.set_factors(f.A.astype(np.float64), f.R.astype(np.float64))
        eng.update_a(float(dt.type(cfg.epsilon)))
        a, _ = eng.get_factors()
    return RescalFactors(a.astype(dt), f.R)


def rel_error(x, f: RescalFactors, engine: "_lib.Engine | None" = None) -> float:
    """|X - A R A^T|_F / |X|_F (rescal.py:269-276), residual on the device."""
    _check_shapes(x, f)
    own = engine is None
    eng = engine if engine is not None else _engine_for(x, f.k, SolverConfig())
    try:
        if eng.k != f.k:
            eng.set_rank(f.k)
        eng.set_factors(np.asarray(f.A, dtype=np.float64), np.asarray(f.R, dtype=np.float64))
        res, nrm = eng.residual()
    finally:
        if own:
            _release_engine(eng)
    if nrm == 0.0:
        raise DataError("relative error undefined: tensor norm is zero")
    return float(np.sqrt(res / nrm))


def regress_r(x, a_fixed: np.ndarray, cfg: SolverConfig | None = None, max_iters: int = 500,
              tol: float | None = 1e-8, engine: "_lib.Engine | None" = None) -> np.ndarray:
    """Refit the cores with A frozen, from all-ones (rescal.py:293-324)."""
    cfg = cfg or SolverConfig()
    a = np.asarray(a_fixed)
    if a.ndim != 2 or a.shape[0] != x.n:
        raise DataError(f"A must be (n, k) with n={x.n}, got {a.shape}")
    if a.size and a.min() < 0:
        raise DataError("A must be non-negative")
    k = a.shape[1]
    own = engine is None
    eng = engine if engine is not None else _engine_for(x, k, cfg)
    try:
        if eng.k != k:
            eng.set_rank(k)
        eng.set_factors(a.astype(np.float64), np.ones((x.m, k, k)))
        eng.regress_r(max_iters, tol, float(a.dtype.type(cfg.epsilon)))
        _, r = eng.get_factors()
    finally:
        if own:
            _release_engine(eng)
    if not (np.isfinite(a).all() and np.isfinite(r).all()):
        raise NumericalError("non-finite value in factors; aborting")
    return r.astype(a.dtype)


def _nndsvd_block(eng, n: int, k: int) -> int:
    if eng.sparse:
        if k > 32:
            raise DataError("nndsvd_init on the sparse engine supports k <= 32")
        return 16 if k + 4 <= 16 else 32
    b = min(n, k + 8)
    if b > 256:
        raise DataError("nndsvd_init on the device supports k <= 248")
    return b


def _leading_singular(eng, n: int, k: int, max_iters: int = 300, rtol: float = 1e-10):
    """Top-k left singular vectors / values of the unfolding M = [X_t | X_t^T]
    by subspace iteration on M M^T (device products, rk_gram_apply) with a
    Rayleigh-Ritz step; the reference takes them from a full LAPACK SVD
    (dense) or ARPACK svds (sparse) of M (rescal.py:341-352). Deterministic:
    fixed start block."""
    b = _nndsvd_block(eng, n, k)

    def orth(z):
        q, _ = np.linalg.qr(z)
        if q.shape[1] < b:  # n < b: keep the block width the kernels expect
            q = np.concatenate([q, np.zeros((n, b - q.shape[1]))], axis=1)
        return q

    v = orth(np.random.default_rng(20220218).standard_normal((n, b)))
    prev = None
    for it in range(max_iters):
        y = eng.gram_apply(v)
        t = v.T @ y
        lam = np.sort(np.linalg.eigvalsh(0.5 * (t + t.T)))[::-1][:k]
        scale = max(abs(lam[0]), np.finfo(float).tiny)
        if prev is not None and it >= 8 and np.max(np.abs(lam - prev)) <= rtol * scale:
            break
        prev = lam
        v = orth(y)
    y = eng.gram_apply(v)
    t = v.T @ y
    w, wv = np.linalg.eigh(0.5 * (t + t.T))
    order = np.argsort(w)[::-1][:k]
    u = v @ wv[:, order]
    s = np.sqrt(np.maximum(w[order], 0.0))
    return u, s, b


def _nndsvd_factor(eng, n: int, k: int) -> np.ndarray:
    """The A of nndsvd_init (rescal.py:354-370) from device singular data."""
    u, s, b = _leading_singular(eng, n, k)
    upad = np.zeros((n, b))
    upad[:, :k] = u
    pos2, neg2 = eng.unfold_sign_norms(upad if eng.sparse else upad[:, :max(k, 1)])
    a = np.zeros((n, k))
    lead = u[:, 0] if u[:, 0].sum() >= 0 else -u[:, 0]
    a[:, 0] = np.sqrt(s[0]) * np.maximum(lead, 0.0)
    for j in range(1, k):
        if s[j] <= 0:
            continue  # rank-deficient direction, filled below
        xu = u[:, j]
        xp, xm = np.maximum(xu, 0.0), np.maximum(-xu, 0.0)
        # right singular vector v_j = M^T u_j / s_j: norms of its +/- parts
        yp, ym = np.sqrt(pos2[j]) / s[j], np.sqrt(neg2[j]) / s[j]
        mu_p = np.linalg.norm(xp) * yp
        mu_m = np.linalg.norm(xm) * ym
        if max(mu_p, mu_m) <= 0:
            continue
        part, norm = (xp, np.linalg.norm(xp)) if mu_p >= mu_m else (xm, np.linalg.norm(xm))
        a[:, j] = np.sqrt(s[j] * max(mu_p, mu_m)) * part / norm
    positives = eng.positive_mean()
    fill = 1e-2 * positives if positives > 0 else 1e-2
    a[a == 0] = fill
    return a


def nndsvd_init(x, k: int, r_update_iters: int = 20, eps: float = 1e-16, cfg: SolverConfig | None = None,
                engine: "_lib.Engine | None" = None) -> RescalFactors:
    """Deterministic NNDSVD start (rescal.py:327-372): A from the non-negative
    parts of the leading singular vectors of [X_1 .. X_m | X_1^T .. X_m^T],
    zeros filled with 1e-2 x the mean positive entry, then `r_update_iters`
    R refits with A fixed. The singular vectors come from a device subspace
    iteration (products with the unfolding on the GPU); ``engine`` (extension)
    reuses a device-resident tensor."""
    if not 1 <= k <= x.n:
        raise DataError(f"need 1 <= k <= n, got k={k}, n={x.n}")
    cfg = cfg or SolverConfig()
    own = engine is None
    eng = engine if engine is not None else _engine_for(x, k, cfg)
    try:
        a = _nndsvd_factor(eng, x.n, k).astype(tensor_dtype(x))
        r = regress_r(x, a, SolverConfig(epsilon=eps, device=cfg.device), max_iters=r_update_iters, tol=None,
                      engine=eng)
    finally:
        if own:
            _release_engine(eng)
    return RescalFactors(a, r)
