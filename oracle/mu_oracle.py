"""numpy restatement of the reference MU arithmetic (oracle; tests only).

Every function cites the reference span it restates (paths relative to
``/root/reference/pkg/src/rescalkit``). The floating-point operation order is
kept identical to the reference so that, on the same numpy/OpenBLAS build, the
results agree bit-for-bit with the golden vectors in ``tests/golden``.

Notation: X is a list of m slice operands (dense (n, n) arrays or scipy CSR),
A is (n, k), R is (m, k, k).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp


@dataclass
class OracleConfig:
    """Mirror of ``SolverConfig`` defaults (rescal.py:30-53)."""

    max_iters: int = 200
    epsilon: float = 1e-16
    tolerance: float | None = None
    seed: int = 0
    track_error: bool = True


# --------------------------------------------------------------------------
# seeds and init


def random_init(n, k, m, seed, dtype=np.float64):
    """rescal.py:173-183 — A from SeedSequence((seed, 1)), R from (seed, 2),
    both drawn as float64 uniforms then cast."""
    ga = np.random.default_rng(np.random.SeedSequence((seed, 1)))
    gr = np.random.default_rng(np.random.SeedSequence((seed, 2)))
    a = ga.random((n, k), dtype=np.float64).astype(dtype)
    r = gr.random((m, k, k), dtype=np.float64).astype(dtype)
    return a, r


# --------------------------------------------------------------------------
# the MU iteration


def mu_iteration(xs, a, r, eps):
    """rescal.py:114-146 with the serial (identity) hooks.

    Gauss-Seidel order: G from the old A once (:124); per slice the core is
    updated first (:128-132) and the NEW core feeds the A numerator and
    denominator (:133-143, eps added per slice at :143); A is updated once
    at the end (:144). ``r`` is updated in place, the new A is returned.
    """
    gram = a.T @ a
    numer = np.zeros_like(a)
    denom = np.zeros_like(a)
    for t, xt in enumerate(xs):
        xa = np.asarray(xt @ a)
        s_t = a.T @ xa
        r_gram = r[t] @ gram
        r[t] = r[t] * s_t / (gram @ r_gram + eps)
        rt = r[t]
        xa_rt = xa @ rt.T
        a_r = a @ rt
        xt_ar = np.asarray(xt.T @ a_r)
        numer += xa_rt + xt_ar
        g_r = gram @ rt
        a_rt = a @ rt.T
        left = a_rt @ g_r
        g_rt = gram @ rt.T
        right = a_r @ g_rt
        denom += left + right + eps
    return a * numer / denom


def sq_residual(xs, a, r):
    """rescal.py:149-157 — sum_t ||X_t - (A R_t) A^T||^2, squared in fp64."""
    acc = 0.0
    for t, xt in enumerate(xs):
        recon = (a @ r[t]) @ a.T
        dense = xt.toarray() if sp.issparse(xt) else xt
        acc += float(np.sum((dense - recon).astype(np.float64) ** 2))
    return acc


def sq_norm(xs):
    """rescal.py:160-165 — stored values squared and summed in fp64."""
    acc = 0.0
    for xt in xs:
        v = xt.data if sp.issparse(xt) else xt
        acc += float(np.sum(np.asarray(v, dtype=np.float64) ** 2))
    return acc


def _finite_or_raise(a, r):
    """rescal.py:168-170."""
    if not (np.isfinite(a).all() and np.isfinite(r).all()):
        raise FloatingPointError("non-finite value in factors")


def solve(xs, k, cfg: OracleConfig | None = None, initial=None, dtype=np.float64):
    """rescal.py:186-225 — returns (A, R, trace).

    ``initial`` is an (A, R) pair (copied, :198-201); otherwise the seeded
    random start of :204-207. The trace holds err_l after iteration l and the
    loop stops as soon as err_l < tolerance (:218-224).
    """
    cfg = cfg or OracleConfig()
    n, m = xs[0].shape[0], len(xs)
    if initial is not None:
        a, r = np.array(initial[0], copy=True), np.array(initial[1], copy=True)
    else:
        a, r = random_init(n, k, m, cfg.seed, dtype=dtype)
    eps = np.dtype(dtype).type(cfg.epsilon)
    norm2 = sq_norm(xs) if cfg.track_error else None
    if cfg.track_error and norm2 == 0.0:
        raise ValueError("zero tensor norm")
    trace = []
    for _ in range(cfg.max_iters):
        a = mu_iteration(xs, a, r, eps)
        _finite_or_raise(a, r)
        if cfg.track_error:
            e = float(np.sqrt(sq_residual(xs, a, r) / norm2))
            trace.append(e)
            if cfg.tolerance is not None and e < cfg.tolerance:
                break
    return a, r, np.asarray(trace)


def update_r(xs, a, r, eps=1e-16):
    """rescal.py:228-240 — one pass over the cores with A fixed."""
    eps = a.dtype.type(eps)
    gram = a.T @ a
    out = r.copy()
    for t, xt in enumerate(xs):
        s_t = a.T @ np.asarray(xt @ a)
        out[t] = out[t] * s_t / (gram @ (out[t] @ gram) + eps)
    return out


def update_a(xs, a, r, eps=1e-16):
    """rescal.py:243-258 — one accumulated A update with the cores fixed."""
    eps = a.dtype.type(eps)
    gram = a.T @ a
    numer = np.zeros_like(a)
    denom = np.zeros_like(a)
    for t, xt in enumerate(xs):
        xa = np.asarray(xt @ a)
        a_r = a @ r[t]
        numer += xa @ r[t].T + np.asarray(xt.T @ a_r)
        a_rt = a @ r[t].T
        denom += a_rt @ (gram @ r[t]) + a_r @ (gram @ r[t].T) + eps
    return a * numer / denom


def rel_error(xs, a, r):
    """rescal.py:269-276."""
    norm2 = sq_norm(xs)
    if norm2 == 0.0:
        raise ValueError("zero tensor norm")
    return float(np.sqrt(sq_residual(xs, a, r) / norm2))


def finalize_normalize(a, r):
    """rescal.py:279-290 — unit column norms for A, D R_t D for the cores."""
    norms = np.linalg.norm(a, axis=0)
    scale = np.where(norms > 0, norms, 1.0).astype(a.dtype)
    return a / scale, r * scale[None, :, None] * scale[None, None, :]


def regress_r(xs, a, eps=1e-16, max_iters=500, tol=1e-8):
    """rescal.py:293-324 — R-only fit from all-ones cores, A frozen.

    S_t = A^T X_t A is formed once (:309); each sweep is Jacobi over t
    (:312-314); the stop test uses the fp64 Frobenius norms (:315-320).
    """
    a = np.asarray(a)
    eps = a.dtype.type(eps)
    k, m = a.shape[1], len(xs)
    gram = a.T @ a
    s = np.stack([a.T @ np.asarray(xt @ a) for xt in xs])
    r = np.ones((m, k, k), dtype=a.dtype)
    for _ in range(max_iters):
        nxt = np.empty_like(r)
        for t in range(m):
            nxt[t] = r[t] * s[t] / (gram @ (r[t] @ gram) + eps)
        if tol is None:
            r = nxt
            continue
        base = float(np.linalg.norm(r.astype(np.float64)))
        step = float(np.linalg.norm((nxt - r).astype(np.float64)))
        r = nxt
        if base == 0.0 or step / base < tol:
            break
    _finite_or_raise(a, r)
    return r


# --------------------------------------------------------------------------
# NNDSVD start


def nndsvd_init(xs, k, r_update_iters=20, eps=1e-16):
    """rescal.py:327-372 — A from the non-negative parts of the leading
    singular triplets of [X_1 .. X_m | X_1^T .. X_m^T] (LAPACK SVD for dense
    slices, ARPACK svds for sparse ones with k < n, :341-352), zeros filled
    with 1e-2 x the mean positive entry (:366-368, :375-383), then
    `r_update_iters` Jacobi R sweeps from all-ones with tol None (:370)."""
    import scipy.sparse.linalg as spla

    n = xs[0].shape[0]
    sparse_input = sp.issparse(xs[0])
    if sparse_input:
        mm = sp.hstack([*(o.tocsr() for o in xs), *(o.T.tocsr() for o in xs)], format="csr")
    else:
        mm = np.concatenate([*xs, *(o.T for o in xs)], axis=1)
    if sparse_input and k < n:
        u, s, vt = spla.svds(mm.astype(np.float64), k=k)
        order = np.argsort(s)[::-1]
        u, s, vt = u[:, order], s[order], vt[order]
    else:
        dense = mm.toarray() if sparse_input else np.asarray(mm, dtype=np.float64)
        u, s, vt = np.linalg.svd(dense, full_matrices=False)
        u, s, vt = u[:, :k], s[:k], vt[:k]
    a = np.zeros((n, k))
    lead = u[:, 0] if u[:, 0].sum() >= 0 else -u[:, 0]
    a[:, 0] = np.sqrt(s[0]) * np.maximum(lead, 0.0)
    for j in range(1, k):
        xu, yv = u[:, j], vt[j]
        xp, xm = np.maximum(xu, 0.0), np.maximum(-xu, 0.0)
        yp, ym = np.maximum(yv, 0.0), np.maximum(-yv, 0.0)
        mu_p = np.linalg.norm(xp) * np.linalg.norm(yp)
        mu_m = np.linalg.norm(xm) * np.linalg.norm(ym)
        if max(mu_p, mu_m) <= 0 or s[j] <= 0:
            continue
        part, norm = (xp, np.linalg.norm(xp)) if mu_p >= mu_m else (xm, np.linalg.norm(xm))
        a[:, j] = np.sqrt(s[j] * max(mu_p, mu_m)) * part / norm
    total, count = 0.0, 0
    for o in xs:
        vals = np.asarray(o.data) if sp.issparse(o) else np.asarray(o).ravel()
        vals = vals[vals > 0]
        total += float(vals.sum())
        count += vals.size
    positives = total / count if count else 0.0
    a[a == 0] = 1e-2 * positives if positives > 0 else 1e-2
    dt = xs[0].dtype
    a = a.astype(dt)
    r = regress_r(xs, a, eps=eps, max_iters=r_update_iters, tol=None)
    return a, r


# --------------------------------------------------------------------------
# perturbation (RESCALk resampling)


def perturbation_field(n, m, delta, base_seed, q, dtype=np.float64):
    """dist_rescal.py:164-171 — 1 + delta*(2u - 1), u from
    PCG64(SeedSequence((base_seed, 3, q))) in C order over (m, n, n)."""
    g = np.random.default_rng(np.random.SeedSequence((base_seed, 3, q)))
    return (1.0 + delta * (2.0 * g.random((m, n, n)) - 1.0)).astype(dtype)


def perturb_dense(x, delta, base_seed, q):
    """dist_rescal.py:205-215 (dense branch): X * field in x.dtype."""
    m, n = x.shape[0], x.shape[1]
    return x * perturbation_field(n, m, delta, base_seed, q, dtype=x.dtype)


def perturb_sparse(slices, delta, base_seed, q):
    """dist_rescal.py:208-214 (sparse branch): stored values only, then the
    SparseRelTensor canonicalisation of the rebuilt CSR."""
    n, m = slices[0].shape[0], len(slices)
    field = perturbation_field(n, m, delta, base_seed, q, dtype=slices[0].dtype)
    out = []
    for t, s in enumerate(slices):
        c = s.tocoo()
        vals = c.data * field[t, c.row, c.col]
        out.append(canonical_csr(sp.csr_matrix((vals, (c.row, c.col)), shape=s.shape, dtype=s.dtype)))
    return out


# --------------------------------------------------------------------------
# CSR index construction


def canonical_csr(s):
    """tensor.py:96-104 — csr_matrix -> sum_duplicates -> sort_indices ->
    eliminate_zeros; negative stored values are rejected."""
    c = sp.csr_matrix(s)
    c.sum_duplicates()
    c.sort_indices()
    c.eliminate_zeros()
    if c.nnz and c.data.min() < 0:
        raise ValueError("negative value in tensor")
    return c
