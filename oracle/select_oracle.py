"""RESCALk oracle (model_select.py:422-503), serial branch only (tests only).

The k x k / r x r host math (assignment, clustering, silhouettes) is restated
here so that selected-k parity of the device driver can be checked on inputs
the reference itself never saw. Paths relative to
``/root/reference/pkg/src/rescalkit``.
"""

from __future__ import annotations

import numpy as np

from .mu_oracle import (
    OracleConfig,
    finalize_normalize,
    perturb_dense,
    random_init,
    regress_r,
    rel_error,
    solve,
)


def hungarian_max(score):
    """model_select.py:52-112 — optimal assignment maximising ``score``.

    Shortest-augmenting-path with row/column potentials (O(k^3)); returns
    perm with perm[row] = column.
    """
    c = -np.asarray(score, dtype=np.float64)
    n = c.shape[0]
    u = np.zeros(n + 1)
    v = np.zeros(n + 1)
    owner = np.zeros(n + 1, dtype=int)   # owner[col] = row (1-based), col 0 virtual
    back = np.zeros(n + 1, dtype=int)
    for row in range(1, n + 1):
        owner[0] = row
        col0 = 0
        best = np.full(n + 1, np.inf)
        seen = np.zeros(n + 1, dtype=bool)
        while True:
            seen[col0] = True
            r0 = owner[col0]
            step, col1 = np.inf, -1
            for col in range(1, n + 1):
                if seen[col]:
                    continue
                red = c[r0 - 1, col - 1] - u[r0] - v[col]
                if red < best[col]:
                    best[col] = red
                    back[col] = col0
                if best[col] < step:
                    step, col1 = best[col], col
            for col in range(n + 1):
                if seen[col]:
                    u[owner[col]] += step
                    v[col] -= step
                else:
                    best[col] -= step
            col0 = col1
            if owner[col0] == 0:
                break
        while col0:
            prev = back[col0]
            owner[col0] = owner[prev]
            col0 = prev
    perm = np.empty(n, dtype=int)
    for col in range(1, n + 1):
        perm[owner[col] - 1] = col - 1
    return perm


def _unit_columns(stack):
    """model_select.py:186-191 (serial)."""
    norms = np.sqrt(np.sum(stack.astype(np.float64) ** 2, axis=0))
    return stack / np.where(norms > 0, norms, 1.0)[None, :, :]


def align_columns(a_stack, max_iters=100):
    """model_select.py:194-241 (serial): returns (aligned, medians, converged)."""
    k, r = a_stack.shape[1], a_stack.shape[2]
    hat = _unit_columns(a_stack)
    aligned = a_stack.copy()
    aligned_hat = hat.copy()
    medoid = aligned[:, :, 0].copy()
    ident = np.arange(k)
    converged = False
    for _ in range(max_iters):
        sim = np.einsum("nc,nlq->clq", medoid, aligned_hat)
        perms = [hungarian_max(sim[:, :, q]) for q in range(r)]
        if all(np.array_equal(p, ident) for p in perms):
            converged = True
            break
        for q, p in enumerate(perms):
            aligned[:, :, q] = aligned[:, p, q]
            aligned_hat[:, :, q] = aligned_hat[:, p, q]
        medoid = np.median(aligned, axis=2)
    return aligned, np.median(aligned, axis=2), converged


def silhouette(a_stack):
    """model_select.py:244-294 (serial): returns (s_min, s_avg)."""
    k, r = a_stack.shape[1], a_stack.shape[2]
    hat = _unit_columns(a_stack)
    within = np.empty((r, r, k))
    for c in range(k):
        u = hat[:, c, :]
        within[:, :, c] = u.T @ u
    i_mat = (1.0 - within).mean(axis=1)
    if k == 1:
        return 1.0, 1.0
    j_mat = np.empty((r, k))
    for c in range(k):
        cross = np.zeros((r, r, k))
        u = hat[:, c, :]
        for o in range(k):
            if o != c:
                cross[:, :, o] = u.T @ hat[:, o, :]
        y = (1.0 - cross).mean(axis=1)
        y[:, c] = np.inf
        j_mat[:, c] = y.min(axis=1)
    peak = np.maximum(j_mat, i_mat)
    with np.errstate(invalid="ignore", divide="ignore"):
        s = np.where(peak > 0, (j_mat - i_mat) / peak, 0.0)
    return float(s.min()), float(s.mean())


def rescalk_oracle(x, k_min, k_max, r, cfg: OracleConfig, delta=0.02, base_seed=0, tau_s=0.75):
    """model_select.py:422-503 (serial, dense, random init).

    Returns dict(k_opt, entries=[(k, s_min, s_avg, rel_error)], medians={k: ...}).
    """
    xs = [x[t] for t in range(x.shape[0])]
    n, m = x.shape[1], x.shape[0]
    entries, medians = [], {}
    for k in range(k_min, k_max + 1):
        cols = []
        for q in range(1, r + 1):
            xq = perturb_dense(x, delta, base_seed, (k, q))
            init = random_init(n, k, m, (cfg.seed, 4, k, q), dtype=x.dtype)
            a, rr, _ = solve([xq[t] for t in range(m)], k, cfg, initial=init, dtype=x.dtype)
            a, rr = finalize_normalize(a, rr)
            cols.append(a)
        stack = np.stack(cols, axis=2)
        aligned, med, _ = align_columns(stack)
        s_min, s_avg = silhouette(aligned)
        core = regress_r(xs, med, eps=cfg.epsilon)
        err = rel_error(xs, med, core)
        entries.append((k, s_min, s_avg, err))
        medians[k] = med
    qualified = [e[0] for e in entries if e[1] >= tau_s]
    k_opt = max(qualified) if qualified else max(entries, key=lambda e: e[1])[0]
    return {"k_opt": k_opt, "entries": entries, "medians": medians}
