"""RESCALk model selection (drop-in for rescalkit.model_select.rescalk).

The expensive part — r perturbed MU solves per k (model_select.py:445-471) —
runs on the device: the tensor is uploaded once, every member resamples it in
place with the bit-exact PCG64 field kernel (dist_rescal.py:164-171) and
solves with the device engine; the per-k refit (regress_r) and its residual
also run on the device against the restored original tensor. The k x k / r x r
host math (assignment, column alignment, silhouettes; SURVEY.md §2.1 marks it
out of the device scope) is numpy/scipy here.

Ensemble spreading across GPUs (``north_star``): pass ``world=(rank, size)``
(one process per GPU, e.g. under torchrun) and an ``allgather`` callable; each
rank solves the members with (index % size == rank) — or takes them
dynamically through ``claim`` — the factors are gathered once for the whole
sweep, and the per-k clustering / refit runs on rank (k - k_min) % size with
the entries gathered after. The tensor is uploaded by rank 0 only; the other
replicas copy its device planes peer-to-peer over NVLink (CUDA IPC,
rk_tensor_export / rk_tensor_import). The iterations themselves exchange
nothing ("replicas only").
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
from scipy.optimize import linear_sum_assignment

from . import _lib
from .containers import dense_slices, is_sparse, tensor_dtype
from .exceptions import DataError, RescalkitError
from .solver import RescalFactors, SolverConfig, drop_cached_engine, finalize_normalize, random_init, rescal_solve

_SEED_TAG_PERTURB = 3
_SEED_TAG_ENSEMBLE = 4
_DENSIFY_MAX = 1 << 28  # elements: a sparse tensor this small may run on the dense engine (k > 32)


@dataclass
class PerturbConfig:
    """Resampling noise U[1-delta, 1+delta] (dist_rescal.py:42-55)."""

    delta: float = 0.02
    base_seed: int = 0

    def __post_init__(self):
        if not self.delta > 0:
            raise DataError(f"delta must be > 0, got {self.delta}")


def _perturb_entropy(pcfg: PerturbConfig, q):
    """SeedSequence entropy of perturbation q (dist_rescal.py:167-168)."""
    return (pcfg.base_seed, _SEED_TAG_PERTURB, q)


def perturbation_field(n: int, m: int, pcfg: PerturbConfig, q, dtype=np.float64, device: int = 0) -> np.ndarray:
    """The full (m, n, n) multiplier field for perturbation q
    (dist_rescal.py:164-171), drawn on the device, bit-exact with numpy."""
    out = np.empty((m, n, n), dtype=np.dtype(dtype))
    if out.dtype not in (np.float32, np.float64):
        raise DataError(f"unsupported field dtype {out.dtype}")
    _lib.perturb_values(_perturb_entropy(pcfg, q), pcfg.delta, out, 0, True, device)
    return out


def perturb(x, pcfg: PerturbConfig, q, device: int = 0):
    """Whole-tensor resampling with the reference's multiplier field
    (dist_rescal.py:205-215): dense x * field.astype(x.dtype); sparse tensors
    keep their pattern and only the stored values are resampled. Computed on
    the device (no (m, n, n) fp64 field on the host)."""
    from .containers import RelTensor, SparseRelTensor, is_sparse
    import scipy.sparse as sps

    key = _perturb_entropy(pcfg, q)
    if is_sparse(x):
        slices = []
        for t, s in enumerate(x.slices):
            data = np.array(s.data, dtype=s.dtype if s.dtype in (np.float32, np.float64) else np.float64)
            _lib.perturb_csr_values(key, pcfg.delta, t, x.n, s.indptr, s.indices, data, device)
            slices.append(sps.csr_matrix((data, s.indices.copy(), s.indptr.copy()), shape=s.shape))
        return SparseRelTensor(slices, n=x.n)
    xs = np.array(x.slices, order="C", copy=True)
    if xs.dtype not in (np.float32, np.float64):
        xs = xs.astype(np.float64)
    _lib.perturb_values(key, pcfg.delta, xs, 0, False, device)
    return RelTensor(xs)


# ---------------------------------------------------------------------------
# host-side k x k math


def lsa(cost: np.ndarray, mode: str = "minimize") -> np.ndarray:
    """Optimal assignment perm[row] = col (model_select.py:52-112 contract)."""
    c = np.asarray(cost, dtype=np.float64)
    if c.ndim != 2 or c.shape[0] != c.shape[1]:
        raise DataError(f"cost matrix must be square, got {c.shape}")
    if not np.all(np.isfinite(c)):
        raise DataError("cost matrix has non-finite entries")
    if mode not in ("minimize", "maximize"):
        raise DataError(f"unknown mode {mode!r}")
    rows, cols = linear_sum_assignment(c, maximize=(mode == "maximize"))
    perm = np.empty(c.shape[0], dtype=int)
    perm[rows] = cols
    return perm


@dataclass
class FactorEnsemble:
    A_stack: np.ndarray
    R_stack: np.ndarray | None = None

    def __post_init__(self):
        self.A_stack = np.asarray(self.A_stack)
        if self.A_stack.ndim != 3:
            raise DataError(f"A_stack must be (n, k, r), got {self.A_stack.shape}")
        if self.A_stack.size and self.A_stack.min() < 0:
            raise DataError("ensemble factors must be non-negative")

    @property
    def k(self) -> int:
        return self.A_stack.shape[1]

    @property
    def r(self) -> int:
        return self.A_stack.shape[2]


@dataclass
class ClusterResult:
    ensemble: FactorEnsemble
    medians: np.ndarray
    permutations: np.ndarray
    iterations: int
    converged: bool


def _unit_columns(stack):
    norms = np.sqrt(np.sum(stack.astype(np.float64) ** 2, axis=0))
    return stack / np.where(norms > 0, norms, 1.0)[None, :, :]


def custom_cluster(ens: FactorEnsemble, ctx=None, max_iters: int = 100) -> ClusterResult:
    """Permutation-constrained k-medians of the ensemble columns
    (model_select.py:194-241): cosine similarity to the medoid, Hungarian
    assignment per solution, elementwise-median medoid, until a sweep applies
    only identity permutations."""
    if ens.r < 2:
        raise DataError(f"need r >= 2 solutions, got {ens.r}")
    k, r = ens.k, ens.r
    hat = _unit_columns(ens.A_stack)
    aligned = ens.A_stack.copy()
    aligned_hat = hat.copy()
    total = np.tile(np.arange(k), (r, 1))
    medoid = aligned[:, :, 0].copy()
    ident = np.arange(k)
    converged, sweeps = False, 0
    for _ in range(max_iters):
        sweeps += 1
        sim = (medoid.T @ aligned_hat.reshape(aligned_hat.shape[0], k * r)).reshape(k, k, r)
        perms = [lsa(sim[:, :, q], mode="maximize") for q in range(r)]
        if all(np.array_equal(p, ident) for p in perms):
            converged = True
            break
        for q, p in enumerate(perms):
            aligned[:, :, q] = aligned[:, p, q]
            aligned_hat[:, :, q] = aligned_hat[:, p, q]
            total[q] = total[q][p]
        medoid = np.median(aligned, axis=2)
    r_stack = None
    if ens.R_stack is not None:
        r_stack = ens.R_stack.copy()
        for q in range(r):
            p = total[q]
            r_stack[:, :, :, q] = r_stack[p][:, p][:, :, :, q]
    return ClusterResult(FactorEnsemble(aligned, r_stack), np.median(aligned, axis=2), total, sweeps,
                         converged)


@dataclass
class SilhouetteStats:
    I: np.ndarray
    J: np.ndarray
    s_points: np.ndarray
    s_min: float
    s_avg: float
    single_cluster: bool = False


def cluster_stability(ens: FactorEnsemble, ctx=None) -> SilhouetteStats:
    """Cosine-distance silhouettes of the aligned clusters (model_select.py:244-294)."""
    if ens.r < 2:
        raise DataError(f"need r >= 2 solutions, got {ens.r}")
    k, r = ens.k, ens.r
    hat = _unit_columns(ens.A_stack)
    inner = np.stack([hat[:, c, :].T @ hat[:, c, :] for c in range(k)], axis=2)  # (r, r, k)
    i_mat = (1.0 - inner).mean(axis=1)
    if k == 1:
        return SilhouetteStats(i_mat, np.ones((r, 1)), np.ones((r, 1)), 1.0, 1.0, True)
    j_mat = np.empty((r, k))
    for c in range(k):
        cross = (hat[:, c, :].T @ hat.reshape(hat.shape[0], k * r)).reshape(r, k, r).transpose(0, 2, 1)
        y = (1.0 - cross).mean(axis=1)
        y[:, c] = np.inf
        j_mat[:, c] = y.min(axis=1)
    peak = np.maximum(j_mat, i_mat)
    with np.errstate(invalid="ignore", divide="ignore"):
        s = np.where(peak > 0, (j_mat - i_mat) / peak, 0.0)
    return SilhouetteStats(i_mat, j_mat, s, float(s.min()), float(s.mean()))


@dataclass
class SelectionEntry:
    k: int
    s_min: float
    s_avg: float
    rel_error: float
    medians: np.ndarray = field(repr=False)
    core: np.ndarray = field(repr=False)
    converged: bool = True


@dataclass
class SelectionReport:
    entries: list
    k_opt: int
    low_confidence: bool
    tau_s: float
    params: dict = field(default_factory=dict)
    timing: dict = field(default_factory=dict)

    def entry(self, k: int) -> SelectionEntry:
        for e in self.entries:
            if e.k == k:
                return e
        raise KeyError(k)

    def to_json_dict(self) -> dict:
        return {
            "k_opt": self.k_opt, "low_confidence": self.low_confidence, "tau_s": self.tau_s,
            "per_k": {str(e.k): {"s_min": e.s_min, "s_avg": e.s_avg, "rel_error": e.rel_error}
                      for e in self.entries},
            "parameters": self.params, "timing": self.timing,
        }


def select_k(entries, tau_s: float = 0.75) -> int:
    """Largest k with s_min >= tau_s, else the best s_min (model_select.py:345-356)."""
    if not entries:
        raise DataError("no selection entries")
    ok = [e.k for e in entries if e.s_min >= tau_s]
    return max(ok) if ok else max(entries, key=lambda e: e.s_min).k


def pearson_correlation(a_est: np.ndarray, a_true: np.ndarray) -> np.ndarray:
    """Column-pair Pearson matrix (model_select.py:510-526)."""
    a_est = np.asarray(a_est, dtype=np.float64)
    a_true = np.asarray(a_true, dtype=np.float64)
    if a_est.shape != a_true.shape:
        raise DataError(f"shape mismatch: {a_est.shape} vs {a_true.shape}")
    e = a_est - a_est.mean(axis=0)
    t = a_true - a_true.mean(axis=0)
    denom = np.outer(np.sqrt((e ** 2).sum(0)), np.sqrt((t ** 2).sum(0)))
    with np.errstate(invalid="ignore", divide="ignore"):
        return np.where(denom > 0, (e.T @ t) / denom, 0.0)


def best_match_diagonal(corr: np.ndarray) -> np.ndarray:
    perm = lsa(corr, mode="maximize")
    return corr[np.arange(corr.shape[0]), perm]


# ---------------------------------------------------------------------------
# the driver


def _solve_member(eng, x, k, q, cfg, pcfg, dt):
    eng.perturb((pcfg.base_seed, _SEED_TAG_PERTURB, (k, q)), pcfg.delta)
    if cfg.init == "nndsvd":  # model_select.py:461-462, on the resampled device tensor
        from .solver import nndsvd_init
        init = nndsvd_init(x, k, eps=cfg.epsilon, cfg=cfg, engine=eng)
    else:
        init = random_init(x.n, k, x.m, (cfg.seed, _SEED_TAG_ENSEMBLE, k, q), dtype=dt)
    f, trace = rescal_solve(x, k, cfg, initial=init, engine=eng)
    f = finalize_normalize(f)
    solved = len(trace) == 0 or bool(np.isfinite(trace[-1]))
    return f.A, f.R, solved


def rescalk(x, k_min: int, k_max: int, r: int, cfg: SolverConfig | None = None,
            pcfg: PerturbConfig | None = None, ctx=None, tau_s: float = 0.75,
            world: tuple | None = None, allgather=None, claim=None) -> SelectionReport:
    """Factorize r resamplings per k, score stability, pick k_opt
    (model_select.py:422-503; serial semantics, device compute).

    ``ctx`` (the reference's in-process grid) is not used: grids here are
    process grids (multigpu.py). ``world``/``allgather`` spread the members
    over GPUs (see module docstring); ``claim`` (optional, with ``world``) is
    a callable shared by all ranks returning 1, 2, 3, ... in turn (e.g. a
    torch.distributed store counter): members are then taken dynamically, so
    a rank whose tensor upload was slow takes fewer. Results do not depend on
    which rank solved a member.
    """
    cfg = cfg or SolverConfig()
    pcfg = pcfg or PerturbConfig()
    if not (1 <= k_min <= k_max <= x.n):
        raise DataError(f"need 1 <= k_min <= k_max <= n, got [{k_min}, {k_max}], n={x.n}")
    if r < 2:
        raise DataError(f"need r >= 2 perturbations, got {r}")
    rank, size = world if world is not None else (0, 1)
    dt = tensor_dtype(x)
    t_start = time.perf_counter()
    # a sparse tensor stays sparse on the device (CSR + device-built CSC,
    # k <= 32): every member resamples the stored values only
    # (dist_rescal.py:205-214), as the reference does
    sparse = is_sparse(x)
    if sparse and k_max > 32:
        if x.m * x.n * x.n > _DENSIFY_MAX:
            raise DataError(f"sparse RESCALk runs on the CSR engine, which supports k <= 32 (k_max={k_max}); "
                            f"a dense copy of this tensor ({x.m}x{x.n}x{x.n}) is too large")
        sparse = False  # small tensor: the dense engine on the densified copy
    drop_cached_engine()  # at most one tensor's device storage per thread
    eng = _lib.Engine(x.n, x.m, k_min, device=cfg.device, engine=cfg.engine, sparse=sparse)
    entries, timing = [], {"per_k_seconds": {}}
    try:
        if sparse:
            eng.upload_csr(list(x.slices))
        elif size > 1 and allgather is not None:
            # the replicas share one tensor: rank 0 uploads it over PCIe, the
            # others copy its device planes peer-to-peer over NVLink (every
            # rank uploading the same tensor contends for the host links);
            # a rank without a peer path uploads its own copy
            if rank == 0:
                eng.upload(dense_slices(x))
            record = allgather(eng.tensor_export() if rank == 0 else None)[0]
            if rank != 0:
                try:
                    eng.tensor_import(record)
                except RescalkitError:
                    eng.upload(dense_slices(x))
            allgather(None)  # rank 0 keeps its planes unperturbed until every copy is done
        else:
            eng.upload(dense_slices(x))
        timing["upload_seconds"] = time.perf_counter() - t_start
        ks = list(range(k_min, k_max + 1))
        # 1) the members: (k, q) in the reference's order, member i on rank
        #    i % size — one gather for the whole sweep, so no rank idles at a
        #    per-k barrier (each member depends only on its (k, q) seeds)
        mine = {}
        order = [(k, q) for k in ks for q in range(1, r + 1)]
        if claim is not None and size > 1:
            while True:
                i = int(claim()) - 1
                if i >= len(order):
                    break
                k, q = order[i]
                mine[(k, q)] = _solve_member(eng, x, k, q, cfg, pcfg, dt)
        else:
            for i, (k, q) in enumerate(order):
                if i % size == rank:
                    mine[(k, q)] = _solve_member(eng, x, k, q, cfg, pcfg, dt)
        timing["members_seconds"] = time.perf_counter() - t_start - timing["upload_seconds"]
        if size > 1:
            t_g = time.perf_counter()
            merged = {}
            for part in allgather(mine):
                merged.update(part)
            mine = merged
            timing["gather_seconds"] = time.perf_counter() - t_g
        eng.restore()
        # 2) per k: clustering, stability, refit and residual on the original
        #    tensor — k on rank (k - k_min) % size, entries gathered after
        from .solver import regress_r, rel_error
        mine_entries = {}
        for i, k in enumerate(ks):
            if i % size != rank:
                continue
            t_k = time.perf_counter()
            a_cols = [mine[(k, q)][0] for q in range(1, r + 1)]
            r_slabs = [mine[(k, q)][1] for q in range(1, r + 1)]
            solved = all(mine[(k, q)][2] for q in range(1, r + 1))
            ens = FactorEnsemble(np.stack(a_cols, axis=2),
                                 np.stack([np.transpose(s, (1, 2, 0)) for s in r_slabs], axis=3))
            clus = custom_cluster(ens)
            stats = cluster_stability(clus.ensemble)
            core = regress_r(x, clus.medians, cfg, engine=eng)
            err = rel_error(x, RescalFactors(clus.medians, core), engine=eng)
            mine_entries[k] = SelectionEntry(k=k, s_min=stats.s_min, s_avg=stats.s_avg, rel_error=err,
                                             medians=clus.medians, core=core,
                                             converged=clus.converged and solved)
            timing["per_k_seconds"][str(k)] = time.perf_counter() - t_k
        if size > 1:
            merged, secs, members_s = {}, {}, []
            for part in allgather((mine_entries, timing["per_k_seconds"], timing["members_seconds"],
                                   timing["upload_seconds"])):
                merged.update(part[0])
                secs.update(part[1])
                members_s.append((round(part[3], 3), round(part[2], 3)))
            mine_entries, timing["per_k_seconds"] = merged, secs
            timing["upload_members_seconds_per_rank"] = members_s
        entries = [mine_entries[k] for k in ks]
    finally:
        eng.close()
    k_opt = select_k(entries, tau_s)
    timing["total_seconds"] = time.perf_counter() - t_start
    params = {"k_min": k_min, "k_max": k_max, "r": r, "delta": pcfg.delta, "seed": cfg.seed,
              "max_iters": cfg.max_iters, "init": cfg.init, "tolerance": cfg.tolerance,
              "grid_p": None, "gpus": size}
    return SelectionReport(entries=entries, k_opt=k_opt,
                           low_confidence=all(e.s_min < tau_s for e in entries), tau_s=tau_s,
                           params=params, timing=timing)
