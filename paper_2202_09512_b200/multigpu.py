"""Multi-GPU RESCAL on a p_r x p_c process grid (one process per GPU).

Generalises the reference's square-grid solver (dist_rescal.py:113-161,
solve_on_grid :237-252) to 1x2 / 2x2 / 2x4 grids with the piece scheme of
SURVEY.md §8(e): A is cut into p = p_r*p_c pieces of b = ceil(n/p) rows, rank
(i, j) owns piece i*p_c + j, holds X[:, I_i, J_j] with row set I_i = pieces
{i*p_c + j'} and column set J_j = pieces {i'*p_c + j}, and per iteration runs
  AllGather(row) / AllGather(col) of A pieces  ->  local K1 on its block
  AllReduce(world) of [G, S_1..S_m, residual]  ->  replicated core update
  ReduceScatter(row) of sum_t P R^T, ReduceScatter(col) of sum_t Q R -> own A piece
all inside librescal_b200.so with NCCL on the engine stream. The cores stay
byte-identical on every rank (the reference invariant, test_dist_rescal.py:65-78).

Call from every rank of an initialised ``torch.distributed`` group (any
backend; it only carries the 128-byte NCCL id). Launch with
``torchrun --nproc-per-node N`` (``--master-addr 127.0.0.1``).
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib
from .containers import dense_slices, is_sparse, tensor_dtype
from .exceptions import DataError, GridError
from .solver import RescalFactors, SolverConfig, random_init


def grid_shape(p: int):
    """Most-square p_r x p_c with p_r <= p_c (1x2, 2x2, 2x4, ...)."""
    pr = int(math.isqrt(p))
    while p % pr:
        pr -= 1
    return pr, p // pr


def block_of(x_dense: np.ndarray, n: int, info: dict) -> np.ndarray:
    """This rank's (m, rows, cols) block of the global tensor, zero padded:
    rows row0 + [0, rows), columns colmap[0, cols) (global indices >= n are
    padding)."""
    m = x_dense.shape[0]
    rows = np.arange(info["row0"], info["row0"] + info["rows"])
    cols = np.asarray(info["colmap"])
    out = np.zeros((m, len(rows), len(cols)), dtype=x_dense.dtype)
    ri = np.nonzero(rows < n)[0]
    ci = np.nonzero(cols < n)[0]
    out[:, ri[:, None], ci[None, :]] = x_dense[:, rows[ri][:, None], cols[ci][None, :]]
    return out


def csr_block_of(slices, n: int, info: dict):
    """This rank's CSR block of canonical CSR slices: rows row0 + [0, rows),
    columns colmap (local column ids), canonical (sorted, no duplicates)."""
    import scipy.sparse as sp

    rows = np.arange(info["row0"], info["row0"] + info["rows"])
    cols = np.asarray(info["colmap"])
    rv = rows[rows < n]
    cmask = cols < n
    local_of = np.nonzero(cmask)[0]
    out = []
    for s in slices:
        sub = sp.csr_matrix(s)[rv][:, cols[cmask]].tocoo()
        blk = sp.csr_matrix((sub.data, (sub.row, local_of[sub.col])), shape=(info["rows"], info["cols"]))
        blk.sum_duplicates()
        blk.sort_indices()
        out.append(blk)
    return out


def piece_layout(n: int, pr: int, pc: int, gi: int, gj: int) -> dict:
    """Host restatement of rk_grid_init's block geometry (for tests/tools)."""
    p = pr * pc
    b = -(-n // p)
    colmap = np.array([(ip * pc + gj) * b + r for ip in range(pr) for r in range(b)], dtype=np.int64)
    return {"gi": gi, "gj": gj, "piece": b, "rows": pc * b, "cols": pr * b,
            "row0": gi * pc * b, "pr": pr, "pc": pc, "colmap": colmap}


def _broadcast_id(dist, rank):
    import torch

    if rank == 0:
        raw = _lib.nccl_unique_id()
        t = torch.tensor(list(raw), dtype=torch.uint8)
    else:
        t = torch.zeros(128, dtype=torch.uint8)
    obj = [bytes(t.tolist())]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def make_grid_engine(n, m, k, grid=None, cfg: SolverConfig | None = None, sparse=False):
    """Create this rank's engine (dense, or the CSR/CSC engine) and join the
    NCCL grid."""
    import torch.distributed as dist

    if not dist.is_initialized():
        raise GridError("solve_on_grid needs an initialised torch.distributed process group")
    cfg = cfg or SolverConfig()
    rank, size = dist.get_rank(), dist.get_world_size()
    pr, pc = grid if grid is not None else grid_shape(size)
    if pr * pc != size:
        raise GridError(f"{pr}x{pc} grid needs {pr * pc} ranks, have {size}")
    eng = _lib.Engine(n, m, k, device=cfg.device, engine=cfg.engine, sparse=sparse)
    nid = _broadcast_id(dist, rank)
    eng.grid_init(pr, pc, rank, nid)
    return eng, eng.grid_block()


def solve_on_grid(x, k: int, cfg: SolverConfig | None = None, p: int | None = None,
                  initial: RescalFactors | None = None, timeout: float = 30.0,
                  with_counters: bool = False, grid=None):
    """Collective solve; returns (factors, trace, info) on every rank
    (dist_rescal.py:237-252 contract; ``grid=(p_r, p_c)`` extension)."""
    import torch.distributed as dist

    cfg = cfg or SolverConfig()
    size = dist.get_world_size() if dist.is_initialized() else 1
    if p is not None and p != size:
        raise GridError(f"p={p} but the process group has {size} ranks")
    if not 1 <= k <= x.n:
        raise DataError(f"need 1 <= k <= n, got k={k}, n={x.n}")
    dt = tensor_dtype(x)
    f0 = initial.copy() if initial is not None else random_init(x.n, k, x.m, cfg.seed, dtype=dt)
    if f0.A.shape != (x.n, k) or f0.R.shape != (x.m, k, k):
        raise DataError("initial factors do not match tensor/k")
    sparse = is_sparse(x) and k <= 32
    eng, info = make_grid_engine(x.n, x.m, k, grid, cfg, sparse=sparse)
    try:
        if sparse:
            eng.upload_csr(csr_block_of(list(x.slices), x.n, info))
        else:
            xd = dense_slices(x)
            sq = float(np.sum(np.asarray(xd, dtype=np.float64) ** 2))
            eng.upload_block(block_of(xd, x.n, info), sq)
        eng.set_factors(f0.A.astype(dt).astype(np.float64), f0.R.astype(dt).astype(np.float64))
        _, trace = eng.run(cfg.max_iters, float(dt.type(cfg.epsilon)), cfg.track_error, cfg.tolerance)
        a, r = eng.get_factors()
        timing = eng.timing()
        exchange = "peer" if eng.info().get("peer_exchange") else "nccl"
    finally:
        eng.close()
    info = {k_: (v.tolist() if isinstance(v, np.ndarray) else v) for k_, v in info.items()}
    info["timing"] = timing
    info["exchange"] = exchange
    return RescalFactors(a.astype(dt), r.astype(dt)), np.asarray(trace), info
