"""Multi-GPU RESCAL on a p_r x p_c process grid (one process per GPU).

Generalises the reference's square-grid solver (dist_rescal.py:113-161,
solve_on_grid :237-252) to 1x2 / 2x2 / 2x4 grids with the piece scheme of
SURVEY.md §8(e): A is cut into p = p_r*p_c pieces of b = ceil(n/p) rows, rank
(i, j) owns piece i*p_c + j, holds X[:, I_i, J_j] with row set I_i = pieces
{i*p_c + j'} and column set J_j = pieces {i'*p_c + j}, and per iteration runs
  AllGather(row) / AllGather(col) of A pieces  ->  local K1 on its block
  AllReduce(world) of [G, S_1..S_m, residual]  ->  replicated core update
  ReduceScatter(row) of sum_t P R^T, ReduceScatter(col) of sum_t Q R -> own A piece
all inside librescal_b200.so (peer-memory stores fused into the kernels, or
NCCL on the engine stream). The cores stay byte-identical on every rank (the
reference invariant, test_dist_rescal.py:65-78).

Layout note. The reference cuts X into sqrt(p) x sqrt(p) contiguous blocks and
re-broadcasts A blocks from the diagonal ranks (dist_rescal.py:74-92). Here the
row set of a rank is contiguous but its column set is strided (one piece per
grid row), so every rank owns exactly one A piece and each axis needs one
all-gather / reduce-scatter instead of diagonal broadcasts. ``grid_block``
cuts a block in this layout; ``partition_block`` is the reference's own
square-grid cut (tensor.py:339-362), kept for callers that use it directly.

Input. ``solve_on_grid`` / ``dist_rescal_solve`` take a whole tensor (every
rank cuts its block from it), a ``TensorBlock`` already cut by ``grid_block``,
or a ``BlockSource``: a per-rank provider (callable, or a memory-mapped RSK1
file via ``BlockSource.from_file``) so that no rank materialises the tensor.

Call from every rank of an initialised ``torch.distributed`` group (any
backend; it carries the 128-byte NCCL id, the norm and the factor gather).
Launch with ``torchrun --nproc-per-node N`` (``--master-addr 127.0.0.1``).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import _lib
from .containers import RelTensor, SparseRelTensor, dense_slices, is_sparse, tensor_dtype
from .exceptions import DataError, GridError
from .solver import KernelCounters, RescalFactors, SolverConfig, random_init


def grid_shape(p: int):
    """Most-square p_r x p_c with p_r <= p_c (1x2, 2x2, 2x4, ...)."""
    pr = int(math.isqrt(p))
    while p % pr:
        pr -= 1
    return pr, p // pr


def piece_layout(n: int, pr: int, pc: int, gi: int, gj: int) -> dict:
    """Host restatement of rk_grid_init's block geometry: rank (gi, gj) holds
    rows row0 + [0, rows) and the global columns colmap (indices >= n are
    zero padding)."""
    p = pr * pc
    b = -(-n // p)
    colmap = np.array([(ip * pc + gj) * b + r for ip in range(pr) for r in range(b)], dtype=np.int64)
    return {"gi": gi, "gj": gj, "piece": b, "rows": pc * b, "cols": pr * b,
            "row0": gi * pc * b, "pr": pr, "pc": pc, "colmap": colmap}


def block_of(x_dense: np.ndarray, n: int, info: dict) -> np.ndarray:
    """This rank's (m, rows, cols) block of a dense (m, n, n) array (a numpy
    array or a read-only memmap: only the block's rows are read), zero padded."""
    m = x_dense.shape[0]
    rows = np.arange(info["row0"], info["row0"] + info["rows"])
    cols = np.asarray(info["colmap"])
    out = np.zeros((m, len(rows), len(cols)), dtype=x_dense.dtype)
    ri = np.nonzero(rows < n)[0]
    ci = np.nonzero(cols < n)[0]
    if len(ri) and len(ci):
        r0, r1 = int(rows[ri[0]]), int(rows[ri[-1]]) + 1
        for t in range(m):  # one contiguous row range per slice, then the column gather
            out[t, ri[:, None], ci[None, :]] = np.asarray(x_dense[t, r0:r1])[:, cols[ci]]
    return out


def csr_block_of(slices, n: int, info: dict):
    """This rank's CSR block of canonical CSR slices: rows row0 + [0, rows),
    columns colmap (local column ids), canonical (sorted, no duplicates)."""
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


# ---------------------------------------------------------------------------
# blocks and block sources


@dataclass
class TensorBlock:
    """One rank's sub-tensor (tensor.py:142-170 fields). ``row_start`` is the
    first global row; ``colmap`` the global column of every local column
    (None: contiguous from ``col_start``, the reference's square-grid cut).
    ``block_dim`` is the row count (the reference's blocks are square)."""

    i: int
    j: int
    block_dim: int
    n_global: int
    m: int
    slices: object = field(repr=False)  # (m, rows, cols) ndarray or list of csr
    row_start: int = 0
    col_start: int = 0
    colmap: np.ndarray | None = field(default=None, repr=False)

    @property
    def is_sparse(self) -> bool:
        return not isinstance(self.slices, np.ndarray)

    @property
    def dtype(self):
        return self.slices.dtype if not self.is_sparse else self.slices[0].dtype

    def slice_ops(self):
        if self.is_sparse:
            return list(self.slices)
        return [self.slices[t] for t in range(self.m)]

    def global_cols(self) -> np.ndarray:
        ncols = self.slices.shape[2] if not self.is_sparse else self.slices[0].shape[1]
        if self.colmap is not None:
            return np.asarray(self.colmap)
        return self.col_start + np.arange(ncols, dtype=np.int64)


def block_dim(n: int, grid_dim: int) -> int:
    """Common padded block edge: ceil(n / grid_dim) (tensor.py:334-336)."""
    return -(-n // grid_dim)


def partition_block(t, grid_dim: int, i: int, j: int) -> TensorBlock:
    """The reference's zero-padded (i, j) block of a grid_dim x grid_dim
    partition (tensor.py:339-362): contiguous rows and columns."""
    if grid_dim < 1:
        raise DataError(f"grid_dim must be >= 1, got {grid_dim}")
    if not (0 <= i < grid_dim and 0 <= j < grid_dim):
        raise DataError(f"block ({i},{j}) outside {grid_dim}x{grid_dim} grid")
    b = block_dim(t.n, grid_dim)
    r0, c0 = i * b, j * b
    r1, c1 = min(r0 + b, t.n), min(c0 + b, t.n)
    if is_sparse(t):
        slices = []
        for s in t.slices:
            blk = sp.csr_matrix(s[r0:r1, c0:c1]) if r1 > r0 and c1 > c0 else sp.csr_matrix((0, 0), dtype=t.dtype)
            blk.resize((b, b))
            blk.sort_indices()
            slices.append(blk)
    else:
        slices = np.zeros((t.m, b, b), dtype=t.dtype)
        if r1 > r0 and c1 > c0:
            slices[:, : r1 - r0, : c1 - c0] = t.slices[:, r0:r1, c0:c1]
    return TensorBlock(i=i, j=j, block_dim=b, n_global=t.n, m=t.m, slices=slices, row_start=r0, col_start=c0)


def grid_block(t, pr: int, pc: int, i: int, j: int) -> TensorBlock:
    """Rank (i, j)'s block of the p_r x p_c piece layout (the engine's)."""
    if not (0 <= i < pr and 0 <= j < pc):
        raise DataError(f"block ({i},{j}) outside {pr}x{pc} grid")
    lay = piece_layout(t.n, pr, pc, i, j)
    if is_sparse(t):
        slices = csr_block_of(list(t.slices), t.n, lay)
    else:
        slices = block_of(np.asarray(t.slices), t.n, lay)
    return TensorBlock(i=i, j=j, block_dim=lay["rows"], n_global=t.n, m=t.m, slices=slices,
                       row_start=lay["row0"], colmap=lay["colmap"])


class BlockSource:
    """Per-rank block provider for the grid solve: ``block(info)`` returns this
    rank's block for the geometry ``info`` (piece_layout keys): a dense
    (m, rows, cols) array or a list of m CSR matrices (rows x cols, local
    column ids). No rank needs the whole tensor. ``sq_norm``: ||X||^2 of the
    whole tensor if known; otherwise the ranks sum their blocks' squares (the
    blocks partition X; padding is zero)."""

    def __init__(self, n: int, m: int, block, dtype=np.float64, sq_norm: float | None = None,
                 sparse: bool = False):
        self.n, self.m = int(n), int(m)
        self._block = block
        self.dtype = np.dtype(dtype)
        self.sq_norm = sq_norm
        self.sparse = bool(sparse)

    def block(self, info: dict):
        return self._block(info)

    @classmethod
    def from_tensor(cls, x) -> "BlockSource":
        if is_sparse(x):
            return cls(x.n, x.m, lambda info: csr_block_of(list(x.slices), x.n, info), dtype=tensor_dtype(x),
                       sparse=True)
        xd = dense_slices(x)
        return cls(x.n, x.m, lambda info: block_of(xd, x.n, info), dtype=tensor_dtype(x))

    @classmethod
    def from_file(cls, path) -> "BlockSource":
        """A dense RSK1 file (tensor_io format), memory-mapped: each rank reads
        only its block's rows."""
        from .tensor_io import DenseFile

        f = DenseFile(path)
        return cls(f.n, f.m, lambda info: block_of(f.array, f.n, info), dtype=f.dtype)


# ---------------------------------------------------------------------------
# the collective solve


@dataclass
class GridContext:
    """One rank's identity on the p_r x p_c grid (the reference's GridContext
    fields, grid.py:305-332; here backed by torch.distributed + NCCL)."""

    p: int
    pr: int
    pc: int
    i: int
    j: int
    counters: KernelCounters | None = None
    exchange: str = ""
    timing: dict = field(default_factory=dict)
    layout: dict = field(default_factory=dict, repr=False)

    @property
    def rank(self) -> int:
        return self.i * self.pc + self.j

    @property
    def grid_dim(self):
        return self.pr if self.pr == self.pc else (self.pr, self.pc)

    @property
    def is_diagonal(self) -> bool:
        return self.i == self.j

    def __getitem__(self, key):  # dict-style access to the block geometry / run info
        if key == "exchange":
            return self.exchange
        if key == "timing":
            return self.timing
        return self.layout[key]

    def get(self, key, default=None):
        try:
            return self[key]
        except KeyError:
            return default


@dataclass
class DistFactors:
    """Per-rank factor state (dist_rescal.py:58-72): this rank's row set of A,
    its column set, the replicated core stack."""

    a_row: np.ndarray
    a_col: np.ndarray
    r: np.ndarray
    i: int
    j: int
    n_global: int

    @property
    def k(self) -> int:
        return self.a_row.shape[1]


def _dist():
    import torch.distributed as dist

    if not dist.is_initialized():
        raise GridError("the grid solve needs an initialised torch.distributed process group")
    return dist


def _broadcast_id(dist, rank):
    obj = [_lib.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def _sum_over_ranks(dist, value: float) -> float:
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, float(value))
    return float(sum(out[r] for r in range(len(out))))  # rank order: identical on every rank


# One idle grid engine per process, kept for the next solve of the same
# shape on the same grid: it owns the NCCL communicators and the mapped peer
# arenas, whose setup (ncclCommInitRank + splits, CUDA IPC) costs seconds per
# call. Kept while its tensor is <= 1/4 of the GPU's memory; dropped by
# release_cached_memory().
_GRID_CACHE = {}


def _grid_key(n, m, k, pr, pc, cfg, sparse, rank):
    return (n, m, k, pr, pc, cfg.device, cfg.engine, bool(sparse), rank)


def release_grid_cache() -> None:
    for eng, _ in list(_GRID_CACHE.values()):
        eng.close()
    _GRID_CACHE.clear()


def _keep_grid_engine(key, eng, lay) -> bool:
    try:
        import torch

        total = torch.cuda.get_device_properties(eng_device(eng)).total_memory
    except Exception:  # noqa: BLE001
        total = 180e9
    dense = 4.0 * eng.m * lay["rows"] * lay["cols"]
    if eng.sparse or dense > total / 4:
        return False
    release_grid_cache()
    _GRID_CACHE[key] = (eng, lay)
    return True


def eng_device(eng) -> int:
    return int(getattr(eng, "device", 0) or 0)


def make_grid_engine(n, m, k, grid=None, cfg: SolverConfig | None = None, sparse=False):
    """Create this rank's engine (dense, or the CSR/CSC engine) and join the
    NCCL grid."""
    dist = _dist()
    cfg = cfg or SolverConfig()
    rank, size = dist.get_rank(), dist.get_world_size()
    pr, pc = grid if grid is not None else grid_shape(size)
    if pr * pc != size:
        raise GridError(f"{pr}x{pc} grid needs {pr * pc} ranks, have {size}")
    eng = _lib.Engine(n, m, k, device=cfg.device, engine=cfg.engine, sparse=sparse)
    try:
        eng.grid_init(pr, pc, rank, _broadcast_id(dist, rank))
    except Exception:
        eng.close()
        raise
    return eng, eng.grid_block()


def _as_source(x) -> BlockSource:
    if isinstance(x, BlockSource):
        return x
    if isinstance(x, TensorBlock):
        blk = x

        def give(info):
            if blk.row_start != info["row0"] or not np.array_equal(blk.global_cols(), info["colmap"]):
                raise GridError(f"block ({blk.i},{blk.j}) is not this rank's grid block: cut it with grid_block()")
            return blk.slices

        return BlockSource(blk.n_global, blk.m, give, dtype=blk.dtype, sparse=blk.is_sparse)
    return BlockSource.from_tensor(x)


def dist_rescal_solve(xblock, k: int, cfg: SolverConfig | None = None, ctx: GridContext | None = None,
                      initial: RescalFactors | None = None, grid=None):
    """Collective RESCAL solve (dist_rescal.py:113-161): every rank returns its
    DistFactors and the trace. ``xblock``: this rank's TensorBlock (grid_block
    layout), a BlockSource, or the whole tensor. Initialisation reproduces the
    serial solver's seeded start (random_init(n, k, m, cfg.seed))."""
    dist = _dist()
    cfg = cfg or SolverConfig()
    src = _as_source(xblock)
    n, m = src.n, src.m
    if not 1 <= k <= n:
        raise DataError(f"need 1 <= k <= n, got k={k}, n={n}")
    if cfg.init == "nndsvd" and initial is None:
        raise DataError("distributed solve needs explicit initial factors for nndsvd init")
    dt = src.dtype
    f0 = initial.copy() if initial is not None else random_init(n, k, m, cfg.seed, dtype=dt, device=cfg.device)
    if f0.A.shape != (n, k) or f0.R.shape != (m, k, k):
        raise DataError("initial factors do not match tensor/k")
    sparse = src.sparse and k <= 32
    t0 = time.perf_counter()
    size = dist.get_world_size()
    pr, pc = grid if grid is not None else grid_shape(size)
    key = _grid_key(n, m, k, pr, pc, cfg, sparse, dist.get_rank())
    cached = _GRID_CACHE.pop(key, None)
    # every rank must agree on reusing (the engine's communicators are collective)
    flags = [None] * size
    dist.all_gather_object(flags, cached is not None)
    if cached is not None and all(flags):
        eng, lay = cached
    else:
        if cached is not None:
            cached[0].close()
        eng, lay = make_grid_engine(n, m, k, (pr, pc), cfg, sparse=sparse)
    phases = {"create_s": time.perf_counter() - t0, "engine_reused": cached is not None and all(flags)}
    counters = ctx.counters if ctx is not None else None
    try:
        t0 = time.perf_counter()
        blk = src.block(lay)
        phases["block_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        if src.sparse and not sparse:  # k > 32: the dense engine on the densified block
            blk = np.stack([np.asarray(s.toarray()) for s in blk])
        if sparse:  # the CSR upload sums ||X||^2 on the device (all-reduced over the grid)
            eng.upload_csr(blk)
        else:
            # no norm given: the ranks sum their blocks' squares on the device
            eng.upload_block(blk, float(src.sq_norm) if src.sq_norm is not None else -1.0)
        del blk
        phases["upload_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        eng.set_factors(f0.A.astype(dt).astype(np.float64), f0.R.astype(dt).astype(np.float64))
        _, trace = eng.run(cfg.max_iters, float(dt.type(cfg.epsilon)), cfg.track_error, cfg.tolerance)
        phases["run_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        a, r = eng.get_factors()
        phases["get_factors_s"] = time.perf_counter() - t0
        timing = dict(eng.timing(), **phases)
        exchange = "peer" if eng.info().get("peer_exchange") else "nccl"
    except BaseException:
        eng.close()
        raise
    if not _keep_grid_engine(key, eng, lay):
        eng.close()
    if counters is not None:
        counters.add_time("device_run", timing["run_ms"] / 1e3)
    a = a.astype(dt)
    rows = np.arange(lay["row0"], lay["row0"] + lay["rows"])
    a_pad = np.zeros((max(n, int(rows[-1]) + 1, int(lay["colmap"].max()) + 1), k), dtype=dt)
    a_pad[:n] = a
    df = DistFactors(a_row=a_pad[rows].copy(), a_col=a_pad[lay["colmap"]].copy(), r=r.astype(dt),
                     i=lay["gi"], j=lay["gj"], n_global=n)
    if ctx is not None:
        ctx.exchange, ctx.timing = exchange, timing
        ctx.layout = {k_: (v.tolist() if isinstance(v, np.ndarray) else v) for k_, v in lay.items()}
    df._layout = lay  # noqa: SLF001 (used by gather_factors)
    df._timing, df._exchange = timing, exchange  # noqa: SLF001
    return df, np.asarray(trace)


def gather_factors(df: DistFactors, ctx: GridContext | None = None) -> RescalFactors:
    """Assemble the global factors; collective (dist_rescal.py:218-234). Row
    sets of the ranks of grid column 0 are stacked in grid-row order with the
    padding trimmed; R is taken from rank 0 after a byte-level replication
    check."""
    dist = _dist()
    payload = (df.i, df.j, df.a_row, df.r.tobytes())
    gathered = [None] * dist.get_world_size()
    dist.all_gather_object(gathered, payload)
    r_ref = gathered[0][3]
    for rank, (_, _, _, r_bytes) in enumerate(gathered):
        if r_bytes != r_ref:
            raise GridError(f"core stack differs on rank {rank}: broken run")
    rows = {i: a for i, j, a, _ in gathered if j == 0}
    a = np.vstack([rows[i] for i in sorted(rows)])[: df.n_global]
    r = np.frombuffer(r_ref, dtype=df.r.dtype).reshape(df.r.shape).copy()
    return RescalFactors(a.copy(), r)


def dist_perturb(xblock: TensorBlock, pcfg, q, ctx: GridContext | None = None, device: int = 0) -> TensorBlock:
    """Elementwise resampling of one rank's block, no communication
    (dist_rescal.py:174-203): element (t, row, col) is multiplied by the
    perturbation field of the WHOLE tensor at its global index, so any grid
    produces the same logical tensor. Sparse blocks keep their pattern
    (stored values only). Runs on the device (PCG64 jump-ahead, bit-exact)."""
    from .selection import _perturb_entropy

    n, m = xblock.n_global, xblock.m
    entropy = _perturb_entropy(pcfg, q)
    r0 = xblock.row_start
    gcols = xblock.global_cols()
    if xblock.is_sparse:
        out = []
        for t, s in enumerate(xblock.slices):
            c = sp.csr_matrix(s)
            rows_local = np.repeat(np.arange(c.shape[0]), np.diff(c.indptr))
            grow = r0 + rows_local
            gcol = gcols[c.indices]
            keep = (grow < n) & (gcol < n)
            if not np.all(keep):
                raise DataError("stored entry in the block's padding")
            # a global-row CSR view of the block's entries (same order) for the device kernel
            counts = np.bincount(grow, minlength=n)
            indptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
            vals = np.ascontiguousarray(c.data.copy())
            _lib.perturb_csr_values(entropy, pcfg.delta, t, n, indptr, gcol.astype(np.int32), vals, device=device)
            blk = sp.csr_matrix((vals, c.indices.copy(), c.indptr.copy()), shape=c.shape)
            out.append(blk)
        slices = out
    else:
        x = np.asarray(xblock.slices)
        slices = x.copy()
        rows = r0 + np.arange(x.shape[1])
        rv = np.nonzero(rows < n)[0]
        cv = np.nonzero(gcols < n)[0]
        if len(rv) and len(cv):
            for t in range(m):
                # the field of the block's full global rows (contiguous), then the column gather
                g0 = int(rows[rv[0]])
                fld = np.empty((len(rv), n), dtype=x.dtype)
                _lib.perturb_values(entropy, pcfg.delta, fld.reshape(-1), e0=(t * n + g0) * n, field_only=True,
                                    device=device)
                slices[t, rv[:, None], cv[None, :]] *= fld[:, gcols[cv]]
    return TensorBlock(i=xblock.i, j=xblock.j, block_dim=xblock.block_dim, n_global=n, m=m, slices=slices,
                       row_start=xblock.row_start, col_start=xblock.col_start, colmap=xblock.colmap)


def solve_on_grid(x, k: int, cfg: SolverConfig | None = None, p: int | None = None,
                  initial: RescalFactors | None = None, timeout: float = 30.0,
                  with_counters: bool = False, grid=None):
    """Collective solve; returns (factors, trace, ctx) with identical factors
    on every rank (dist_rescal.py:237-252 contract; ``grid=(p_r, p_c)``
    extension). ``x``: a RelTensor / SparseRelTensor (each rank cuts its own
    block), a TensorBlock from grid_block, or a BlockSource."""
    dist = _dist()
    cfg = cfg or SolverConfig()
    size = dist.get_world_size()
    if p is not None and p != size:
        raise GridError(f"p={p} but the process group has {size} ranks")
    pr, pc = grid if grid is not None else grid_shape(size)
    rank = dist.get_rank()
    ctx = GridContext(p=size, pr=pr, pc=pc, i=rank // pc, j=rank % pc,
                      counters=KernelCounters() if with_counters else None)
    df, trace = dist_rescal_solve(x, k, cfg, ctx, initial=initial, grid=(pr, pc))
    t0 = time.perf_counter()
    factors = gather_factors(df, ctx)
    ctx.timing["gather_s"] = time.perf_counter() - t0
    return factors, trace, ctx
