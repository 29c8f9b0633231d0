"""Multi-GPU parity check (run under torchrun, one rank per GPU): the NCCL
p_r x p_c grid path vs the CPU oracle on identical inputs."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch.distributed as dist

import oracle
import paper_2202_09512_b200 as rk

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
# GRID_SHAPE=PRxPC forces a grid (e.g. 1x4 on 4 GPUs exercises 4-rank row
# communicators, the row-side shape of the 2x4 grid of an 8-GPU box)
_gs = os.environ.get("GRID_SHAPE")
GRID = tuple(int(v) for v in _gs.lower().split("x")) if _gs else None
results = []
ok = True
for (n, m, k, iters, engine) in [(300, 3, 5, 30, "auto"), (1000, 2, 16, 20, "auto"), (700, 2, 32, 12, "auto"),
                                 (257, 2, 4, 25, "simt"), (300, 2, 40, 8, "auto"),
                                 (600, 2, 64, 6, "auto")]:
    x = np.random.default_rng(n).random((m, n, n), dtype=np.float32).astype(np.float64)
    f0 = rk.random_init(n, k, m, 1)
    f, tr, info = rk.solve_on_grid(rk.RelTensor(x), k, rk.SolverConfig(max_iters=iters, engine=engine),
                                   initial=f0, grid=GRID)
    rb = [None] * world
    dist.all_gather_object(rb, f.R.tobytes())
    if rank == 0:
        ao, ro, tro = oracle.solve([x[t] for t in range(m)], k, oracle.OracleConfig(max_iters=iters),
                                   initial=(f0.A, f0.R))
        rel_a = float(np.linalg.norm(f.A - ao) / np.linalg.norm(ao))
        rel_r = float(np.linalg.norm(f.R - ro) / np.linalg.norm(ro))
        derr = float(np.max(np.abs(tr - tro)))
        same_r = len(set(rb)) == 1
        good = rel_a <= 1e-4 and rel_r <= 1e-4 and derr <= 1e-5 and same_r and len(tr) == iters
        ok = ok and good
        results.append(dict(n=n, m=m, k=k, iters=iters, engine=engine, grid=[info["pr"], info["pc"]],
                            exchange=info.get("exchange"),
                            relA=rel_a, relR=rel_r, dErr=derr, R_replicated=same_r, ok=good))
# the same solve again (the kept grid engine is reused: no NCCL / IPC setup),
# and from a memory-mapped RSK1 file through BlockSource.from_file: the
# factors must be byte-identical to the first solve of the list
import tempfile
n, m, k, iters = 1000, 2, 16, 20
x = np.random.default_rng(n).random((m, n, n), dtype=np.float32).astype(np.float64)
f0 = rk.random_init(n, k, m, 1)
ref, _, _ = rk.solve_on_grid(rk.RelTensor(x), k, rk.SolverConfig(max_iters=iters), initial=f0, grid=GRID)
again, _, ctx2 = rk.solve_on_grid(rk.RelTensor(x), k, rk.SolverConfig(max_iters=iters), initial=f0, grid=GRID)
path = os.path.join(tempfile.gettempdir(), f"grid_check_{os.getpid() if rank == 0 else 0}.rsk")
paths = [None] * world
dist.all_gather_object(paths, path)
if rank == 0:
    rk.save_tensor(rk.RelTensor(x), paths[0])
dist.barrier()
ff, _, _ = rk.solve_on_grid(rk.BlockSource.from_file(paths[0]), k, rk.SolverConfig(max_iters=iters), initial=f0,
                            grid=GRID)
dist.barrier()
if rank == 0:
    os.remove(paths[0])
    good = (np.array_equal(again.A, ref.A) and np.array_equal(again.R, ref.R) and np.array_equal(ff.A, ref.A)
            and np.array_equal(ff.R, ref.R) and bool(ctx2.timing.get("engine_reused")))
    ok = ok and good
    results.append(dict(n=n, m=m, k=k, iters=iters, engine="reuse+file", exchange=ctx2.exchange,
                        reused=bool(ctx2.timing.get("engine_reused")),
                        grid=[ctx2.pr, ctx2.pc], ok=good))
# sparse CSR/CSC grid engine
import scipy.sparse as sp
for (n, m, k, dens, iters) in [(600, 2, 8, 0.02, 20), (1000, 3, 16, 0.01, 15), (555, 2, 32, 0.03, 10)]:
    rng = np.random.default_rng(n + 7)
    slices = []
    for _ in range(m):
        nnz = int(dens * n * n)
        slices.append(sp.coo_matrix((rng.random(nnz) + 0.01, (rng.integers(0, n, nnz), rng.integers(0, n, nnz))),
                                    shape=(n, n)))
    xs = rk.SparseRelTensor(slices)
    f0 = rk.random_init(n, k, m, 2)
    f, tr, info = rk.solve_on_grid(xs, k, rk.SolverConfig(max_iters=iters), initial=f0, grid=GRID)
    rb = [None] * world
    dist.all_gather_object(rb, f.R.tobytes())
    if rank == 0:
        ao, ro, tro = oracle.solve(list(xs.slices), k, oracle.OracleConfig(max_iters=iters), initial=(f0.A, f0.R))
        rel_a = float(np.linalg.norm(f.A - ao) / np.linalg.norm(ao))
        rel_r = float(np.linalg.norm(f.R - ro) / np.linalg.norm(ro))
        derr = float(np.max(np.abs(tr - tro)))
        same_r = len(set(rb)) == 1
        good = rel_a <= 1e-4 and rel_r <= 1e-4 and derr <= 1e-5 and same_r and len(tr) == iters
        ok = ok and good
        results.append(dict(n=n, m=m, k=k, iters=iters, engine="sparse", grid=[info["pr"], info["pc"]],
                            relA=rel_a, relR=rel_r, dErr=derr, R_replicated=same_r, ok=good))
if rank == 0:
    print(json.dumps({"world": world, "ok": ok, "cases": results}))
dist.destroy_process_group()
sys.exit(0 if ok or rank != 0 else 1)
