"""Grid parity at a north-star block size (run with one rank per GPU, e.g.
`python -m torch.distributed.run --nproc-per-node 2 tools/grid_check_big.py`):
n = 32768, k = 32 (cfg3's shape, m = 2 so the host oracle stays affordable),
3 iterations through solve_on_grid with a BlockSource (every rank uploads only
its own block of the synthetic tensor), against the fp64 oracle on rank 0.
RK_PEER=0|1 picks the NCCL or the peer-memory exchange."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch.distributed as dist

import oracle
import paper_2202_09512_b200 as rk
from paper_2202_09512_b200 import _lib
from paper_2202_09512_b200.multigpu import make_grid_engine

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
n, m, k, iters, seed = int(os.environ.get("BIG_N", 32768)), 2, 32, 3, 13
cfg = rk.SolverConfig(max_iters=iters, device=int(os.environ.get("LOCAL_RANK", "0")))
eg, lay = make_grid_engine(n, m, k, cfg=cfg)
blk = eg.block_uniform(seed, lay["rows"], lay["cols"])  # this rank's block of the synthetic tensor
eg.close()
sq = [None] * world
dist.all_gather_object(sq, float(np.sum(blk.astype(np.float64) ** 2)))
src = rk.BlockSource(n, m, lambda info: blk, dtype=np.float32)
f0 = rk.random_init(n, k, m, 5)
t0 = time.perf_counter()
f, tr, ctx = rk.solve_on_grid(src, k, cfg, initial=f0)
secs = time.perf_counter() - t0
rb = [None] * world
dist.all_gather_object(rb, f.R.tobytes())
ok = True
if rank == 0:
    xs = []
    for t in range(m):
        xs.append(_lib.uniform_values(seed, t * n * n, n * n).reshape(n, n).astype(np.float64))
    a, r = f0.A.copy(), f0.R.copy()
    for _ in range(iters):
        a = oracle.mu_iteration(xs, a, r, 1e-16)
    err = float(np.sqrt(oracle.sq_residual(xs, a, r) / oracle.sq_norm(xs)))
    rel_a = float(np.linalg.norm(f.A - a) / np.linalg.norm(a))
    rel_r = float(np.linalg.norm(f.R - r) / np.linalg.norm(r))
    same_r = len(set(rb)) == 1
    ok = rel_a <= 1e-4 and rel_r <= 1e-4 and abs(tr[-1] - err) <= 1e-5 and same_r and len(tr) == iters
    print(json.dumps({"world": world, "grid": [ctx.pr, ctx.pc], "exchange": ctx.exchange, "n": n, "m": m, "k": k,
                      "iters": iters, "block": [lay["rows"], lay["cols"]], "relA": rel_a, "relR": rel_r,
                      "err_dev": float(tr[-1]), "err_oracle": err, "R_replicated": same_r,
                      "sum_block_sq_over_ranks": float(sum(sq)), "solve_s": secs, "ok": bool(ok)}), flush=True)
dist.destroy_process_group()
sys.exit(0 if ok else 1)
