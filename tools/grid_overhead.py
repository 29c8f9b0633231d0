"""Grid-iteration cost split (per-phase CUDA events); CFG=cfg4 runs the sparse
CSR/CSC grid engine on the cfg4 tensor (n=2^20, m=32, density 1e-5, k=16)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import math
import torch.distributed as dist
import paper_2202_09512_b200 as rk
from paper_2202_09512_b200.multigpu import make_grid_engine

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
SPARSE = os.environ.get("CFG") == "cfg4"
if SPARSE:
    n, m, k = 1 << 20, 32, 16
    eng, info = make_grid_engine(n, m, k, sparse=True)
    eng.fill_sparse_uniform(1, int(round(1e-5 * n * n)))
else:
    n = int(round(8192 * math.sqrt(world)))
    m, k = 16, 16
    eng, info = make_grid_engine(n, m, k)
    eng.fill_uniform(1)
f0 = rk.random_init(n, k, m, 0)
out = {}
eng.set_factors(f0.A, f0.R)
eng.run(5, 1e-16, False)
dist.barrier()
eng.set_factors(f0.A, f0.R)
eng.set_option(1, 1)
eng.run(30, 1e-16, False)
out["profiled_ms_per_iter"] = eng.timing()["run_ms"] / 30
out["phases"] = eng.phase_timing()
eng.set_option(1, 0)
eng.set_factors(f0.A, f0.R)
eng.run(30, 1e-16, False)
out["graph_or_direct_ms_per_iter"] = eng.timing()["run_ms"] / 30
allv = [None] * world
dist.all_gather_object(allv, out)
if rank == 0:
    print(json.dumps({"world": world, "n": n, "per_rank": allv}))
eng.close()
dist.destroy_process_group()
