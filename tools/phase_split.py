"""Per-phase device time of one MU iteration on one GPU (CUDA events between
phases, profiled run): python tools/phase_split.py [cfg2|cfg3|cfg4]."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_09512_b200 as rk
from paper_2202_09512_b200 import _lib

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n, m, k, sparse = {"cfg1": (256, 8, 4, False), "cfg5": (16384, 8, 16, False),
                   "cfg2": (8192, 16, 16, False), "k48": (8192, 16, 48, False), "k64": (8192, 16, 64, False), "cfg3": (32768, 16, 32, False), "k32m": (16384, 16, 32, False),
                   "cfg4": (1 << 20, 32, 16, True), "cfg4k32": (1 << 20, 32, 32, True)}[cfg]
eng = _lib.Engine(n, m, k, device=0, sparse=sparse)
if sparse:
    eng.fill_sparse_uniform(1, int(round(1e-5 * n * n)))
else:
    eng.fill_uniform(1)
f0 = rk.random_init(n, k, m, 0)
eng.set_factors(f0.A, f0.R)
eng.run(5, 1e-16, False)
eng.set_factors(f0.A, f0.R)
eng.set_option(1, 1)
eng.run(20, 1e-16, False)
out = {"cfg": cfg, "profiled_ms_per_iter": eng.timing()["run_ms"] / 20,
       "phases_ms": {a: round(b, 4) for a, b in eng.phase_timing().items()}}
eng.set_option(1, 0)
eng.set_factors(f0.A, f0.R)
eng.run(20, 1e-16, False)
out["graph_ms_per_iter"] = eng.timing()["run_ms"] / 20
print(json.dumps(out))
eng.close()
