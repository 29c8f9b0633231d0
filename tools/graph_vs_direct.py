"""Graph-replayed vs directly launched iterations on the same engine (cfg3):
does the CUDA-graph path cost time? Alternates the modes twice."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_09512_b200 as rk
from paper_2202_09512_b200 import _lib
n, m, k = {"cfg3": (32768, 16, 32), "cfg2": (8192, 16, 16)}[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
eng = _lib.Engine(n, m, k, device=0)
eng.fill_uniform(1)
f0 = rk.random_init(n, k, m, 0)
eng.set_factors(f0.A, f0.R)
eng.run(40, 1e-16, False)
out = []
for rep in range(3):
    for mode in ("graph", "profiled", "direct"):
        eng.set_option(1, 1 if mode == "profiled" else 0)
        eng.set_option(2, 0 if mode == "direct" else 1)
        eng.set_factors(f0.A, f0.R)
        eng.run(steps, 1e-16, False)
        out.append((mode, round(eng.timing()["run_ms"] / steps, 4)))
eng.set_option(1, 0)
eng.set_option(2, 1)
print(json.dumps(out))
