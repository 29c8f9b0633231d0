"""cfg1 (n = 256, m = 8, k = 4): graph-replayed ms/iteration, tcgen05 vs SIMT engine."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_09512_b200 as rk
from paper_2202_09512_b200 import _lib
for (n, m, k) in ((256, 8, 4), (512, 8, 8), (1024, 8, 16)):
    for engine in ("tc", "simt"):
        e = _lib.Engine(n, m, k, device=0, engine=engine)
        e.fill_uniform(1)
        f0 = rk.random_init(n, k, m, 0)
        e.set_factors(f0.A, f0.R)
        e.run(50, 1e-16, False)
        e.set_factors(f0.A, f0.R)
        e.run(2000, 1e-16, False)
        print(n, m, k, engine, round(e.timing()["run_ms"] / 2000 * 1000, 2), "us/it", flush=True)
        e.close()
