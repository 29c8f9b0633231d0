"""K1 bandwidth experiments (results are NOT valid factorizations): time the
tcgen05 slice contraction alone under debug switches."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_09512_b200 import _lib
import paper_2202_09512_b200 as rk

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n, m, k = {"cfg2": (8192, 16, 16), "cfg3": (32768, 16, 32)}[cfg]
eng = _lib.Engine(n, m, k)
eng.fill_uniform(1)
f = rk.random_init(n, k, m, 0)
eng.set_factors(f.A, f.R)
out = {"info": eng.info()}
for dbg, name in [(0, "full"), (2, "no_q_drain_wait"), (1, "no_mma"), (3, "no_mma_no_wait")]:
    eng.set_option(3, dbg)
    ms = eng.time_k1(10 if cfg == "cfg2" else 3)
    out[name] = {"ms": ms, "GBps": 4.0 * m * n * n / (ms / 1e3) / 1e9}
eng.set_option(3, 0)
print(json.dumps(out))
