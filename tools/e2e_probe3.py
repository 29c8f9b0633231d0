"""Sparse engine phases (diagnostics): set_factors / run / get_factors."""
import sys
import time

sys.path.insert(0, ".")
import paper_2202_09512_b200 as rk  # noqa: E402
from paper_2202_09512_b200 import _lib  # noqa: E402

n, m, k, steps = 1 << 20, 32, 16, 10
f0 = rk.random_init(n, k, m, 0)
e = _lib.Engine(n, m, k, sparse=True)
e.fill_sparse_uniform(20220218, int(round(1e-5 * n * n)))
for rep in range(3):
    t = {}
    t0 = time.perf_counter()
    e.set_factors(f0.A, f0.R)
    t["set_factors"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    e.run(steps, 1e-16, track_error=False)
    t["run"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    e.get_factors()
    t["get"] = time.perf_counter() - t0
    print(rep, {a: round(b * 1e3, 1) for a, b in t.items()}, "ms", e.timing())
e.close()
