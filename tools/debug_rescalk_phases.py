import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2202_09512_b200 as rk
from paper_2202_09512_b200 import _lib

m, n, k = 8, 16384, 16
eng = _lib.Engine(n, m, k)
eng.fill_uniform(1)
def t(label, fn):
    t0 = time.perf_counter(); r = fn(); print(f"{label:40s} {time.perf_counter() - t0:8.4f} s", flush=True); return r
x = rk.RelTensor(np.zeros((m, 2, 2)))  # placeholder shape checks bypassed below
f0 = rk.random_init(n, k, m, 0)
for q in range(3):
    t(f"perturb q={q}", lambda: eng.perturb((0, 3, (k, q)), 0.02))
    t("set_factors", lambda: eng.set_factors(f0.A, f0.R))
    t("run 200 tracked", lambda: eng.run(200, 1e-16, True))
    print("  timing", eng.timing(), flush=True)
    t("get_factors", lambda: eng.get_factors())
t("restore", lambda: eng.restore())
t("set_rank 15", lambda: eng.set_rank(15))
f1 = rk.random_init(n, 15, m, 0)
t("set_factors k15", lambda: eng.set_factors(f1.A, f1.R))
t("run 200 tracked k15", lambda: eng.run(200, 1e-16, True))
t("regress", lambda: eng.regress_r(500, 1e-8, 1e-16))
t("residual", lambda: eng.residual())
