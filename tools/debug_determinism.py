import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2202_09512_b200 as rk
from paper_2202_09512_b200 import _lib
from conftest import golden

g = golden("rescalk16")
x = g["X"]
def solve_once(eng, k, q):
    eng.perturb((6, 3, (k, q)), 0.02)
    init = rk.random_init(16, k, 3, (6, 4, k, q))
    f, tr = rk.rescal_solve(rk.RelTensor(x), k, rk.SolverConfig(max_iters=120, seed=6), initial=init, engine=eng)
    return f.A.copy(), f.R.copy(), tr.copy()

for engine in ("tc", "simt"):
    eng = _lib.Engine(16, 3, 2, engine=engine)
    eng.upload(x)
    ref = solve_once(eng, 2, 1)
    bad = 0
    for rep in range(30):
        a, r, tr = solve_once(eng, 2, 1 + (rep % 4))
        if rep % 4 == 0:
            if not (np.array_equal(a, ref[0]) and np.array_equal(r, ref[1]) and np.array_equal(tr, ref[2])):
                bad += 1
                print(engine, "rep", rep, "A diff", np.abs(a - ref[0]).max(), "trace diff", np.abs(tr - ref[2]).max(), flush=True)
    print(engine, "nondeterministic repeats:", bad, flush=True)
    # regress / rel_error determinism
    eng.restore()
    med = g["medians_k2"]
    vals = []
    for rep in range(20):
        core = rk.regress_r(rk.RelTensor(x), med, engine=eng)
        e = rk.rel_error(rk.RelTensor(x), rk.RescalFactors(med, core), engine=eng)
        vals.append((e, core.copy()))
    es = [v[0] for v in vals]
    print(engine, "regress/rel_error spread", max(es) - min(es), "core spread", max(np.abs(v[1] - vals[0][1]).max() for v in vals), flush=True)
    eng.close()
# bigger problem determinism (multi-tile, multi-segment TC schedule)
xb = np.random.default_rng(0).random((4, 1024, 1024), dtype=np.float32)
eng = _lib.Engine(1024, 4, 16, engine="tc")
eng.upload(xb)
f0 = rk.random_init(1024, 16, 4, 0)
outs = []
for rep in range(10):
    eng.set_factors(f0.A, f0.R)
    _, tr = eng.run(20, 1e-16, True)
    a, r = eng.get_factors()
    outs.append((a, r, tr))
print("big tc repeats differ:", sum(not np.array_equal(o[0], outs[0][0]) for o in outs), "max", max(np.abs(o[0]-outs[0][0]).max() for o in outs))
