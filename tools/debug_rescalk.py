import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle
import paper_2202_09512_b200 as rk
from conftest import golden

g = golden("rescalk16")
x = g["X"]; xs = [x[t] for t in range(3)]
rep = rk.rescalk(rk.RelTensor(x), 2, 4, r=4, cfg=rk.SolverConfig(max_iters=120, seed=6),
                 pcfg=rk.PerturbConfig(delta=0.02, base_seed=6))
for e in rep.entries:
    med_ref = g[f"medians_k{e.k}"]
    r_or = oracle.regress_r(xs, e.medians)
    e_or = oracle.rel_error(xs, e.medians, r_or)
    r_dev = rk.regress_r(rk.RelTensor(x), e.medians)
    e_dev = rk.rel_error(rk.RelTensor(x), rk.RescalFactors(e.medians, r_dev))
    e_dev2 = rk.rel_error(rk.RelTensor(x), rk.RescalFactors(e.medians, r_or))
    print(e.k, "rel_err ours", e.rel_error, "golden", g["rel_error"][e.k - 2],
          "| med diff", np.abs(e.medians - med_ref).max(),
          "| oracle on our medians", e_or, "| dev regress fresh", e_dev, "dev relerr w/ oracle R", e_dev2,
          "| core diff vs oracle", np.linalg.norm(e.core - r_or) / np.linalg.norm(r_or),
          "| fresh core diff", np.linalg.norm(r_dev - r_or) / np.linalg.norm(r_or))
