"""Two engines on one GPU running K1 at the same time (two host threads, two
streams): strip-group K1 is launched cooperatively, so its members are
co-resident and the concurrent solves finish (no inter-CTA wait deadlock)."""
import os, sys, threading, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2202_09512_b200 as rk
from paper_2202_09512_b200 import _lib

n, m, k = 16384, 4, 32
res = {}
def work(i):
    e = _lib.Engine(n, m, k, device=0)
    e.fill_uniform(3 + i)
    f0 = rk.random_init(n, k, m, 2)
    e.set_factors(f0.A, f0.R)
    t = time.perf_counter()
    e.run(20, 1e-16, track_error=False)
    res[i] = (time.perf_counter() - t, e.info()["k1_group"], e.get_factors()[1].sum())
    e.close()
th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
for t in th: t.start()
for t in th: t.join(timeout=240)
print("alive after join:", [t.is_alive() for t in th], res, flush=True)
os._exit(0 if not any(t.is_alive() for t in th) else 3)
