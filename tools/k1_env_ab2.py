"""Like k1_env_ab.py with several RK_* variables per setting:
python tools/k1_env_ab2.py 'A=1,B=2' 'A=2,B=0' ... [n m k via RK_SHAPE=n,m,k]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_09512_b200 as rk
from paper_2202_09512_b200 import _lib
n, m, k = (int(v) for v in os.environ.get("RK_SHAPE", "32768,16,32").split(","))
for s in sys.argv[1:]:
    for kv in s.split(","):
        a, b = kv.split("=")
        os.environ[a] = b
    e = _lib.Engine(n, m, k, device=0)
    e.fill_uniform(7)
    f0 = rk.random_init(n, k, m, 2)
    e.set_factors(f0.A, f0.R)
    e.run(3, 1e-16, track_error=False)
    print(s, e.info(), flush=True)
    e.close()
