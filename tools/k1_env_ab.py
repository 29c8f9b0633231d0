"""One process, several settings of an RK_* switch read at engine creation:
per-kernel time / DRAM bytes under ncu for each. Usage:
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    python tools/k1_env_ab.py VAR v1,v2,... [n m k]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_09512_b200 as rk
from paper_2202_09512_b200 import _lib
var, vals = sys.argv[1], sys.argv[2].split(",")
n, m, k = (int(v) for v in (sys.argv[3:6] if len(sys.argv) > 5 else (32768, 16, 32)))
for v in vals:
    os.environ[var] = v
    e = _lib.Engine(n, m, k, device=0)
    e.fill_uniform(7)
    f0 = rk.random_init(n, k, m, 2)
    e.set_factors(f0.A, f0.R)
    e.run(3, 1e-16, track_error=False)
    print(var, v, e.info(), flush=True)
    e.close()
