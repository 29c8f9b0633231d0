"""K1 DRAM traffic and duration with rotating Q drains off / on (RK_K1_QROT),
one process. Run under
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k1_tc
(profiles/r02_q_rotation.md)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2202_09512_b200 as rk
from paper_2202_09512_b200 import _lib
n, m, k = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (32768, 16, 32)))
for qr in ("0", "1", "4", "0"):
    os.environ["RK_K1_QROT"] = qr
    e = _lib.Engine(n, m, k, device=0)
    e.fill_uniform(7)
    f0 = rk.random_init(n, k, m, 2)
    e.set_factors(f0.A, f0.R)
    e.run(3, 1e-16, track_error=False)
    print("qrot", qr, "slots", e.info()["slots"], flush=True)
    e.close()
