"""K1 P / Q accuracy vs fp64 at one shape, with and without rotating Q drains
(RK_K1_QROT). python tools/q_accuracy.py n m k -> one line per setting."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if len(sys.argv) > 4:  # child: one measurement
    import numpy as np
    import paper_2202_09512_b200 as rk
    from paper_2202_09512_b200 import _lib
    n, m, k = map(int, sys.argv[1:4])
    x = np.random.default_rng(1).random((m, n, n), dtype=np.float32)
    f0 = rk.random_init(n, k, m, 2)
    e = _lib.Engine(n, m, k, device=0)
    e.upload(x)
    e.set_factors(f0.A, f0.R)
    e.update_r(1e-16)
    p, q = e.debug_read_pq()
    a = f0.A
    ep = eq = 0.0
    for t in range(m):
        xt = x[t].astype(np.float64)
        pr, qr = xt @ a, xt.T @ a
        ep = max(ep, np.linalg.norm(p[t, :n, :k] - pr) / np.linalg.norm(pr))
        eq = max(eq, np.linalg.norm(q[t, :n, :k] - qr) / np.linalg.norm(qr))
    inf = e.info()
    print(f"n={n} m={m} k={k} qrot={os.environ.get('RK_K1_QROT')} slots={inf['slots']} strip_tiles={inf['strip_tiles']}"
          f"  P relerr {ep:.3e}  Q relerr {eq:.3e}", flush=True)
    sys.exit(0)
for qr in ("0", "1", "2", "4"):
    subprocess.run([sys.executable, __file__, *sys.argv[1:4], "child"], env=dict(os.environ, RK_K1_QROT=qr), check=True)
