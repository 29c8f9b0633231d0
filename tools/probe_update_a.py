import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2202_09512_b200 as rk
import oracle
for n, m, k in ((256, 8, 4), (256, 8, 16), (1024, 4, 16), (640, 3, 32), (768, 2, 27)):
    rng = np.random.default_rng(n + k)
    x = rng.random((m, n, n), dtype=np.float32).astype(np.float64)
    a0, r0 = oracle.random_init(n, k, m, 3)
    f = rk.update_a(rk.RelTensor(x), rk.RescalFactors(a0, r0))
    # oracle update_a: numerator/denominator with fixed cores (rescal.py:243-258)
    g = a0.T @ a0
    num = np.zeros_like(a0); den = np.zeros_like(a0)
    for t in range(m):
        xa = x[t] @ a0; ar = a0 @ r0[t]
        num += xa @ r0[t].T + x[t].T @ ar
        den += (a0 @ r0[t].T) @ (g @ r0[t]) + ar @ (g @ r0[t].T) + 1e-16
    ao = a0 * num / den
    rel = np.abs(f.A - ao) / np.abs(ao)
    i, j = np.unravel_index(np.argmax(rel), rel.shape)
    print(n, m, k, "max rel %.3e at (%d,%d)  median %.3e  relfro %.3e" % (rel.max(), i, j, np.median(rel), np.linalg.norm(f.A-ao)/np.linalg.norm(ao)))
