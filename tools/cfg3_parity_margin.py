"""relA / relR of the cfg3-shape parity test (n = 32768, m = 2, k = 32, 3
iterations vs the fp64 oracle) under several RK_* settings: how much room
the 1e-4 tolerance leaves. python tools/cfg3_parity_margin.py 'RK_K1_GRP=1' 'RK_K1_GRP=2' ..."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import test_gpu_north_star as t
    iters = int(os.environ.get("ITERS", "3"))
    a_dev, r_dev, trace, a, r, err, info = t._device_vs_oracle(32768, 2, 32, iters, 13)
    print(f"{os.environ.get('SETTING')} iters {iters}: relA {t.rel_fro(a_dev, a):.3e} relR {t.rel_fro(r_dev, r):.3e} "
          f"dErr {abs(trace[-1] - err):.2e} strips {info['strips']} group {info['k1_group']}", flush=True)
    sys.exit(0)
for s in sys.argv[1:]:
    env = dict(os.environ, SETTING=s)
    for kv in s.split(","):
        k, v = kv.split("=")
        env[k] = v
    subprocess.run([sys.executable, __file__, "child"], env=env, check=False)
