"""Factor hash + graph-replayed timing probe for library A/Bs
(tools/ab_hash.sh runs it against two builds via RK_LIB_PATH):
python tools/k2af_check.py cfgX. Prints the ms/iteration (untracked and
tracked), the trace tail and a hash of the factor bytes after 20 iterations
(two builds that keep the arithmetic must agree bit for bit). Named after
its first use, the fused K2a+K2f A/B of round 2."""
import hashlib, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2202_09512_b200 as rk
from paper_2202_09512_b200 import _lib

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n, m, k = {"cfg1": (256, 8, 4), "cfg5": (16384, 8, 16), "cfg2": (8192, 16, 16),
           "cfg3": (32768, 16, 32), "k32s": (4096, 8, 32), "k20": (2048, 4, 20),
           "k32m": (16384, 16, 32), "k48": (8192, 16, 48), "k64": (8192, 16, 64)}[cfg]
eng = _lib.Engine(n, m, k, device=0)
eng.fill_uniform(1)
f0 = rk.random_init(n, k, m, 0)
out = {"cfg": cfg, "env": {a: b for a, b in os.environ.items() if a.startswith("RK_")}}
for track in (False, True):
    eng.set_factors(f0.A, f0.R)
    done, tr = eng.run(20, 1e-16, track)
    a, r = eng.get_factors()
    out[f"hash_track{int(track)}"] = hashlib.sha1(a.tobytes() + r.tobytes()).hexdigest()[:16]
    out[f"trace_track{int(track)}"] = [float(x) for x in np.asarray(tr)[-3:]]
    reps = 200 if n <= 8192 else 20
    eng.set_factors(f0.A, f0.R)
    eng.run(reps, 1e-16, track)
    out[f"ms_per_iter_track{int(track)}"] = eng.timing()["run_ms"] / reps
print(json.dumps(out))
eng.close()
