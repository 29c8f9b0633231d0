"""Diagnostics for the fused k-wide chain (k2_chain.cuh): per-phase edges of
one launch (RK_CHAIN_STAMPS=1) and graph-replayed it/s with the chain on / off."""
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2202_09512_b200 as rk
from paper_2202_09512_b200 import _lib

lib = _lib.load()
lib.rk_chain_stamps.restype = ctypes.c_int
lib.rk_chain_stamps.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)]
out = {"env": {k: os.environ.get(k) for k in ("RK_CHAIN_COOP", "RK_CHAIN_SLEEP")}}
CFGS = {"cfg1": (256, 8, 4, 3000), "cfg2": (8192, 16, 16, 200), "cfg5": (16384, 8, 16, 100),
        "cfg3": (32768, 16, 32, 20), "n2048k32": (2048, 8, 32, 1000)}
for name in os.environ.get("CHAIN_CFGS", "cfg1,cfg2,cfg5").split(","):
    n, m, k, iters = CFGS[name]
    eng = _lib.Engine(n, m, k, device=0)
    eng.fill_uniform(7)
    f0 = rk.random_init(n, k, m, 0)
    res = {}
    for chain in (1, 0):
        eng.set_option(5, chain)
        eng.set_factors(f0.A, f0.R)
        eng.run(50, 1e-16, track_error=False)
        eng.set_factors(f0.A, f0.R)
        eng.run(iters, 1e-16, track_error=False)
        res[f"chain{chain}_it_s"] = iters / (eng.timing()["run_ms"] / 1e3)
        if chain and os.environ.get("RK_CHAIN_STAMPS"):
            st = (ctypes.c_double * 5)()
            if lib.rk_chain_stamps(eng._h, st) == 0:
                res["phase_edges_us"] = dict(zip(["A_end", "bar1_exit", "B_end", "bar2_exit", "C_end"], list(st)))
    eng.close()
    out[name] = res
print(json.dumps(out))
