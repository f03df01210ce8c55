"""Run one config through the public API a few times (target for ncu)."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2402_14821_b200 as G
from paper_2402_14821_b200 import workloads as W, _native

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg5")
ap.add_argument("--nodes", type=int, default=296)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--mode", default="full")
a = ap.parse_args()
eng = _native.default_engine()
if a.cfg in ("cfg2", "cfg5"):
    c, k, flat, off = (W.cfg2_nodes if a.cfg == "cfg2" else W.cfg5_nodes)(a.nodes)
    kk = 2**62 if a.mode == "full" else k
    for _ in range(a.reps):
        t = time.perf_counter()
        eng.check_batch(flat, off, c, kk, list(range(6)), {"full": 0, "seq": 1, "cancel": 2}[a.mode] | _native.F_TIMING)
        print(a.cfg, "wall ms", (time.perf_counter() - t) * 1e3, "device ms", eng.last_device_ms(), flush=True)
else:
    c, w = {"cfg1": W.cfg1, "cfg3": W.cfg3, "cfg3u": W.cfg3u, "cfg4": W.cfg4}[a.cfg]()
    for _ in range(a.reps):
        t = time.perf_counter()
        res = eng.check(w, c, 2**62, list(range(6)), _native.F_TIMING | {"full": 0, "seq": 1, "cancel": 2}[a.mode])
        print(a.cfg, "wall ms", (time.perf_counter() - t) * 1e3, "device ms", eng.last_device_ms(), "lb", res.lb, flush=True)
