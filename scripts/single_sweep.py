import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2402_14821_b200 as G
from paper_2402_14821_b200 import workloads as W, _native
eng = _native.default_engine()
for cfg in ("cfg1", "cfg3"):
    c, w = {"cfg1": W.cfg1, "cfg3": W.cfg3}[cfg]()
    red = G.ReducedInstance.from_array(c, w)
    for _ in range(10):
        G.lower_bound_seq(red, 2**62)
    ts, ds = [], []
    for _ in range(100):
        t = time.perf_counter(); eng.check(w, c, 2**62, list(range(6)), _native.F_PHASED | _native.F_TIMING)
        ts.append(time.perf_counter() - t); ds.append(eng.last_device_ms())
    print(f"DIV={os.environ.get('BPLB_CELLS_DIV','16384')} {cfg}: wall {np.median(ts)*1e6:.1f} us device {np.median(ds)*1e3:.1f} us")
