"""Single drop-in checks (lower_bound_par, no cancellation = full collection):
device ms (F_TIMING) and host wall us per call, cfg1 / cfg3 / cfg3u / cfg4."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2402_14821_b200 as G  # noqa: E402
from paper_2402_14821_b200 import _native, workloads as W  # noqa: E402

if os.environ.get("BPLB_LIB"):  # a development build
    _native.load_library(os.environ["BPLB_LIB"])
eng = _native.default_engine(0)
cfgs = (("cfg1", W.cfg1), ("cfg3", W.cfg3), ("cfg3u", W.cfg3u), ("cfg4", W.cfg4))
if os.environ.get("ONLY"):
    cfgs = [x for x in cfgs if x[0] in os.environ["ONLY"].split(",")]
for name, gen in cfgs:
    c, w = gen()
    red = G.ReducedInstance.from_array(c, w)
    for _ in range(3):
        G.lower_bound_par(red, 2**62, cancellation=False)
    reps = 50 if name != "cfg4" else 10
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        res = G.lower_bound_par(red, 2**62, cancellation=False)
        ts.append(time.perf_counter() - t)
    eng.check(w, c, 2**62, list(range(6)), _native.F_TIMING)
    dms = eng.last_device_ms()
    print(f"{name:6s} wall {1e6 * statistics.median(ts):9.1f} us  device {1e3 * dms:9.1f} us  lb {res.lb} "
          f"path {eng.last_path()}")
