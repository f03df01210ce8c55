"""cfg4 single check: one engine vs the lambda-split check over several
engines of the same / different devices (bplb_check_multi), wall time."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_14821_b200 import _native, workloads as W  # noqa: E402

c, w = W.cfg4()
eng = _native.Engine(0)
for name, run in [("1 engine", lambda: eng.check(w, c, 2**62, list(range(6)), 0))] + [
        (f"split {devs}", (lambda m: (lambda: m.check(w, c, 2**62, list(range(6)), 0)))(_native.MultiEngine(devs)))
        for devs in ((0, 0), (0, 0, 0, 0))]:
    for _ in range(3):
        r = run()
    ts = []
    for _ in range(20):
        t = time.perf_counter()
        r = run()
        ts.append(time.perf_counter() - t)
    print(f"{name:20s} {1e6 * statistics.median(ts):8.1f} us  lb {r.lb}")
