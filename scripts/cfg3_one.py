"""ncu target: two cfg3 single checks (full collection, multi-CTA node
path); scripts/ncu_cfg4_metrics.py keeps the second launch sequence."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_14821_b200 import _native, workloads as W  # noqa: E402

c, w = W.cfg3()
eng = _native.Engine(0)
for _ in range(2):
    r = eng.check(w, c, 2**62, list(range(6)), 0)
print("lb", r.lb, "path", eng.last_path())
