"""cfg4 single check (r = 1e5, c = 1e6): device time of the grid-wide path,
pruned (default, full collection) vs dense (F_NOPRUNE), and the per-kind
maxima against the reference goldens (tests/golden/configs.npz,
cfg4_vb2.npz)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2402_14821_b200 import _native, workloads as W  # noqa: E402

if os.environ.get("BPLB_LIB"):  # a development build (e.g. another launch-bounds variant)
    _native.load_library(os.environ["BPLB_LIB"])
c, w = W.cfg4()
eng = _native.Engine(0)
g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "configs.npz"))
modes = (("pruned", 0),) if os.environ.get("PRUNED_ONLY") else (("pruned", 0), ("dense", _native.F_NOPRUNE))
for label, fl in modes:
    eng.check(w, c, 2**62, list(range(6)), fl | _native.F_TIMING)
    ts = []
    for _ in range(9):
        r = eng.check(w, c, 2**62, list(range(6)), fl | _native.F_TIMING)
        ts.append(eng.last_device_ms())
    best = [int(r.best[i]) for i in range(6)]
    print(f"{label:7s} device ms median {np.median(ts):8.3f}  best {best} lb {r.lb} evals {[int(r.evals[i]) for i in range(6)]} "
          f"path {eng.last_path()}")
print("golden non-VB2 best", g["cfg4_best_nonvb2"].tolist())
