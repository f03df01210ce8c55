import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2402_14821_b200 import _native
_native.load_library(os.path.join("paper_2402_14821_b200", os.environ.get("LIBN", "libbplb_wtrace.so")))
eng = _native.Engine(0)
c = 1_000_000
w = np.random.default_rng(0).integers(1, c + 1, int(os.environ.get("R", "3000"))).astype(np.int32)
print("start", flush=True)
r = eng.check(w, c, 2**62, list(range(6)), 0)
print("lb", r.lb, eng.last_path(), flush=True)
