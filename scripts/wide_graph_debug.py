"""Debug: repeated grid-wide checks of two instance sizes (graph capture / replay, table reuse)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2402_14821_b200 import _native  # noqa: E402

eng = _native.Engine(0)
if os.environ.get("NOGRAPH"):
    eng.profile_kernel(True)
rng = np.random.default_rng(11)
a = (1_000_000, rng.integers(1, 1_000_001, 30_000).astype(np.int32))
b = (200_003, rng.integers(1, 200_004, 20_000).astype(np.int32))
seq = os.environ.get("SEQ", "abaabbaba")
for i, ch in enumerate(seq):
    c, w = a if ch == "a" else b
    res = eng.check(w, c, 2**62, list(range(6)), 0)
    print(i, ch, res.lb, list(res.best), flush=True)
