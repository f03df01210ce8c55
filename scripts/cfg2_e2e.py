"""cfg2 e2e through the public batch API with pinned host buffers (wall us)."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_14821_b200 import _native, workloads as W  # noqa: E402

c, k, flat, off = W.cfg2_nodes(10_000)
n = len(off) - 1
eng = _native.Engine(0)
h_w = torch.from_numpy(flat.astype(np.uint8)).pin_memory().numpy()
h_off = torch.from_numpy(off).pin_memory().numpy()
h_lb = torch.empty(n, dtype=torch.int64).pin_memory().numpy()
h_ex = torch.empty(n, dtype=torch.uint8).pin_memory().numpy()
for _ in range(3):
    eng.check_batch(h_w, h_off, c, 2**62, list(range(6)), 0, out=(h_lb, h_ex))
ts = []
for _ in range(30):
    t = time.perf_counter()
    eng.check_batch(h_w, h_off, c, 2**62, list(range(6)), 0, out=(h_lb, h_ex))
    ts.append(time.perf_counter() - t)
print(f"e2e pinned {1e6 * statistics.median(ts):.1f} us per 10^4 nodes, path {eng.last_path()}")
