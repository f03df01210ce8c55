"""Distribution of e2e (pinned host in/out) batch-call times, cfg2 10^4 nodes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2402_14821_b200 import _native, workloads as W

c, k, flat, off = W.cfg2_nodes(10_000)
flat = flat.astype(np.uint8)
eng = _native.Engine(0)
h_w = torch.from_numpy(flat).pin_memory().numpy()
h_off = torch.from_numpy(off).pin_memory().numpy()
n = len(off) - 1
h_lb = torch.empty(n, dtype=torch.int64).pin_memory().numpy()
h_ex = torch.empty(n, dtype=torch.uint8).pin_memory().numpy()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
for mode in ("noflush", "flush"):
    ts = []
    for i in range(60):
        if mode == "flush":
            flush.fill_(i)
            torch.cuda.synchronize()
        t = time.perf_counter()
        eng.check_batch(h_w, h_off, c, 2**62, list(range(6)), 0, out=(h_lb, h_ex))
        ts.append((time.perf_counter() - t) * 1e6)
    ts = np.array(ts[5:])
    print(f"{mode}: p10 {np.percentile(ts,10):.0f} p50 {np.percentile(ts,50):.0f} p90 {np.percentile(ts,90):.0f} max {ts.max():.0f} us")
