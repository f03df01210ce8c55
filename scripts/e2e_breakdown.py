"""e2e (host buffers) timing of the batched API vs. the pure pinned H2D copy."""
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
for _ in range(5):
    eng.check_batch(h_w, h_off, c, 2**62, list(range(6)), 0, out=(h_lb, h_ex))
ts, ds = [], []
for _ in range(20):
    t = time.perf_counter()
    eng.check_batch(h_w, h_off, c, 2**62, list(range(6)), _native.F_TIMING, out=(h_lb, h_ex))
    ts.append(time.perf_counter() - t)
    ds.append(eng.last_device_ms())
print(f"e2e wall {np.median(ts)*1e6:.1f} us, device-timed {np.median(ds)*1e3:.1f} us")
d = torch.empty(flat.nbytes + off.nbytes, dtype=torch.uint8, device="cuda")
src = torch.from_numpy(np.concatenate([flat.view(np.uint8), off.view(np.uint8)])).pin_memory()
for _ in range(3):
    d.copy_(src, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20):
    d.copy_(src, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 20
print(f"pure pinned H2D of {src.numel()/1e6:.2f} MB: {dt*1e6:.1f} us = {src.numel()/dt/1e9:.1f} GB/s")

if os.environ.get("TRACE"):
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(2):
            eng.check_batch(h_w, h_off, c, 2**62, list(range(6)), 0, out=(h_lb, h_ex))
    evs = [e for e in prof.events() if e.device_type.name == "CUDA" or "cuda" in e.name.lower()]
    t0 = None
    for e in sorted(prof.events(), key=lambda e: e.time_range.start)[-60:]:
        if t0 is None:
            t0 = e.time_range.start
        print(f"{e.time_range.start - t0:9.1f} {e.time_range.elapsed_us():8.1f} {e.device_type.name[:4]} {e.name[:70]}")
