"""Timeline of single drop-in checks (cfg1 / cfg3) through lower_bound_seq."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2402_14821_b200 as G
from paper_2402_14821_b200 import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
c, w = {"cfg1": W.cfg1, "cfg3": W.cfg3}[cfg]()
red = G.ReducedInstance.from_array(c, w)
for _ in range(20):
    G.lower_bound_seq(red, 2**62)
ts = []
for _ in range(200):
    t = time.perf_counter(); G.lower_bound_seq(red, 2**62); ts.append(time.perf_counter() - t)
print(f"{cfg}: median {np.median(ts)*1e6:.1f} us, min {min(ts)*1e6:.1f} us")
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        G.lower_bound_seq(red, 2**62)
t0 = None
for e in sorted(prof.events(), key=lambda e: e.time_range.start)[-40:]:
    if t0 is None:
        t0 = e.time_range.start
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.elapsed_us():8.1f} {e.device_type.name[:4]} {e.name[:70]}")
