"""Timeline of the assignment-path batch call (device-side reduce_packing)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2402_14821_b200 as G
from paper_2402_14821_b200 import workloads as W

c, k, w, a = W.cfg2_assignments(10_000)
ha = torch.from_numpy(a).pin_memory().numpy()
for _ in range(3):
    G.lower_bound_batch_assign(c, w, ha, k, 2**62)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    G.lower_bound_batch_assign(c, w, ha, k, 2**62)
t0 = None
for e in sorted(prof.events(), key=lambda e: e.time_range.start):
    if t0 is None:
        t0 = e.time_range.start
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.elapsed_us():8.1f} {e.device_type.name[:4]} {e.name[:70]}")
