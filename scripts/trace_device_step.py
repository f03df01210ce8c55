"""Timeline of the bench's device-resident step (flush, hist, tab, fin)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2402_14821_b200 import _native, workloads as W

c, k, flat, off = W.cfg2_nodes(10_000)
w8 = flat.astype(np.uint8)
eng = _native.Engine(0)
dev = torch.device("cuda", 0)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
d_w = torch.from_numpy(w8).to(dev)
d_off = torch.from_numpy(off).to(dev)
n = len(off) - 1
d_lb = torch.empty(n, dtype=torch.int64, device=dev)
d_ex = torch.empty(n, dtype=torch.uint8, device=dev)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)
mr = int(np.diff(off).max())
def step(i):
    flush.fill_(i)
    eng.check_batch_device(d_w.data_ptr(), d_off.data_ptr(), n, mr, c, 2**62, list(range(6)), 0,
                           d_lb.data_ptr(), d_ex.data_ptr(), stream_ptr=st.cuda_stream, wbytes=1)
for i in range(5):
    step(i)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(3):
        step(i)
    torch.cuda.synchronize()
t0 = None
for e in sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start):
    if t0 is None:
        t0 = e.time_range.start
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - t0:9.1f} {e.time_range.elapsed_us():8.1f} {e.name[:60]}")
