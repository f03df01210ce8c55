"""Device-resident batched check (the bench's `value` path) a few times; a
target for ncu.  --notab selects the warp-per-node kernel."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2402_14821_b200 import _native, workloads as W

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg2")
ap.add_argument("--nodes", type=int, default=10_000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--notab", action="store_true")
ap.add_argument("--kinds", default="0,1,2,3,4,5")
a = ap.parse_args()
c, k, flat, off = (W.cfg2_nodes if a.cfg == "cfg2" else W.cfg5_nodes)(a.nodes)
wdt = np.uint8 if c <= 255 else (np.uint16 if c <= 65535 else np.int32)
eng = _native.Engine(0)
dev = torch.device("cuda", 0)
d_w = torch.from_numpy(flat.astype(wdt)).to(dev)
d_off = torch.from_numpy(off).to(dev)
n = len(off) - 1
d_lb = torch.empty(n, dtype=torch.int64, device=dev)
d_ex = torch.empty(n, dtype=torch.uint8, device=dev)
fl = _native.F_NOTAB if a.notab else 0
st = torch.cuda.Stream()  # a real stream handle (the legacy default stream reads as "engine stream")
torch.cuda.set_stream(st)
for i in range(a.reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(st)
    eng.check_batch_device(d_w.data_ptr(), d_off.data_ptr(), n, int(np.diff(off).max()), c, 2**62,
                           [int(x) for x in a.kinds.split(",")], fl, d_lb.data_ptr(), d_ex.data_ptr(), wbytes=np.dtype(wdt).itemsize,
                           stream_ptr=st.cuda_stream)
    e.record(st)
    torch.cuda.synchronize()
    print(f"{a.cfg} nodes={n} rep={i} ms={s.elapsed_time(e):.4f}", flush=True)
