"""Device-resident timing of the cfg5 batch (native generator nodes) through
bplb_check_batch_device: pruned (default) vs dense (F_NOPRUNE) sweep."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2402_14821_b200 import _native, workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
ndense = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
if os.environ.get("BPLB_LIB"):  # a development build
    _native.load_library(os.environ["BPLB_LIB"])
c, k, w = W.cfg5_instance()
t = time.time()
flat, off = W.gen_nodes_device(w, c, k, W.CFG5_SEED, n, device="cuda:0")
torch.cuda.synchronize()
print(f"gen {n} nodes on device: {time.time()-t:.3f}s; mean r {float((off[1:]-off[:-1]).double().mean()):.1f}")
max_r = int((off[1:] - off[:-1]).max())
eng = _native.Engine(0)
lb = torch.empty(n, dtype=torch.int64, device="cuda:0")
ex = torch.empty(n, dtype=torch.uint8, device="cuda:0")
best = torch.empty(n * 6, dtype=torch.int64, device="cuda:0")
arg = torch.empty(n * 6, dtype=torch.int64, device="cuda:0")
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)  # a real stream handle (the legacy default stream's 0 means "engine stream")
s = stream.cuda_stream

def run(nn, flags, kk=2**62, want=False):
    eng.check_batch_device(flat.data_ptr(), off.data_ptr(), nn, max_r, c, kk, list(range(6)), flags,
                           lb.data_ptr(), ex.data_ptr(), best.data_ptr() if want else 0,
                           arg.data_ptr() if want else 0, s)

def timeit(nn, flags, reps=3, **kw):
    run(nn, flags, **kw); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record(stream); run(nn, flags, **kw); e1.record(stream); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)

for label, nn, fl, kw in [("prune lb-mode full", n, 0, {}), ("prune key-mode full", n, 0, {"want": True}),
                          ("prune decision k=334 (seq)", n, _native.F_PHASED, {"kk": 334}),
                          ("prune decision k=334 (cancel)", n, _native.F_CANCEL, {"kk": 334}),
                          ("dense (NOPRUNE) full", ndense, _native.F_NOPRUNE, {})]:
    ms = timeit(nn, fl, **kw)
    print(f"{label:32s} {nn:8d} nodes {ms:9.3f} ms  {1e3*ms/nn:8.3f} us/node  {nn/ms*1e3:12.0f} checks/s  path={eng.last_path()}")
# consistency prune vs dense on the first ndense nodes
run(ndense, 0); torch.cuda.synchronize(); a = lb[:ndense].cpu().clone()
run(ndense, _native.F_NOPRUNE); torch.cuda.synchronize(); b = lb[:ndense].cpu().clone()
print("prune == dense on", ndense, "nodes:", bool((a == b).all()))
