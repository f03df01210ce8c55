"""cfg2 batch (10^4 Scholl-1 nodes, c = 150, uint8 weights): device time of the
table path on the tensor cores (default) vs the FP32 pipe (F_NOTC), CUDA
events on the launching stream, L2 flushed before each call; parity of the
two paths and against the oracle on the first 500 nodes."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_14821_b200 import _native, workloads as W  # noqa: E402

c, k, flat, off = W.cfg2_nodes(10_000)
n = len(off) - 1
dev = torch.device("cuda", 0)
d_w = torch.from_numpy(flat.astype(np.uint8)).to(dev)
d_off = torch.from_numpy(off).to(dev)
lb = torch.empty(n, dtype=torch.int64, device=dev)
ex = torch.empty(n, dtype=torch.uint8, device=dev)
eng = _native.Engine(0)
s = torch.cuda.Stream()
flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)
max_r = int(np.diff(off).max())
res = {}
for label, fl in (("tc", 0), ("fp32", _native.F_NOTC)):
    for _ in range(3):
        eng.check_batch_device(d_w.data_ptr(), d_off.data_ptr(), n, max_r, c, 2**62, list(range(6)), fl,
                               lb.data_ptr(), ex.data_ptr(), stream_ptr=s.cuda_stream, wbytes=1)
    ts = []
    for i in range(20):
        with torch.cuda.stream(s):
            flush.fill_(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        eng.check_batch_device(d_w.data_ptr(), d_off.data_ptr(), n, max_r, c, 2**62, list(range(6)), fl,
                               lb.data_ptr(), ex.data_ptr(), stream_ptr=s.cuda_stream, wbytes=1)
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    res[label] = lb.cpu().numpy().copy()
    print(f"{label:5s} {statistics.median(ts):8.1f} us per 10^4 nodes  path {eng.last_path()}")
print("tc == fp32:", bool(np.array_equal(res["tc"], res["fp32"])))
# the contraction kernel alone (events around the launch inside the C ABI;
# graph replay off), same L2 flush
eng._lib.bplb_profile_kernel(eng.handle, 1)
ks = []
for i in range(20):
    with torch.cuda.stream(s):
        flush.fill_(i)
    eng.check_batch_device(d_w.data_ptr(), d_off.data_ptr(), n, max_r, c, 2**62, list(range(6)), 0,
                           lb.data_ptr(), ex.data_ptr(), stream_ptr=s.cuda_stream, wbytes=1)
    s.synchronize()
    ks.append(eng.last_kernel_ms() * 1e3)
eng._lib.bplb_profile_kernel(eng.handle, 0)
print(f"tc kernel alone {statistics.median(ks):8.1f} us per 10^4 nodes")
from oracle import oracle as O  # noqa: E402

O.set_threads(O.max_threads())
lbo, _ = O.check_batch(flat[:off[500]], off[:501], c, 2**62)
print("tc == oracle (500 nodes):", bool(np.array_equal(res["tc"][:500], lbo)))
