"""cfg2 batches back to back: (a) the same batch with an L2 flush (torch fill)
before each call, (b) 32 distinct copies of the batch cycled (160 MB of CSR,
larger than the 126 MB L2, no flush kernel between the batches), (c) the same
batch back to back (L2-warm).  CUDA events on the launching stream."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_14821_b200 import _native, workloads as W  # noqa: E402

c, k, flat, off = W.cfg2_nodes(10_000)
n = len(off) - 1
dev = torch.device("cuda", 0)
NC = 32
ws = [torch.from_numpy(flat.astype(np.uint8)).to(dev) for _ in range(NC)]
offs = [torch.from_numpy(off).to(dev) for _ in range(NC)]
lb = torch.empty(n, dtype=torch.int64, device=dev)
ex = torch.empty(n, dtype=torch.uint8, device=dev)
eng = _native.Engine(0)
s = torch.cuda.Stream()
flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)
max_r = int(np.diff(off).max())
fl = int(os.environ.get("FLAGS", "0"))


def call(i):
    eng.check_batch_device(ws[i].data_ptr(), offs[i].data_ptr(), n, max_r, c, 2**62, list(range(6)), fl,
                           lb.data_ptr(), ex.data_ptr(), stream_ptr=s.cuda_stream, wbytes=1)


for i in range(NC):
    call(i)
torch.cuda.synchronize()
import ctypes  # noqa: E402

peaks = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2402_14821_b200",
                                 "libbplb_peaks.so"))
peaks.bplb_flush_l2.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_int]
for label in ("flush", "flush_smem", "flush_smem_only", "cycle", "warm"):
    if label.startswith("flush_smem"):
        sm = int(os.environ.get("FLUSH_SMEM", str(200 * 1024)))
        tot = 0.0
        for i in range(20):
            peaks.bplb_flush_l2(flush.data_ptr(), flush.numel() * 4, s.cuda_stream, sm)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            if label == "flush_smem":
                call(0)
            e1.record(s)
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        print(f"{label:6s} {tot / 20 * 1e3:8.1f} us per 10^4-node batch")
        continue
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if label == "flush":
        tot = 0.0
        for i in range(20):
            with torch.cuda.stream(s):
                flush.fill_(i)
            e0.record(s)
            call(0)
            e1.record(s)
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        us = tot / 20 * 1e3
    else:
        reps = 3 * NC
        e0.record(s)
        for j in range(reps):
            call(j % NC if label == "cycle" else 0)
        e1.record(s)
        e1.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
    print(f"{label:6s} {us:8.1f} us per 10^4-node batch  path {eng.last_path()}")
