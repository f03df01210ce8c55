"""ncu target: ONE bplb_check_batch_device launch over the first N nodes of
the cfg5 stream (device-generated), lb mode (default) / key / dense / seq.
    python scripts/cfg5_one_launch.py N [lb|key|dense|seq]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_14821_b200 import _native, workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
mode = sys.argv[2] if len(sys.argv) > 2 else "lb"
c, k, w = W.cfg5_instance()
flat, off = W.gen_nodes_device(w, c, k, W.CFG5_SEED, n, device="cuda:0")
max_r = int((off[1:] - off[:-1]).max())
eng = _native.Engine(0)
lb = torch.empty(n, dtype=torch.int64, device="cuda:0")
ex = torch.empty(n, dtype=torch.uint8, device="cuda:0")
best = torch.empty(n * 6, dtype=torch.int64, device="cuda:0") if mode == "key" else None
arg = torch.empty(n * 6, dtype=torch.int64, device="cuda:0") if mode == "key" else None
s = torch.cuda.Stream()
torch.cuda.synchronize()
fl = {"lb": 0, "key": 0, "dense": _native.F_NOPRUNE, "seq": _native.F_PHASED}[mode]
kk = k if mode == "seq" else 2**62
eng.check_batch_device(flat.data_ptr(), off.data_ptr(), n, max_r, c, kk, list(range(6)), fl, lb.data_ptr(),
                       ex.data_ptr(), best.data_ptr() if best is not None else 0,
                       arg.data_ptr() if arg is not None else 0, stream_ptr=s.cuda_stream)
s.synchronize()
print("nodes", n, "items", int(off[-1]), "path", eng.last_path(), "lb sum", int(lb.sum()))
