"""Prune-path timing on batch shapes other than cfg5 (cost-model A/B):
cfg2 nodes (c = 150) forced off the table path, random uniform nodes at
c = 1e4 and c = 1e5; lb and key mode, device-resident, CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_14821_b200 import _native, workloads as W  # noqa: E402

if os.environ.get("BPLB_LIB"):
    _native.load_library(os.environ["BPLB_LIB"])
eng = _native.Engine(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)  # the engine launches on this stream (events must see it)
rng = np.random.default_rng(1)


def uniform_nodes(c, n, rlo, rhi, wlo, whi):
    r = rng.integers(rlo, rhi + 1, n)
    off = np.concatenate([[0], np.cumsum(r)]).astype(np.int64)
    w = rng.integers(max(1, int(wlo * c)), int(whi * c) + 1, int(off[-1])).astype(np.int32)
    return w, off


shapes = []
c2, k2, f2, o2 = W.cfg2_nodes(10_000)
shapes.append(("cfg2 c=150 (NOTAB)", 150, f2.astype(np.int32), o2, _native.F_NOTAB))
shapes.append(("uniform c=1e4 r~300", 10_000, *uniform_nodes(10_000, 20_000, 200, 400, 0.05, 0.6), 0))
shapes.append(("uniform c=1e5 r~800", 100_000, *uniform_nodes(100_000, 20_000, 600, 1000, 0.01, 0.5), 0))
for name, c, w, off, fl in shapes:
    n = len(off) - 1
    d_w = torch.from_numpy(w).cuda()
    d_off = torch.from_numpy(off).cuda()
    lb = torch.empty(n, dtype=torch.int64, device="cuda")
    ex = torch.empty(n, dtype=torch.uint8, device="cuda")
    best = torch.empty(n * 6, dtype=torch.int64, device="cuda")
    arg = torch.empty(n * 6, dtype=torch.int64, device="cuda")
    max_r = int(np.diff(off).max())
    for key in (False, True):
        def run():
            eng.check_batch_device(d_w.data_ptr(), d_off.data_ptr(), n, max_r, c, 2**62, list(range(6)), fl,
                                   lb.data_ptr(), ex.data_ptr(), best.data_ptr() if key else 0,
                                   arg.data_ptr() if key else 0, stream.cuda_stream)
        run(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(3):
            e0.record(stream); run(); e1.record(stream); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        print(f"{name:24s} {'key' if key else 'lb '} {min(ts) * 1e3 / n:8.3f} us/node path={eng.last_path()}")
