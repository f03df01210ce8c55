"""Per-unit cycle trace of prune_kernel (development build with -DPRUNE_TRACE).

    python scripts/prune_trace.py build        # here: builds paper_2402_14821_b200/libbplb_trace.so
    python scripts/prune_trace.py run [N]      # GPU box: one lb-mode launch over N cfg5 nodes, summary

Summary per (kind, unit type): units, total / max cycles, and per CTA the
unit-sweep span vs the drain span (what the barrier waits on)."""
import collections
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "paper_2402_14821_b200", "libbplb_trace.so")
KN = ["MT", "RAD2", "FS1", "CCM1", "VB2", "BJ1"]
TN = ["CAND", "LOOK", "WALK", "PRUNE", "BLK"]

if sys.argv[1] == "build":
    from paper_2402_14821_b200 import build_native as B

    cmd = ["/usr/local/cuda/bin/nvcc", *B.NVCC_FLAGS, "-DPRUNE_TRACE", "-shared", "-o", LIB,
           os.path.join(B.CSRC, "bplb_capi.cu"), "-lcudart"]
    subprocess.run(cmd, check=True, capture_output=True)
    print("built", LIB)
    sys.exit(0)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_14821_b200 import _native, workloads as W  # noqa: E402

n = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
key_mode = len(sys.argv) > 3 and sys.argv[3] == "key"
_native.load_library(LIB)
lib = _native.load_library()
lib.bplb_prune_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
c, k, w = W.cfg5_instance()
flat, off = W.gen_nodes_device(w, c, k, W.CFG5_SEED, n, device="cuda:0")
max_r = int((off[1:] - off[:-1]).max())
eng = _native.Engine(0)
lb = torch.empty(n, dtype=torch.int64, device="cuda:0")
ex = torch.empty(n, dtype=torch.uint8, device="cuda:0")
s = torch.cuda.Stream()
torch.cuda.synchronize()
buf = np.zeros((1 << 16, 4), dtype=np.int64)
lib.bplb_prune_trace(buf.ctypes.data, 1 << 16)  # reset
best = torch.empty(n * 6, dtype=torch.int64, device="cuda:0")
arg = torch.empty(n * 6, dtype=torch.int64, device="cuda:0")
eng.check_batch_device(flat.data_ptr(), off.data_ptr(), n, max_r, c, 2**62, list(range(6)), 0, lb.data_ptr(),
                       ex.data_ptr(), best.data_ptr() if key_mode else 0, arg.data_ptr() if key_mode else 0,
                       stream_ptr=s.cuda_stream)
s.synchronize()
m = lib.bplb_prune_trace(buf.ctypes.data, 1 << 16)
rec = buf[:m]
tag = rec[:, 0] & 0xFFFF0000
units = rec[(tag != 0xFFFF0000) & (tag != 0xFFFE0000)]
drains = rec[tag == 0xFFFF0000]
items = rec[tag == 0xFFFE0000]
agg = collections.defaultdict(list)
for r in units:
    kind, typ = int(r[1]) >> 8, int(r[1]) & 0xFF
    agg[(KN[kind], TN[typ])].append(int(r[3] - r[2]))
tot = sum(sum(v) for v in agg.values())
print(f"{m} records ({len(units)} units, {len(drains)} warp drains) over the first CTAs' nodes")
print(f"{'kind/type':14s} {'units':>7s} {'cycles%':>8s} {'mean':>9s} {'max':>9s}")
for key, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{key[0]+'/'+key[1]:14s} {len(v):7d} {100*sum(v)/tot:7.1f}% {np.mean(v):9.0f} {max(v):9d}")
agg = collections.defaultdict(list)
for r in items:
    kind, typ = (int(r[1]) >> 8) & 0xFF, int(r[1]) & 0xFF
    agg[(KN[kind], "q" + TN[typ])].append(int(r[3] - r[2]))
tot = sum(sum(v) for v in agg.values()) or 1
print("queue items (drain phase):")
for key, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{key[0]+'/'+key[1]:14s} {len(v):7d} {100*sum(v)/tot:7.1f}% {np.mean(v):9.0f} {max(v):9d}")
if len(drains):
    d = drains[:, 3] - drains[:, 2]
    print("drain per warp: mean", int(d.mean()), "max", int(d.max()), "queue sizes mean", float(drains[:, 1].mean()))
