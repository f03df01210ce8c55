"""Phase timeline of the multi-CTA node kernel (development build with -DNODE_TRACE).

    python scripts/node_trace.py build     # here: builds paper_2402_14821_b200/libbplb_ntrace.so
    python scripts/node_trace.py run [cfg3|cfg3u]   # GPU box: per-phase spans over the CTAs of one check
"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "paper_2402_14821_b200", "libbplb_ntrace.so")
if sys.argv[1] == "build":
    from paper_2402_14821_b200 import build_native as B

    cmd = ["/usr/local/cuda/bin/nvcc", *B.NVCC_FLAGS, "-DNODE_TRACE", "-shared", "-o", LIB,
           os.path.join(B.CSRC, "bplb_capi.cu"), "-lcudart"]
    subprocess.run(cmd, check=True, capture_output=True)
    print("built", LIB)
    sys.exit(0)

import numpy as np  # noqa: E402

from paper_2402_14821_b200 import _native, workloads as W  # noqa: E402

_native.load_library(LIB)
lib = _native.load_library()
lib.bplb_node_trace.argtypes = [ctypes.c_void_p]
c, w = (W.cfg3u if len(sys.argv) > 2 and sys.argv[2] == "cfg3u" else W.cfg3)()
eng = _native.Engine(0)
buf = np.zeros((1024, 8), dtype=np.uint64)
for _ in range(3):
    r = eng.check(w, c, 2**62, list(range(6)), 0)
lib.bplb_node_trace(buf.ctypes.data)
g = eng.last_path()[1]
t = buf[:g, :7].astype(np.int64)
t0 = t[:, 0].min()
rel = (t - t0) / 1e3
print("lb", r.lb, "path", eng.last_path())
names = ["start", "staged", "stats", "tables+plan", "sweep end", "bucket sort", "prefix+vb2"]
for i, nm in enumerate(names):
    col = rel[:, i]
    print(f"{nm:12s} min {col.min():7.1f}  median {np.median(col):7.1f}  max {col.max():7.1f} us")
