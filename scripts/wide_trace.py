"""Per-unit trace of the grid-wide path (development build with -DWIDE_TRACE).

    python scripts/wide_trace.py build     # here: builds paper_2402_14821_b200/libbplb_wtrace.so
    python scripts/wide_trace.py run [cfg4|cfg3]  # GPU box: one warm check, summary per (launch, kind, type)
"""
import collections
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "paper_2402_14821_b200", "libbplb_wtrace.so")
KN = ["MT", "RAD2", "FS1", "CCM1", "VB2", "BJ1"]
TN = ["LOOKUP", "MOD", "DIV", "WLOOK", "HSL"]

if sys.argv[1] == "build":
    from paper_2402_14821_b200 import build_native as B

    cmd = ["/usr/local/cuda/bin/nvcc", *B.NVCC_FLAGS, "-DWIDE_TRACE", "-shared", "-o", LIB,
           os.path.join(B.CSRC, "bplb_capi.cu"), "-lcudart"]
    subprocess.run(cmd, check=True, capture_output=True)
    print("built", LIB)
    sys.exit(0)

import faulthandler  # noqa: E402

import numpy as np  # noqa: E402

if os.environ.get("WT_TIMEOUT"):
    faulthandler.dump_traceback_later(int(os.environ["WT_TIMEOUT"]), exit=True)

from paper_2402_14821_b200 import _native, workloads as W  # noqa: E402

which = sys.argv[2] if len(sys.argv) > 2 else "cfg4"
_native.load_library(LIB)
lib = _native.load_library()
lib.bplb_wide_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
c, w = W.cfg4() if which == "cfg4" else W.cfg3()
eng = _native.Engine(0)
buf = np.zeros((1 << 18, 4), dtype=np.int64)
print("engine up", flush=True)
for it in range(2):
    lib.bplb_wide_trace(buf.ctypes.data, 1 << 18)  # reset
    print("reset", flush=True)
    r = eng.check(w, c, 2**62, list(range(6)), int(os.environ.get("FLAGS", "0")))
    print("checked", r.lb, flush=True)
    m = lib.bplb_wide_trace(buf.ctypes.data, 1 << 18)
print("lb", r.lb, "per_dff", r.per_dff if hasattr(r, "per_dff") else "", "path", eng.last_path(), "records", m)
rec = buf[:m]
x = rec[:, 0]
seg = x & 0xFF
part = (x >> 8) & 0xFF
sm = (x >> 16) & 0xFFFF
kind = (x >> 32) & 0xFF
typ = (x >> 40) & 0xFF
t0, t1 = rec[:, 2], rec[:, 3]
for p in sorted(set(part.tolist())):
    sel = part == p
    T0, T1 = t0[sel].min(), t1[sel].max()
    print(f"\n== launch part {p}: {sel.sum()} units, span {(T1 - T0) / 1e3:.1f} us")
    # per-SM busy time
    busy = collections.defaultdict(int)
    for s_, a, b in zip(sm[sel], t0[sel], t1[sel]):
        busy[int(s_)] += int(b - a)
    bs = np.array(list(busy.values())) / 1e3
    print(f"   per-SM summed warp-busy us: mean {bs.mean():.1f} max {bs.max():.1f} (SMs {len(bs)})")
    agg = collections.defaultdict(lambda: [0, 0, 0, 2**62, 0])
    for sg, k, t, a, b in zip(seg[sel], kind[sel], typ[sel], t0[sel], t1[sel]):
        e = agg[(int(sg), int(k), int(t))]
        d = int(b - a)
        e[0] += 1
        e[1] += d
        e[2] = max(e[2], d)
        e[3] = min(e[3], int(a))
        e[4] = max(e[4], int(b))
    for (sg, k, t), e in sorted(agg.items()):
        print(f"   seg {sg:2d} {KN[k]:5s} {TN[t] if t < 5 else t:7s} units {e[0]:7d} sum {e[1] / 1e3:10.1f} us "
              f"max {e[2] / 1e3:8.1f} us  window [{(e[3] - T0) / 1e3:8.1f}, {(e[4] - T0) / 1e3:8.1f}] us")
