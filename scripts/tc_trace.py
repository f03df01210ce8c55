"""Phase timeline of tc_kernel's CTA 0 (development build with -DTC_TRACE).
    python scripts/tc_trace.py build     # here
    python scripts/tc_trace.py run       # GPU box: cfg2 batch, prints ns offsets"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "paper_2402_14821_b200", "libbplb_tctrace.so")
if sys.argv[1] == "build":
    from paper_2402_14821_b200 import build_native as B

    subprocess.run(["/usr/local/cuda/bin/nvcc", *B.NVCC_FLAGS, "-DTC_TRACE", "-shared", "-o", LIB,
                    os.path.join(B.CSRC, "bplb_capi.cu"), "-lcudart"], check=True, capture_output=True)
    print("built", LIB)
    sys.exit(0)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_14821_b200 import _native, workloads as W  # noqa: E402

lib = _native.load_library(LIB)
lib.bplb_tc_trace.argtypes = [ctypes.c_void_p]
c, k, flat, off = W.cfg2_nodes(10_000)
n = len(off) - 1
d_w = torch.from_numpy(flat.astype(np.uint8)).cuda()
d_off = torch.from_numpy(off).cuda()
lb = torch.empty(n, dtype=torch.int64, device="cuda")
ex = torch.empty(n, dtype=torch.uint8, device="cuda")
eng = _native.Engine(0)
s = torch.cuda.Stream()
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
for i in range(3):
    if os.environ.get("FLUSH"):
        with torch.cuda.stream(s):
            flush.fill_(i)
    eng.check_batch_device(d_w.data_ptr(), d_off.data_ptr(), n, int(np.diff(off).max()), c, 2**62, list(range(6)), 0,
                           lb.data_ptr(), ex.data_ptr(), stream_ptr=s.cuda_stream, wbytes=1)
    s.synchronize()
buf = np.zeros(64 + 256 * 3, dtype=np.uint64)
lib.bplb_tc_trace(buf.ctypes.data)
t0 = int(buf[0])
names = {0: "start", 1: "hist done", 2: "A planes done", 40: "epilogues done", 41: "outputs done"}
for nt in range(8):
    names[3 + 4 * nt] = f"tile {nt} B landed"
    names[4 + 4 * nt] = f"tile {nt} MMA done"
    names[5 + 4 * nt] = f"tile {nt} epilogue (thread 0)"
    names[6 + 4 * nt] = f"tile {nt} all threads"
for i in sorted(names):
    if buf[i]:
        print(f"{names[i]:28s} {(int(buf[i]) - t0) / 1e3:8.2f} us")
print("path", eng.last_path())
cta = buf[64:].reshape(256, 3).astype(np.int64)
g = int(eng.last_path()[1]) if False else int((cta[:, 0] > 0).sum())
cta = cta[:g]
base = cta[:, 0].min()
st, hd, en = (cta[:, 0] - base) / 1e3, (cta[:, 1] - base) / 1e3, (cta[:, 2] - base) / 1e3
print(f"CTAs {g}: start min/median/max {st.min():.2f}/{np.median(st):.2f}/{st.max():.2f} us; "
      f"hist done {np.median(hd):.2f}/{hd.max():.2f}; end median {np.median(en):.2f} max {en.max():.2f} us")
