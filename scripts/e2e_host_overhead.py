"""Host-side overhead of the e2e batch call: Python wrapper vs the raw C
call with pre-built ctypes arguments vs the device-timed span (F_TIMING)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2402_14821_b200 import _native, workloads as W

c, k, flat, off = W.cfg2_nodes(10_000)
eng = _native.Engine(0)
h_w = torch.from_numpy(flat.astype(np.uint8)).pin_memory().numpy()
h_off = torch.from_numpy(off).pin_memory().numpy()
n = len(off) - 1
h_lb = torch.empty(n, dtype=torch.int64).pin_memory().numpy()
h_ex = torch.empty(n, dtype=torch.uint8).pin_memory().numpy()
ks = np.arange(6, dtype=np.int32)
lib = eng._lib
args = [eng.handle, h_w.ctypes.data, 1, h_off.ctypes.data, n, c, 2**62, ks.ctypes.data, 6, 0,
        h_lb.ctypes.data, h_ex.ctypes.data, None, None]
f = lib.bplb_check_batch_ex
for _ in range(10):
    eng.check_batch(h_w, h_off, c, 2**62, list(range(6)), 0, out=(h_lb, h_ex))


def med(fn, reps=50):
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return np.median(ts) * 1e6


raw = med(lambda: f(*args))
wrap = med(lambda: eng.check_batch(h_w, h_off, c, 2**62, list(range(6)), 0, out=(h_lb, h_ex)))
raw = min(raw, med(lambda: f(*args)))
args[9] = _native.F_TIMING
devs = []
def timed():
    f(*args)
    devs.append(eng.last_device_ms())
rawt = med(timed)
print(f"wrapper {wrap:.1f} us, raw ctypes {raw:.1f} us, raw+timing {rawt:.1f} us, device span {np.median(devs)*1e3:.1f} us")
