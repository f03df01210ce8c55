"""Where the time of one drop-in check (cfg1) goes: the public call, the
engine wrapper, the raw C call, and the kernel span (F_TIMING)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2402_14821_b200 as G
from paper_2402_14821_b200 import _native, workloads as W

import os
c, w = (W.cfg3 if os.environ.get("CFG") == "cfg3" else W.cfg1)()
red = G.ReducedInstance.from_array(c, w)
eng = _native.default_engine()
wa = red.array()


def med(fn, reps=300):
    for _ in range(20):
        fn()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return np.median(ts) * 1e6


kinds = list(range(6))
res = _native.BplbResult()
ks = (ctypes.c_int32 * 6)(*kinds)
f = eng._lib.bplb_check
a_pub = med(lambda: G.lower_bound_seq(red, 2**62))
a_par = med(lambda: G.lower_bound_par(red, 2**62))
a_eng = med(lambda: eng.check(wa, c, 2**62, kinds, 0))
a_raw = med(lambda: f(eng.handle, wa.ctypes.data, len(wa), c, 2**62, ctypes.addressof(ks), 6, 0, ctypes.addressof(res)))
devs = []
def timed():
    f(eng.handle, wa.ctypes.data, len(wa), c, 2**62, ctypes.addressof(ks), 6, _native.F_TIMING, ctypes.addressof(res))
    devs.append(eng.last_device_ms())
a_t = med(timed)
print(f"lower_bound_seq {a_pub:.1f} us | lower_bound_par {a_par:.1f} | Engine.check {a_eng:.1f} | raw C {a_raw:.1f} | "
      f"raw+timing {a_t:.1f} | device span {np.median(devs)*1e3:.1f} us (r={len(wa)}, c={c})")
