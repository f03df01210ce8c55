"""Quick wall-clock timing of the drop-in API on the configs (dev aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2402_14821_b200 as G
from paper_2402_14821_b200 import workloads as W, _native

eng = _native.default_engine()

def t(fn, reps):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e3, min(ts) * 1e3

c, w = W.cfg1(); red = G.ReducedInstance.from_array(c, w)
print("cfg1 seq ms", t(lambda: G.lower_bound_seq(red, 2**62), 200))
print("cfg1 par ms", t(lambda: G.lower_bound_par(red, 2**62), 200))
c, k, flat, off = W.cfg2_nodes(10000)
print("cfg2 full ms", t(lambda: G.lower_bound_batch(c, flat, off, 2**62), 20))
print("cfg2 seq ms", t(lambda: G.lower_bound_batch(c, flat, off, k, mode='seq'), 20))
for name, gen in (("cfg3", W.cfg3), ("cfg3u", W.cfg3u), ("cfg4", W.cfg4)):
    c, w = gen(); red = G.ReducedInstance.from_array(c, w)
    print(name, "par ms", t(lambda: G.lower_bound_par(red, 2**62, cancellation=False), 10))
    print(name, "seq ms", t(lambda: G.lower_bound_seq(red, 2**62), 5))
c, k, flat, off = W.cfg5_nodes(2048)
print("cfg5 2048 nodes full ms", t(lambda: G.lower_bound_batch(c, flat, off, 2**62), 3))
print("launches", eng.launch_count())
