import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2402_14821_b200 import _native, workloads as W
mode = sys.argv[1]
c, k, w = W.cfg5_instance()
if mode == "gen":
    import torch
    flat, off = W.gen_nodes_host(w, c, k, W.CFG5_SEED, 300)
    df, do = W.gen_nodes_device(w, c, k, W.CFG5_SEED, 300, device="cuda:0")
    print("off equal", np.array_equal(do.cpu().numpy(), off), "w equal", np.array_equal(df.cpu().numpy()[:off[-1]], flat))
    d = df.cpu().numpy(); print("device min/max", d.min(), d.max(), "host min/max", flat.min(), flat.max())
    sys.exit(0)
flat, off = W.gen_nodes_host(w, c, k, W.CFG5_SEED, int(sys.argv[2]))
eng = _native.Engine(0)
fl = {"key": 0, "phased": _native.F_PHASED, "lb": 0}[mode]
print(eng.check_batch(flat, off, c, 2**62 if mode != "phased" else k, list(range(6)), fl, want_best=(mode == "key"))[0][:8])
