"""Summarise a per-warp tab_kernel globaltimer trace (debug builds that dump
[grid, nw, P] + [cta][warp][16] stamps: t0, table ready, end of each tile)."""
import numpy as np, os, sys
f = sys.argv[1]
raw = np.fromfile(f, dtype=np.int64)
pos = 0; k = 0
while pos < len(raw):
    g, nw, P = raw[pos:pos+3]; pos += 3
    a = raw[pos:pos + g*nw*16].reshape(g, nw, 16).astype(np.float64); pos += g*nw*16
    k += 1
    if k < 3: continue
    t0 = a[:, :, 0][a[:, :, 0] > 0].min()
    a = np.where(a > 0, (a - t0) / 1e3, np.nan)
    ntile = np.sum(~np.isnan(a[:, :, 2:]), axis=2)
    end = np.nanmax(a, axis=2)
    print(f"launch {k}: grid {g} nw {nw} P {P}")
    print(f"  start {np.nanmin(a[:,:,0]):.2f}..{np.nanmax(a[:,:,0]):.2f} us; table ready {np.nanmin(a[:,:,1]):.2f}..{np.nanmax(a[:,:,1]):.2f}")
    print(f"  tiles/warp hist {np.bincount(ntile.ravel())}; warp end min/med/max {np.nanmin(end):.2f}/{np.nanmedian(end):.2f}/{np.nanmax(end):.2f}")
    d = np.diff(a[:, :, 1:], axis=2)
    print(f"  per-tile us: median {np.nanmedian(d):.2f}, first tile median {np.nanmedian(d[:,:,0]):.2f}, p10 {np.nanpercentile(d,10):.2f} p90 {np.nanpercentile(d,90):.2f}")
    for ti in range(5):
        col = d[:, :, ti]
        print(f"   tile#{ti}: n={np.sum(~np.isnan(col))} median {np.nanmedian(col):.2f} end med {np.nanmedian(a[:,:,2+ti]):.2f} max {np.nanmax(a[:,:,2+ti]):.2f}")
