"""Summarise tab_kernel globaltimer traces written by a TAB_TRACE build of
libbplb.so (nvcc ... -DTAB_TRACE; load it with BPLB_LIB=... and set
BPLB_TAB_TRACE=<file>).  Per launch the file holds [grid, nw, P, ntiles, 0],
[cta][warp][16] stamps (start, table ready, end of each tile) and [tile]
publish stamps of the histogram pass.  Times are µs from the first stamp."""
import sys

import numpy as np

raw = np.fromfile(sys.argv[1], dtype=np.int64)
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 2
pos = k = 0
while pos < len(raw):
    g, nw, P, nt, _ = raw[pos:pos + 5]
    pos += 5
    a = raw[pos:pos + g * nw * 16].reshape(g, nw, 16).astype(np.float64)
    pos += g * nw * 16
    pub = raw[pos:pos + nt].astype(np.float64)
    pos += nt
    k += 1
    if k <= skip:
        continue
    t0 = min(a[:, :, 0][a[:, :, 0] > 0].min(), pub[pub > 0].min() if (pub > 0).any() else np.inf)
    a = np.where(a > 0, (a - t0) / 1e3, np.nan)
    pub = np.where(pub > 0, (pub - t0) / 1e3, np.nan)
    ntile = np.sum(~np.isnan(a[:, :, 2:]), axis=2)
    end = np.nanmax(a, axis=2)
    print(f"launch {k}: grid {g} nw {nw} P {P} tiles {nt}")
    print(f"  tab start {np.nanmin(a[:, :, 0]):.2f}..{np.nanmax(a[:, :, 0]):.2f} us; table ready "
          f"{np.nanmin(a[:, :, 1]):.2f}..{np.nanmax(a[:, :, 1]):.2f}")
    print(f"  tiles published: first {np.nanmin(pub):.2f}, median {np.nanmedian(pub):.2f}, last {np.nanmax(pub):.2f} us")
    q = np.nanpercentile(pub, [10, 25, 50, 75, 90])
    print("  publish p10/25/50/75/90: " + " ".join(f"{x:.2f}" for x in q))
    print(f"  tiles/warp {np.bincount(ntile.ravel())}; warp end min/med/max "
          f"{np.nanmin(end):.2f}/{np.nanmedian(end):.2f}/{np.nanmax(end):.2f}")
    d = np.diff(a[:, :, 1:], axis=2)
    for ti in range(6):
        col = d[:, :, ti]
        if np.all(np.isnan(col)):
            break
        print(f"   tile#{ti}: n={np.sum(~np.isnan(col))} dur median {np.nanmedian(col):.2f} "
              f"end med {np.nanmedian(a[:, :, 2 + ti]):.2f} max {np.nanmax(a[:, :, 2 + ti]):.2f}")
