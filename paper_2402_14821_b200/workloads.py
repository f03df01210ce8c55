"""Synthetic workloads of BASELINE.json's configs (definitions: SURVEY.md 8(d)).

  cfg1  Falkenauer-U-shaped: r=120, w ~ U{20..100}, c=150 (rng(0))
  cfg2  Scholl-1-shaped: n=500, w ~ U{20..100}, c=150 (seed 0); search-node
        residual states (seed 1), bins k = L2(root) + 2
  cfg3  AI/ANI-shaped: n=1000, c=1e5, triplets in (c/4, c/2) summing to c
        (333 triplets + 1 extra item, seed 0); cfg3u: U{c/4+1..c/2-1} variant
  cfg4  large: r=1e5, w ~ U{1..1e6}, c=1e6 (rng(0))
  cfg5  search-node states of the cfg3 instance (seed 2), k = 334 bins

Search-node generator (one node): draw depth d ~ U{0..n}; the d heaviest
items (stable by index) are each committed to a uniformly random bin among
those with load + w <= c (or stay open if none fits); the reduced instance is
the open weights in item order followed by the positive bin loads in bin
order -- exactly the layout of reduce_packing (instances.py:262-282).
Nodes are generated in independent blocks (seeded by (seed, block)) so a
rank can generate only its own shard.

All workload code is data generation, not the bound path.
"""

from __future__ import annotations

import os

import numpy as np

__all__ = ["cfg1", "cfg2_instance", "cfg3", "cfg3u", "cfg4", "node_batch", "l2_host", "CONFIGS"]

BLOCK = 1024


def cfg1() -> tuple[int, np.ndarray]:
    return 150, np.random.default_rng(0).integers(20, 101, 120).astype(np.int32)


def cfg2_instance() -> tuple[int, np.ndarray]:
    return 150, np.random.default_rng(0).integers(20, 101, 500).astype(np.int32)


def cfg3(seed: int = 0, n: int = 1000, c: int = 100_000) -> tuple[int, np.ndarray]:
    rng = np.random.default_rng(seed)
    q = c // 4
    items = []
    for _ in range(n // 3):
        a = int(rng.integers(q + 2, c // 2 - 1))
        b_lo = max(q + 1, c // 2 - a + 1)
        b_hi = min(c // 2 - 1, 3 * q - a - 1)
        b = int(rng.integers(b_lo, b_hi + 1))
        items += [a, b, c - a - b]
    while len(items) < n:
        items.append(int(rng.integers(q + 1, c // 2)))
    w = np.array(items, dtype=np.int32)
    rng.shuffle(w)
    return c, w


def cfg3u(seed: int = 0, n: int = 1000, c: int = 100_000) -> tuple[int, np.ndarray]:
    rng = np.random.default_rng(seed)
    return c, rng.integers(c // 4 + 1, c // 2, n).astype(np.int32)


def cfg4() -> tuple[int, np.ndarray]:
    return 1_000_000, np.random.default_rng(0).integers(1, 10**6 + 1, 10**5).astype(np.int32)


def l2_host(c: int, w: np.ndarray) -> int:
    """Martello-Toth L2 of a root instance (generator helper only: it picks
    the bin count of the synthetic search nodes).  max over lambda of the
    f_MT bound via prefix sums."""
    w = np.asarray(w, dtype=np.int64)
    if w.size == 0:
        return 0
    cnt = np.bincount(w, minlength=c + 1)
    n_le = np.concatenate([[0], np.cumsum(cnt)])
    w_le = np.concatenate([[0], np.cumsum(cnt * np.arange(c + 1))])
    lam = np.arange(0, (c + 1) // 2 + 1, dtype=np.int64)
    idx = lambda v: np.clip(v, -1, c) + 1  # noqa: E731
    s = c * (w.size - n_le[idx(c - lam)]) + w_le[idx(c - lam)] - w_le[idx(lam - 1)]
    return int(((s + c - 1) // c).max())


def _node_block(w: np.ndarray, c: int, k: int, rng: np.random.Generator, nb: int):
    n = w.size
    order = np.argsort(-w.astype(np.int64), kind="stable")
    ws = w[order].astype(np.int64)
    d = rng.integers(0, n + 1, nb)
    loads = np.zeros((nb, k), dtype=np.int64)
    assign_sorted = np.full((nb, n), -1, dtype=np.int64)
    for i in range(n):
        rows = np.nonzero(d > i)[0]
        if rows.size == 0:
            break
        fits = loads[rows] + ws[i] <= c
        cnt = fits.sum(axis=1)
        pick = (rng.random(rows.size) * cnt).astype(np.int64)
        cs = np.cumsum(fits, axis=1)
        j = np.argmax(cs > pick[:, None], axis=1)
        ok = cnt > 0
        rr, jj = rows[ok], j[ok]
        loads[rr, jj] += ws[i]
        assign_sorted[rr, i] = jj
    assign = np.empty_like(assign_sorted)
    assign[:, order] = assign_sorted
    out = []
    for b in range(nb):
        open_w = w[assign[b] < 0]
        ld = loads[b][loads[b] > 0]
        out.append(np.concatenate([open_w.astype(np.int64), ld]).astype(np.int32))
    return out, assign


def node_batch(w: np.ndarray, c: int, k: int, n_nodes: int, seed: int, first_node: int = 0):
    """CSR (weights int32, offsets int64) of search-node states
    [first_node, first_node + n_nodes) of the generator stream ``seed``."""
    nodes = []
    b0 = first_node // BLOCK
    b1 = (first_node + n_nodes + BLOCK - 1) // BLOCK
    for b in range(b0, b1):
        rng = np.random.default_rng([seed, b])
        blk, _ = _node_block(w, c, k, rng, BLOCK)
        lo = max(first_node, b * BLOCK) - b * BLOCK
        hi = min(first_node + n_nodes, (b + 1) * BLOCK) - b * BLOCK
        nodes.extend(blk[lo:hi])
    lens = np.fromiter((x.size for x in nodes), dtype=np.int64, count=len(nodes))
    off = np.zeros(len(nodes) + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    flat = np.concatenate(nodes) if nodes else np.zeros(0, dtype=np.int32)
    return flat.astype(np.int32), off


def node_assignments(w: np.ndarray, c: int, k: int, n_nodes: int, seed: int, first_node: int = 0):
    """The same node states as :func:`node_batch`, as bin assignments
    (uint8 when k < 255, else uint16; open items = all ones): the input of
    the device-side reduction (``lower_bound_batch_assign``)."""
    dt = np.uint8 if k < 255 else np.uint16
    openv = np.iinfo(dt).max
    rows = []
    b0 = first_node // BLOCK
    b1 = (first_node + n_nodes + BLOCK - 1) // BLOCK
    for b in range(b0, b1):
        rng = np.random.default_rng([seed, b])
        _, assign = _node_block(w, c, k, rng, BLOCK)
        lo = max(first_node, b * BLOCK) - b * BLOCK
        hi = min(first_node + n_nodes, (b + 1) * BLOCK) - b * BLOCK
        rows.append(assign[lo:hi])
    a = np.concatenate(rows) if rows else np.zeros((0, w.size), dtype=np.int64)
    return np.where(a < 0, openv, a).astype(dt)


def cfg2_assignments(n_nodes: int = 10_000, first_node: int = 0):
    """cfg2 search nodes as (c, k, instance weights, bin assignments)."""
    c, w = cfg2_instance()
    k = l2_host(c, w) + 2
    return c, k, w, node_assignments(w, c, k, n_nodes, seed=1, first_node=first_node)


def cfg2_nodes(n_nodes: int = 10_000, first_node: int = 0):
    c, w = cfg2_instance()
    k = l2_host(c, w) + 2
    flat, off = node_batch(w, c, k, n_nodes, seed=1, first_node=first_node)
    return c, k, flat, off


def cfg5_nodes(n_nodes: int = 1_000_000, first_node: int = 0):
    c, w = cfg3()
    k = 334
    flat, off = node_batch(w, c, k, n_nodes, seed=2, first_node=first_node)
    return c, k, flat, off


CONFIGS = {
    "cfg1": "Falkenauer-U-shaped synthetic instance: 120 items, sizes U[20,100], capacity 150",
    "cfg2": "Scholl-1-shaped instance: 500 items, capacity 150, batch of 10k search-node residual states",
    "cfg3": "AI/ANI-shaped hard instance: 1000 items, capacity 1e5",
    "cfg4": "large instance: 1e5 items, capacity 1e6, single check",
    "cfg5": "batched search-node sweep of the 1000-item cfg3 instance",
}


# ---------------------------------------------------------------------------
# Native node generator (csrc/bplb_gen.cu -> libbplb_gen.so): the same
# search-node definition as above with a splitmix64 stream per node keyed by
# (seed, node), identical on the host and on the device, fast enough for the
# 10^6-node batches of cfg5 (the numpy generator above needs minutes).
# ---------------------------------------------------------------------------

GEN_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libbplb_gen.so")
CFG5_SEED = 5  # node stream of the cfg5 headline batch (native generator)
_gen = None


def _gen_lib():
    global _gen
    if _gen is None:
        import ctypes

        if not os.path.exists(GEN_LIB_PATH):
            raise RuntimeError(f"{GEN_LIB_PATH} missing: build with paper_2402_14821_b200/build_native.py")
        lib = ctypes.CDLL(GEN_LIB_PATH)
        vp, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
        lib.bplbgen_nodes_host.argtypes = [vp, i32, vp, i64, i32, u64, i64, i64, vp, vp, vp, i32]
        lib.bplbgen_sizes_device.argtypes = [vp, i32, vp, i64, i32, u64, i64, i64, vp, vp]
        lib.bplbgen_fill_device.argtypes = [vp, i32, vp, i64, i32, u64, i64, i64, vp, vp, vp, vp]
        for f in (lib.bplbgen_nodes_host, lib.bplbgen_sizes_device, lib.bplbgen_fill_device):
            f.restype = ctypes.c_int
        _gen = lib
    return _gen


def heavy_order(w: np.ndarray) -> np.ndarray:
    """Item indices by weight descending, stable by index (the commit order)."""
    return np.argsort(-np.asarray(w, dtype=np.int64), kind="stable").astype(np.int32)


def gen_nodes_host(w: np.ndarray, c: int, k: int, seed: int, n_nodes: int, first_node: int = 0,
                   want_assign: bool = False, threads: int | None = None):
    """CSR (int32 weights, int64 offsets) of native-generator nodes
    [first_node, first_node + n_nodes); with ``want_assign`` also the bin
    assignments (uint16, 0xFFFF = open) of the same nodes."""
    w = np.ascontiguousarray(w, dtype=np.int32)
    order = heavy_order(w)
    off = np.zeros(n_nodes + 1, dtype=np.int64)
    nt = threads or max(1, min(32, os.cpu_count() or 1))
    lib = _gen_lib()
    rc = lib.bplbgen_nodes_host(w.ctypes.data, w.size, order.ctypes.data, c, k, seed, first_node, n_nodes,
                                off.ctypes.data, None, None, nt)
    if rc:
        raise ValueError("bad generator arguments")
    flat = np.empty(max(1, int(off[-1])), dtype=np.int32)
    asg = np.empty((n_nodes, w.size), dtype=np.uint16) if want_assign else None
    rc = lib.bplbgen_nodes_host(w.ctypes.data, w.size, order.ctypes.data, c, k, seed, first_node, n_nodes,
                                off.ctypes.data, flat.ctypes.data, asg.ctypes.data if want_assign else None, nt)
    if rc:
        raise ValueError("bad generator arguments")
    flat = flat[:off[-1]]
    return (flat, off, asg) if want_assign else (flat, off)


def gen_nodes_device(w: np.ndarray, c: int, k: int, seed: int, n_nodes: int, first_node: int = 0,
                     device=None, want_assign: bool = False):
    """The same nodes generated on the GPU: torch tensors (weights int32,
    offsets int64[, assignments uint16 as int16 storage]) on ``device``."""
    import torch

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    wt = torch.as_tensor(np.ascontiguousarray(w, dtype=np.int32), device=dev)
    order = torch.as_tensor(heavy_order(w), device=dev)
    off = torch.empty(n_nodes + 1, dtype=torch.int64, device=dev)
    s = torch.cuda.current_stream(dev).cuda_stream
    lib = _gen_lib()
    with torch.cuda.device(dev):
        rc = lib.bplbgen_sizes_device(wt.data_ptr(), wt.numel(), order.data_ptr(), c, k, seed, first_node, n_nodes,
                                      off.data_ptr(), s)
        if rc:
            raise RuntimeError(f"bplbgen_sizes_device failed ({rc})")
        total = int(off[-1].item())
        flat = torch.empty(max(1, total), dtype=torch.int32, device=dev)
        asg = torch.empty((n_nodes, wt.numel()), dtype=torch.int16, device=dev) if want_assign else None
        rc = lib.bplbgen_fill_device(wt.data_ptr(), wt.numel(), order.data_ptr(), c, k, seed, first_node, n_nodes,
                                     off.data_ptr(), flat.data_ptr(), asg.data_ptr() if want_assign else None, s)
        if rc:
            raise RuntimeError(f"bplbgen_fill_device failed ({rc})")
    return (flat, off, asg) if want_assign else (flat, off)


def cfg5_instance():
    """cfg5: the cfg3 instance (1000 items, c = 1e5) and k = 334 bins."""
    c, w = cfg3()
    return c, 334, w


def knapsack_bins_workload(which: str, n_bins: int, seed: int = 21):
    """Synthetic per-bin knapsack states (SURVEY.md 8(f)4 measurement): the
    dirty bins a propagate() pass hands to _knapsack_bin
    (propagator.py:259-260), drawn from a BASELINE instance's items.

    which = "cfg2": the Scholl-1-shaped instance (c = 150, warp-per-bin path);
            "cfg5": the AI/ANI-shaped 1000-item instance (c = 10^5, CTA path).
    Per bin: 8..64 open candidate items, a committed load of a few items
    (<= c), and an interval above the committed load (so the item filter
    runs, propagator.py:208-212): lo in (committed, c], hi = lo + up to c/8.
    Returns (c, committed, lo, hi, weights_concat int32, offsets int64)."""
    if which == "cfg2":
        c, inst = cfg2_instance()
    elif which == "cfg5":
        c, _, inst = cfg5_instance()
    else:
        raise ValueError(which)
    inst = np.asarray(inst, dtype=np.int64)
    rng = np.random.default_rng(seed)
    m = rng.integers(8, 65, n_bins)
    off = np.concatenate([[0], np.cumsum(m)]).astype(np.int64)
    w = inst[rng.integers(0, len(inst), int(off[-1]))].astype(np.int32)
    k_c = rng.integers(0, 4, n_bins)
    cl = np.zeros(n_bins, np.int64)
    for t in range(4):
        add = inst[rng.integers(0, len(inst), n_bins)]
        sel = (k_c > t) & (cl + add <= c)
        cl[sel] += add[sel]
    lo = np.minimum(c, cl + 1 + (rng.random(n_bins) * (c - cl)).astype(np.int64))
    hi = np.minimum(c, lo + (rng.random(n_bins) * (c // 8 + 1)).astype(np.int64))
    return c, cl, lo, hi, w, off


def knapsack_shift_count(m: int) -> int:
    """Bitset shifts _knapsack_bin performs for m open items when the item
    filter runs: m for the reach pass plus m per level of the exclusion-sum
    recursion (propagator.py:171-187, 201-202)."""
    def rec(n: int) -> int:
        return 0 if n <= 1 else n + rec(n // 2) + rec(n - n // 2)
    return m + rec(m)
