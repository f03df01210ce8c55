"""Exact knapsack reasoning per bin on the GPU.

Drop-in mirror of the reference's bitset subset-sum DP,
/root/reference/pkg/src/binpack/propagator.py:98-227 -- the same names,
argument meaning, store mutations and ``Wipeout`` messages:

  reachable_sums(store, j)            propagator.py:105-110
  packability(store, j)               :130-133
  knapsack_load_tightening(store, j)  :136-143
  knapsack_item_filter(store, i, j)   :153-168
  knapsack_bin(store, j)              :190-227 (``_knapsack_bin``, what
                                      propagate() calls per dirty bin, :259-260)

plus the batched form the GPU is for, ``knapsack_bins`` -- many independent
bins (e.g. the dirty bins of many search nodes) in one launch of the
``bplb_knapsack_bins`` C entry (include/bplb.h, kernels in
csrc/bplb_knap.cuh).  The paper tried this reasoning on the GPU and kept the
CPU version; here it is exact and batched, with the
store-level decisions applied on the host in the reference's item order.
There is no CPU fallback: the bitsets are computed by libbplb.so only.
"""

from __future__ import annotations

import sys
from typing import NamedTuple

import numpy as np

from . import _native

# per-item action codes (include/bplb.h)
KEEP, REMOVE, COMMIT, WIPEOUT = 0, 1, 2, 3


class KnapsackBatch(NamedTuple):
    status: np.ndarray   # int32 per bin: 0 ok, 1 no reachable load in [lo, hi] (Wipeout)
    lo: np.ndarray       # int32 per bin: tightened lower load bound (input lo when status is 1)
    hi: np.ndarray       # int32 per bin: tightened upper load bound
    action: np.ndarray   # uint8 per open item (CSR positions): KEEP / REMOVE / COMMIT / WIPEOUT
    reach: np.ndarray | None  # uint32 [n_bins, (c + 32) // 32] reachable-load bitsets, when requested


def _engine(engine):
    return engine if engine is not None else _native.default_engine()


def knapsack_bins(c: int, committed, lo, hi, weights_concat, offsets, *, tighten: bool = True,
                  reach_only: bool = False, want_reach: bool = False, engine=None) -> KnapsackBatch:
    """``_knapsack_bin``'s bitset reasoning for many independent bins at once.

    Bin b has committed load ``committed[b]``, interval ``[lo[b], hi[b]]`` and
    open items ``weights_concat[offsets[b]:offsets[b+1]]`` (reference order,
    ``DomainStore.open_items_of_bin``).  ``tighten=False`` filters items on the
    input interval with no committed-load skip (``knapsack_item_filter``);
    ``reach_only`` stops after the reach pass and the tightening."""
    flags = (0 if tighten else _native.KN_NO_TIGHTEN) | (_native.KN_REACH_ONLY if reach_only else 0)
    st, l, h, act, reach = _engine(engine).knapsack_bins(c, committed, lo, hi, weights_concat, offsets, flags,
                                                         want_reach)
    return KnapsackBatch(st, l, h, act, reach)


def _wipeout(store):
    """The reference store module's Wipeout exception (store.py:17)."""
    mod = sys.modules.get(type(store).__module__)
    exc = getattr(mod, "Wipeout", None)
    if exc is None:
        raise TypeError("store does not come from a module defining Wipeout (binpack.store)")
    return exc


def _open(store, j: int):
    items = store.open_items_of_bin(j)
    return items, [store.weights[i] for i in items]


def _one(store, j: int, ws, flags: int, want_reach: bool = False, engine=None):
    return _engine(engine).knapsack_bins(store.c, [store.committed_load[j]], [store.load_lo[j]],
                                         [store.load_hi[j]], ws, [0, len(ws)], flags, want_reach)


def _bits(reach_row: np.ndarray) -> int:
    return int.from_bytes(np.ascontiguousarray(reach_row, dtype="<u4").tobytes(), "little")


def reachable_sums(store, j: int, engine=None) -> int:
    """propagator.py:105-110: committed load plus any subset of bin j's open
    candidates, cut at c, as a Python int bitset."""
    _, ws = _open(store, j)
    if not ws:  # the reference returns the bare base, even above c (:109-110)
        return 1 << store.committed_load[j]
    *_, reach = _one(store, j, ws, _native.KN_REACH_ONLY, True, engine)
    return _bits(reach[0])


def packability(store, j: int, engine=None) -> bool:
    """propagator.py:130-133: some reachable load lies in bin j's interval."""
    _, ws = _open(store, j)
    st, *_ = _one(store, j, ws, _native.KN_REACH_ONLY, False, engine)
    return int(st[0]) == 0


def knapsack_load_tightening(store, j: int, engine=None) -> bool:
    """propagator.py:136-143: clamp bin j's interval to its reachable loads."""
    _, ws = _open(store, j)
    st, lo, hi, _, _ = _one(store, j, ws, _native.KN_REACH_ONLY, False, engine)
    if int(st[0]) == 1:
        raise _wipeout(store)(f"bin {j} has no reachable load in its interval")
    changed = store.set_lo(j, int(lo[0]))
    changed |= store.set_hi(j, int(hi[0]))
    return changed


def _use_avoid_bits(sums_without: int, w: int, lo: int, hi: int) -> tuple[bool, bool]:
    def window(a: int, b: int) -> int:
        return 0 if b < a else ((1 << (b - a + 1)) - 1) << a
    use = bool(sums_without & window(max(0, lo - w), hi - w)) if hi >= w else False
    return use, bool(sums_without & window(lo, hi))


def knapsack_item_filter(store, i: int, j: int, engine=None) -> bool:
    """propagator.py:153-168: remove bin j from item i when no reachable load
    in the interval uses it; commit when none avoids it."""
    items, ws = _open(store, j)
    if i in items:
        pos = items.index(i)
        st, _, _, act, _ = _one(store, j, ws, _native.KN_NO_TIGHTEN, False, engine)
        a = WIPEOUT if int(st[0]) == 1 else int(act[pos])
        use, avoid = a in (KEEP, COMMIT), a in (KEEP, REMOVE)
    else:  # item i is not an open candidate of j: its sums-without are the full reach
        use, avoid = _use_avoid_bits(reachable_sums(store, j, engine), store.weights[i], store.load_lo[j],
                                     store.load_hi[j])
    if not use and not avoid:
        raise _wipeout(store)(f"bin {j} unpackable with or without item {i}")
    if not use:
        return store.remove_bin(i, j)
    if not avoid:
        return store.commit(i, j)
    return False


def knapsack_bin(store, j: int, engine=None) -> bool:
    """``_knapsack_bin`` (propagator.py:190-227): packability, load tightening
    and item filtering for one bin from one GPU pass; the decisions are
    applied to the store in the reference's item order."""
    items, ws = _open(store, j)
    st, lo, hi, act, _ = _one(store, j, ws, 0, False, engine)
    W = _wipeout(store)
    if int(st[0]) == 1:
        raise W(f"bin {j} has no reachable load in its interval")
    changed = store.set_lo(j, int(lo[0]))
    changed |= store.set_hi(j, int(hi[0]))
    for pos, i in enumerate(items):
        if not store.has_candidate(i, j):
            continue
        a = int(act[pos])
        if a == WIPEOUT:
            raise W(f"bin {j} unpackable with or without item {i}")
        if a == REMOVE:
            changed |= store.remove_bin(i, j)
        elif a == COMMIT:
            changed |= store.commit(i, j)
    return changed


def install_knapsack_gpu(propagator_module, engine=None):
    """Route the reference propagator's per-bin knapsack reasoning
    (``propagate`` -> ``_knapsack_bin``, propagator.py:259-260) through the
    GPU without editing the reference.  Returns a function that restores the
    original."""
    orig = propagator_module._knapsack_bin

    def gpu_knapsack_bin(store, j):
        return knapsack_bin(store, j, engine)

    propagator_module._knapsack_bin = gpu_knapsack_bin

    def restore():
        propagator_module._knapsack_bin = orig

    return restore
