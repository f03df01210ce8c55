"""Array-native batched feasibility checks over many search-node states.

No reference counterpart: the reference evaluates one node per engine call
(propagator.py:274-276).  A batch is a CSR of reduced weights
(``weights[offsets[i]:offsets[i+1]]`` = node i) sharing capacity ``c`` and
bin budget ``k``.  One call = one upload + one kernel launch (the paper's
"batch all copies and launches into a single API call").
"""

from __future__ import annotations

from typing import Sequence

import numpy as np

from . import _native
from .bounds import DEFAULT_DFF_ORDER, kind_ids

__all__ = ["lower_bound_batch", "lower_bound_batch_multi", "csr_from_lists"]


def csr_from_lists(nodes: Sequence[Sequence[int]]) -> tuple[np.ndarray, np.ndarray]:
    lens = np.fromiter((len(n) for n in nodes), dtype=np.int64, count=len(nodes))
    off = np.zeros(len(nodes) + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    w = np.fromiter((x for n in nodes for x in n), dtype=np.int32, count=int(off[-1]))
    return w, off


def lower_bound_batch(c: int, weights: np.ndarray, offsets: np.ndarray, k: int,
                      kinds: Sequence = DEFAULT_DFF_ORDER, *, mode: str = "full",
                      want_best: bool = False, dense: bool = False,
                      engine: _native.Engine | None = None):
    """Evaluate the LB collection for every node of a CSR batch on the GPU.

    ``weights`` may be int32, or -- to cut host->device bytes -- uint16
    (c <= 65535) / uint8 (c <= 255); values are validated on the device.

    mode: ``"full"`` (every kind completes; lb = max over kinds),
          ``"seq"`` (kinds in order, early exit once lb > k -- per node
          identical to lower_bound_seq's lb/exceeded_k),
          ``"cancel"`` (units skip once the node's lb > k; decision bit
          identical, lb any computed value > k).
    Returns ``(lb int64[n], exceeded bool[n])`` and, with ``want_best``,
    also ``best int64[n, 6]`` and ``arg_lambda int64[n, 6]`` indexed by kind
    id (MT, RAD2, FS1, CCM1, VB2, BJ1).

    ``dense=True`` evaluates every lambda of the grid (the paper's sweep)
    instead of skipping the lambdas whose integer upper bound provably
    cannot change the outputs (bplb_prune.cuh); both are bit-exact.
    """
    flags = {"full": 0, "seq": _native.F_PHASED, "cancel": _native.F_CANCEL}[mode]
    if dense:
        flags |= _native.F_NOPRUNE
    eng = engine or _native.default_engine()
    return eng.check_batch(weights, offsets, c, k, kind_ids(kinds), flags, want_best=want_best)


def lower_bound_batch_multi(c: int, weights: np.ndarray, offsets: np.ndarray, k: int,
                            kinds: Sequence = DEFAULT_DFF_ORDER, *, devices: Sequence[int] | None = None,
                            mode: str = "full", want_best: bool = False, dense: bool = False,
                            engine: "_native.MultiEngine | None" = None):
    """:func:`lower_bound_batch` over several GPUs in ONE call from one
    process (``bplb_check_batch_multi``): the nodes are sharded over
    ``devices`` (default: every visible GPU) in contiguous ranges balanced by
    item count, checked concurrently, and returned in node order."""
    flags = {"full": 0, "seq": _native.F_PHASED, "cancel": _native.F_CANCEL}[mode]
    if dense:
        flags |= _native.F_NOPRUNE
    if engine is None:
        if devices is None:
            import torch

            devices = list(range(max(1, torch.cuda.device_count())))
        engine = _native.MultiEngine(devices)
        try:
            return engine.check_batch(weights, offsets, c, k, kind_ids(kinds), flags, want_best=want_best)
        finally:
            engine.close()
    return engine.check_batch(weights, offsets, c, k, kind_ids(kinds), flags, want_best=want_best)


def open_marker(dtype) -> int:
    """Assignment value of an open item (all ones of the element type)."""
    return int(np.iinfo(np.dtype(dtype)).max)


def lower_bound_batch_assign(c: int, inst_weights, assign: np.ndarray, n_bins: int, k: int,
                             kinds: Sequence = DEFAULT_DFF_ORDER, *, mode: str = "full",
                             want_best: bool = False, engine: _native.Engine | None = None):
    """The feasibility check of many search nodes given as bin assignments.

    ``assign[node, i]`` is the bin item ``i`` is committed to, or
    ``open_marker(assign.dtype)`` (uint8: 255, uint16: 65535) while it is
    open.  Each node is reduced on the GPU exactly as ``reduce_packing``
    (instances.py:262-282) -- open weights in item order, then positive bin
    loads in bin order; a load above ``c`` raises ValueError -- and checked as
    in :func:`lower_bound_batch` (same modes and outputs)."""
    flags = {"full": 0, "seq": _native.F_PHASED, "cancel": _native.F_CANCEL}[mode]
    eng = engine or _native.default_engine()
    return eng.check_batch_assign(inst_weights, assign, n_bins, c, k, kind_ids(kinds), flags, want_best=want_best)


def reduce_packing_batch(c: int, inst_weights, assign: np.ndarray, n_bins: int,
                         engine: _native.Engine | None = None):
    """Device-side ``reduce_packing`` of a batch of node states: the reduced
    instances as CSR (int32 weights, int64 offsets), reference order."""
    eng = engine or _native.default_engine()
    return eng.reduce_batch(inst_weights, assign, n_bins, c)
