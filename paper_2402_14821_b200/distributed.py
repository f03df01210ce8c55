"""Multi-GPU batched feasibility checks: one process per GPU, search nodes
sharded contiguously, one exchange step (an all-gather of per-node verdicts).

The batched path shards naturally: nodes are independent,
so each rank evaluates ``[rank*N/G, (rank+1)*N/G)`` on its own GPU with no
data-path collective, then the verdicts -- ``lb`` and ``exceeded`` packed
into one int64 per node (``lb | exceeded << 62``) -- are all-gathered so every
rank (in particular the search driver on rank 0) sees the whole batch.  On
NCCL this is one all-gather of 8 bytes per node over NVLink/NVSwitch.

``compute`` is injectable so the sharding and gather logic is testable on
CPU with the gloo backend (tests/test_distributed_gloo.py); the default is
the GPU engine (``lower_bound_batch``).
"""

from __future__ import annotations

from typing import Callable, Sequence

import numpy as np

from .bounds import DEFAULT_DFF_ORDER

__all__ = ["shard_range", "pack_verdicts", "unpack_verdicts", "lower_bound_batch_sharded"]

EXCEEDED_BIT = 62


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous node range of ``rank`` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def pack_verdicts(lb: np.ndarray, exceeded: np.ndarray) -> np.ndarray:
    lb = np.asarray(lb, dtype=np.int64)
    if lb.size and (lb.min() < 0 or lb.max() >= (1 << EXCEEDED_BIT)):
        raise ValueError("lb outside the packable range")
    return lb | (np.asarray(exceeded, dtype=np.int64) << EXCEEDED_BIT)


def unpack_verdicts(v: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    v = np.asarray(v, dtype=np.int64)
    return v & ((1 << EXCEEDED_BIT) - 1), (v >> EXCEEDED_BIT).astype(bool)


def _default_compute(c, w, off, k, kinds):
    from .batch import lower_bound_batch

    return lower_bound_batch(c, w, off, k, kinds)


def lower_bound_batch_sharded(c: int, weights: np.ndarray, offsets: np.ndarray, k: int,
                              kinds: Sequence = DEFAULT_DFF_ORDER, *, group=None,
                              compute: Callable | None = None, device=None):
    """Evaluate a CSR batch across all ranks of ``group``.

    Every rank passes the same full batch (or at least the same offsets);
    each evaluates only its shard, then the packed verdicts are all-gathered.
    Returns ``(lb, exceeded)`` for the whole batch on every rank.
    """
    import torch
    import torch.distributed as dist

    compute = compute or _default_compute
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    offsets = np.asarray(offsets, dtype=np.int64)
    n = len(offsets) - 1
    lo, hi = shard_range(n, world, rank)
    w0, w1 = int(offsets[lo]), int(offsets[hi])
    sub_w = np.ascontiguousarray(np.asarray(weights)[w0:w1])
    sub_off = offsets[lo:hi + 1] - w0
    lb, ex = compute(c, sub_w, sub_off, k, kinds)
    packed = pack_verdicts(lb, ex)
    # equal-size buffers for all_gather (shards differ by at most one node)
    width = -(-n // world)
    buf = np.zeros(width, dtype=np.int64)
    buf[:hi - lo] = packed
    backend = dist.get_backend(group)
    dev = torch.device("cpu")
    if backend == "nccl":
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    t = torch.from_numpy(buf).to(dev)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    out = np.empty(n, dtype=np.int64)
    for r_, part in enumerate(parts):
        a, b = shard_range(n, world, r_)
        out[a:b] = part[:b - a].cpu().numpy()
    return unpack_verdicts(out)
