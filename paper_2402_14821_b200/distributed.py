"""Multi-GPU batched feasibility checks: one process per GPU, search nodes
sharded contiguously, one exchange step (an all-gather of per-node verdicts).

The batched path shards naturally: nodes are independent,
so rank g evaluates ``[g*N/G, (g+1)*N/G)`` on its own GPU with no data-path
collective.  Every rank holds only its own shard (host or device); the
verdicts -- ``lb`` and ``exceeded`` packed into one int64 per node
(``lb | exceeded << 62``) -- are all-gathered so every rank (in particular
the search driver on rank 0) sees the whole batch.  On NCCL the packing and
the all-gather run on the GPU (8 bytes per node over NVLink/NVSwitch); the
only host copy is the final read of the gathered verdicts.

The per-shard ``compute`` is injectable so the sharding, packing and gather
logic -- the exact code path bench.py times -- is testable on CPU with the
gloo backend (tests/test_distributed_gloo.py).  The default compute is the
GPU engine of this rank's device (``LOCAL_RANK`` / the current CUDA device).
"""

from __future__ import annotations

import os
from typing import Callable, Sequence

import numpy as np

from .bounds import DEFAULT_DFF_ORDER

__all__ = ["shard_range", "pack_verdicts", "unpack_verdicts", "lower_bound_batch_sharded",
           "check_shard_device", "rank_engine"]

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


def _kind_ids(kinds) -> list[int]:
    from .bounds import DffKind

    return [int(k.value) if isinstance(k, DffKind) else int(k) for k in kinds]


def rank_engine(device=None):
    """The engine of this rank's GPU: ``device`` if given, else LOCAL_RANK
    (torchrun), else the current CUDA device."""
    from . import _native

    if device is None:
        if "LOCAL_RANK" in os.environ:
            device = int(os.environ["LOCAL_RANK"])
        else:
            import torch

            device = torch.cuda.current_device()
    idx = device.index if hasattr(device, "index") else int(device)
    return _native.default_engine(idx)


def check_shard_device(engine, d_w, d_off, n: int, max_r: int, c: int, k: int, kinds, flags: int,
                       d_lb, d_ex, stream, *, group=None, gathered=None, wbytes: int = 4):
    """Device-resident step: check this rank's shard (CSR already in HBM)
    on ``stream``; with ``gathered`` (a [world * ceil(N/world)] int64 CUDA
    tensor), pack the verdicts on the device and all-gather them into it.
    Nothing is copied to the host."""
    import torch

    engine.check_batch_device(d_w.data_ptr(), d_off.data_ptr(), n, max_r, c, k, _kind_ids(kinds), flags,
                              d_lb.data_ptr(), d_ex.data_ptr(), stream_ptr=stream.cuda_stream, wbytes=wbytes)
    if gathered is None:
        return None
    import torch.distributed as dist

    width = gathered.numel() // dist.get_world_size(group)
    with torch.cuda.stream(stream):
        verdict = torch.zeros(width, dtype=torch.int64, device=d_lb.device)
        verdict[:n] = d_lb[:n] | (d_ex[:n].to(torch.int64) << EXCEEDED_BIT)
        dist.all_gather_into_tensor(gathered, verdict, group=group)
    return gathered


def _default_compute(c, w, off, k, kinds, engine=None):
    """This rank's shard on this rank's GPU (the public batch path)."""
    from .batch import lower_bound_batch

    return lower_bound_batch(c, w, off, k, kinds, engine=engine or rank_engine())


def lower_bound_batch_sharded(c: int, weights: np.ndarray, offsets: np.ndarray, k: int,
                              kinds: Sequence = DEFAULT_DFF_ORDER, *, n_total: int | None = None,
                              group=None, compute: Callable | None = None, engine=None):
    """Check this rank's SHARD of a CSR batch and all-gather the verdicts.

    ``weights`` / ``offsets`` are the rank's own nodes ``shard_range(n_total,
    world, rank)`` (offsets rebased to 0; pinned host arrays go to the GPU
    without a staging copy).  ``n_total`` is the whole batch size (default:
    the sum of the shard sizes, from one small all-reduce).  Returns
    ``(lb, exceeded)`` for the WHOLE batch, in node order, on every rank.
    """
    import torch
    import torch.distributed as dist

    offsets = np.asarray(offsets, dtype=np.int64)
    n = len(offsets) - 1
    if not (dist.is_available() and dist.is_initialized()):  # one process: the whole batch is the shard
        if n_total is not None and n_total != n:
            raise ValueError(f"single process holds {n} nodes, n_total is {n_total}")
        if compute is not None:
            return compute(c, weights, offsets, k, kinds)
        return _default_compute(c, weights, offsets, k, kinds, engine)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    backend = dist.get_backend(group)
    dev = torch.device("cpu")
    if backend == "nccl":
        if engine is None:
            engine = rank_engine()
        dev = torch.device("cuda", engine.device)
    if n_total is None:
        t = torch.tensor([n], dtype=torch.int64, device=dev)
        dist.all_reduce(t, group=group)
        n_total = int(t.item())
    lo, hi = shard_range(n_total, world, rank)
    if hi - lo != n:
        raise ValueError(f"rank {rank} holds {n} nodes, its shard of {n_total} is [{lo}, {hi})")
    if compute is not None:
        lb, ex = compute(c, weights, offsets, k, kinds)
    else:
        lb, ex = _default_compute(c, weights, offsets, k, kinds, engine)
    # equal-size buffers for the all-gather (shards differ by at most one node)
    width = -(-n_total // world)
    buf = torch.zeros(width, dtype=torch.int64, device=dev)
    if n:
        buf[:n] = torch.from_numpy(pack_verdicts(lb, ex)).to(dev, non_blocking=True)
    parts = torch.empty(world * width, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(parts, buf, group=group)
    host = parts.cpu().numpy().reshape(world, width)
    out = np.empty(n_total, dtype=np.int64)
    for r_ in range(world):
        a, b = shard_range(n_total, world, r_)
        out[a:b] = host[r_, :b - a]
    return unpack_verdicts(out)
