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
           "check_shard_device", "rank_engine", "lambda_slices", "lower_bound_lambda_split"]

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


# ---------------------------------------------------------------------------
# One large check split over ranks by lambda (optional row)
# ---------------------------------------------------------------------------
def lambda_slices(c: int, red, kinds, world: int, rank: int):
    """Per-kind lambda slice ``(lo[6], hi[6])`` of ``rank``: each kind's range
    (``lambda_range``, VB2 cap included) cut into ``world`` contiguous
    near-equal parts; kinds outside ``kinds`` are empty (hi < lo).  Also
    returns the full ranges ``(dlo[6], dhi[6])``."""
    from .bounds import DEFAULT_DFF_ORDER as ORDER, lambda_range, resolve_kinds

    kinds_t, ids = resolve_kinds(kinds)
    dlo = np.zeros(6, dtype=np.int64)
    dhi = np.full(6, -1, dtype=np.int64)
    for kd, kind in enumerate(ORDER):
        lr = lambda_range(kind, c, red)
        dlo[kd] = lr.lo
        dhi[kd] = lr.hi if kd in ids else lr.lo - 1
    n = np.maximum(0, dhi - dlo + 1)
    lo = dlo + n * rank // world
    hi = dlo + n * (rank + 1) // world - 1
    return lo, hi, dlo, dhi


def _slice_compute_gpu(c, w, k, ids, lo, hi, engine=None):
    r = (engine or rank_engine()).check_ranges(w, c, k, ids, 0, lo, hi)
    return (np.array(r.best[:], dtype=np.int64), np.array(r.arg_lambda[:], dtype=np.int64),
            np.array(r.evals[:], dtype=np.int64), np.array(r.evaluated[:], dtype=np.int64))


def lower_bound_lambda_split(red, k: int, kinds: Sequence = DEFAULT_DFF_ORDER, *, group=None,
                             compute: Callable | None = None, engine=None):
    """Every rank checks its lambda slice of the SAME instance (bound pruning
    inside the slice) and the ranks meet in ONE exchange step: an
    all-reduce(MAX) of six packed keys ``best << 32 | ~(arg - lo)`` (plus the
    per-kind evals / evaluated, summed / max-ed in the same collective).
    Returns a lower_bound_par(cancellation=False) ``BoundResult`` on every
    rank.  ``compute(c, w, k, ids, lo, hi) -> (best, arg, evals, evaluated)``
    is injectable (the gloo tests); the default is this rank's GPU
    (``bplb_check_ranges``)."""
    import torch
    import torch.distributed as dist

    from .bounds import resolve_kinds
    from .instances import as_reduced
    from .parallel import _result_par
    from ._native import BplbResult

    kinds_t, ids = resolve_kinds(kinds)
    c, w = as_reduced(red)
    init = dist.is_available() and dist.is_initialized()
    world = dist.get_world_size(group) if init else 1
    rank = dist.get_rank(group) if init else 0
    lo, hi, dlo, dhi = lambda_slices(c, red, kinds_t, world, rank)
    fn = compute or (lambda *a: _slice_compute_gpu(*a, engine=engine))
    best, arg, evals, ev = fn(c, w, k, list(ids), lo, hi)
    keys = np.where(ev > 0, (best << 32) | (0xFFFFFFFF - (arg - dlo)), 0).astype(np.int64)
    if init:
        dev = torch.device("cpu")
        if dist.get_backend(group) == "nccl":
            dev = torch.device("cuda", (engine or rank_engine()).device)
        t = torch.from_numpy(np.concatenate([keys, ev])).to(dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        e = torch.from_numpy(evals.copy()).to(dev)
        dist.all_reduce(e, group=group)
        t, e = t.cpu().numpy(), e.cpu().numpy()
        keys, ev, evals = t[:6], t[6:], e
    res = BplbResult()
    for kd in range(6):
        res.evaluated[kd] = int(ev[kd] > 0)
        res.best[kd] = int(keys[kd] >> 32) if ev[kd] else 0
        res.arg_lambda[kd] = int(dlo[kd] + (0xFFFFFFFF - (int(keys[kd]) & 0xFFFFFFFF))) if ev[kd] else int(dlo[kd])
        res.evals[kd] = int(evals[kd])
        res.n_lambda[kd] = int(max(0, dhi[kd] - dlo[kd] + 1))
    res.evals_total = int(evals.sum())
    return _result_par(res, kinds_t, ids, k)
