"""Multi-rank batched path on CPU: world_size 2 with the gloo backend, the
oracle as the per-shard compute.  Checks the contiguous sharding, the verdict
packing and the all-gather reassembly (the GPU version swaps in NCCL and the
CUDA engine; bench.py exercises that path on the B200)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from conftest import ROOT


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_compute(c, w, off, k, kinds):
    import sys

    sys.path.insert(0, ROOT)
    from oracle import oracle as O

    return O.check_batch(w, off, c, k)


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2402_14821_b200 import distributed as D
    from paper_2402_14821_b200 import workloads as W

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        # (1) Python-generator nodes: each rank slices only its own shard
        c, k, flat, off = W.cfg2_nodes(37)  # odd count: uneven shards
        lo, hi = D.shard_range(37, world, rank)
        sw, so = flat[off[lo]:off[hi]], off[lo:hi + 1] - off[lo]
        lb, ex = D.lower_bound_batch_sharded(c, sw, so, k, compute=_oracle_compute)
        out.append((lb.tolist(), ex.tolist()))
        # (2) the bench's own path: each rank GENERATES only its shard
        # [lo, hi) of the native node stream (first_node = lo), n_total given
        c2, w2 = W.cfg2_instance()
        k2 = W.l2_host(c2, w2) + 2
        lo, hi = D.shard_range(41, world, rank)
        sw, so = W.gen_nodes_host(w2, c2, k2, 7, hi - lo, first_node=lo)
        lb, ex = D.lower_bound_batch_sharded(c2, sw, so, k2, n_total=41, compute=_oracle_compute)
        out.append((lb.tolist(), ex.tolist()))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_shard_range_covers_everything():
    from paper_2402_14821_b200.distributed import shard_range

    for n in (0, 1, 5, 37, 1000):
        for world in (1, 2, 3, 8):
            got = [shard_range(n, world, r) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            assert max(b - a for a, b in got) - min(b - a for a, b in got) <= 1


def test_pack_roundtrip():
    from paper_2402_14821_b200.distributed import pack_verdicts, unpack_verdicts

    lb = np.array([0, 1, 5, 2**40])
    ex = np.array([False, True, False, True])
    a, b = unpack_verdicts(pack_verdicts(lb, ex))
    assert (a == lb).all() and (b == ex).all()


def test_two_rank_gloo_matches_single_process():
    import multiprocessing as mp

    import sys

    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    from paper_2402_14821_b200 import workloads as W

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c, k, flat, off = W.cfg2_nodes(37)
    want = [O.check_batch(flat, off, c, k)]
    c2, w2 = W.cfg2_instance()
    k2 = W.l2_host(c2, w2) + 2
    f2, o2 = W.gen_nodes_host(w2, c2, k2, 7, 41)
    want.append(O.check_batch(f2, o2, c2, k2))
    for rank, out in res:
        for (lbr, exr), (lb, ex) in zip(out, want):
            assert lbr == lb.tolist(), rank
            assert exr == ex.tolist(), rank


def test_shard_size_mismatch_raises():
    """A rank passing the wrong number of nodes for its shard is an error."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bad_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == [(0, "ValueError"), (1, "ValueError")]


def _bad_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2402_14821_b200 import distributed as D
    from paper_2402_14821_b200 import workloads as W

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c, k, flat, off = W.cfg2_nodes(6)
        try:  # every rank passes the WHOLE batch but claims n_total = 6
            D.lower_bound_batch_sharded(c, flat, off, k, n_total=6, compute=_oracle_compute)
            q.put((rank, "ok"))
        except ValueError:
            q.put((rank, "ValueError"))
    finally:
        dist.destroy_process_group()
