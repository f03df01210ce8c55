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
        c, k, flat, off = W.cfg2_nodes(37)  # odd count: uneven shards
        lb, ex = D.lower_bound_batch_sharded(c, flat, off, k, compute=_oracle_compute)
        q.put((rank, lb.tolist(), ex.tolist()))
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
    lb, ex = O.check_batch(flat, off, c, k)
    for rank, lbr, exr in res:
        assert lbr == lb.tolist(), rank
        assert exr == ex.tolist(), rank
