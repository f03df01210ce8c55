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


# ---------------------------------------------------------------------------
# One check split over ranks by lambda: slice results from the
# oracle's per-lambda vectors, one all-reduce(MAX) of packed keys
# ---------------------------------------------------------------------------
_KN = ["MT", "RAD2", "FS1", "CCM1", "VB2", "BJ1"]


def _oracle_slice(c, w, k, ids, lo, hi):
    import sys

    sys.path.insert(0, ROOT)
    from oracle import oracle as O

    best = np.zeros(6, dtype=np.int64)
    arg = lo.copy()
    evals = np.zeros(6, dtype=np.int64)
    ev = np.zeros(6, dtype=np.int64)
    for kd in ids:
        if hi[kd] < lo[kd]:
            continue
        v = O.dff_bound_batch(_KN[kd], w, c, int(lo[kd]), int(hi[kd]))
        j = int(np.argmax(v))  # first maximum: the lowest lambda
        best[kd], arg[kd], evals[kd], ev[kd] = v[j], lo[kd] + j, len(v), 1
    return best, arg, evals, ev


def _split_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2402_14821_b200 import ReducedInstance
    from paper_2402_14821_b200 import distributed as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        rng = np.random.default_rng(5)
        for c, n in ((150, 120), (997, 300), (5000, 200)):
            w = rng.integers(1, c + 1, n).astype(np.int32)
            res = D.lower_bound_lambda_split(ReducedInstance.from_array(c, w), 2**62, compute=_oracle_slice)
            out.append(({kk.name: v for kk, v in res.per_dff.items()}, {kk.name: v for kk, v in res.arg.items()},
                        res.lb, res.evals))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_lambda_split_gloo_matches_oracle(world):
    import multiprocessing as mp

    import sys

    sys.path.insert(0, ROOT)
    from oracle import oracle as O

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_split_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(5)
    want = []
    for c, n in ((150, 120), (997, 300), (5000, 200)):
        w = rng.integers(1, c + 1, n).astype(np.int32)
        o = O.lower_bound_seq(w, c, 2**62)
        want.append((o.per_dff, o.arg, o.lb, o.evals))
    for rank, out in res:
        for got, exp in zip(out, want):
            assert got == exp, rank


def test_lambda_slices_cover_every_range():
    from paper_2402_14821_b200 import DEFAULT_DFF_ORDER, ReducedInstance
    from paper_2402_14821_b200.distributed import lambda_slices

    red = ReducedInstance.from_array(1000, np.arange(1, 400, dtype=np.int32))
    for world in (1, 2, 3, 8):
        parts = [lambda_slices(1000, red, DEFAULT_DFF_ORDER, world, r) for r in range(world)]
        dlo, dhi = parts[0][2], parts[0][3]
        for kd in range(6):
            assert parts[0][0][kd] == dlo[kd] and parts[-1][1][kd] == dhi[kd]
            for a, b in zip(parts, parts[1:]):
                assert a[1][kd] + 1 == b[0][kd]
