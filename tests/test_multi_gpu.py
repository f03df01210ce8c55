"""The multi-GPU C entry (bplb_check_batch_multi): one call shards a host CSR
batch over several engines (contiguous node ranges balanced by item count,
one host thread per shard) and gathers the verdicts in node order.  On the
one-GPU test box the device list repeats device 0 (several engines on one
GPU), which exercises the sharding, the per-shard offsets and the gather."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2402_14821_b200 import _native, workloads as W

pytestmark = pytest.mark.gpu
ALL = list(range(6))


@pytest.mark.parametrize("ndev", [1, 2, 3, 4])
def test_multi_matches_single_engine(ndev):
    c, k, w = W.cfg5_instance()
    flat, off = W.gen_nodes_host(w, c, k, W.CFG5_SEED, 777, first_node=40_000)
    single = _native.default_engine(0)
    want = single.check_batch(flat, off, c, 2**62, ALL, 0, want_best=True)
    m = _native.MultiEngine([0] * ndev)
    try:
        got = m.check_batch(flat, off, c, 2**62, ALL, 0, want_best=True)
        for a, b in zip(got, want):
            np.testing.assert_array_equal(a, b)
        b = m.last_bounds()
        assert b[0] == 0 and b[-1] == len(off) - 1 and np.all(np.diff(b) >= 0)
        items = off[b[1:]] - off[b[:-1]]
        assert items.max() - items.min() <= 2 * 1000  # balanced by items (max node = 1000 items)
        # decision mode and the cfg2 table path through the same entry
        got = m.check_batch(flat, off, c, k, ALL, _native.F_PHASED)
        want = single.check_batch(flat, off, c, k, ALL, _native.F_PHASED)
        np.testing.assert_array_equal(got[0], want[0])
        c2, k2, f2, o2 = W.cfg2_nodes(3000)
        got = m.check_batch(f2.astype(np.uint8), o2, c2, 2**62, ALL, 0)
        want = single.check_batch(f2.astype(np.uint8), o2, c2, 2**62, ALL, 0)
        np.testing.assert_array_equal(got[0], want[0])
    finally:
        m.close()


def test_multi_errors_and_edge_cases():
    m = _native.MultiEngine([0, 0])
    try:
        lb, ex = m.check_batch(np.zeros(0, np.int32), np.zeros(1, np.int64), 100, 5, ALL, 0)
        assert lb.size == 0
        # fewer nodes than engines, empty nodes
        lb, ex = m.check_batch(np.array([60, 70], np.int32), np.array([0, 2], np.int64), 100, 1, ALL, 0)
        assert lb.tolist() == [2] and ex.tolist() == [True]
        with pytest.raises(ValueError):  # a bad weight in the second shard surfaces as ValueError
            m.check_batch(np.array([5, 7, 3, 101], np.int32), np.array([0, 1, 2, 3, 4], np.int64), 100, 5, ALL, 0)
    finally:
        m.close()
    with pytest.raises(ValueError):
        _native.MultiEngine([])


def test_lower_bound_batch_multi_api():
    import paper_2402_14821_b200 as G

    c, k, w = W.cfg5_instance()
    flat, off = W.gen_nodes_host(w, c, k, W.CFG5_SEED, 200)
    lb, ex = G.lower_bound_batch_multi(c, flat, off, k, devices=[0, 0], mode="seq")
    lb2, ex2 = G.lower_bound_batch(c, flat, off, k, mode="seq")
    np.testing.assert_array_equal(lb, lb2)
    np.testing.assert_array_equal(ex, ex2)
