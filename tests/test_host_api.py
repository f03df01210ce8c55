"""Host-side pieces of the drop-in API that need no GPU: lambda ranges,
scalar transforms, ReducedInstance validation, engine argument checks,
SharedMax -- restated from the reference's own tests (test_bounds.py,
test_parallel.py, test_instances.py)."""

from __future__ import annotations

import random
import threading

import numpy as np
import pytest

from paper_2402_14821_b200 import (DffKind, ParallelBoundEngine, ReducedInstance, SharedMax,
                                   VB2_ACCUMULATOR_MAX, dff_value, l1, l2_partition, l2_value,
                                   lambda_range, lower_bound_par)


@pytest.mark.parametrize("w,expected", [(140, 150), (75, 75), (20, 0)])
def test_mt_values(w, expected):
    assert dff_value(DffKind.MT, w, 150, 30) == expected


@pytest.mark.parametrize("w,expected", [(6, 4), (5, 3), (4, 2)])
def test_ccm1_values(w, expected):
    assert dff_value(DffKind.CCM1, w, 10, 3) == expected


def test_other_value_kats():
    assert dff_value(DffKind.BJ1, 7, 10, 4) == 3
    assert dff_value(DffKind.FS1, 5, 10, 3) == 15
    assert dff_value(DffKind.FS1, 4, 10, 3) == 10
    assert dff_value(DffKind.VB2, 6, 10, 2) == 2
    assert dff_value(DffKind.VB2, 4, 10, 2) == 0


@pytest.mark.parametrize("kind", list(DffKind))
def test_zero_maps_to_zero(kind):
    for c in (1, 7, 10, 33):
        for lam in lambda_range(kind, c):
            assert dff_value(kind, 0, c, lam) == 0


@pytest.mark.parametrize("kind", list(DffKind))
def test_lambda_range_matches_domain_predicate(kind):
    def valid(c, lam):
        if kind is DffKind.MT:
            return 0 <= lam and (2 * lam <= c or (2 * lam == c + 1 and c > 1))
        if kind is DffKind.RAD2:
            return 4 * lam > c and 3 * lam <= c
        if kind is DffKind.FS1:
            return 1 <= lam <= 100
        if kind is DffKind.CCM1:
            return 1 <= lam and 2 * lam <= c
        if kind is DffKind.VB2:
            return 2 <= lam <= c
        return 1 <= lam <= c

    for c in range(1, 130):
        assert list(lambda_range(kind, c)) == [lam for lam in range(0, max(c, 100) + 1) if valid(c, lam)]


def test_lambda_range_examples():
    assert (lambda_range(DffKind.RAD2, 150).lo, lambda_range(DffKind.RAD2, 150).hi) == (38, 50)
    assert lambda_range(DffKind.RAD2, 4).is_empty
    assert (lambda_range(DffKind.MT, 1).lo, lambda_range(DffKind.MT, 1).hi) == (0, 0)
    c = 10**13
    red = ReducedInstance(c, (c - 1, c - 2, c // 2) + (10**12,) * 7)
    rng = lambda_range(DffKind.VB2, c, red)
    assert rng.hi == VB2_ACCUMULATOR_MAX // (red.r * red.max_weight) < c
    assert lambda_range(DffKind.VB2, 100).hi == 100


def test_l2_partition_and_value():
    red = ReducedInstance(10, (9, 6, 5, 4, 2, 1))
    p = l2_partition(red, 2)
    assert sorted(p.w1) == [9] and sorted(p.w2) == [6] and sorted(p.w3) == [2, 4, 5]
    assert l2_value(ReducedInstance(10, (6, 6, 4, 4, 2)), 0) == 3


def test_l1_host():
    assert l1(ReducedInstance(9, (4, 4, 3, 3, 2, 2))) == 2
    assert l1(ReducedInstance(9, ())) == 0


def test_reduced_instance_validation():
    with pytest.raises(ValueError):
        ReducedInstance(0, ())
    with pytest.raises(ValueError):
        ReducedInstance(10, (11,))
    with pytest.raises(ValueError):
        ReducedInstance(10, (0,))
    a = ReducedInstance.from_array(10, [3, 4])
    assert a.r == 2 and a.max_weight == 4 and a.weights == (3, 4)
    with pytest.raises(ValueError):
        ReducedInstance.from_array(10, [3, 40])


def test_capacity_envelope_is_explicit():
    # the GPU path refuses (ValueError) instead of silently falling back to the CPU
    from paper_2402_14821_b200.instances import as_reduced

    with pytest.raises(ValueError):
        as_reduced(ReducedInstance(2**31, (5,)))


def test_engine_rejects_bad_workers():
    with pytest.raises(ValueError):
        ParallelBoundEngine(workers=0)
    with pytest.raises(ValueError):
        lower_bound_par(ReducedInstance(5, (1,)), 1, workers=0)


def test_shared_max():
    shared = SharedMax(0)
    assert shared.offer(5) == 5 and shared.offer(3) == 5 and shared.get() == 5
    values = list(range(1000))
    random.Random(0).shuffle(values)
    shared = SharedMax(0)
    ts = [threading.Thread(target=lambda ch: [shared.offer(v) for v in ch], args=(values[i::8],)) for i in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert shared.get() == 999


def test_from_name():
    assert DffKind.from_name(" vb2 ") is DffKind.VB2
    with pytest.raises(ValueError):
        DffKind.from_name("nope")


def test_workloads_deterministic():
    from paper_2402_14821_b200 import workloads as W

    c, k, f1, o1 = W.cfg2_nodes(20)
    c2, k2, f2, o2 = W.cfg2_nodes(20)
    assert (f1 == f2).all() and (o1 == o2).all() and k == 209
    _, _, f3, o3 = W.cfg2_nodes(5, first_node=10)
    assert (f3 == f1[o1[10]:o1[15]]).all()
    c3, w3 = W.cfg3()
    assert w3.size == 1000 and ((w3 > c3 // 4) & (w3 < c3 // 2)).all() and -(-int(w3.sum()) // c3) == 334


def test_node_assignments_reduce_to_node_batch():
    """The assignment form of the cfg2 node generator reduces (reduce_packing
    semantics) to exactly the CSR nodes the benchmark uses."""
    from paper_2402_14821_b200 import workloads as W
    from paper_2402_14821_b200.instances import reduce_packing_arrays

    c, k, w, a = W.cfg2_assignments(40, first_node=3)
    _, _, flat, off = W.cfg2_nodes(40, first_node=3)
    openv = np.iinfo(a.dtype).max
    for i in range(40):
        asg = np.where(a[i] == openv, -1, a[i].astype(np.int64))
        red = reduce_packing_arrays(w, asg, k, c)
        np.testing.assert_array_equal(red, flat[off[i]:off[i + 1]])


def test_addr_helper_matches_ctypes_data():
    """_native._addr (the cheap pointer read on the batch-call path) returns
    the array's data pointer for writable, read-only and empty arrays."""
    import numpy as np

    from paper_2402_14821_b200._native import _addr

    a = np.arange(100, dtype=np.int64)
    assert _addr(a) == a.ctypes.data
    ro = np.frombuffer(b"\x01\x02\x03\x04", dtype=np.uint8)
    assert not ro.flags.writeable and _addr(ro) == ro.ctypes.data
    e = np.zeros(0, dtype=np.uint8)
    assert _addr(e) == e.ctypes.data
    v = a[10:]
    assert _addr(v) == v.ctypes.data
