"""GPU parity of the bound-pruned sweep (csrc/bplb_prune.cuh).

The pruned kernel skips lambdas whose integer upper bound cannot change the
outputs; every output must still be bit-exact with the reference's full
sweep.  Checked against the pinned C oracle (oracle/, restating bounds.py) on
fresh seeded nodes -- including >= 1000 nodes of the cfg5 headline batch --
and against the dense (every-lambda) GPU kernels for the arg lambdas, in all
three modes, and the tests assert that the pruned kernel actually served the
call (bplb_last_path)."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2402_14821_b200 import _native, workloads as W
from paper_2402_14821_b200.batch import lower_bound_batch
from oracle import oracle as O

pytestmark = pytest.mark.gpu
ALL = list(range(6))


@pytest.fixture(scope="module")
def eng():
    e = _native.Engine(0)
    yield e
    e.close()


def _oracle_best(flat, off, c, k=2**62):
    lbo, exo, besto = O.check_batch(flat, off, c, k, want_best=True)
    return lbo, exo, besto


def _rand_batch(rng, c, n, rmax, special=True):
    nodes = []
    for _ in range(n):
        r = int(rng.integers(0, rmax + 1))
        w = rng.integers(1, c + 1, r)
        if special and r and rng.random() < 0.3:
            pick = rng.integers(0, r, max(1, r // 4))
            w[pick] = rng.choice([c, max(1, c // 2), max(1, (c + 1) // 2), 1], pick.size)
        nodes.append(w.astype(np.int32))
    off = np.zeros(n + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(x) for x in nodes])
    flat = np.concatenate(nodes) if off[-1] else np.zeros(0, np.int32)
    return flat.astype(np.int32), off


def test_cfg5_1000_nodes_lb_mode(eng):
    """cfg5 (1000-item c=1e5 instance, native generator): 1200 nodes, lb mode."""
    c, k, w = W.cfg5_instance()
    flat, off = W.gen_nodes_host(w, c, k, W.CFG5_SEED, 1200)
    lb, ex = eng.check_batch(flat, off, c, 2**62, ALL, 0)
    assert eng.last_path() == ("prune", 1)
    O.set_threads(O.max_threads())
    lbo, exo = O.check_batch(flat, off, c, 2**62)
    np.testing.assert_array_equal(lb, lbo)
    # decision mode k = 334 (lower_bound_seq early exit)
    lb2, ex2 = eng.check_batch(flat, off, c, k, ALL, _native.F_PHASED)
    lbo2, exo2 = O.check_batch(flat, off, c, k)
    np.testing.assert_array_equal(lb2, lbo2)
    np.testing.assert_array_equal(ex2, exo2)


def test_cfg5_key_mode_best_and_arg(eng):
    """Per-kind best (oracle) and lowest arg lambda (dense GPU sweep) on 200 cfg5 nodes."""
    c, k, w = W.cfg5_instance()
    flat, off = W.gen_nodes_host(w, c, k, W.CFG5_SEED, 200, first_node=5000)
    lb, ex, best, arg = eng.check_batch(flat, off, c, 2**62, ALL, 0, want_best=True)
    assert eng.last_path() == ("prune", 0)
    lbo, exo, besto = _oracle_best(flat, off, c)
    np.testing.assert_array_equal(lb, lbo)
    np.testing.assert_array_equal(best, besto)
    lbd, exd, bestd, argd = eng.check_batch(flat, off, c, 2**62, ALL, _native.F_NOPRUNE, want_best=True)
    assert eng.last_path()[0] != "prune"
    np.testing.assert_array_equal(bestd, besto)
    np.testing.assert_array_equal(arg, argd)


@pytest.mark.parametrize("c", [2, 3, 4, 5, 7, 8, 31, 150, 151, 289, 500, 1000, 1001, 4095, 65536, 99991,
                               100000, 262144])
def test_random_nodes_vs_oracle(eng, c):
    rng = np.random.default_rng(c)
    rmax = 300 if c >= 65536 else 600
    flat, off = _rand_batch(rng, c, 96, rmax)
    flags_list = [0, _native.F_PHASED, _native.F_CANCEL]
    lbo, exo, besto = _oracle_best(flat, off, c)
    # lb mode (full)
    lb, ex = eng.check_batch(flat, off, c, 2**62, ALL, _native.F_NOTAB)
    assert eng.last_path()[0] == "prune"
    np.testing.assert_array_equal(lb, lbo)
    # key mode (full) vs oracle best and dense arg
    lb, ex, best, arg = eng.check_batch(flat, off, c, 2**62, ALL, _native.F_NOTAB, want_best=True)
    np.testing.assert_array_equal(best, besto)
    _, _, bestd, argd = eng.check_batch(flat, off, c, 2**62, ALL, _native.F_NOTAB | _native.F_NOPRUNE,
                                        want_best=True)
    np.testing.assert_array_equal(bestd, besto)
    np.testing.assert_array_equal(arg, argd)
    # decision modes at a k inside the bound range
    kk = int(np.median(lbo)) if len(lbo) else 0
    lbs, exs = O.check_batch(flat, off, c, kk)
    for fl in flags_list[1:]:
        lb, ex = eng.check_batch(flat, off, c, kk, ALL, fl | _native.F_NOTAB)
        np.testing.assert_array_equal(ex, exs)
        if fl == _native.F_PHASED:
            np.testing.assert_array_equal(lb, lbs)
        else:  # cancel: exact when not exceeded, any computed value > k otherwise
            np.testing.assert_array_equal(lb[~exs], lbs[~exs])
            assert np.all(lb[exs] > kk) and np.all(lb[exs] <= lbo[exs])


@pytest.mark.parametrize("kinds", [[4], [5, 3], [0, 1], [2], [3, 4, 5], [5, 4, 3, 2, 1, 0]])
def test_kind_subsets_and_orders(eng, kinds):
    rng = np.random.default_rng(len(kinds) * 7 + kinds[0])
    c = 99991
    flat, off = _rand_batch(rng, c, 64, 400)
    names = [O.KIND_NAMES[i] for i in kinds]
    lbo, exo, besto = O.check_batch(flat, off, c, 2**62, kinds=names, want_best=True)
    lb, ex = eng.check_batch(flat, off, c, 2**62, kinds, 0)
    np.testing.assert_array_equal(lb, lbo)
    lb, ex, best, arg = eng.check_batch(flat, off, c, 2**62, kinds, 0, want_best=True)
    np.testing.assert_array_equal(best[:, kinds], besto)
    kk = int(np.median(lbo))
    lbs, exs = O.check_batch(flat, off, c, kk, kinds=names)
    lb, ex = eng.check_batch(flat, off, c, kk, kinds, _native.F_PHASED)
    np.testing.assert_array_equal(lb, lbs)
    np.testing.assert_array_equal(ex, exs)


def test_bad_weight_raises(eng):
    flat = np.array([5, 7, 0, 3], dtype=np.int32)
    off = np.array([0, 2, 4], dtype=np.int64)
    with pytest.raises(ValueError):
        eng.check_batch(flat, off, 1000, 2**62, ALL, 0)
    flat = np.array([5, 1001], dtype=np.int32)
    with pytest.raises(ValueError):
        eng.check_batch(flat, np.array([0, 2], dtype=np.int64), 1000, 2**62, ALL, 0)


def test_device_generator_matches_host():
    import torch

    c, k, w = W.cfg5_instance()
    flat, off = W.gen_nodes_host(w, c, k, W.CFG5_SEED, 3000, first_node=12345)
    df, do = W.gen_nodes_device(w, c, k, W.CFG5_SEED, 3000, first_node=12345, device="cuda:0")
    torch.cuda.synchronize()
    np.testing.assert_array_equal(do.cpu().numpy(), off)
    np.testing.assert_array_equal(df.cpu().numpy()[:off[-1]], flat)


def test_lower_bound_batch_dense_flag():
    c, k, w = W.cfg5_instance()
    flat, off = W.gen_nodes_host(w, c, k, W.CFG5_SEED, 64, first_node=777)
    a = lower_bound_batch(c, flat, off, 2**62)
    b = lower_bound_batch(c, flat, off, 2**62, dense=True)
    np.testing.assert_array_equal(a[0], b[0])


def test_cfg5_reference_golden(eng):
    """The headline batch's reference outputs (96 nodes across the 10^6-node
    stream, tests/golden/cfg5_ref.npz, made by the reference itself): the
    pruned kernel in lb mode, key mode and decision mode (k = 334, the
    lower_bound_seq early exit), and the dense sweep."""
    import os

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "cfg5_ref.npz"))
    c, k = int(g["c"]), int(g["k"])
    w, off = g["weights"], g["offsets"]
    lb, ex = eng.check_batch(w, off, c, 2**62, ALL, 0)
    assert eng.last_path() == ("prune", 1)
    np.testing.assert_array_equal(lb, g["lb"])
    lb, ex, best, arg = eng.check_batch(w, off, c, 2**62, ALL, 0, want_best=True)
    assert eng.last_path() == ("prune", 0)
    np.testing.assert_array_equal(best, g["best"])
    lb, ex = eng.check_batch(w, off, c, k, ALL, _native.F_PHASED)
    assert eng.last_path()[0] == "prune"
    np.testing.assert_array_equal(lb, g["dec_lb"])
    np.testing.assert_array_equal(ex, g["dec_exceeded"].astype(bool))
    lb, ex, best, arg = eng.check_batch(w, off, c, 2**62, ALL, _native.F_NOPRUNE, want_best=True)
    np.testing.assert_array_equal(best, g["best"])


def test_cfg5_device_batch_matches_golden_nodes(eng):
    """The bench's device-resident path: nodes generated on the GPU at the
    golden node ids, checked by bplb_check_batch_device, equal the
    reference's outputs."""
    import os

    import torch

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "cfg5_ref.npz"))
    c, k, w = W.cfg5_instance()
    ids = g["node_ids"]
    s = torch.cuda.Stream()
    for j in (0, 50, 95):
        df, do = W.gen_nodes_device(w, c, k, W.CFG5_SEED, 1, first_node=int(ids[j]), device="cuda:0")
        lb = torch.empty(1, dtype=torch.int64, device="cuda:0")
        ex = torch.empty(1, dtype=torch.uint8, device="cuda:0")
        torch.cuda.synchronize()
        eng.check_batch_device(df.data_ptr(), do.data_ptr(), 1, int(do[1] - do[0]), c, 2**62, ALL, 0,
                               lb.data_ptr(), ex.data_ptr(), stream_ptr=s.cuda_stream)
        s.synchronize()
        assert int(lb[0]) == int(g["lb"][j])


@pytest.mark.parametrize("shape", [("cfg4", 0, 0), ("u", 30_000, 1_000_000), ("u", 20_000, 262_147),
                                   ("tri", 9_000, 99_991), ("small", 40_000, 700_001)])
def test_wide_path_pruned_equals_dense(eng, shape):
    """Single checks on the grid-wide path (r > 16384 or c large): the pruned
    full collection (seed launch, keys snapshot, pruned launch) returns the
    same per-kind best, arg lambda, lb and evals as the dense sweep; cfg4
    also against the reference goldens (VB2: 50011 at lambda 3)."""
    kind, r, c = shape
    rng = np.random.default_rng(r + c)
    if kind == "cfg4":
        c, w = W.cfg4()
    elif kind == "u":
        w = rng.integers(1, c + 1, r)
    elif kind == "tri":
        w = rng.integers(c // 4 + 1, c // 2, r)
    else:
        w = rng.integers(1, c // 50, r)
    w = w.astype(np.int32)
    a = eng.check(w, c, 2**62, ALL, 0)
    assert eng.last_path()[0] == "wide"
    b = eng.check(w, c, 2**62, ALL, _native.F_NOPRUNE)
    for f in ("best", "arg_lambda", "evals", "evaluated"):
        assert list(getattr(a, f)) == list(getattr(b, f)), f
    assert a.lb == b.lb
    if kind == "cfg4":
        import os

        g = np.load(os.path.join(os.path.dirname(__file__), "golden", "configs.npz"))
        want = g["cfg4_best_nonvb2"].tolist()
        got = list(a.best)
        assert [x for i, x in enumerate(got) if i != 4] == [x for i, x in enumerate(want) if i != 4]
        assert got[4] == 50011 and a.arg_lambda[4] == 3


@pytest.mark.parametrize("shape", [("cfg3", 0, 0), ("cfg3u", 0, 0), ("u", 3_000, 200_003), ("u", 900, 65_537),
                                   ("tri", 2_000, 99_991)])
def test_multi_cta_node_vb2_pruned_equals_dense(eng, shape):
    """Single full-collection checks on the multi-CTA node kernel: the VB2
    rest is tested chunk by chunk against the best VB2 key any CTA has
    published (seed chunk first); per-kind best, arg lambda, evals and lb equal
    the dense sweep's (F_NOPRUNE)."""
    kind, r, c = shape
    rng = np.random.default_rng(r + c + 7)
    if kind == "cfg3":
        c, w = W.cfg3()
    elif kind == "cfg3u":
        c, w = W.cfg3u()
    elif kind == "u":
        w = rng.integers(1, c + 1, r)
    else:
        w = rng.integers(c // 4 + 1, c // 2, r)
    w = w.astype(np.int32)
    a = eng.check(w, c, 2**62, ALL, 0)
    path = eng.last_path()[0]
    b = eng.check(w, c, 2**62, ALL, _native.F_NOPRUNE)
    for f in ("best", "arg_lambda", "evals", "evaluated"):
        assert list(getattr(a, f)) == list(getattr(b, f)), (f, path)
    assert a.lb == b.lb


def test_wide_graph_replay_and_table_reuse(eng):
    """The grid-wide single check is captured into a CUDA graph on the second
    call with an argument set and replayed after; instances of another size in
    between reuse the table buffer (the histogram counts are re-zeroed before a
    replay).  Every repeat returns the first call's result."""
    rng = np.random.default_rng(11)
    a = (1_000_000, rng.integers(1, 1_000_001, 30_000).astype(np.int32))
    b = (200_003, rng.integers(1, 200_004, 20_000).astype(np.int32))
    want = {}
    for c, w in (a, b, a, a, b, b, a, b, a):
        res = eng.check(w, c, 2**62, ALL, 0)
        assert eng.last_path()[0] == "wide"
        got = (res.lb, list(res.best), list(res.arg_lambda), list(res.evals))
        want.setdefault(c, got)
        assert got == want[c], c
    # a different weight vector of the same size (same argument set: replayed)
    w2 = rng.integers(1, 1_000_001, 30_000).astype(np.int32)
    r1 = eng.check(w2, a[0], 2**62, ALL, 0)
    r2 = eng.check(w2, a[0], 2**62, ALL, _native.F_NOPRUNE)
    assert r1.lb == r2.lb and list(r1.best) == list(r2.best)


@pytest.mark.parametrize("devices", [(0, 0), (0, 0, 0)])
def test_lambda_split_multi_device(devices):
    """bplb_check_multi: one instance, each kind's lambda range split over the
    engines (a repeated device id stands in for several GPUs), per-kind keys
    merged -- identical to the single-engine full check (grid-wide cfg4 and a
    node-path instance), and lower_bound_seq semantics replayed."""
    import paper_2402_14821_b200 as G
    from paper_2402_14821_b200 import _native as N

    m = N.MultiEngine(devices)
    try:
        eng = N.Engine(0)
        rng = np.random.default_rng(3)
        for c, w in (W.cfg4(), (100_000, rng.integers(1, 100_001, 900).astype(np.int32)), W.cfg3()):
            a = m.check(w, c, 2**62, ALL, 0)
            b = eng.check(w, c, 2**62, ALL, 0)
            for f in ("best", "arg_lambda", "evals", "evaluated", "n_lambda"):
                assert list(getattr(a, f)) == list(getattr(b, f)), (c, f)
            assert a.lb == b.lb and a.exceeded == b.exceeded
            red = G.ReducedInstance.from_array(c, w)
            for k in (2**62, int(b.lb) - 1):
                s1 = G.lower_bound_multi(red, k, devices, mode="seq")
                s2 = G.lower_bound_seq(red, k)
                assert s1.per_dff == s2.per_dff and s1.lb == s2.lb and s1.evals == s2.evals, (c, k)
        eng.close()
    finally:
        m.close()
