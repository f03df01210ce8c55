"""Batched knapsack reasoning on the B200: the
bplb_knapsack_bins kernels (csrc/bplb_knap.cuh) through the C ABI, against
the reference's own outputs (tests/golden/knap_ref.npz, propagator.py:98-227)
and the pinned oracle (oracle/bplb_oracle.c) on random batches, the
store-level drop-ins against the reference functions, and the reference
search run with the GPU knapsack reasoning inside propagate()."""

from __future__ import annotations

import copy
import os
import random

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
from oracle import oracle as O

pytestmark = pytest.mark.gpu
UNREACHED = 255
REF_SITE = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def eng():
    from paper_2402_14821_b200 import _native

    return _native.default_engine()


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(GOLDEN, "knap_ref.npz"))


def _golden_batch(g, name):
    return (g[f"{name}_c"], g[f"{name}_cl"], g[f"{name}_lo"], g[f"{name}_hi"], g[f"{name}_w"], g[f"{name}_off"])


def _run_per_c(eng, g, name, flags=0, want_reach=False):
    """Group the golden bins by capacity (one launch per capacity)."""
    from paper_2402_14821_b200 import knapsack as K

    cs, cl, lo, hi, w, off = _golden_batch(g, name)
    out = {}
    for c in np.unique(cs):
        idx = np.nonzero(cs == c)[0]
        ws = [w[off[b]:off[b + 1]] for b in idx]
        o = np.concatenate([[0], np.cumsum([len(x) for x in ws])]).astype(np.int64)
        wcat = np.concatenate(ws) if o[-1] else np.zeros(0, np.int32)
        res = K.knapsack_bins(int(c), cl[idx], lo[idx], hi[idx], wcat, o,
                              tighten=not (flags & 0x200), reach_only=bool(flags & 0x100), want_reach=want_reach,
                              engine=eng)
        for t, b in enumerate(idx):
            out[int(b)] = (int(res.status[t]), int(res.lo[t]), int(res.hi[t]), res.action[o[t]:o[t + 1]],
                           None if res.reach is None else res.reach[t])
    return out


@pytest.mark.parametrize("name", ["rnd", "sol"])
def test_knapsack_bins_match_reference_goldens(eng, g, name):
    res = _run_per_c(eng, g, name)
    off = g[f"{name}_off"]
    for b, (st, lo, hi, act, _) in res.items():
        gst = int(g[f"{name}_status"][b])
        if gst == 1:
            assert st == 1, b
            continue
        assert st == 0 and (lo, hi) == (int(g[f"{name}_lo_out"][b]), int(g[f"{name}_hi_out"][b])), b
        want = g[f"{name}_act"][off[b]:off[b + 1]]
        seen = want != UNREACHED
        assert np.array_equal(act[seen], want[seen]), b
    assert len(res) == len(g[f"{name}_c"])


def test_reach_tightening_item_filter_match_reference(eng, g):
    reach = _run_per_c(eng, g, "rnd", flags=0x100, want_reach=True)
    filt = _run_per_c(eng, g, "rnd", flags=0x200)
    rb = g["rnd_reach"]
    off = g["rnd_off"]
    pos = 0
    for b in range(len(g["rnd_c"])):
        c = int(g["rnd_c"][b])
        nbytes = (c + 64) // 64 * 8
        want = int.from_bytes(rb[pos:pos + nbytes].tobytes(), "little")
        pos += nbytes
        st, lo, hi, _, words = reach[b]
        assert int.from_bytes(words.astype("<u4").tobytes(), "little") == want, b   # reachable_sums
        t = g["rnd_tight"][b]
        assert st == int(t[0]) and (st == 1 or (lo, hi) == (int(t[1]), int(t[2]))), b  # tightening
        st2, _, _, act, _ = filt[b]
        got = np.full(len(act), 3, np.uint8) if st2 == 1 else act
        assert np.array_equal(got, g["rnd_filt"][off[b]:off[b + 1]]), b                 # item filter


def _random_bins(rng: np.random.Generator, c: int, n: int, max_m: int):
    m = rng.integers(0, max_m + 1, n)
    off = np.concatenate([[0], np.cumsum(m)]).astype(np.int64)
    w = rng.integers(1, max(2, c // 3) + 1, int(off[-1])).astype(np.int32)
    w = np.minimum(w, c).astype(np.int32)
    cl = rng.integers(0, c // 2 + 1, n).astype(np.int64)
    cl[rng.random(n) < 0.03] = c + 1  # committed load above c
    lo = np.zeros(n, np.int64)
    hi = np.zeros(n, np.int64)
    for b in range(n):
        ws = w[off[b]:off[b + 1]]
        pick = ws[rng.random(len(ws)) < 0.5]
        target = min(c, int(cl[b]) + int(pick.sum()))
        r = rng.random()
        if r < 0.4:      # a narrow window around a reachable load: commits and removals
            lo[b] = max(0, target - int(rng.integers(0, 3)))
            hi[b] = min(c, target + int(rng.integers(0, 3)))
        elif r < 0.8:    # random interval
            lo[b] = int(rng.integers(0, c + 1))
            hi[b] = int(rng.integers(lo[b], c + 1))
        else:            # the initial [0, c]
            lo[b], hi[b] = 0, c
    return cl, lo, hi, w, off


@pytest.mark.parametrize("c,n,max_m,detail", [
    (1, 200, 6, 8), (31, 500, 12, 8), (150, 3000, 40, 8), (150, 300, 400, 8), (255, 1001, 30, 8),
    (256, 999, 30, 16), (511, 700, 30, 16), (512, 700, 30, 32), (1023, 1000, 30, 32),
    (1024, 500, 30, 256), (5000, 400, 60, 256), (100000, 96, 40, 256)])
@pytest.mark.parametrize("flags", [0, 0x200])
def test_knapsack_bins_vs_oracle(eng, c, n, max_m, detail, flags):
    rng = np.random.default_rng(c * 7 + max_m + flags)
    cl, lo, hi, w, off = _random_bins(rng, c, n, max_m)
    st, lo_o, hi_o, act, _ = eng.knapsack_bins(c, cl, lo, hi, w, off, flags)
    assert eng.last_path() == ("knap", detail)
    O.set_threads(O.max_threads())
    ost, olo, ohi, oact = O.knapsack_bins(c, cl, lo, hi, w, off, flags)
    assert np.array_equal(st, ost)
    ok = ost == 0
    assert np.array_equal(lo_o[ok], olo[ok]) and np.array_equal(hi_o[ok], ohi[ok])
    assert np.array_equal(act, oact)  # (both write a Wipeout bin's actions as 0)
    if flags == 0 and c >= 150:  # the batch exercises every decision
        assert (act == 1).any() and (act == 2).any() and (st == 1).any()


def test_knapsack_reach_vs_oracle_large_c(eng):
    rng = np.random.default_rng(9)
    c = 70001
    cl, lo, hi, w, off = _random_bins(rng, c, 40, 25)
    st, lo_o, hi_o, _, reach = eng.knapsack_bins(c, cl, lo, hi, w, off, 0x100, want_reach=True)
    for b in range(40):
        ost, olo, ohi, _, bits = O.knapsack_bin(c, cl[b], lo[b], hi[b], w[off[b]:off[b + 1]], flags=0x100)
        assert int.from_bytes(reach[b].astype("<u4").tobytes(), "little") == bits, b
        assert st[b] == ost and (ost == 1 or (lo_o[b], hi_o[b]) == (olo, ohi))


def test_knapsack_edge_cases_and_errors(eng):
    from paper_2402_14821_b200 import knapsack as K

    empty = K.knapsack_bins(10, [], [], [], [], [0], engine=eng)
    assert len(empty.status) == 0
    # no open items: the committed load alone
    r = K.knapsack_bins(10, [4, 4, 11], [0, 5, 0], [10, 10, 10], [], [0, 0, 0, 0], engine=eng)
    assert r.status.tolist() == [0, 1, 1] and (r.lo[0], r.hi[0]) == (4, 4)
    for bad in (dict(w=[0]), dict(w=[11]), dict(lo=[5], hi=[4]), dict(hi=[11]), dict(cl=[-1])):
        args = dict(cl=[0], lo=[0], hi=[10], w=[3])
        args.update(bad)
        with pytest.raises(ValueError):
            K.knapsack_bins(10, args["cl"], args["lo"], args["hi"], args["w"], [0, len(args["w"])], engine=eng)
    with pytest.raises(ValueError):  # bitsets of 2^20 loads x a 1000-item recursion exceed shared memory
        K.knapsack_bins(1 << 20, [0], [0], [1 << 20], np.ones(1000, np.int32), [0, 1000], engine=eng)


def _ref():
    if not os.path.isdir(os.path.join(REF_SITE, "binpack")):
        pytest.skip("baseline/_ref (reference install) not present")
    import sys

    if REF_SITE not in sys.path:
        sys.path.insert(0, REF_SITE)
    from binpack import propagator, search
    from binpack.instances import Instance
    from binpack.store import DomainStore, Wipeout

    return propagator, search, Instance, DomainStore, Wipeout


def _state(st):
    return (list(st.masks), list(st.load_lo), list(st.load_hi), list(st.committed_load))


def test_store_dropins_match_reference(eng):
    """reachable_sums / packability / knapsack_load_tightening /
    knapsack_item_filter / _knapsack_bin on DomainStores, GPU vs reference:
    same return value, same store mutations, same Wipeout."""
    P, _, _, DomainStore, Wipeout = _ref()
    from paper_2402_14821_b200 import knapsack as K

    rng = random.Random(17)
    for t in range(300):
        c = rng.choice([rng.randint(1, 60), rng.randint(61, 400), rng.randint(1024, 3000)])
        n = rng.randint(1, 12)
        k = rng.randint(2, 4)
        store = DomainStore(tuple(rng.randint(1, c) for _ in range(n)), c, k)
        for i in range(n):  # commit / remove a few
            if rng.random() < 0.25:
                try:
                    store.commit(i, rng.randrange(k))
                except Exception:
                    pass
        j = rng.randrange(k)
        lo = rng.randint(0, c)
        hi = rng.randint(lo, c)
        try:
            store.set_lo(j, lo)
            store.set_hi(j, hi)
        except Wipeout:
            continue
        assert K.reachable_sums(store, j, eng) == P.reachable_sums(store, j), t
        assert K.packability(store, j, eng) == P.packability(store, j), t

        def both(fa, fb):
            s1, s2 = copy.deepcopy(store), copy.deepcopy(store)
            try:
                r1 = fa(s1)
            except Wipeout as e:
                r1 = ("W", str(e))
            try:
                r2 = fb(s2)
            except Wipeout as e:
                r2 = ("W", str(e))
            assert r1 == r2 and _state(s1) == _state(s2), (t, r1, r2)

        both(lambda s: K.knapsack_load_tightening(s, j, eng), lambda s: P.knapsack_load_tightening(s, j))
        both(lambda s: K.knapsack_bin(s, j, eng), lambda s: P._knapsack_bin(s, j))
        for i in range(n):
            both(lambda s: K.knapsack_item_filter(s, i, j, eng), lambda s: P.knapsack_item_filter(s, i, j))


def test_reference_search_with_gpu_knapsack(eng):
    """The reference's minimize with the GPU knapsack reasoning inside
    propagate() makes exactly the recorded search (node / fail / bound-call
    counts of tests/golden/solver_calls.npz)."""
    P, search, Instance, _, _ = _ref()
    from paper_2402_14821_b200.knapsack import install_knapsack_gpu

    calls = np.load(os.path.join(GOLDEN, "solver_calls.npz"))
    off = calls["inst_off"]
    insts = [Instance(int(c), tuple(int(x) for x in calls["inst_w"][off[i]:off[i + 1]]))
             for i, c in enumerate(calls["inst_c"])]
    undo = install_knapsack_gpu(P, eng)
    l0 = eng.launch_count()
    try:
        for row in calls["outcomes"][:14]:
            i, c, bins, nodes, fails, bound_calls, solved = (int(x) for x in row)
            res = search.minimize(insts[i], search.SearchConfig(bound_mode=search.BoundMode.DFFS_SEQ,
                                                                time_limit=120.0))
            assert (res.bins, res.stats.nodes, res.stats.fails, res.stats.bound_calls) == \
                   (bins, nodes, fails, bound_calls), i
    finally:
        undo()
    assert eng.launch_count() > l0
