"""The oracle's knapsack restatement (oracle/bplb_oracle.c, or_knapsack_bin)
pinned to goldens the REFERENCE produced (tests/golden/make_golden_knap.py:
propagator.py:98-227 on random bins and on every _knapsack_bin call of the
reference's own minimize).  CPU only."""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import oracle as O

UNREACHED = 255


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(GOLDEN, "knap_ref.npz"))


def _bins(g, name):
    off = g[f"{name}_off"]
    for b in range(len(g[f"{name}_c"])):
        yield b, int(g[f"{name}_c"][b]), int(g[f"{name}_cl"][b]), int(g[f"{name}_lo"][b]), \
            int(g[f"{name}_hi"][b]), g[f"{name}_w"][off[b]:off[b + 1]], int(off[b]), int(off[b + 1])


def _knap_bin_matches(g, name, b, st, lo, hi, act, s, e):
    gst = int(g[f"{name}_status"][b])
    if gst == 1:
        assert st == 1, (name, b)
        return
    assert st == 0, (name, b)
    assert (lo, hi) == (int(g[f"{name}_lo_out"][b]), int(g[f"{name}_hi_out"][b])), (name, b)
    want = g[f"{name}_act"][s:e]
    seen = want != UNREACHED
    assert np.array_equal(act[seen], want[seen]), (name, b)


@pytest.mark.parametrize("name", ["rnd", "sol"])
def test_oracle_knapsack_bin_matches_reference(g, name):
    n = 0
    for b, c, cl, lo, hi, w, s, e in _bins(g, name):
        st, lo_o, hi_o, act, _ = O.knapsack_bin(c, cl, lo, hi, w)
        _knap_bin_matches(g, name, b, st, lo_o, hi_o, act, s, e)
        n += 1
    assert n > 1000


def test_oracle_reach_tightening_item_filter_match_reference(g):
    reach = g["rnd_reach"]
    pos = 0
    for b, c, cl, lo, hi, w, s, e in _bins(g, "rnd"):
        nbytes = (c + 64) // 64 * 8
        want_bits = int.from_bytes(reach[pos:pos + nbytes].tobytes(), "little")
        pos += nbytes
        st, lo_o, hi_o, _, bits = O.knapsack_bin(c, cl, lo, hi, w, flags=O.KN_REACH_ONLY)
        assert bits == want_bits, b                                  # reachable_sums
        t = g["rnd_tight"][b]
        assert st == int(t[0]) and (st == 1 or (lo_o, hi_o) == (int(t[1]), int(t[2]))), b  # tightening
        st2, _, _, act, _ = O.knapsack_bin(c, cl, lo, hi, w, flags=O.KN_NO_TIGHTEN)
        got = np.full(len(w), 3, np.uint8) if st2 == 1 else act      # knapsack_item_filter
        assert np.array_equal(got, g["rnd_filt"][s:e]), b
    assert pos == len(reach)


def test_oracle_batch_equals_single(g):
    c = 150
    rng = np.random.default_rng(3)
    n = 300
    m = rng.integers(0, 30, n)
    off = np.concatenate([[0], np.cumsum(m)])
    w = rng.integers(1, c + 1, int(off[-1])).astype(np.int32)
    cl = rng.integers(0, c + 1, n)
    lo = rng.integers(0, c + 1, n)
    hi = np.minimum(c, lo + rng.integers(0, c, n))
    st, lo_o, hi_o, act = O.knapsack_bins(c, cl, lo, hi, w, off)
    for b in range(n):
        s1, l1, h1, a1, _ = O.knapsack_bin(c, cl[b], lo[b], hi[b], w[off[b]:off[b + 1]])
        assert (st[b], lo_o[b], hi_o[b]) == (s1, l1, h1)
        assert np.array_equal(act[off[b]:off[b + 1]], a1)
