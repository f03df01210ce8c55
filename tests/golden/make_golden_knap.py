"""Knapsack-reasoning goldens, produced by the REFERENCE.

Run in the build container (the reference is importable only here):
    python tests/golden/make_golden_knap.py

Two sets of bins, each recorded as (c, committed load, lo, hi, open item
weights in open_items_of_bin order) -> what the reference does:
  * random bins: a DomainStore with k = 2 bins whose bin 0 gets a committed
    item (weight = the committed load), its interval set by set_lo / set_hi,
    and a few open items; recorded per bin:
      - reachable_sums(store, 0)            (propagator.py:105-110)
      - knapsack_load_tightening(store, 0)  (:136-143) -> lo, hi or Wipeout
      - knapsack_item_filter(store, i, 0) for every open item (:153-168)
      - _knapsack_bin(store, 0)             (:190-227) -> lo, hi, per-item
        action (mask diff: commit / remove / keep), or the Wipeout (no
        reachable load, or the item it names) -- later items unrecorded (255)
  * every _knapsack_bin call the reference's own propagate() makes
    (:259-260) while minimize() solves the solver-golden instances
    (tests/golden/make_golden_solver.py), same record.
Action codes as include/bplb.h: 0 keep, 1 remove, 2 commit, 3 Wipeout.
Output: tests/golden/knap_ref.npz.
"""

from __future__ import annotations

import copy
import os
import re
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, HERE)

from binpack import propagator as P  # noqa: E402  (reference)
from binpack import search as S  # noqa: E402
from binpack.store import DomainStore, Wipeout  # noqa: E402

UNREACHED = 255
_KNAP_BIN = P._knapsack_bin  # the reference function (solver_bins wraps the module name)


class Rec:
    def __init__(self):
        self.c, self.cl, self.lo, self.hi, self.off, self.w = [], [], [], [], [0], []
        self.status, self.lo_out, self.hi_out, self.act = [], [], [], []
        self.reach = []          # bytes of the reachable bitset (random set only)
        self.tight = []          # (status, lo, hi) of knapsack_load_tightening
        self.filt = []           # knapsack_item_filter codes per item

    def add_bin(self, c, cl, lo, hi, ws):
        self.c.append(c); self.cl.append(cl); self.lo.append(lo); self.hi.append(hi)
        self.w.extend(ws); self.off.append(len(self.w))


def knap_bin_outcome(store: DomainStore, j: int):
    """Run the reference _knapsack_bin on a copy; return (status, lo, hi, actions)."""
    items = store.open_items_of_bin(j)
    s2 = copy.deepcopy(store)
    acts = [UNREACHED] * len(items)
    status = 0
    try:
        _KNAP_BIN(s2, j)
    except Wipeout as e:
        msg = str(e)
        if "no reachable load" in msg:
            return 1, store.load_lo[j], store.load_hi[j], [0] * len(items)
        m = re.search(r"unpackable with or without item (\d+)", msg)
        assert m, msg
        bad = int(m.group(1))
        status = 2
        for pos, i in enumerate(items):
            if i == bad:
                acts[pos] = 3
                break
            acts[pos] = code(store, s2, i, j)
        return status, s2.load_lo[j], s2.load_hi[j], acts
    acts = [code(store, s2, i, j) for i in items]
    return status, s2.load_lo[j], s2.load_hi[j], acts


def code(before: DomainStore, after: DomainStore, i: int, j: int) -> int:
    if after.masks[i] == before.masks[i]:
        return 0
    if not after.has_candidate(i, j):
        return 1
    assert after.masks[i] == 1 << j
    return 2


def record(rec: Rec, store: DomainStore, j: int, extras: bool):
    items = store.open_items_of_bin(j)
    ws = [store.weights[i] for i in items]
    rec.add_bin(store.c, store.committed_load[j], store.load_lo[j], store.load_hi[j], ws)
    st, lo, hi, acts = knap_bin_outcome(store, j)
    rec.status.append(st); rec.lo_out.append(lo); rec.hi_out.append(hi); rec.act.extend(acts)
    if not extras:
        return
    # loads 0..c only: a committed load above c (no open items) is a bit no
    # window inside [0, c] can see (propagator.py:109-110)
    bits = P.reachable_sums(store, j) & ((1 << (store.c + 1)) - 1)
    rec.reach.append(bits.to_bytes((store.c + 64) // 64 * 8, "little"))
    s3 = copy.deepcopy(store)
    try:
        P.knapsack_load_tightening(s3, j)
        rec.tight.append((0, s3.load_lo[j], s3.load_hi[j]))
    except Wipeout:
        rec.tight.append((1, store.load_lo[j], store.load_hi[j]))
    for i in items:
        s4 = copy.deepcopy(store)
        try:
            P.knapsack_item_filter(s4, i, j)
            rec.filt.append(code(store, s4, i, j))
        except Wipeout:
            rec.filt.append(3)


def random_bins(rec: Rec, n: int, seed: int):
    rng = np.random.default_rng(seed)
    for t in range(n):
        band = t % 4
        c = int([rng.integers(1, 61), rng.integers(61, 1024), rng.integers(1024, 4000), rng.integers(1, 200)][band])
        m = int(rng.integers(0, 13 if band < 3 else 40))
        ws = [int(x) for x in rng.integers(1, c + 1, m)]
        cl = int(rng.integers(0, c + 1)) if rng.random() < 0.9 else int(rng.integers(c + 1, 2 * c + 2))
        weights = tuple(ws + ([cl] if cl > 0 else []))
        store = DomainStore(weights, c, 2)
        if cl > 0:
            store.commit(len(ws), 0)
        lo = int(rng.integers(0, c + 1))
        hi = int(rng.integers(lo, c + 1))
        if rng.random() < 0.3:
            lo = int(rng.integers(0, max(1, c // 4)))
            hi = int(rng.integers(max(lo, c - c // 4), c + 1))
        store.set_lo(0, lo)
        store.set_hi(0, hi)
        record(rec, store, 0, True)


def solver_bins(rec: Rec):
    import make_golden_solver as MS

    orig = P._knapsack_bin

    def recording(store, j):
        record(rec, store, j, False)
        return orig(store, j)

    P._knapsack_bin = recording
    try:
        for inst in MS.instances()[:14]:
            S.minimize(inst, S.SearchConfig(bound_mode=S.BoundMode.DFFS_SEQ, time_limit=60.0))
    finally:
        P._knapsack_bin = orig


def main() -> None:
    rnd = Rec()
    random_bins(rnd, 1200, 11)
    sol = Rec()
    solver_bins(sol)
    out = {}
    for name, r in (("rnd", rnd), ("sol", sol)):
        out[f"{name}_c"] = np.array(r.c, np.int64)
        out[f"{name}_cl"] = np.array(r.cl, np.int64)
        out[f"{name}_lo"] = np.array(r.lo, np.int64)
        out[f"{name}_hi"] = np.array(r.hi, np.int64)
        out[f"{name}_off"] = np.array(r.off, np.int64)
        out[f"{name}_w"] = np.array(r.w, np.int32)
        out[f"{name}_status"] = np.array(r.status, np.int32)
        out[f"{name}_lo_out"] = np.array(r.lo_out, np.int64)
        out[f"{name}_hi_out"] = np.array(r.hi_out, np.int64)
        out[f"{name}_act"] = np.array(r.act, np.uint8)
    out["rnd_reach"] = np.frombuffer(b"".join(rnd.reach), np.uint8)
    out["rnd_tight"] = np.array(rnd.tight, np.int64).reshape(-1, 3)
    out["rnd_filt"] = np.array(rnd.filt, np.uint8)
    np.savez_compressed(os.path.join(HERE, "knap_ref.npz"), **out)
    print("random bins", len(rnd.c), "solver bins", len(sol.c),
          "statuses", np.bincount(out["sol_status"], minlength=3), np.bincount(out["rnd_status"], minlength=3),
          "actions", np.bincount(out["sol_act"], minlength=4)[:4], np.bincount(out["rnd_act"], minlength=4)[:4])


if __name__ == "__main__":
    main()
