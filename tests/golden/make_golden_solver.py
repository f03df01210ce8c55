"""Solver-integration goldens, produced by the REFERENCE.

Run in the build container (the reference is importable only here):
    python tests/golden/make_golden_solver.py

For small Falkenauer-U- and Scholl-shaped instances it runs the reference's
own ``minimize`` (search.py:339-381) with ``BoundMode.DFFS_SEQ`` and records
EVERY bound-engine call the solver makes -- the root call (search.py:352)
and the feasibility checks inside ``propagate`` (propagator.py:266-276) --
as (instance, reduced weights, k) -> BoundResult (lb, exceeded_k, evals,
per_dff in order), plus the solve's outcome (bins, nodes, fails,
bound_calls).  tests/test_solver_gpu.py replays the calls through the GPU
engine (identical results in order => identical search) and re-runs the
reference search end to end with the GPU engine plugged in.
Output: tests/golden/solver_calls.npz.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from binpack import search as S  # noqa: E402  (reference)
from binpack.bounds import DEFAULT_DFF_ORDER, lower_bound_seq  # noqa: E402
from binpack.instances import Instance  # noqa: E402

KIND_IDS = {k: i for i, k in enumerate(DEFAULT_DFF_ORDER)}


def instances():
    out = []
    for s in range(6):  # Falkenauer-U-shaped: c = 150, w ~ U{20..100}
        rng = np.random.default_rng(100 + s)
        n = 18 + 4 * s
        out.append(Instance(150, tuple(int(x) for x in rng.integers(20, 101, n)), f"fu{s}"))
    for s in range(4):  # Scholl-1-shaped: c in {100, 120, 150}, w ~ U{1..100} / U{20..100} / U{30..100}
        rng = np.random.default_rng(200 + s)
        c = (100, 120, 150, 150)[s]
        lo = (1, 20, 30, 20)[s]
        n = 20 + 5 * s
        out.append(Instance(c, tuple(int(x) for x in rng.integers(lo, 101, n)), f"sch{s}"))
    for s in range(4):  # triplet-shaped (no slack): c = 1000, bins of three items in (250, 500)
        rng = np.random.default_rng(300 + s)
        items = []
        for _ in range(5 + s):
            a = int(rng.integers(252, 499))
            b = int(rng.integers(max(251, 501 - a), min(499, 749 - a) + 1))
            items += [a, b, 1000 - a - b]
        rng.shuffle(items)
        out.append(Instance(1000, tuple(items), f"trip{s}"))
    for s in range(3):  # larger, lightly slack random: c = 150, U{40..100}
        rng = np.random.default_rng(400 + s)
        out.append(Instance(150, tuple(int(x) for x in rng.integers(40, 101, 45 + 5 * s)), f"fu_big{s}"))
    # seeds whose search hits bound failures (engine(red, k).lb > k inside
    # propagate, propagator.py:275): picked by scanning seeds 0..161
    for seed in (10, 39, 78, 86, 89, 93, 98, 137, 140, 146, 151, 161):
        rng = np.random.default_rng(seed)
        kind = seed % 4
        c = [100, 120, 1000, 150][kind]
        n = int(rng.integers(12, 30))
        lo, hi = [(20, 50), (25, 60), (200, 500), (30, 80)][kind]
        out.append(Instance(c, tuple(int(x) for x in rng.integers(lo, hi + 1, n)), f"hard{seed}"))
    return out


def main() -> None:
    calls = []  # (instance idx, c, weights, k, lb, exceeded, evals, per_dff[6] or -1, order mask)
    outcomes = []
    orig = S.make_bound_engine
    cur = {"i": -1}

    def recording_factory(cfg):
        def engine(red, k):
            res = lower_bound_seq(red, k, cfg.dff_order)
            per = [-1] * 6
            order = []
            for kd, v in res.per_dff.items():
                per[KIND_IDS[kd]] = v
                order.append(KIND_IDS[kd])
            calls.append((cur["i"], red.c, tuple(red.weights), k, res.lb, int(res.exceeded_k), res.evals, per,
                          order))
            return res

        return engine, lambda: None

    S.make_bound_engine = recording_factory
    try:
        for i, inst in enumerate(instances()):
            cur["i"] = i
            t = time.time()
            cfg = S.SearchConfig(bound_mode=S.BoundMode.DFFS_SEQ, time_limit=120.0)
            res = S.minimize(inst, cfg)
            n_calls = sum(1 for x in calls if x[0] == i)
            outcomes.append((i, inst.c, res.bins if res.bins is not None else -1, res.stats.nodes, res.stats.fails,
                             res.stats.bound_calls, int(res.status is S.SolveStatus.SOLUTION)))
            print(f"{inst.name}: n={inst.n} bins={res.bins} nodes={res.stats.nodes} fails={res.stats.fails} "
                  f"bound_calls={res.stats.bound_calls} recorded={n_calls} {time.time() - t:.1f}s")
    finally:
        S.make_bound_engine = orig
    insts = instances()
    iw = [np.array(x.weights, dtype=np.int32) for x in insts]
    ioff = np.zeros(len(iw) + 1, dtype=np.int64)
    ioff[1:] = np.cumsum([len(x) for x in iw])
    woff = np.zeros(len(calls) + 1, dtype=np.int64)
    woff[1:] = np.cumsum([len(x[2]) for x in calls])
    np.savez_compressed(
        os.path.join(HERE, "solver_calls.npz"),
        inst_c=np.array([x.c for x in insts], dtype=np.int64), inst_w=np.concatenate(iw), inst_off=ioff,
        call_inst=np.array([x[0] for x in calls], dtype=np.int64),
        call_c=np.array([x[1] for x in calls], dtype=np.int64),
        call_w=np.concatenate([np.array(x[2], dtype=np.int32) for x in calls]) if calls else np.zeros(0, np.int32),
        call_off=woff, call_k=np.array([x[3] for x in calls], dtype=np.int64),
        call_lb=np.array([x[4] for x in calls], dtype=np.int64),
        call_exceeded=np.array([x[5] for x in calls], dtype=np.int64),
        call_evals=np.array([x[6] for x in calls], dtype=np.int64),
        call_per_dff=np.array([x[7] for x in calls], dtype=np.int64).reshape(-1, 6),
        call_order=np.array([x[8] + [-1] * (6 - len(x[8])) for x in calls], dtype=np.int64).reshape(-1, 6),
        outcomes=np.array(outcomes, dtype=np.int64),
    )
    print("wrote", len(calls), "calls")


if __name__ == "__main__":
    main()
