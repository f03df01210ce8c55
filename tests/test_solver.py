"""Solver integration: the GPU engine plugged into the
reference's search through the ``dffs-gpu`` bound mode.

Fixture tests/golden/solver_calls.npz (tests/golden/make_golden_solver.py)
records every ``engine(red, k)`` call the REFERENCE's ``minimize``
(search.py:339-381) makes with ``BoundMode.DFFS_SEQ`` -- the root call
(search.py:352) and the feasibility checks of ``propagate``
(propagator.py:266-276) -- on 29 small Falkenauer-U / Scholl / triplet
instances (33 of the 929 calls are bound failures, lb > k), plus each
solve's bins / nodes / fails / bound_calls.

* CPU: the oracle reproduces every recorded call; the reference search
  (installed copy in baseline/_ref) run through ``install_dffs_gpu`` with the
  oracle injected as the engine reproduces every recorded outcome (shim
  mechanics, CLI parsing of ``--bound dffs-gpu``).
* GPU: ``GpuBoundEngine(mode="seq")`` reproduces every recorded call in
  order (lb, exceeded_k, evals, per_dff keys / order / values) -- hence the
  same search -- and the reference search end to end with the B200 engine
  (``--bound dffs-gpu``) gives the recorded node counts.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

REF_SITE = os.path.join(ROOT, "baseline", "_ref")
KIND_NAMES = ("MT", "RAD2", "FS1", "CCM1", "VB2", "BJ1")


@pytest.fixture(scope="module")
def calls():
    return np.load(os.path.join(GOLDEN, "solver_calls.npz"))


def _ref():
    """The reference package installed in baseline/_ref (skip if absent)."""
    if not os.path.isdir(os.path.join(REF_SITE, "binpack")):
        pytest.skip("baseline/_ref (reference install) not present")
    if REF_SITE not in sys.path:
        sys.path.insert(0, REF_SITE)
    from binpack import cli, search
    from binpack.instances import Instance

    return search, cli, Instance


def _instances(g, Instance):
    off = g["inst_off"]
    return [Instance(int(c), tuple(int(x) for x in g["inst_w"][off[i]:off[i + 1]]))
            for i, c in enumerate(g["inst_c"])]


def _call(g, i):
    off = g["call_off"]
    return int(g["call_c"][i]), g["call_w"][off[i]:off[i + 1]], int(g["call_k"][i])


def _want(g, i):
    order = [int(x) for x in g["call_order"][i] if x >= 0]
    per = {KIND_NAMES[j]: int(g["call_per_dff"][i, j]) for j in order}
    return int(g["call_lb"][i]), bool(g["call_exceeded"][i]), int(g["call_evals"][i]), per


class _OracleEngine:
    """Test-only BoundEngine backed by the C oracle (lower_bound_seq)."""

    def __init__(self, kinds):
        self.kinds = [k.name for k in kinds]
        self.n = 0

    def __call__(self, red, k):
        from oracle import oracle as O

        self.n += 1
        return O.lower_bound_seq(np.asarray(red.weights, dtype=np.int64), red.c, k, self.kinds)


def test_oracle_reproduces_recorded_calls(calls, oracle):
    for i in range(len(calls["call_k"])):
        c, w, k = _call(calls, i)
        r = oracle.lower_bound_seq(w, c, k)
        lb, ex, ev, per = _want(calls, i)
        assert (r.lb, r.exceeded_k, r.evals) == (lb, ex, ev), i
        assert list(r.per_dff.items()) == list(per.items()), i


def test_install_shim_reproduces_reference_solves(calls):
    """The shim routes ``dffs-gpu`` to the injected factory and leaves the
    other modes on the reference's own factory; the search through it makes
    the recorded number of nodes / fails / bound calls."""
    search, cli, Instance = _ref()
    from paper_2402_14821_b200.solver import DFFS_GPU, BoundModeGPU, install_dffs_gpu

    made = []

    def factory(cfg):
        e = _OracleEngine(cfg.dff_order)
        made.append(e)
        return e, lambda: None

    undo = install_dffs_gpu(search, cli, factory=factory)
    try:
        insts = _instances(calls, Instance)
        for row in calls["outcomes"]:
            i, c, bins, nodes, fails, bound_calls, solved = (int(x) for x in row)
            cfg = search.SearchConfig(bound_mode=BoundModeGPU.from_name(DFFS_GPU), time_limit=120.0)
            res = search.minimize(insts[i], cfg)
            assert (res.bins, res.stats.nodes, res.stats.fails, res.stats.bound_calls) == \
                   (bins, nodes, fails, bound_calls), insts[i]
        assert sum(e.n for e in made) == len(calls["call_k"])
        # the reference modes still go to the reference factory
        cfg = search.SearchConfig(bound_mode=BoundModeGPU.DFFS_SEQ, time_limit=30.0)
        n_made = len(made)
        res = search.minimize(insts[0], cfg)
        assert len(made) == n_made and res.bins == int(calls["outcomes"][0][2])
        # cli: --bound dffs-gpu parses to the GPU mode
        import argparse

        p = argparse.ArgumentParser()
        cli._add_solver_flags(p, 10.0)
        args = p.parse_args(["--bound", "dffs-gpu"])
        assert cli._config_from_args(args).bound_mode is BoundModeGPU.DFFS_GPU
    finally:
        undo()
    assert search.make_bound_engine.__module__ == "binpack.search"


@pytest.mark.gpu
def test_gpu_engine_replays_recorded_calls(calls):
    """Every recorded solver call through the B200 engine (lower_bound_seq
    semantics): identical BoundResult fields in order."""
    from paper_2402_14821_b200 import ReducedInstance
    from paper_2402_14821_b200.solver import make_gpu_bound_engine

    eng, close = make_gpu_bound_engine()
    try:
        for i in range(len(calls["call_k"])):
            c, w, k = _call(calls, i)
            r = eng(ReducedInstance(c, tuple(int(x) for x in w)), k)
            lb, ex, ev, per = _want(calls, i)
            assert (r.lb, r.exceeded_k, r.evals) == (lb, ex, ev), i
            assert [(kd.name, v) for kd, v in r.per_dff.items()] == list(per.items()), i
    finally:
        close()


@pytest.mark.gpu
def test_reference_search_with_dffs_gpu(calls):
    """The reference's minimize with ``--bound dffs-gpu`` (the B200 engine
    inside propagate) makes exactly the recorded dffs-seq search."""
    search, cli, Instance = _ref()
    from paper_2402_14821_b200.solver import BoundModeGPU, install_dffs_gpu

    undo = install_dffs_gpu(search, cli)
    try:
        insts = _instances(calls, Instance)
        for row in calls["outcomes"]:
            i, c, bins, nodes, fails, bound_calls, solved = (int(x) for x in row)
            cfg = search.SearchConfig(bound_mode=BoundModeGPU.DFFS_GPU, time_limit=120.0)
            res = search.minimize(insts[i], cfg)
            assert (res.bins, res.stats.nodes, res.stats.fails, res.stats.bound_calls) == \
                   (bins, nodes, fails, bound_calls), i
    finally:
        undo()
