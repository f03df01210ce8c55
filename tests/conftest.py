"""Shared test helpers.  GPU tests are marked ``gpu``; everything else runs on
CPU (the driver runs ``pytest -m "not gpu"`` in the GPU-less build container
and ``pytest -m gpu`` on a B200)."""

from __future__ import annotations

import os
import random
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libbplb.so")


def random_reduced_pair(rng: random.Random, max_r: int = 12, max_c: int = 100):
    """conftest.py:18-21 of the reference, as (c, weights)."""
    c = rng.randint(1, max_c)
    r = rng.randint(0, max_r)
    return c, tuple(rng.randint(1, c) for _ in range(r))


def random_reduced(rng: random.Random, max_r: int = 12, max_c: int = 100):
    from paper_2402_14821_b200 import ReducedInstance

    c, w = random_reduced_pair(rng, max_r, max_c)
    return ReducedInstance(c=c, weights=w)


def brute_optimum(c: int, weights) -> int:
    """Exact minimum bin count by enumeration (oracle.py:34-75 shape), n <= 10."""
    ws = sorted(weights, reverse=True)
    n = len(ws)
    best = [n]
    loads: list[int] = []

    def place(i):
        if len(loads) >= best[0]:
            return
        if i == n:
            best[0] = len(loads)
            return
        w = ws[i]
        for j in range(len(loads)):
            if loads[j] + w <= c:
                loads[j] += w
                place(i + 1)
                loads[j] -= w
        loads.append(w)
        place(i + 1)
        loads.pop()

    place(0)
    return best[0] if n else 0


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.lib()
    return O
