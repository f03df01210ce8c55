"""Golden fixture for the batched dffstats path, produced by the REFERENCE.

Run in the build container (the reference is importable only here):
    python tests/golden/make_golden_dffstats.py

Builds 60 small seeded instances (three capacities, so the batched path
groups them), fake optima around the root L2 bound, and records the
reference's own ``binpack.cli._root_bounds`` per instance and
``binpack.cli.dffstats_table`` (cli.py:334-370) into dffstats.json.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from binpack.cli import _root_bounds, dffstats_table  # noqa: E402  (reference)
from binpack.bounds import DEFAULT_DFF_ORDER  # noqa: E402
from binpack.instances import Instance  # noqa: E402


def main():
    rng = np.random.default_rng(2024)
    insts, optima = [], {}
    for i in range(60):
        c = [150, 1000, 10_007][i % 3]
        n = int(rng.integers(5, 80))
        lo = max(1, c // 20)
        w = tuple(int(x) for x in rng.integers(lo, c + 1, n))
        name = f"g{i:02d}"
        inst = Instance(c=c, weights=w, name=name)
        insts.append(inst)
        rb = _root_bounds(inst, DEFAULT_DFF_ORDER)
        optima[name] = max(rb.values()) + int(rng.integers(0, 2))
    table = dffstats_table(insts, optima, DEFAULT_DFF_ORDER)
    roots = [{k.name: v for k, v in _root_bounds(x, DEFAULT_DFF_ORDER).items()} for x in insts]
    out = {"instances": [{"name": x.name, "c": x.c, "weights": list(x.weights)} for x in insts],
           "optima": optima, "root_bounds": roots, "table": table}
    with open(os.path.join(HERE, "dffstats.json"), "w") as f:
        json.dump(out, f)
    print("wrote", len(insts), "instances")


if __name__ == "__main__":
    main()
