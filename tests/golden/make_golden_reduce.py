"""Goldens for reduce_packing (instances.py:262-282), produced by the REFERENCE.

Run in the build container (the reference is importable only here):
    python tests/golden/make_golden_reduce.py

Random instances and random partial packings built through the reference's
own DomainStore (store.py): items committed to bins (commit) and items whose
candidate set is narrowed to one bin (remove_bin) -- both count as assigned
(is_assigned: a single candidate), including overloaded bins, for which
reduce_packing raises ValueError.  Recorded per state: the assignment vector
(bin, or -1 while open) and the reference's reduced weights, or the error.
Output: tests/golden/reduce_ref.npz (read by tests/test_reduce_golden.py).
"""

from __future__ import annotations

import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from binpack.instances import Instance, reduce_packing  # noqa: E402  (reference)
from binpack.store import DomainStore, Wipeout  # noqa: E402


def main() -> None:
    rng = random.Random(77)
    cases = []  # (c, k, inst weights, assignment, reduced or None)
    for case in range(150):
        c = rng.choice([1, 2, 7, 100, 150, 151, 1000, 99991, 100000])
        n = rng.randint(1, 60)
        k = rng.randint(1, 40)
        w = [rng.randint(1, c) for _ in range(n)]
        for _state in range(3):  # three search-node states of the same instance
            st = DomainStore(tuple(w), c, k)
            try:
                for _ in range(rng.randint(0, 2 * n)):
                    i = rng.randrange(n)
                    if rng.random() < 0.6:
                        j = rng.randrange(k)
                        # mostly feasible commits; a few overload a bin (reduce_packing's error)
                        fits = st.committed_load[j] + w[i] <= c or rng.random() < 0.03
                        if st.has_candidate(i, j) and not st.is_assigned(i) and fits:
                            st.commit(i, j)
                    else:
                        cands = list(st.candidates(i))
                        if len(cands) > 1:
                            st.remove_bin(i, rng.choice(cands))
            except Wipeout:
                continue
            asg = [st.assigned_bin(i) if st.is_assigned(i) else -1 for i in range(n)]
            try:
                red = list(reduce_packing(Instance(c, tuple(w)), st).weights)
            except ValueError:
                red = None
            cases.append((c, k, w, asg, red))
    ok = [x for x in cases if x[4] is not None]
    print(f"{len(cases)} states, {len(cases) - len(ok)} raise ValueError (overloaded bin)")
    woff = np.zeros(len(cases) + 1, dtype=np.int64)
    woff[1:] = np.cumsum([len(x[2]) for x in cases])
    roff = np.zeros(len(cases) + 1, dtype=np.int64)
    roff[1:] = np.cumsum([len(x[4]) if x[4] is not None else 0 for x in cases])
    np.savez_compressed(
        os.path.join(HERE, "reduce_ref.npz"),
        c=np.array([x[0] for x in cases], dtype=np.int64), k=np.array([x[1] for x in cases], dtype=np.int64),
        w=np.concatenate([np.array(x[2], dtype=np.int32) for x in cases]), woff=woff,
        asg=np.concatenate([np.array(x[3], dtype=np.int64) for x in cases]),
        red=np.concatenate([np.array(x[4] or [], dtype=np.int64) for x in cases]), roff=roff,
        error=np.array([x[4] is None for x in cases], dtype=bool),
    )


if __name__ == "__main__":
    main()
