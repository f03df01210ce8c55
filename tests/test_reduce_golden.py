"""reduce_packing (instances.py:262-282) pinned to the REFERENCE's own outputs
(tests/golden/reduce_ref.npz, made by tests/golden/make_golden_reduce.py from
partial packings built through the reference's DomainStore: commits and
candidate removals, including overloaded bins -> ValueError).

CPU: the host restatement (instances.reduce_packing_arrays).  GPU: the
device reduction (bplb_reduce_batch, the front of bplb_check_batch_assign) on
the same states, one batch per (c, k)."""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLDEN, "reduce_ref.npz"))


def _case(g, i):
    w = g["w"][g["woff"][i]:g["woff"][i + 1]]
    a = g["asg"][g["woff"][i]:g["woff"][i + 1]]
    red = None if g["error"][i] else g["red"][g["roff"][i]:g["roff"][i + 1]]
    return int(g["c"][i]), int(g["k"][i]), w, a, red


def test_host_restatement_matches_reference(gold):
    from paper_2402_14821_b200.instances import reduce_packing_arrays

    n_err = 0
    for i in range(len(gold["c"])):
        c, k, w, a, red = _case(gold, i)
        if red is None:
            n_err += 1
            with pytest.raises(ValueError):
                reduce_packing_arrays(w, a, k, c)
        else:
            np.testing.assert_array_equal(reduce_packing_arrays(w, a, k, c), red)
    assert n_err > 0


@pytest.mark.gpu
def test_device_reduction_matches_reference(gold):
    from paper_2402_14821_b200.batch import reduce_packing_batch

    for i in range(len(gold["c"])):
        c, k, w, a, red = _case(gold, i)
        asg = np.where(a < 0, 0xFFFF, a).astype(np.uint16)[None, :]
        if red is None:
            with pytest.raises(ValueError):
                reduce_packing_batch(c, w, asg, k)
            continue
        rw, roff = reduce_packing_batch(c, w, asg, k)
        assert roff.tolist() == [0, len(red)]
        np.testing.assert_array_equal(rw, red)
    # several states of one instance shape in one batch (same c, k, n)
    idx = [i for i in range(len(gold["c"])) if not gold["error"][i]]
    by_shape = {}
    for i in idx:
        c, k, w, a, red = _case(gold, i)
        by_shape.setdefault((c, k, tuple(w)), []).append((a, red))
    for (c, k, w), rows in by_shape.items():
        if len(rows) < 2:
            continue
        asg = np.stack([np.where(a < 0, 0xFFFF, a).astype(np.uint16) for a, _ in rows])
        rw, roff = reduce_packing_batch(c, np.array(w, np.int32), asg, k)
        for j, (_, red) in enumerate(rows):
            np.testing.assert_array_equal(rw[roff[j]:roff[j + 1]], red)
