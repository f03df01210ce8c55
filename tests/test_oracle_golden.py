"""Pin the C oracle (oracle/bplb_oracle.c) to golden vectors produced by the
reference itself (tests/golden/make_golden.py).  CPU only.

If these pass, the oracle is a faithful restatement of the reference on
every recorded input, and the GPU parity tests may use it as the checker
on fresh seeded inputs."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

KINDS = ("MT", "RAD2", "FS1", "CCM1", "VB2", "BJ1")


@pytest.fixture(scope="module")
def small():
    return np.load(os.path.join(GOLDEN, "small.npz"))


@pytest.fixture(scope="module")
def configs():
    return np.load(os.path.join(GOLDEN, "configs.npz"))


def _case(small, i):
    off = small["offsets"]
    return int(small["c"][i]), small["weights"][off[i]:off[i + 1]]


def test_small_vectors(small, oracle):
    meta, vals = small["vec_meta"], small["vec_vals"]
    for case, kid, lo, hi, o in meta:
        c, w = _case(small, case)
        assert oracle.lambda_range(KINDS[kid], c, w) == (lo, hi)
        got = oracle.dff_bound_batch(KINDS[kid], w, c, lo, hi)
        np.testing.assert_array_equal(got, vals[o:o + hi - lo + 1], err_msg=f"case {case} kind {KINDS[kid]}")


def test_small_seq(small, oracle):
    orders = json.loads(str(small["orders"]))
    for row in small["seq_rows"]:
        case, k, oi, lb, ex, evals, nd = (int(x) for x in row[:7])
        per = [int(x) for x in row[7:7 + nd]]
        c, w = _case(small, case)
        kinds = [KINDS[i] for i in orders[oi]]
        res = oracle.lower_bound_seq(w, c, k, kinds)
        assert res.lb == lb and res.exceeded_k == bool(ex) and res.evals == evals
        assert list(res.per_dff) == kinds[:nd]
        assert list(res.per_dff.values()) == per


def test_cfg1(configs, oracle):
    w = configs["cfg1_w"]
    res = oracle.lower_bound_seq(w, 150, 2**62)
    assert list(res.per_dff.values()) == list(configs["cfg1_best"])
    vec = np.concatenate([oracle.dff_bound_batch(k, w, 150, *oracle.lambda_range(k, 150, w)) for k in KINDS])
    np.testing.assert_array_equal(vec, configs["cfg1_vec"])


def test_cfg2_nodes(configs, oracle):
    from paper_2402_14821_b200 import workloads as W

    c, k, flat, off = W.cfg2_nodes(300)
    assert k == int(configs["cfg2_k"][0])
    lb, ex, best = oracle.check_batch(flat, off, c, 2**62, want_best=True)
    np.testing.assert_array_equal(best, configs["cfg2_best"])
    lbd, exd = oracle.check_batch(flat, off, c, k)
    np.testing.assert_array_equal(lbd, configs["cfg2_dec"][:, 0])
    np.testing.assert_array_equal(exd, configs["cfg2_dec"][:, 1].astype(bool))


@pytest.mark.parametrize("name", ["cfg3", "cfg3u"])
def test_cfg3_windows_and_best(configs, oracle, name):
    w = configs[f"{name}_w"]
    c = 100_000
    vals = configs[f"{name}_win_vals"]
    for kid, lo, hi, o in configs[f"{name}_win_meta"]:
        got = oracle.dff_bound_batch(KINDS[kid], w, c, lo, hi)
        np.testing.assert_array_equal(got, vals[o:o + hi - lo + 1])
    oracle.set_threads(oracle.max_threads())
    try:
        res = oracle.lower_bound_seq(w, c, 2**62)
    finally:
        oracle.set_threads(1)
    assert list(res.per_dff.values()) == list(configs[f"{name}_best"])


def test_cfg4_windows_and_nonvb2_best(configs, oracle):
    from paper_2402_14821_b200 import workloads as W

    c, w = W.cfg4()
    vals = configs["cfg4_win_vals"]
    for kid, lo, hi, o in configs["cfg4_win_meta"]:
        got = oracle.dff_bound_batch(KINDS[kid], w, c, lo, hi)
        np.testing.assert_array_equal(got, vals[o:o + hi - lo + 1])
    best = configs["cfg4_best_nonvb2"]
    oracle.set_threads(oracle.max_threads())
    try:
        for kid, kind in enumerate(KINDS):
            if kind == "VB2":
                continue
            lo, hi = oracle.lambda_range(kind, c, w)
            assert int(oracle.dff_bound_batch(kind, w, c, lo, hi).max()) == int(best[kid]), kind
    finally:
        oracle.set_threads(1)


def test_oracle_known_answers(oracle):
    # test_bounds.py / test_oracle.py KATs restated against the oracle
    assert oracle.dff_value("MT", 140, 150, 30) == 150
    assert oracle.dff_value("CCM1", 6, 10, 3) == 4
    assert oracle.dff_value("BJ1", 7, 10, 4) == 3
    assert oracle.dff_value("FS1", 5, 10, 3) == 15
    assert oracle.dff_value("VB2", 6, 10, 2) == 2
    assert oracle.dff_bound("MT", (6, 6, 6), 10, 4) == 2
    assert oracle.dff_bound("MT", (6, 6, 6), 10, 5) == 3
    assert oracle.dff_bound("FS1", (5, 5), 10, 3) == 1
    assert oracle.lambda_range("RAD2", 150) == (38, 50)
    assert oracle.lambda_range("RAD2", 4)[0] > oracle.lambda_range("RAD2", 4)[1]
    res = oracle.lower_bound_seq((6, 6, 6), 10, 1)
    assert res.exceeded_k and list(res.per_dff) == ["MT"]
    res = oracle.lower_bound_seq((6, 6, 6), 10, 3)
    assert res.lb == 3 and not res.exceeded_k


def test_oracle_pins_dffstats_golden(oracle):
    """The C oracle's per-kind maxima equal the reference's root bounds in
    tests/golden/dffstats.json (the fixture of the batched dffstats test)."""
    import json
    import os

    with open(os.path.join(GOLDEN, "dffstats.json")) as f:
        g = json.load(f)
    kinds = ("MT", "RAD2", "FS1", "CCM1", "VB2", "BJ1")
    for x, roots in zip(g["instances"], g["root_bounds"]):
        w = np.asarray(x["weights"], dtype=np.int64)
        _, _, best = oracle.check_batch(w, np.array([0, len(w)]), x["c"], 2**62, want_best=True)
        assert {k: int(best[0, i]) for i, k in enumerate(kinds)} == roots, x["name"]


def test_oracle_pins_cfg5_reference_golden(oracle):
    """96 nodes of the cfg5 headline batch (native generator, spread over all
    10^6 nodes) with the reference's lower_bound_seq outputs
    (tests/golden/make_golden_cfg5.py): full-mode per-kind maxima and
    decision-mode (k = 334) lb / exceeded; the committed node weights are the
    generator's output (regenerated here)."""
    import os

    from paper_2402_14821_b200 import workloads as W

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "cfg5_ref.npz"))
    c, k, w = W.cfg5_instance()
    assert int(g["c"]) == c and int(g["k"]) == k
    off = g["offsets"]
    for j, i in enumerate(g["node_ids"][::8]):
        f, o = W.gen_nodes_host(w, c, k, W.CFG5_SEED, 1, first_node=int(i))
        np.testing.assert_array_equal(f, g["weights"][off[8 * j]:off[8 * j + 1]])
    oracle.set_threads(oracle.max_threads())
    lb, ex, best = oracle.check_batch(g["weights"], off, c, 2**62, want_best=True)
    np.testing.assert_array_equal(best, g["best"])
    np.testing.assert_array_equal(lb, g["lb"])
    lb, ex = oracle.check_batch(g["weights"], off, c, k)
    np.testing.assert_array_equal(lb, g["dec_lb"])
    np.testing.assert_array_equal(ex, g["dec_exceeded"].astype(bool))
