"""GPU parity: the CUDA path (through the C ABI / drop-in API) against the
golden vectors recorded from the reference and against the pinned C oracle
on fresh seeded inputs.  Bit-exact equality everywhere (all integer)."""

from __future__ import annotations

import json
import os
import random

import numpy as np
import pytest

import paper_2402_14821_b200 as G
from paper_2402_14821_b200 import DffKind, ReducedInstance, workloads as W
from conftest import GOLDEN, random_reduced_pair

pytestmark = pytest.mark.gpu
KINDS = ("MT", "RAD2", "FS1", "CCM1", "VB2", "BJ1")


@pytest.fixture(scope="module")
def small():
    return np.load(os.path.join(GOLDEN, "small.npz"))


@pytest.fixture(scope="module")
def configs():
    return np.load(os.path.join(GOLDEN, "configs.npz"))


def _case(small, i):
    off = small["offsets"]
    return int(small["c"][i]), tuple(int(x) for x in small["weights"][off[i]:off[i + 1]])


def test_small_vectors_golden(small):
    meta, vals = small["vec_meta"], small["vec_vals"]
    for case, kid, lo, hi, o in meta:
        c, w = _case(small, case)
        red = ReducedInstance(c, w)
        got = G.dff_bound_batch(DffKind[KINDS[kid]], red, int(lo), int(hi))
        np.testing.assert_array_equal(got, vals[o:o + hi - lo + 1], err_msg=f"case {case} {KINDS[kid]} c={c} w={w}")


def test_small_seq_golden(small):
    orders = json.loads(str(small["orders"]))
    for row in small["seq_rows"]:
        case, k, oi, lb, ex, evals, nd = (int(x) for x in row[:7])
        per = [int(x) for x in row[7:7 + nd]]
        c, w = _case(small, case)
        kinds = [DffKind[KINDS[i]] for i in orders[oi]]
        res = G.lower_bound_seq(ReducedInstance(c, w), k, kinds)
        assert (res.lb, res.exceeded_k, res.evals) == (lb, bool(ex), evals), (case, k, oi)
        assert list(res.per_dff) == kinds[:nd]
        assert list(res.per_dff.values()) == per


def test_small_par_golden(small):
    for row in small["par_rows"]:
        case, lb, evals, mask = (int(x) for x in row[:4])
        c, w = _case(small, case)
        res = G.lower_bound_par(ReducedInstance(c, w), 5, workers=1, cancellation=False)
        assert res.lb == lb and res.evals == evals
        want = {DffKind[KINDS[i]]: int(row[4 + i]) for i in range(6) if mask >> i & 1}
        assert res.per_dff == want


def test_batch_matches_single(small):
    """All golden small cases as one CSR batch: per-node best == singles."""
    n = len(small["c"])
    # batch API needs one capacity: group by c
    by_c: dict[int, list[int]] = {}
    for i in range(n):
        by_c.setdefault(int(small["c"][i]), []).append(i)
    meta = small["vec_meta"]
    vals = small["vec_vals"]
    best_ref = {}
    for case, kid, lo, hi, o in meta:
        best_ref[(int(case), int(kid))] = int(vals[o:o + hi - lo + 1].max())
    for c, cases in by_c.items():
        nodes = [_case(small, i)[1] for i in cases]
        w, off = G.csr_from_lists(nodes)
        lb, ex, best, arg = G.lower_bound_batch(c, w, off, 2**62, want_best=True)
        for j, case in enumerate(cases):
            for kid in range(6):
                assert best[j, kid] == best_ref.get((case, kid), 0), (case, kid, c)


def test_cfg1(configs):
    c, w = W.cfg1()
    red = ReducedInstance.from_array(c, w)
    res = G.lower_bound_seq(red, 2**62)
    assert [res.per_dff[k] for k in G.DEFAULT_DFF_ORDER] == list(configs["cfg1_best"])
    vec = np.concatenate([G.dff_bound_batch(k, red, *(lambda r: (r.lo, r.hi))(G.lambda_range(k, c, red)))
                          for k in G.DEFAULT_DFF_ORDER])
    np.testing.assert_array_equal(vec, configs["cfg1_vec"])
    dec = G.lower_bound_seq(red, res.lb - 1)
    assert dec.exceeded_k and dec.lb == int(configs["cfg1_l2m1"][0]) and list(dec.per_dff) == [DffKind.MT]


@pytest.mark.parametrize("mode", ["full", "seq", "cancel"])
def test_cfg2_nodes(configs, mode):
    c, k, flat, off = W.cfg2_nodes(300)
    if mode == "full":
        lb, ex, best, arg = G.lower_bound_batch(c, flat, off, 2**62, want_best=True)
        np.testing.assert_array_equal(best, configs["cfg2_best"])
        np.testing.assert_array_equal(lb, configs["cfg2_best"].max(axis=1))
    else:
        lb, ex = G.lower_bound_batch(c, flat, off, k, mode=mode)
        np.testing.assert_array_equal(ex, configs["cfg2_dec"][:, 1].astype(bool))
        if mode == "seq":
            np.testing.assert_array_equal(lb, configs["cfg2_dec"][:, 0])


@pytest.mark.parametrize("name", ["cfg3", "cfg3u"])
def test_cfg3(configs, name):
    w = configs[f"{name}_w"].astype(np.int32)
    c = 100_000
    red = ReducedInstance.from_array(c, w)
    vals = configs[f"{name}_win_vals"]
    for kid, lo, hi, o in configs[f"{name}_win_meta"]:
        got = G.dff_bound_batch(DffKind[KINDS[kid]], red, int(lo), int(hi))
        np.testing.assert_array_equal(got, vals[o:o + hi - lo + 1], err_msg=KINDS[kid])
    res = G.lower_bound_seq(red, 2**62)
    assert [res.per_dff[k] for k in G.DEFAULT_DFF_ORDER] == list(configs[f"{name}_best"])
    par = G.lower_bound_par(red, 2**62, cancellation=False)
    assert [par.per_dff[k] for k in G.DEFAULT_DFF_ORDER] == list(configs[f"{name}_best"])


def test_cfg4(configs):
    c, w = W.cfg4()
    red = ReducedInstance.from_array(c, w)
    vals = configs["cfg4_win_vals"]
    for kid, lo, hi, o in configs["cfg4_win_meta"]:
        got = G.dff_bound_batch(DffKind[KINDS[kid]], red, int(lo), int(hi))
        np.testing.assert_array_equal(got, vals[o:o + hi - lo + 1], err_msg=KINDS[kid])
    res = G.lower_bound_par(red, 2**62, cancellation=False)
    best = configs["cfg4_best_nonvb2"]
    for kid, kind in enumerate(G.DEFAULT_DFF_ORDER):
        if kind is DffKind.VB2:
            continue
        assert res.per_dff[kind] == int(best[kid]), kind
    vb2_path = os.path.join(GOLDEN, "cfg4_vb2.npz")
    if os.path.exists(vb2_path):
        vb = np.load(vb2_path)["cfg4_vb2_best"]
        assert res.per_dff[DffKind.VB2] == int(vb[0])
        assert res.arg[DffKind.VB2] == int(vb[1])


def test_cfg5_nodes(configs):
    c, k, flat, off = W.cfg5_nodes(12)
    lb, ex, best, arg = G.lower_bound_batch(c, flat, off, 2**62, want_best=True)
    np.testing.assert_array_equal(best, configs["cfg5_best"])


# ---------------------------------------------------------------------------
# Fresh seeded inputs against the pinned oracle
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("max_c,max_r,n", [(150, 40, 300), (5000, 300, 60), (200_000, 800, 12),
                                           (4094, 2000, 20), (4096, 3000, 10)])
def test_random_vs_oracle(oracle, max_c, max_r, n):
    rng = random.Random(max_c * 7 + max_r)
    for _ in range(n):
        c, w = random_reduced_pair(rng, max_r, max_c)
        red = ReducedInstance(c, w)
        got = G.lower_bound_seq(red, 2**62)
        want = oracle.lower_bound_seq(w, c, 2**62)
        assert {k.name: v for k, v in got.per_dff.items()} == want.per_dff, (c, len(w))
        assert {k.name: v for k, v in got.arg.items()} == want.arg, (c, len(w))


@pytest.mark.parametrize("max_c,max_r,n", [(200_000, 800, 12), (60_000, 2000, 8), (4096, 3000, 10),
                                           (1_000_000, 600, 6)])
def test_random_full_collection_vs_oracle(oracle, max_c, max_r, n):
    """Full-collection single checks (lower_bound_par without cancellation):
    the bound-pruned multi-CTA node kernel / grid-wide path, per-kind best and
    arg lambda against the oracle's full sweep."""
    rng = random.Random(max_c * 11 + max_r)
    for _ in range(n):
        c, w = random_reduced_pair(rng, max_r, max_c)
        red = ReducedInstance(c, w)
        got = G.lower_bound_par(red, 2**62, cancellation=False)
        want = oracle.lower_bound_seq(w, c, 2**62)
        assert {k.name: v for k, v in got.per_dff.items()} == want.per_dff, (c, len(w))
        assert {k.name: v for k, v in got.arg.items()} == want.arg, (c, len(w))
        assert got.lb == want.lb


def test_random_batch_vs_oracle(oracle):
    rng = np.random.default_rng(7)
    for c in (1, 2, 3, 7, 8, 150, 1000, 4094, 4095, 65536, 100_000, 999_983):
        n = 64
        lens = rng.integers(0, 300, n)
        lens[0] = 0
        nodes = []
        for L in lens:
            x = rng.integers(1, c + 1, L)
            if L > 2:
                x[0] = c
                if c % 2 == 0:
                    x[1] = c // 2
            nodes.append(x)
        w, off = G.csr_from_lists(nodes)
        lb, ex, best, arg = G.lower_bound_batch(c, w, off, 2**62, want_best=True)
        lbo, exo, besto = oracle.check_batch(w, off, c, 2**62, want_best=True)
        np.testing.assert_array_equal(best, besto, err_msg=f"c={c}")
        np.testing.assert_array_equal(lb, lbo)
        kk = int(np.median(lbo))
        lb2, ex2 = G.lower_bound_batch(c, w, off, kk, mode="seq")
        lbo2, exo2 = oracle.check_batch(w, off, c, kk)
        np.testing.assert_array_equal(lb2, lbo2)
        np.testing.assert_array_equal(ex2, exo2)
        lb3, ex3 = G.lower_bound_batch(c, w, off, kk, mode="cancel")
        np.testing.assert_array_equal(ex3, exo2)
        assert (lb3[~ex3] == lbo2[~exo2]).all()


def test_invalid_weight_raises():
    with pytest.raises(ValueError):
        G.lower_bound_batch(10, np.array([3, 11], dtype=np.int32), np.array([0, 2]), 5)
    with pytest.raises(ValueError):
        G.dff_bound_batch(DffKind.MT, (10, np.array([0, 4], dtype=np.int32)), 0, 3)


def test_launch_counter_moves():
    from paper_2402_14821_b200 import _native

    eng = _native.default_engine()
    before = eng.launch_count()
    G.lower_bound_seq(ReducedInstance(10, (6, 6, 6)), 3)
    assert eng.launch_count() > before


def test_compact_weight_dtypes(oracle):
    """uint16 / uint8 CSR weights give the same verdicts as int32."""
    c, k, flat, off = W.cfg2_nodes(300)
    ref = G.lower_bound_batch(c, flat, off, 2**62, want_best=True)
    for dt in (np.uint16, np.uint8):
        got = G.lower_bound_batch(c, flat.astype(dt), off, 2**62, want_best=True)
        for a, b in zip(ref, got):
            np.testing.assert_array_equal(a, b)
    rng = np.random.default_rng(3)
    c2 = 60000
    nodes = [rng.integers(1, c2 + 1, int(L)) for L in rng.integers(0, 400, 40)]
    w, off2 = G.csr_from_lists(nodes)
    lb16, ex16 = G.lower_bound_batch(c2, w.astype(np.uint16), off2, 2**62)
    lbo, exo = oracle.check_batch(w, off2, c2, 2**62)
    np.testing.assert_array_equal(lb16, lbo)
    with pytest.raises(ValueError):  # 0 is not a valid weight
        G.lower_bound_batch(10, np.array([0, 3], dtype=np.uint8), np.array([0, 2]), 5)


# ---------------------------------------------------------------------------
# Batched small-capacity path (histogram x table kernel, bplb_tab.cuh)
# ---------------------------------------------------------------------------
def _tab_batch(rng, c, n, max_r):
    lens = rng.integers(0, max_r + 1, n)
    lens[:3] = [0, 1, max_r]
    nodes = []
    for L in lens:
        x = rng.integers(1, c + 1, L)
        if L > 2:
            x[0] = c
            if c % 2 == 0:
                x[1] = c // 2
        nodes.append(x)
    return G.csr_from_lists(nodes)


TAB_ENVELOPE = 1 << 23  # max_r * max f < 2^23 (csrc/bplb_capi.cu tab_path)


def _tab_case(oracle, c, max_r, kinds, n=517, seed=None):
    """One table-path batch against the oracle (all outputs, three modes) and
    against the warp-per-node kernel (arg lambdas, per-kind best); asserts the
    table kernel actually served every call (bplb_last_path)."""
    from paper_2402_14821_b200 import _native

    rng = np.random.default_rng(c if seed is None else seed)
    w, off = _tab_batch(rng, c, n, max_r)
    eng = _native.default_engine()
    lb, ex, best, arg = eng.check_batch(w, off, c, 2**62, kinds, 0, want_best=True)
    path = eng.last_path()
    assert path[0] in ("tab", "tc"), path
    # the tensor-core contraction and the FP32-pipe contraction: identical outputs
    fp = eng.check_batch(w, off, c, 2**62, kinds, _native.F_NOTC, want_best=True)
    assert eng.last_path()[0] == "tab" and eng.last_path()[1] >= 2
    for a, b in zip((lb, ex, best, arg), fp):
        np.testing.assert_array_equal(a, b)
    lbo, exo, besto = oracle.check_batch(w, off, c, 2**62, want_best=True, kinds=kinds)
    np.testing.assert_array_equal(best[:, kinds], besto, err_msg=f"c={c}")
    np.testing.assert_array_equal(lb, lbo)
    # same arg-lambdas as the dense warp-per-node kernel
    lbw, exw, bestw, argw = eng.check_batch(w, off, c, 2**62, kinds, _native.F_NOTAB | _native.F_NOPRUNE,
                                            want_best=True)
    assert eng.last_path()[0] == "warp"
    np.testing.assert_array_equal(arg, argw)
    np.testing.assert_array_equal(best, bestw)
    kk = int(np.median(lbo))
    for mode, fl in (("seq", _native.F_PHASED), ("cancel", _native.F_CANCEL)):
        got = eng.check_batch(w, off, c, kk, kinds, fl, want_best=True)
        assert eng.last_path()[0] in ("tab", "tc")
        lbo2, exo2 = oracle.check_batch(w, off, c, kk, kinds=kinds)
        np.testing.assert_array_equal(got[1], exo2)
        if mode == "seq":
            np.testing.assert_array_equal(got[0], lbo2)
        # kinds in order with the same guard as the warp kernel: identical outputs
        ref = eng.check_batch(w, off, c, kk, kinds, fl | _native.F_NOTAB | _native.F_NOPRUNE, want_best=True)
        for a, b in zip(got, ref):
            np.testing.assert_array_equal(a, b)
    return path


@pytest.mark.parametrize("c", [1, 2, 3, 7, 8, 100, 150, 151, 200, 255, 280, 288])
def test_tab_batch_vs_oracle(oracle, c):
    """The table kernel (>= 256 nodes, small c) against the oracle in all
    three modes, with ragged node sizes (r = 0 included) and a partial tile,
    at the fp32 envelope edge (max_r * 101c just below 2^23)."""
    max_r = min(500, (TAB_ENVELOPE - 1) // (101 * c))
    _tab_case(oracle, c, max_r, list(range(6)))


@pytest.mark.parametrize("c", [200, 255, 288])
def test_tab_batch_large_c_without_fs1(oracle, c):
    """Without FS1 (max f = 2c) nodes of 500 items stay inside the envelope:
    the 4-6-warp contraction CTAs of the largest capacities, with max_r = 500
    and at the envelope edge."""
    kinds = [0, 1, 3, 4, 5]
    widths = set()
    # (nodes above 16384 items leave the node-resident paths: per-node grid-wide checks)
    for max_r in (500, min(16384, (TAB_ENVELOPE - 1) // (2 * c))):
        widths.add(_tab_case(oracle, c, max_r, kinds, n=300, seed=c + max_r)[1])
    assert widths


def test_tab_kind_subsets_and_orders():
    """Kind subsets / orders (the table is re-tabulated per kind mask) match
    the warp-per-node kernel, every output."""
    from paper_2402_14821_b200 import _native

    eng = _native.default_engine()
    rng = np.random.default_rng(11)
    w, off = _tab_batch(rng, 150, 300, 400)
    for kinds in ([4], [2, 0], [5, 3, 1], [1], [3, 4, 5, 0, 1, 2]):
        for fl in (0, _native.F_PHASED, _native.F_CANCEL):
            got = eng.check_batch(w, off, 150, 190, kinds, fl, want_best=True)
            ref = eng.check_batch(w, off, 150, 190, kinds, fl | _native.F_NOTAB | _native.F_NOPRUNE,
                                  want_best=True)
            for a, b in zip(got, ref):
                np.testing.assert_array_equal(a, b, err_msg=f"{kinds} {fl}")


def test_tab_exactness_envelope_fallback(oracle):
    """Nodes too large for exact fp32 sums (max_r * 101 c > 2^24) take the
    integer kernels; results are unchanged."""
    rng = np.random.default_rng(5)
    c = 250
    nodes = [rng.integers(1, c + 1, 700) for _ in range(260)]
    w, off = G.csr_from_lists(nodes)
    lb, ex = G.lower_bound_batch(c, w, off, 2**62)
    lbo, exo = oracle.check_batch(w, off, c, 2**62)
    np.testing.assert_array_equal(lb, lbo)


def test_tab_large_batch_device_api(oracle):
    """10^4 cfg2 nodes through the device-resident entry (the bench path)."""
    import torch

    from paper_2402_14821_b200 import _native

    c, k, flat, off = W.cfg2_nodes(10_000)
    eng = _native.default_engine()
    dev = torch.device("cuda", 0)
    d_w = torch.from_numpy(flat.astype(np.uint8)).to(dev)
    d_off = torch.from_numpy(off).to(dev)
    d_lb = torch.empty(len(off) - 1, dtype=torch.int64, device=dev)
    d_ex = torch.empty(len(off) - 1, dtype=torch.uint8, device=dev)
    eng.check_batch_device(d_w.data_ptr(), d_off.data_ptr(), len(off) - 1, int(np.diff(off).max()), c,
                           2**62, list(range(6)), 0, d_lb.data_ptr(), d_ex.data_ptr(), wbytes=1)
    torch.cuda.synchronize()
    lb = d_lb.cpu().numpy()
    m = 1500
    lbo, _ = oracle.check_batch(flat[:off[m]], off[:m + 1], c, 2**62)
    np.testing.assert_array_equal(lb[:m], lbo)
    lbh, _ = G.lower_bound_batch(c, flat, off, 2**62)
    np.testing.assert_array_equal(lb, lbh)


# ---------------------------------------------------------------------------
# Device-side reduce_packing of node states (bplb_reduce.cuh)
# ---------------------------------------------------------------------------
def _random_assignments(rng, n, k, c, n_nodes, dtype=np.uint8):
    w = rng.integers(1, c // 3 + 1, n)
    openv = np.iinfo(dtype).max
    a = np.full((n_nodes, n), openv, dtype=dtype)
    for r in range(n_nodes):
        loads = np.zeros(k, dtype=np.int64)
        depth = rng.integers(0, n + 1)
        for i in rng.permutation(n)[:depth]:
            j = rng.integers(0, k)
            if loads[j] + w[i] <= c:
                loads[j] += w[i]
                a[r, i] = j
    return w.astype(np.int32), a


@pytest.mark.parametrize("c,n,k,dt", [(150, 500, 209, np.uint8), (1000, 300, 120, np.uint8),
                                      (100_000, 200, 300, np.uint16), (7, 40, 30, np.uint8)])
def test_reduce_batch_matches_reduce_packing(c, n, k, dt):
    """Device reduction == reduce_packing_arrays (reference order) per node."""
    from paper_2402_14821_b200.instances import reduce_packing_arrays

    rng = np.random.default_rng(c + n)
    w, a = _random_assignments(rng, n, k, c, 120, dt)
    flat, off = G.reduce_packing_batch(c, w, a, k)
    openv = np.iinfo(dt).max
    for i in range(a.shape[0]):
        asg = np.where(a[i] == openv, -1, a[i].astype(np.int64))
        np.testing.assert_array_equal(flat[off[i]:off[i + 1]], reduce_packing_arrays(w, asg, k, c))


def test_check_batch_assign_matches_csr_path(oracle):
    """cfg2 nodes as assignments through the device reduction give the same
    verdicts / per-kind bests as the CSR path and the oracle."""
    c, k, w, a = W.cfg2_assignments(600)
    _, _, flat, off = W.cfg2_nodes(600)
    got = G.lower_bound_batch_assign(c, w, a, k, 2**62, want_best=True)
    ref = G.lower_bound_batch(c, flat, off, 2**62, want_best=True)
    for x, y in zip(got, ref):
        np.testing.assert_array_equal(x, y)
    lbo, _ = oracle.check_batch(flat[:off[100]], off[:101], c, 2**62)
    np.testing.assert_array_equal(got[0][:100], lbo)
    for mode in ("seq", "cancel"):
        g = G.lower_bound_batch_assign(c, w, a, k, 209, mode=mode)
        r = G.lower_bound_batch(c, flat, off, 209, mode=mode)
        np.testing.assert_array_equal(g[1], r[1])


def test_reduce_errors():
    """A committed load above c and an out-of-range bin id raise ValueError."""
    w = np.array([60, 60, 40], dtype=np.int32)
    a = np.array([[0, 0, 255]], dtype=np.uint8)  # bin 0 holds 120 > 100
    with pytest.raises(ValueError):
        G.lower_bound_batch_assign(100, w, a, 4, 5)
    a2 = np.array([[7, 255, 255]], dtype=np.uint8)  # bin 7 >= n_bins = 4
    with pytest.raises(ValueError):
        G.reduce_packing_batch(100, w, a2, 4)
    # all open: the reduced instance is the instance itself
    flat, off = G.reduce_packing_batch(100, w, np.full((2, 3), 255, dtype=np.uint8), 4)
    np.testing.assert_array_equal(flat, np.concatenate([w, w]))


# ---------------------------------------------------------------------------
# Solver integration: GPU bound mode and batched dffstats
# ---------------------------------------------------------------------------
def _dffstats_golden():
    with open(os.path.join(GOLDEN, "dffstats.json")) as f:
        return json.load(f)


def test_dffstats_batched_matches_reference():
    """Root bounds and the dffstats table of 60 instances (3 capacities, one
    batched launch each) equal the reference's cli._root_bounds / dffstats_table."""
    from paper_2402_14821_b200 import solver

    g = _dffstats_golden()
    insts = [(x["c"], x["weights"], x["name"]) for x in g["instances"]]
    roots = solver.root_bounds_batch(insts)
    assert [{k.name: v for k, v in r.items()} for r in roots] == g["root_bounds"]
    assert solver.dffstats_table(insts, g["optima"]) == g["table"]


def test_gpu_bound_mode_engine():
    """make_gpu_bound_engine gives a BoundEngine with lower_bound_seq semantics."""
    from paper_2402_14821_b200 import solver

    eng, close = solver.make_gpu_bound_engine(mode="seq")
    rng = random.Random(3)
    for _ in range(20):
        c, w = random_reduced_pair(rng, 60, 300)
        red = ReducedInstance(c, w)
        k = rng.randint(0, 40)
        got, want = eng(red, k), G.lower_bound_seq(red, k)
        assert (got.lb, got.exceeded_k, got.evals, list(got.per_dff.items())) == \
            (want.lb, want.exceeded_k, want.evals, list(want.per_dff.items()))
    close()


def test_assign_table_path_errors_and_modes(oracle):
    """>= 256 nodes from assignments take the table path (histograms straight
    from the assignments): errors as reduce_packing, uint16 assignments, and
    all modes against the CSR path."""
    c, k, w, a = W.cfg2_assignments(300)
    _, _, flat, off = W.cfg2_nodes(300)
    a16 = np.where(a == 255, 65535, a.astype(np.uint16)).astype(np.uint16)
    for mode, kk in (("full", 2**62), ("seq", 209), ("cancel", 209)):
        got = G.lower_bound_batch_assign(c, w, a16, k, kk, mode=mode, want_best=True)
        ref = G.lower_bound_batch(c, flat, off, kk, mode=mode, want_best=True)
        for x, y in zip(got, ref):
            np.testing.assert_array_equal(x, y)
    bad = a.copy()
    bad[17, :] = 0  # every item committed to bin 0: load far above c
    with pytest.raises(ValueError):
        G.lower_bound_batch_assign(c, w, bad, k, 2**62)
    bad = a.copy()
    bad[5, 3] = k + 2  # bin id >= n_bins
    with pytest.raises(ValueError):
        G.lower_bound_batch_assign(c, w, bad, k, 2**62)


def test_pinned_zero_copy_batch_paths(oracle):
    """Pinned caller buffers take the zero-copy path (the histogram pass reads
    the weights across PCIe, kernels write the outputs into the pinned
    arrays); results equal the pageable path, errors still raise."""
    import torch

    from paper_2402_14821_b200 import _native

    eng = _native.default_engine()
    c, k, flat, off = W.cfg2_nodes(2000)
    w8 = flat.astype(np.uint8)
    ref = eng.check_batch(w8, off, c, 2**62, list(range(6)), 0, want_best=True)
    pw = torch.from_numpy(w8).pin_memory().numpy()
    po = torch.from_numpy(off).pin_memory().numpy()
    n = len(off) - 1
    lb = torch.empty(n, dtype=torch.int64).pin_memory().numpy()
    ex = torch.empty(n, dtype=torch.uint8).pin_memory().numpy()
    for inputs in ((pw, po), (w8, off)):
        for outputs in ((lb, ex), None):
            got = eng.check_batch(inputs[0], inputs[1], c, 2**62, list(range(6)), 0, out=outputs)
            np.testing.assert_array_equal(got[0], ref[0])
            np.testing.assert_array_equal(got[1], ref[1])
    got = eng.check_batch(pw, po, c, 209, list(range(6)), _native.F_PHASED, want_best=True)
    want = eng.check_batch(w8, off, c, 209, list(range(6)), _native.F_PHASED, want_best=True)
    for a, b in zip(got, want):
        np.testing.assert_array_equal(a, b)
    bad = pw.copy()
    bad[off[7] + 3] = 0  # weight 0 is outside [1, c]
    pbad = torch.from_numpy(bad).pin_memory().numpy()
    with pytest.raises(ValueError):
        eng.check_batch(pbad, po, c, 2**62, list(range(6)), 0, out=(lb, ex))


def test_device_batch_graph_replay(oracle):
    """Repeated device-resident calls with the same arguments replay a
    captured CUDA graph: new buffer contents are picked up, and a changed
    argument (node count) re-captures."""
    import torch

    from paper_2402_14821_b200 import _native

    eng = _native.Engine(0)
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream()
    c, k, flat, off = W.cfg2_nodes(1200)
    n = len(off) - 1
    d_w = torch.from_numpy(flat.astype(np.uint8)).to(dev)
    d_off = torch.from_numpy(off).to(dev)
    d_lb = torch.zeros(n, dtype=torch.int64, device=dev)
    d_ex = torch.zeros(n, dtype=torch.uint8, device=dev)
    mr = int(np.diff(off).max())

    def run(nn):
        eng.check_batch_device(d_w.data_ptr(), d_off.data_ptr(), nn, mr, c, 2**62, list(range(6)), 0,
                               d_lb.data_ptr(), d_ex.data_ptr(), stream_ptr=st.cuda_stream, wbytes=1)
        st.synchronize()
        return d_lb.cpu().numpy().copy()

    first = run(n)
    lbo, _ = oracle.check_batch(flat, off, c, 2**62)
    np.testing.assert_array_equal(first, lbo)
    # same arguments, new contents: nodes shifted by one (weights rotated)
    flat2, off2 = flat.copy(), off.copy()
    perm = np.roll(np.arange(n), 1)
    nodes = [flat[off[i]:off[i + 1]] for i in perm]
    flat2, off2 = G.csr_from_lists(nodes)
    d_w.copy_(torch.from_numpy(flat2.astype(np.uint8)))
    d_off.copy_(torch.from_numpy(off2))
    second = run(n)
    np.testing.assert_array_equal(second, lbo[perm])
    third = run(n - 100)  # different argument set -> new capture
    np.testing.assert_array_equal(third[:n - 100], lbo[perm][:n - 100])
    eng.close()


def test_interleaved_streams_share_engine(oracle):
    """An asynchronous device-resident call on a caller stream followed at
    once (no synchronisation) by host-buffer calls on the engine's stream:
    the engine orders the second after the first (shared scratch), so both
    results stay exact, repeatedly."""
    import torch

    from paper_2402_14821_b200 import _native

    eng = _native.Engine(0)
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream()
    c, k, flat, off = W.cfg2_nodes(3000)
    n = len(off) - 1
    w8 = flat.astype(np.uint8)
    d_w = torch.from_numpy(w8).to(dev)
    d_off = torch.from_numpy(off).to(dev)
    d_lb = torch.zeros(n, dtype=torch.int64, device=dev)
    d_ex = torch.zeros(n, dtype=torch.uint8, device=dev)
    mr = int(np.diff(off).max())
    lbo, _ = oracle.check_batch(flat, off, c, 2**62)
    for _ in range(6):
        eng.check_batch_device(d_w.data_ptr(), d_off.data_ptr(), n, mr, c, 2**62, list(range(6)), 0,
                               d_lb.data_ptr(), d_ex.data_ptr(), stream_ptr=st.cuda_stream, wbytes=1)
        lb, _ = eng.check_batch(w8, off, c, 2**62, list(range(6)), 0)
        np.testing.assert_array_equal(lb, lbo)
        st.synchronize()
        np.testing.assert_array_equal(d_lb.cpu().numpy(), lbo)


def test_chunked_pageable_batch_matches_oracle(oracle):
    """Pageable host buffers large enough for the chunked upload (4 chunks,
    sub-ranges starting at node0 > 0 on 16-node tiles): per-tile ready flags
    and keys are offset per chunk; every node matches the oracle, twice in a
    row (flags cleared between calls), and again interleaved with a pinned
    zero-copy call."""
    import torch

    from paper_2402_14821_b200 import _native

    eng = _native.Engine(0)
    c, k, flat, off = W.cfg2_nodes(6000)
    w8 = flat.astype(np.uint8)
    lbo, _ = oracle.check_batch(flat, off, c, 2**62)
    lbs, exs = oracle.check_batch(flat, off, c, k)  # lower_bound_seq early exit at k
    for _ in range(2):
        lb, _ = eng.check_batch(w8, off, c, 2**62, list(range(6)), 0)
        np.testing.assert_array_equal(lb, lbo)
        lb, ex = eng.check_batch(w8, off, c, k, list(range(6)), _native.F_PHASED)
        np.testing.assert_array_equal(lb, lbs)
        np.testing.assert_array_equal(ex, exs)
    pw = torch.from_numpy(w8).pin_memory().numpy()
    po = torch.from_numpy(off).pin_memory().numpy()
    lb2, _ = eng.check_batch(pw, po, c, 2**62, list(range(6)), 0)
    lb3, _ = eng.check_batch(w8, off, c, 2**62, list(range(6)), 0)
    np.testing.assert_array_equal(lb2, lbo)
    np.testing.assert_array_equal(lb3, lbo)


@pytest.mark.parametrize("c", [1, 2, 3, 100, 150, 255, 256, 280, 288])
def test_single_check_cluster_kernel(oracle, c):
    """Drop-in single checks on the cached table (one thread-block cluster of
    up to 16 CTAs; c = 288 needs the full 16) equal the oracle's
    lower_bound_seq and every field of the node kernel's result (full and
    early-exit modes; the cancel mode's verdict); an invalid weight raises."""
    from paper_2402_14821_b200 import _native

    eng = _native.default_engine()
    rng = np.random.default_rng(1000 + c)
    for r in (0, 1, 17, 120, 400):
        if r * 101 * c >= 1 << 23:
            continue
        w = rng.integers(1, c + 1, size=r).astype(np.int32)
        red = ReducedInstance.from_array(c, w)
        want = oracle.lower_bound_seq(w, c, 2**62)
        got = G.lower_bound_seq(red, 2**62)
        assert {k.name: v for k, v in got.per_dff.items()} == want.per_dff, (c, r)
        assert {k.name: v for k, v in got.arg.items()} == want.arg, (c, r)
        k = max(0, got.lb - 1)
        a = eng.check(w, c, k, list(range(6)), _native.F_CANCEL)
        b = eng.check(w, c, k, list(range(6)), _native.F_CANCEL | _native.F_NOTAB)
        assert a.exceeded == b.exceeded  # which units a cancelled sweep skips is path-specific
        for fl in (0, _native.F_PHASED):
            a = eng.check(w, c, k, list(range(6)), fl)
            b = eng.check(w, c, k, list(range(6)), fl | _native.F_NOTAB)
            for f in ("lb", "exceeded", "n_done", "evals_total"):
                assert getattr(a, f) == getattr(b, f), (c, r, fl, f)
            for f in ("best", "arg_lambda", "n_lambda", "evals", "evaluated"):
                assert list(getattr(a, f)) == list(getattr(b, f)), (c, r, fl, f)
    bad = np.array([1, c + 1], dtype=np.int32)
    with pytest.raises(ValueError):
        eng.check(bad, c, 2**62, list(range(6)), 0)


@pytest.mark.parametrize("c", [510, 1022, 262_142, 262_143, 1_048_574, 1_048_577])
def test_wide_scan_tiles_dff_vectors(oracle, c):
    """The grid-wide path's cumulative table (adaptive scan tile: c + 2
    entries split into <= ~512 blocks, boundaries exercised by c) gives the
    oracle's per-lambda bounds: MT over its whole range, VB2 and BJ1 over a
    window at both ends."""
    rng = np.random.default_rng(c % 9973)
    w = rng.integers(1, c + 1, size=300).astype(np.int32)
    red = ReducedInstance.from_array(c, w)
    for kind, lo, hi in (("MT", 0, min(4000, (c + 1) // 2)), ("VB2", 2, min(600, c)), ("BJ1", max(1, c - 500), c)):
        got = G.dff_bound_batch(kind, red, lo, hi)
        want = oracle.dff_bound_batch(kind, w, c, lo, hi)
        np.testing.assert_array_equal(got, want, err_msg=f"{kind} c={c}")


@pytest.mark.parametrize("c,r", [(1_000_000, 300), (1_048_577, 20_000), (4_000_037, 5_000)])
def test_wide_sliced_harmonic_vectors(oracle, c, r):
    """CCM1 / BJ1 at small lambda on the grid-wide path: every lambda whose
    harmonic loop is longer than HSL_TS terms is cut into term slices on
    many warps (partial sums per lambda, finished in wide_final), the rest by
    one warp per lambda; both against the oracle's per-lambda bounds."""
    rng = np.random.default_rng(c + r)
    w = rng.integers(1, c + 1, size=r).astype(np.int32)
    red = ReducedInstance.from_array(c, w)
    for kind in ("CCM1", "BJ1"):
        got = G.dff_bound_batch(kind, red, 1, 1200)
        want = oracle.dff_bound_batch(kind, w, c, 1, 1200)
        np.testing.assert_array_equal(got, want, err_msg=f"{kind} c={c} r={r}")
