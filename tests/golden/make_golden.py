"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container (the reference is importable only here):
    python tests/golden/make_golden.py            # everything except cfg4 VB2
    python tests/golden/make_golden.py --cfg4-vb2 # the ~730 core-second part

It imports /root/reference/pkg/src/binpack (read-only) and records
dff_bound_batch / lower_bound_seq / lower_bound_par outputs on seeded inputs
into tests/golden/*.npz.  The committed fixtures pin both the C oracle
(tests/test_oracle_golden.py, CPU) and the CUDA path (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import argparse
import json
import os
import random
import sys
import time
from multiprocessing import Pool

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

from binpack import ReducedInstance  # noqa: E402  (reference)
from binpack.bounds import DEFAULT_DFF_ORDER, DffKind, dff_bound_batch, lambda_range, lower_bound_seq  # noqa: E402
from binpack.parallel import lower_bound_par  # noqa: E402

from paper_2402_14821_b200 import workloads as W  # noqa: E402  (input generators only)

KIND_NAMES = [k.name for k in DEFAULT_DFF_ORDER]


def random_reduced(rng: random.Random, max_r: int, max_c: int):
    # conftest.py:18-21 shape
    c = rng.randint(1, max_c)
    r = rng.randint(0, max_r)
    return c, [rng.randint(1, c) for _ in range(r)]


def small_cases(out_path: str) -> None:
    """Random small reduced instances: full per-lambda vectors of every kind,
    lower_bound_seq for several k / kind orders, lower_bound_par without
    cancellation."""
    rng = random.Random(2024)
    cs, offs, ws = [], [0], []
    vec_vals, vec_meta = [], []  # meta rows: case, kind, lo, hi, offset
    seq_rows = []  # case, k, order-id, lb, exceeded, evals, n_done, per_dff[6] (by position)
    par_rows = []  # case, lb, evals, present-mask, per_dff by kind id
    orders = [list(range(6)), [3, 0], [5, 4, 3, 2, 1, 0], [2], [4, 1]]
    shapes = [(12, 130)] * 900 + [(40, 600)] * 150 + [(10, 3000)] * 50
    for case, (mr, mc) in enumerate(shapes):
        c, w = random_reduced(rng, mr, mc)
        if case % 7 == 0 and c % 2 == 0 and w:
            w[0] = c // 2  # exercise 2w == c
        if case % 5 == 0 and w:
            w[-1] = c      # exercise w == c
        red = ReducedInstance(c, tuple(w))
        cs.append(c)
        ws.extend(w)
        offs.append(len(ws))
        for kid, kind in enumerate(DEFAULT_DFF_ORDER):
            rg = lambda_range(kind, c, red)
            if rg.is_empty:
                continue
            v = dff_bound_batch(kind, red, rg.lo, rg.hi)
            vec_meta.append([case, kid, rg.lo, rg.hi, len(vec_vals)])
            vec_vals.extend(int(x) for x in v)
        for k in (0, 1, 3, rng.randint(0, 8), 10**9):
            for oi, order in enumerate(orders):
                kinds = [DEFAULT_DFF_ORDER[i] for i in order]
                res = lower_bound_seq(red, k, kinds)
                per = [int(res.per_dff[kd]) for kd in res.per_dff] + [-1] * (6 - len(res.per_dff))
                seq_rows.append([case, k, oi, res.lb, int(res.exceeded_k), res.evals, len(res.per_dff), *per])
        par = lower_bound_par(red, 5, workers=1, cancellation=False)
        mask = sum(1 << KIND_NAMES.index(kd.name) for kd in par.per_dff)
        per = [int(par.per_dff.get(kd, -1)) for kd in DEFAULT_DFF_ORDER]
        par_rows.append([case, par.lb, par.evals, mask, *per])
    np.savez_compressed(
        out_path,
        c=np.array(cs, dtype=np.int64), offsets=np.array(offs, dtype=np.int64),
        weights=np.array(ws, dtype=np.int64),
        vec_meta=np.array(vec_meta, dtype=np.int64), vec_vals=np.array(vec_vals, dtype=np.int64),
        seq_rows=np.array(seq_rows, dtype=np.int64), par_rows=np.array(par_rows, dtype=np.int64),
        orders=json.dumps(orders))


def windows(kind, c, red, n_win=3, width=200):
    rg = lambda_range(kind, c, red)
    if rg.is_empty:
        return []
    if len(rg) <= n_win * width:
        return [(rg.lo, rg.hi)]
    mids = [rg.lo, (rg.lo + rg.hi) // 2 - width // 2, rg.hi - width + 1]
    return [(m, m + width - 1) for m in mids[:n_win]]


def config_cases(out_path: str) -> None:
    data = {}
    # cfg1: full vectors
    c, w = W.cfg1()
    red = ReducedInstance(c, tuple(int(x) for x in w))
    res = lower_bound_seq(red, 2**62)
    data["cfg1_w"] = w.astype(np.int64)
    data["cfg1_best"] = np.array([res.per_dff[k] for k in DEFAULT_DFF_ORDER], dtype=np.int64)
    vals = []
    for kind in DEFAULT_DFF_ORDER:
        rg = lambda_range(kind, c, red)
        vals.append(dff_bound_batch(kind, red, rg.lo, rg.hi))
    data["cfg1_vec"] = np.concatenate(vals)
    data["cfg1_l2m1"] = np.array([lower_bound_seq(red, res.lb - 1).lb], dtype=np.int64)
    # cfg2: first 300 nodes, full mode + decision mode
    c, k, flat, off = W.cfg2_nodes(300)
    best, dec = [], []
    for i in range(300):
        red = ReducedInstance(c, tuple(int(x) for x in flat[off[i]:off[i + 1]]))
        r = lower_bound_seq(red, 2**62)
        best.append([r.per_dff[kd] for kd in DEFAULT_DFF_ORDER])
        d = lower_bound_seq(red, k)
        dec.append([d.lb, int(d.exceeded_k), d.evals, len(d.per_dff)])
    data["cfg2_k"] = np.array([k])
    data["cfg2_best"] = np.array(best, dtype=np.int64)
    data["cfg2_dec"] = np.array(dec, dtype=np.int64)
    # cfg3 / cfg3u: per-kind maxima + lambda windows
    for name, gen in (("cfg3", W.cfg3), ("cfg3u", W.cfg3u)):
        c, w = gen()
        red = ReducedInstance(c, tuple(int(x) for x in w))
        t = time.time()
        res = lower_bound_seq(red, 2**62)
        data[f"{name}_w"] = w.astype(np.int64)
        data[f"{name}_best"] = np.array([res.per_dff[k] for k in DEFAULT_DFF_ORDER], dtype=np.int64)
        meta, vals = [], []
        for kid, kind in enumerate(DEFAULT_DFF_ORDER):
            for lo, hi in windows(kind, c, red):
                v = dff_bound_batch(kind, red, lo, hi)
                meta.append([kid, lo, hi, len(vals)])
                vals.extend(int(x) for x in v)
        data[f"{name}_win_meta"] = np.array(meta, dtype=np.int64)
        data[f"{name}_win_vals"] = np.array(vals, dtype=np.int64)
        print(name, "done", time.time() - t, flush=True)
    # cfg4: per-kind maxima except VB2 (full), and windows for every kind
    c, w = W.cfg4()
    red = ReducedInstance(c, tuple(int(x) for x in w))
    best4 = []
    for kind in DEFAULT_DFF_ORDER:
        if kind is DffKind.VB2:
            best4.append(-1)
            continue
        rg = lambda_range(kind, c, red)
        t = time.time()
        best4.append(int(dff_bound_batch(kind, red, rg.lo, rg.hi).max()))
        print("cfg4", kind.name, time.time() - t, flush=True)
    data["cfg4_best_nonvb2"] = np.array(best4, dtype=np.int64)
    meta, vals = [], []
    for kid, kind in enumerate(DEFAULT_DFF_ORDER):
        for lo, hi in windows(kind, c, red, n_win=3, width=100):
            v = dff_bound_batch(kind, red, lo, hi)
            meta.append([kid, lo, hi, len(vals)])
            vals.extend(int(x) for x in v)
    data["cfg4_win_meta"] = np.array(meta, dtype=np.int64)
    data["cfg4_win_vals"] = np.array(vals, dtype=np.int64)
    # cfg5: first 12 nodes, full mode
    c, k, flat, off = W.cfg5_nodes(12)
    best5 = []
    for i in range(12):
        red = ReducedInstance(c, tuple(int(x) for x in flat[off[i]:off[i + 1]]))
        r = lower_bound_seq(red, 2**62)
        best5.append([r.per_dff[kd] for kd in DEFAULT_DFF_ORDER])
    data["cfg5_best"] = np.array(best5, dtype=np.int64)
    np.savez_compressed(out_path, **data)


def _vb2_chunk(args):
    lo, hi = args
    c, w = W.cfg4()
    red = ReducedInstance(c, tuple(int(x) for x in w))
    v = dff_bound_batch(DffKind.VB2, red, lo, hi)
    j = int(np.argmax(v))
    return int(v[j]), lo + j


def cfg4_vb2(out_path: str, procs: int) -> None:
    c, w = W.cfg4()
    red = ReducedInstance(c, tuple(int(x) for x in w))
    rg = lambda_range(DffKind.VB2, c, red)
    step = 2000
    chunks = [(lo, min(lo + step - 1, rg.hi)) for lo in range(rg.lo, rg.hi + 1, step)]
    t = time.time()
    with Pool(procs) as pool:
        res = pool.map(_vb2_chunk, chunks, chunksize=1)
    best = max(r[0] for r in res)
    arg = min(r[1] for r in res if r[0] == best)
    np.savez_compressed(out_path, cfg4_vb2_best=np.array([best, arg], dtype=np.int64))
    print("cfg4 VB2", best, arg, time.time() - t, flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg4-vb2", action="store_true")
    ap.add_argument("--procs", type=int, default=max(1, (os.cpu_count() or 2) - 1))
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    if a.cfg4_vb2:
        cfg4_vb2(os.path.join(HERE, "cfg4_vb2.npz"), a.procs)
    else:
        if a.only in ("", "small"):
            t = time.time()
            small_cases(os.path.join(HERE, "small.npz"))
            print("small done", time.time() - t, flush=True)
        if a.only in ("", "configs"):
            config_cases(os.path.join(HERE, "configs.npz"))
            print("configs done", flush=True)
