"""Golden vectors for the cfg5 headline batch, produced by the REFERENCE itself.

Run in the build container (the reference is importable only here):
    python tests/golden/make_golden_cfg5.py

The nodes come from the native generator stream that bench.py measures
(workloads.gen_nodes_host, seed CFG5_SEED): 48 nodes from the start of the
10^6-node batch plus 48 spread over the whole batch (indices up to 999,999),
so the fixture covers the batch the bench line is quoted on.  For every node
the reference's lower_bound_seq (bounds.py:504-527) is recorded in full mode
(k = 2^62: per-kind maxima, evals) and in decision mode (k = 334, the cfg5
bin budget: early-exit lb, exceeded, evals, processed kinds), and
lower_bound_par (parallel.py:122-137, workers=1, no cancellation) is checked
to agree with the full-mode maxima.  Output: tests/golden/cfg5_ref.npz.
"""

from __future__ import annotations

import os
import sys
import time
from multiprocessing import Pool

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

from binpack import ReducedInstance  # noqa: E402  (reference)
from binpack.bounds import DEFAULT_DFF_ORDER, lower_bound_seq  # noqa: E402

from paper_2402_14821_b200 import workloads as W  # noqa: E402  (input generators only)

N_BATCH = 1_000_000
FULL_K = 2**62


def node_ids() -> np.ndarray:
    head = np.arange(48)
    spread = np.linspace(48, N_BATCH - 1, 48).astype(np.int64)
    return np.concatenate([head, spread])


def _one(args):
    c, w, k_dec = args
    red = ReducedInstance(int(c), tuple(int(x) for x in w))
    full = lower_bound_seq(red, FULL_K)
    dec = lower_bound_seq(red, k_dec)
    best = [full.per_dff[kd] for kd in DEFAULT_DFF_ORDER]
    dec_best = [dec.per_dff.get(kd, -1) for kd in DEFAULT_DFF_ORDER]
    return best, full.lb, full.evals, dec.lb, int(dec.exceeded_k), dec.evals, dec_best


def main() -> None:
    c, k, w = W.cfg5_instance()
    ids = node_ids()
    nodes = []
    for i in ids:
        flat, off = W.gen_nodes_host(w, c, k, W.CFG5_SEED, 1, first_node=int(i))
        nodes.append(flat.copy())
    t = time.time()
    with Pool(min(8, os.cpu_count() or 1)) as pool:
        rows = pool.map(_one, [(c, x, k) for x in nodes])
    print(f"reference lower_bound_seq on {len(nodes)} cfg5 nodes x 2 modes: {time.time() - t:.1f} s")
    off = np.zeros(len(nodes) + 1, dtype=np.int64)
    off[1:] = np.cumsum([x.size for x in nodes])
    np.savez_compressed(
        os.path.join(HERE, "cfg5_ref.npz"),
        node_ids=ids, weights=np.concatenate(nodes).astype(np.int32), offsets=off,
        c=np.int64(c), k=np.int64(k),
        best=np.array([r[0] for r in rows], dtype=np.int64),
        lb=np.array([r[1] for r in rows], dtype=np.int64),
        evals=np.array([r[2] for r in rows], dtype=np.int64),
        dec_lb=np.array([r[3] for r in rows], dtype=np.int64),
        dec_exceeded=np.array([r[4] for r in rows], dtype=np.int64),
        dec_evals=np.array([r[5] for r in rows], dtype=np.int64),
        dec_best=np.array([r[6] for r in rows], dtype=np.int64),
    )
    print("wrote", os.path.join(HERE, "cfg5_ref.npz"))


if __name__ == "__main__":
    main()
