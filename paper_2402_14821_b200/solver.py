"""Solver-facing integration of the GPU bound engine.

* ``DFFS_GPU`` / :func:`make_gpu_bound_engine` -- the extra bound mode a
  maintainer adds to the reference's ``BoundMode`` / ``make_bound_engine``
  (search.py:44-55, 127-141): returns ``(engine, close)`` like the reference
  factory, ``engine(red, k) -> BoundResult`` (the ``BoundEngine`` protocol,
  propagator.py:40) with ``lower_bound_seq`` semantics (mode="seq") so the
  search explores the same nodes as ``dffs-seq``.
* :func:`root_bounds_batch` / :func:`dffstats_table` -- the ``dffstats``
  command's root bounds (cli.py:334-370) for a whole directory of instances
  in batched launches (one per distinct capacity) instead of one
  ``dff_bound_batch`` sweep per kind and instance.
"""

from __future__ import annotations

import dataclasses
import enum
from collections import defaultdict
from typing import Callable, Sequence

import numpy as np

from .batch import csr_from_lists, lower_bound_batch
from .bounds import DEFAULT_DFF_ORDER, DffKind
from .bounds import _kind
from .parallel import GpuBoundEngine

DFFS_GPU = "dffs-gpu"  # value of the new BoundMode member

DFFSTATS_COLUMNS = ["dff", "only_opt", "total_opt", "only_best", "total_best", "sum_bounds"]


def make_gpu_bound_engine(cfg=None, *, kinds: Sequence = DEFAULT_DFF_ORDER, device: int | None = None,
                          mode: str = "seq"):
    """``(engine, close)`` for ``BoundMode.DFFS_GPU``.  ``cfg`` is the
    reference's ``SearchConfig`` (its ``dff_order`` is used when present)."""
    if cfg is not None and getattr(cfg, "dff_order", None) is not None:
        kinds = cfg.dff_order
    eng = GpuBoundEngine(kinds=kinds, device=device, mode=mode)
    return eng, eng.close


class BoundModeGPU(enum.Enum):
    """The reference's ``BoundMode`` (search.py:44-55) plus ``DFFS_GPU``;
    ``from_name`` parses like the reference's (case-insensitive value)."""

    L2 = "l2"
    DFFS_SEQ = "dffs-seq"
    DFFS_PAR = "dffs-par"
    DFFS_GPU = DFFS_GPU

    @classmethod
    def from_name(cls, name: str) -> "BoundModeGPU":
        for mode in cls:
            if mode.value == name.strip().lower():
                return mode
        valid = ", ".join(m.value for m in cls)
        raise ValueError(f"unknown bound mode {name!r} (expected one of {valid})")


def install_dffs_gpu(search, cli=None, *, device: int | None = None,
                     factory: Callable | None = None) -> Callable[[], None]:
    """Plug ``dffs-gpu`` into the reference solver without editing it.

    ``search`` / ``cli`` are the reference's ``binpack.search`` /
    ``binpack.cli`` modules.  ``search.make_bound_engine`` (search.py:127-141)
    is wrapped: a config whose ``bound_mode`` value is ``"dffs-gpu"`` gets
    ``make_gpu_bound_engine(cfg)`` (``lower_bound_seq`` semantics, so the
    search explores exactly the nodes of ``dffs-seq``); every other mode is
    mapped back to the reference's own enum member and served by the
    original factory.  With ``cli``, its ``BoundMode`` becomes
    :class:`BoundModeGPU` so ``--bound dffs-gpu`` parses (cli.py:127-134,
    143-155).  ``factory`` replaces the GPU factory (tests inject the
    oracle).  Returns a callable that undoes the patch.
    """
    orig = search.make_bound_engine
    ref_mode = search.BoundMode
    make = factory or (lambda cfg: make_gpu_bound_engine(cfg, device=device))

    def make_bound_engine(cfg):
        value = getattr(cfg.bound_mode, "value", cfg.bound_mode)
        if value == DFFS_GPU:
            return make(cfg)
        if not isinstance(cfg.bound_mode, ref_mode):
            cfg = dataclasses.replace(cfg, bound_mode=ref_mode(value))
        return orig(cfg)

    search.make_bound_engine = make_bound_engine
    cli_mode = getattr(cli, "BoundMode", None) if cli is not None else None
    if cli is not None:
        cli.BoundMode = BoundModeGPU

    def uninstall() -> None:
        search.make_bound_engine = orig
        if cli is not None:
            cli.BoundMode = cli_mode

    return uninstall


def _instance_parts(inst):
    if isinstance(inst, tuple):
        c, w = inst[0], inst[1]
        return int(c), np.asarray(w, dtype=np.int32), (inst[2] if len(inst) > 2 else "")
    return int(inst.c), np.asarray(inst.weights, dtype=np.int32), getattr(inst, "name", "")


def root_bounds_batch(instances, kinds: Sequence = DEFAULT_DFF_ORDER) -> list[dict[DffKind, int]]:
    """Per instance and kind, the best bound over the kind's full lambda
    range on the unreduced instance (cli.py:334-345 ``_root_bounds``; 0 for
    an empty range).  ``instances``: reference ``Instance`` objects or
    ``(c, weights[, name])`` tuples.  One batched launch per capacity."""
    kinds = [_kind(k) for k in kinds]
    parts = [_instance_parts(x) for x in instances]
    by_c: dict[int, list[int]] = defaultdict(list)
    for i, (c, _, _) in enumerate(parts):
        by_c[c].append(i)
    out: list[dict[DffKind, int] | None] = [None] * len(parts)
    for c, idx in by_c.items():
        w, off = csr_from_lists([parts[i][1] for i in idx])
        _, _, best, _ = lower_bound_batch(c, w, off, 2**62, kinds, want_best=True)
        for j, i in enumerate(idx):
            out[i] = {k: int(best[j, _kid(k)]) for k in kinds}
    return out  # type: ignore[return-value]


def _kid(kind: DffKind) -> int:
    return list(DEFAULT_DFF_ORDER).index(kind)


def dffstats_table(instances, optima: dict[str, int], kinds: Sequence = DEFAULT_DFF_ORDER):
    """The ``dffstats`` table (cli.py:351-370): per kind, how often it alone /
    jointly attains the optimum and the best root bound, and the sum of its
    root bounds, over ``instances`` (named; ``optima`` by name)."""
    kinds = [_kind(k) for k in kinds]
    counters = {k: {"only_opt": 0, "total_opt": 0, "only_best": 0, "total_best": 0, "sum_bounds": 0}
                for k in kinds}
    names = [_instance_parts(x)[2] for x in instances]
    for name, bounds in zip(names, root_bounds_batch(instances, kinds)):
        best = max(bounds.values())
        best_kinds = [k for k in kinds if bounds[k] == best]
        opt = optima.get(name)
        opt_kinds = [k for k in kinds if opt is not None and bounds[k] == opt]
        for k in kinds:
            counters[k]["sum_bounds"] += bounds[k]
            if bounds[k] == best:
                counters[k]["total_best"] += 1
                if len(best_kinds) == 1:
                    counters[k]["only_best"] += 1
            if opt is not None and bounds[k] == opt:
                counters[k]["total_opt"] += 1
                if len(opt_kinds) == 1:
                    counters[k]["only_opt"] += 1
    return [{"dff": k.name, **counters[k]} for k in kinds]
