"""Drop-in mirror of the reference's parallel engine, GPU-backed.

Reference: /root/reference/pkg/src/binpack/parallel.py.  ``lower_bound_par``
and ``ParallelBoundEngine`` keep their signatures and contracts
(parallel.py:122-174): the decision bit equals the
sequential engine's, the value equals the completed sweep whenever the bound
stays within budget, ``cancellation=False`` evaluates every grid point, and
with cancellation work units that observe ``lb > k`` are skipped (the
in-kernel form of Alg. 4's guard ``if lb <= k``).  ``workers``
is accepted and validated for compatibility; the parallelism is the GPU's.

``GpuBoundEngine`` is the ``BoundEngine`` callable (propagator.py:40) a
search plugs in; ``ParallelBoundEngine`` is an alias-compatible subclass.
"""

from __future__ import annotations

import os
import threading
from typing import Sequence

from . import _native
from .bounds import DEFAULT_DFF_ORDER, BoundResult, DffKind, _kind, _result_seq, resolve_kinds
from .instances import as_reduced

__all__ = ["SharedMax", "lower_bound_par", "lower_bound_multi", "GpuBoundEngine", "ParallelBoundEngine",
           "default_workers", "CHUNK"]

#: Reference cancellation granularity (parallel.py:33); the GPU checks its
#: guard once per work unit (32-128 lambdas).
CHUNK = 64


def default_workers() -> int:
    return os.cpu_count() or 1


class SharedMax:
    """Thread-safe non-decreasing maximum (parallel.py:40-55).  The GPU
    engine's equivalent is the in-kernel atomicMax on the node's bound."""

    def __init__(self, value: int = 0):
        self._value = value
        self._lock = threading.Lock()

    def offer(self, value: int) -> int:
        with self._lock:
            if value > self._value:
                self._value = value
            return self._value

    def get(self) -> int:
        with self._lock:
            return self._value


def _result_par(res: _native.BplbResult, kinds: Sequence[DffKind], ids: Sequence[int], k: int) -> BoundResult:
    # parallel.py:105-119: kinds with at least one evaluated unit, in kinds
    # order; empty ranges never appear.
    best, ev, arg = res.best[:], res.evaluated[:], res.arg_lambda[:]
    out = BoundResult(lb=0, evals=int(res.evals_total))
    per, args = out.per_dff, out.arg
    lb = 0
    for kind, kid in zip(kinds, ids):
        if ev[kid]:
            b = best[kid]
            per[kind] = b
            args[kind] = arg[kid]
            if b > lb:
                lb = b
    out.lb, out.exceeded_k = lb, lb > k
    return out


def _run_par(engine: _native.Engine, red, k: int, kinds, cancellation: bool) -> BoundResult:
    kinds, ids = resolve_kinds(kinds)
    c, w = as_reduced(red)
    if not kinds:
        return BoundResult(lb=0, exceeded_k=0 > k)
    res = engine.check(w, c, k, ids, _native.F_CANCEL if cancellation else 0)
    return _result_par(res, kinds, ids, k)


def lower_bound_par(red, k: int, kinds: Sequence = DEFAULT_DFF_ORDER, workers: int = 1,
                    cancellation: bool = True) -> BoundResult:
    """Parallel counterpart of the sequential sweep (parallel.py:122-137)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    return _run_par(_native.default_engine(), red, k, kinds, cancellation)


_multi_engines: dict = {}
_multi_lock = threading.Lock()


def lower_bound_multi(red, k: int, devices: Sequence[int], kinds: Sequence = DEFAULT_DFF_ORDER,
                      mode: str = "par") -> BoundResult:
    """One check of one (large) reduced instance over several GPUs in one call
    (SURVEY.md 8(e)): every kind's lambda range is cut into one contiguous
    slice per device, each slice a bound-pruned check on its own device, the
    per-kind (best, lowest arg lambda) merged like an allreduce(MAX) of packed
    keys (``bplb_check_multi``).  The multi-device counterpart of the
    reference's lambda-chunk dispatch of one check (parallel.py:84-119).
    ``mode="par"``: lower_bound_par(cancellation=False) semantics (the full
    collection); ``mode="seq"``: lower_bound_seq semantics (kinds in order,
    early exit replayed on the merged per-kind results)."""
    if mode not in ("par", "seq"):
        raise ValueError("mode must be 'par' or 'seq'")
    kinds, ids = resolve_kinds(kinds)
    c, w = as_reduced(red)
    if not kinds:
        return BoundResult(lb=0, exceeded_k=0 > k)
    key = tuple(int(d) for d in devices)
    with _multi_lock:
        eng = _multi_engines.get(key)
        if eng is None:
            eng = _multi_engines[key] = _native.MultiEngine(key)
    res = eng.check(w, c, k, ids, _native.F_PHASED if mode == "seq" else 0)
    return _result_seq(res, kinds, ids, k) if mode == "seq" else _result_par(res, kinds, ids, k)


class GpuBoundEngine:
    """Reusable B200 bound engine: ``engine(red, k) -> BoundResult``.

    ``mode="par"`` (default) has lower_bound_par semantics (concurrent
    kinds, cancellation guard); ``mode="seq"`` has lower_bound_seq
    semantics (kinds in order, early exit).  Owns one libbplb engine (CUDA
    stream + resident buffers) on ``device``; ``close()`` releases it.
    """

    def __init__(self, kinds: Sequence = DEFAULT_DFF_ORDER, device: int | None = None,
                 cancellation: bool = True, mode: str = "par"):
        self.kinds = tuple(_kind(x) for x in kinds)
        self.cancellation = cancellation
        if mode not in ("par", "seq"):
            raise ValueError("mode must be 'par' or 'seq'")
        self.mode = mode
        self.device = int(os.environ.get("BPLB_DEVICE", "0")) if device is None else int(device)
        self._engine: _native.Engine | None = None
        self._lock = threading.Lock()

    def _eng(self) -> _native.Engine:
        with self._lock:
            if self._engine is None:
                self._engine = _native.Engine(self.device)
            return self._engine

    def __call__(self, red, k: int) -> BoundResult:
        eng = self._eng()
        if self.mode == "seq":
            kinds, ids = resolve_kinds(self.kinds)
            c, w = as_reduced(red)
            if not kinds:
                return BoundResult(lb=0, exceeded_k=0 > k)
            res = eng.check(w, c, k, ids, _native.F_PHASED)
            return _result_seq(res, kinds, ids, k)
        return _run_par(eng, red, k, self.kinds, self.cancellation)

    def close(self) -> None:
        with self._lock:
            if self._engine is not None:
                self._engine.close()
                self._engine = None

    def __enter__(self):
        return self

    def __exit__(self, *exc) -> None:
        self.close()


class ParallelBoundEngine(GpuBoundEngine):
    """Signature-compatible stand-in for parallel.py:140-174."""

    def __init__(self, kinds: Sequence = DEFAULT_DFF_ORDER, workers: int | None = None,
                 cancellation: bool = True):
        self.workers = workers if workers is not None else default_workers()
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        super().__init__(kinds=kinds, cancellation=cancellation, mode="par")
