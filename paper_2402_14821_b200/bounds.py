"""Drop-in mirror of the reference's lower-bound module, GPU-backed.

Reference: /root/reference/pkg/src/binpack/bounds.py.  Same names, argument
meaning, return types and error behaviour; the sweeps behind
``dff_bound_batch``, ``dff_bound``, ``lower_bound_seq`` and ``l2`` run in
libbplb.so on the B200 (there is no CPU path for them).  ``lambda_range``,
``dff_value``, ``l1``, ``l2_partition`` and ``l2_value`` are O(1)/O(r)
scalar metadata helpers and stay in Python, as SURVEY.md section 7.1(2) plans.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import Iterator, Sequence

import numpy as np

from . import _native
from .instances import ReducedInstance, as_reduced

__all__ = [
    "DffKind",
    "DEFAULT_DFF_ORDER",
    "LambdaRange",
    "L2Partition",
    "BoundResult",
    "VB2_ACCUMULATOR_MAX",
    "l1",
    "l2",
    "l2_partition",
    "l2_value",
    "dff_value",
    "lambda_range",
    "dff_bound",
    "dff_bound_batch",
    "lower_bound_seq",
    "kind_ids",
]

#: bounds.py:38-40 -- cap of the VB2 sweep keeps r * max_weight * lambda in 64 bits.
VB2_ACCUMULATOR_MAX = 2**64 - 1


class DffKind(enum.Enum):
    """The six weight transformations, in default priority order (bounds.py:48-64)."""

    MT = "MT"
    RAD2 = "RAD2"
    FS1 = "FS1"
    CCM1 = "CCM1"
    VB2 = "VB2"
    BJ1 = "BJ1"

    @classmethod
    def from_name(cls, name: str) -> "DffKind":
        try:
            return cls[name.strip().upper()]
        except KeyError:
            valid = ", ".join(k.name for k in cls)
            raise ValueError(f"unknown DFF {name!r} (expected one of {valid})") from None

    @property
    def id(self) -> int:
        return _KIND_ID[self.name]


_KIND_ID = {"MT": 0, "RAD2": 1, "FS1": 2, "CCM1": 3, "VB2": 4, "BJ1": 5}
_BY_ID = {v: DffKind[k] for k, v in _KIND_ID.items()}

DEFAULT_DFF_ORDER: tuple[DffKind, ...] = tuple(DffKind)
_DEFAULT_RESOLVED = (DEFAULT_DFF_ORDER, tuple(_KIND_ID[x.name] for x in DEFAULT_DFF_ORDER))


def _kind(k) -> DffKind:
    """Accept our DffKind, the reference's DffKind (same names) or a name."""
    if isinstance(k, DffKind):
        return k
    name = getattr(k, "name", k)
    return DffKind.from_name(str(name))


def kind_ids(kinds: Sequence) -> list[int]:
    return [_kind(k).id for k in kinds]


_RESOLVED: dict = {}


def resolve_kinds(kinds: Sequence) -> tuple[tuple, tuple]:
    """(DffKind tuple, id tuple) for a kinds sequence, cached: the drop-in
    single-check calls sit on a solver's per-node path."""
    if kinds is DEFAULT_DFF_ORDER:
        return _DEFAULT_RESOLVED
    try:
        key = tuple(kinds)
        hit = _RESOLVED.get(key)
    except TypeError:
        key, hit = None, None
    if hit is None:
        ks = tuple(_kind(x) for x in kinds)
        hit = (ks, tuple(_KIND_ID[x.name] for x in ks))
        if key is not None and len(_RESOLVED) < 256:
            _RESOLVED[key] = hit
    return hit


@dataclass(frozen=True)
class LambdaRange:
    """Inclusive integer parameter interval; empty when lo > hi (bounds.py:70-88)."""

    lo: int
    hi: int

    @property
    def is_empty(self) -> bool:
        return self.lo > self.hi

    def __len__(self) -> int:
        return max(0, self.hi - self.lo + 1)

    def __iter__(self) -> Iterator[int]:
        return iter(range(self.lo, self.hi + 1))

    def __contains__(self, lam: int) -> bool:
        return self.lo <= lam <= self.hi


@dataclass(frozen=True)
class L2Partition:
    """Weights split by the two thresholds lambda and c/2 (bounds.py:91-98)."""

    w1: tuple[int, ...]
    w2: tuple[int, ...]
    w3: tuple[int, ...]
    lam: int


@dataclass
class BoundResult:
    """Outcome of a bound sweep (bounds.py:101-108).  ``arg`` (extra) maps
    each evaluated kind to the lowest lambda attaining its best bound."""

    lb: int
    per_dff: dict = field(default_factory=dict)
    exceeded_k: bool = False
    evals: int = 0
    arg: dict = field(default_factory=dict, compare=False, repr=False)


def _ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def l1(red) -> int:
    """Total weight over capacity, rounded up; 0 for no weights (bounds.py:115-119)."""
    c, w = as_reduced(red)
    if w.size == 0:
        return 0
    return _ceil_div(int(w.sum(dtype=np.int64)), c)


def l2_partition(red, lam: int) -> L2Partition:
    """bounds.py:122-127 (host metadata helper)."""
    c = red.c
    ws = tuple(int(x) for x in red.weights)
    return L2Partition(
        w1=tuple(w for w in ws if c - lam < w),
        w2=tuple(w for w in ws if 2 * w > c and w <= c - lam),
        w3=tuple(w for w in ws if lam <= w and 2 * w <= c),
        lam=lam,
    )


def l2_value(red, lam: int) -> int:
    """bounds.py:130-136 (host metadata helper, one threshold)."""
    p = l2_partition(red, lam)
    slack = red.c * len(p.w2) - sum(p.w2)
    overflow = _ceil_div(sum(p.w3) - slack, red.c)
    return len(p.w1) + len(p.w2) + max(0, overflow)


def l2(red, full_sweep: bool = False) -> int:
    """Martello-Toth L2 (bounds.py:139-152).  Computed on the GPU as the best
    f_MT bound over lambda in [0, ceil(c/2)], which equals L2 (the reference
    tests this equivalence, test_bounds.py:62-81); ``full_sweep`` is accepted
    for signature compatibility -- the GPU always sweeps the full range."""
    c, w = as_reduced(red)
    if w.size == 0:
        return 0
    res = _native.default_engine().check(w, c, 0, [0], 0)
    return int(res.best[0])


# ---------------------------------------------------------------------------
# Scalar transforms (bounds.py:155-250): host metadata, one cell at a time.
# ---------------------------------------------------------------------------
def _mt(w, c, lam):
    if c - lam < w:
        return c
    if w < lam:
        return 0
    return w


def _rad2(w, c, lam):
    def base(v):
        if v < lam:
            return 0
        return c // 3 if v <= c - 2 * lam else c // 2

    return c - base(c - w) if w >= 2 * lam else base(w)


def _fs1(w, c, lam):
    q, rem = divmod(w * (lam + 1), c)
    return w * lam if rem == 0 else q * c


def _ccm1(w, c, lam):
    if 2 * w > c:
        return 2 * (c // lam - (c - w) // lam)
    if 2 * w == c:
        return c // lam
    return 2 * (w // lam)


def _vb2(w, c, lam):
    def piece(v):
        return max(0, -(-(v * lam) // c) - 1)

    if 2 * w > c:
        return 2 * piece(c) - 2 * piece(c - w)
    if 2 * w == c:
        return piece(c)
    return 2 * piece(w)


def _bj1(w, c, lam):
    cm = c % lam
    base = (w // lam) * (lam - cm)
    wm = w % lam
    return base if wm <= cm else base + wm - cm


_VALUE_FN = {DffKind.MT: _mt, DffKind.RAD2: _rad2, DffKind.FS1: _fs1,
             DffKind.CCM1: _ccm1, DffKind.VB2: _vb2, DffKind.BJ1: _bj1}


def _mt_hi(c: int) -> int:
    # odd-capacity midpoint ceil(c/2) (bounds.py:219-225)
    return 0 if c == 1 else (c + 1) // 2


def _domain_ok(kind: DffKind, c: int, lam: int) -> bool:
    if kind is DffKind.MT:
        return 0 <= lam <= _mt_hi(c)
    if kind is DffKind.RAD2:
        return 4 * lam > c and 3 * lam <= c
    if kind is DffKind.FS1:
        return 1 <= lam <= 100
    if kind is DffKind.CCM1:
        return 1 <= lam and 2 * lam <= c
    if kind is DffKind.VB2:
        return 2 <= lam <= c
    return 1 <= lam <= c


def dff_value(kind, w: int, c: int, lam: int) -> int:
    """Transformed weight for one grid point (bounds.py:242-250)."""
    kind = _kind(kind)
    assert 0 <= w <= c, f"weight {w} outside [0, {c}]"
    assert _domain_ok(kind, c, lam), f"{kind.name}: lambda {lam} outside domain for c={c}"
    return _VALUE_FN[kind](w, c, lam)


def lambda_range(kind, c: int, red=None) -> LambdaRange:
    """Integer parameter interval swept for ``kind`` at capacity ``c``
    (bounds.py:253-273), with the VB2 accumulator cap when ``red`` is given."""
    kind = _kind(kind)
    if kind is DffKind.MT:
        return LambdaRange(0, _mt_hi(c))
    if kind is DffKind.RAD2:
        return LambdaRange(c // 4 + 1, c // 3)
    if kind is DffKind.FS1:
        return LambdaRange(1, 100)
    if kind is DffKind.CCM1:
        return LambdaRange(1, c // 2)
    if kind is DffKind.VB2:
        hi = c
        if red is not None and red.r > 0:
            hi = min(hi, VB2_ACCUMULATOR_MAX // (red.r * red.max_weight))
        return LambdaRange(2, hi)
    return LambdaRange(1, c)


# ---------------------------------------------------------------------------
# GPU-backed sweeps
# ---------------------------------------------------------------------------
def dff_bound_batch(kind, red, lo: int, hi: int) -> np.ndarray:
    """Per-lambda bounds for the inclusive grid [lo, hi] as int64
    (bounds.py:463-501), evaluated on the GPU in one call."""
    kind = _kind(kind)
    if hi < lo:
        return np.zeros(0, dtype=np.int64)
    c, w = as_reduced(red)
    return _native.default_engine().dff_bound_batch(kind.id, w, c, lo, hi)


def dff_bound(kind, red, lam: int) -> int:
    """Bound from a single grid point: ceil(sum f(w) / f(c)) (bounds.py:276-290)."""
    return int(dff_bound_batch(kind, red, lam, lam)[0])


def _result_seq(res: _native.BplbResult, kinds: Sequence[DffKind], ids: Sequence[int], k: int) -> BoundResult:
    best, ev, arg, nl = res.best[:], res.evaluated[:], res.arg_lambda[:], res.n_lambda[:]
    out = BoundResult(lb=0)
    per, args = out.per_dff, out.arg
    lb = evals = 0
    for i in range(res.n_done):
        kind, kid = kinds[i], ids[i]
        b = best[kid] if ev[kid] else 0
        per[kind] = b
        args[kind] = arg[kid]
        evals += nl[kid]
        if b > lb:
            lb = b
    out.lb, out.evals, out.exceeded_k = lb, evals, lb > k
    return out


def lower_bound_seq(red, k: int, kinds: Sequence = DEFAULT_DFF_ORDER) -> BoundResult:
    """Sequential sweep (Alg. 2, bounds.py:504-527): kinds in order, each over
    its full parameter grid, early exit once the bound exceeds ``k``.

    The GPU runs the kinds in order (one phase per kind, the Alg. 3/4
    "launch per DFF, guard lb <= k" shape) and stops after the first kind
    whose best exceeds ``k``; ``per_dff`` / ``evals`` / ``lb`` then match the
    reference's early-exit semantics exactly (0 for empty ranges, keys in
    evaluation order)."""
    kinds, ids = resolve_kinds(kinds)
    c, w = as_reduced(red)
    if not kinds:
        return BoundResult(lb=0, exceeded_k=0 > k)
    res = _native.default_engine().check(w, c, k, ids, _native.F_PHASED)
    return _result_seq(res, kinds, ids, k)
