"""The path's input type: a reduced instance (capacity + reduced weights).

Mirrors ``ReducedInstance`` (/root/reference/pkg/src/binpack/instances.py:75-97):
same fields, same validation (``c >= 1`` and every weight in ``[1, c]``,
ValueError otherwise), same ``r`` / ``max_weight`` properties.  Every bound
function of this package also accepts the reference's own ReducedInstance
(any object with ``.c`` and ``.weights``) and an array-native form
(``ReducedInstance.from_array``) that keeps the weights as a contiguous
int32 array so no per-call tuple conversion is paid on the hot path.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["ReducedInstance", "ArrayReducedInstance", "as_reduced", "reduce_packing_arrays"]


@dataclass(frozen=True)
class ReducedInstance:
    """Weights derived from a partial packing: unpacked items plus one
    virtual item per non-empty bin.  May be empty."""

    c: int
    weights: tuple = ()
    _array: np.ndarray | None = field(default=None, repr=False, compare=False, hash=False)

    def __post_init__(self) -> None:
        if self.c < 1:
            raise ValueError(f"capacity must be >= 1, got {self.c}")
        if self._array is None:
            for w in self.weights:
                if not 1 <= w <= self.c:
                    raise ValueError(f"reduced weight {w} outside [1, {self.c}]")
            object.__setattr__(self, "weights", tuple(self.weights))

    @classmethod
    def from_array(cls, c: int, weights: np.ndarray) -> "ArrayReducedInstance":
        """Array-native instance (vectorised validation, no Python tuple)."""
        return ArrayReducedInstance(c, weights)

    @property
    def r(self) -> int:
        return len(self.weights)

    @property
    def max_weight(self) -> int:
        if self._array is not None:
            return int(self._array.max()) if self._array.size else 0
        return max(self.weights) if self.weights else 0

    def array(self) -> np.ndarray:
        """Weights as a contiguous int32 array (cached)."""
        if self._array is None:
            object.__setattr__(self, "_array", np.asarray(self.weights, dtype=np.int64).astype(np.int32))
        return self._array


class ArrayReducedInstance:
    """Reduced instance whose weights stay a contiguous int32 array; the
    ``weights`` tuple is only built if someone asks for it."""

    __slots__ = ("c", "_array", "_tuple")

    def __init__(self, c: int, weights):
        c = int(c)
        if c < 1:
            raise ValueError(f"capacity must be >= 1, got {c}")
        a = np.ascontiguousarray(np.asarray(weights).reshape(-1))
        if a.size and (a.min() < 1 or a.max() > c):
            bad = a[(a < 1) | (a > c)][0]
            raise ValueError(f"reduced weight {int(bad)} outside [1, {c}]")
        self.c = c
        self._array = a.astype(np.int32, copy=False)
        self._tuple = None

    @property
    def weights(self) -> tuple:
        if self._tuple is None:
            self._tuple = tuple(self._array.tolist())
        return self._tuple

    @property
    def r(self) -> int:
        return int(self._array.size)

    @property
    def max_weight(self) -> int:
        return int(self._array.max()) if self._array.size else 0

    def array(self) -> np.ndarray:
        return self._array


MAX_C = 1 << 30  # BPLB_MAX_C (include/bplb.h)


def as_reduced(red) -> tuple[int, np.ndarray]:
    """(c, int32 weights) from our ReducedInstance, the reference's, or a pair."""
    c0 = int(red[0]) if isinstance(red, tuple) and not hasattr(red, "c") else int(red.c)
    if c0 > MAX_C:
        raise ValueError(f"capacity {c0} exceeds the GPU integer envelope (2^30); see DESIGN.md")
    if isinstance(red, (ReducedInstance, ArrayReducedInstance)):
        return red.c, red.array()
    if isinstance(red, tuple) and len(red) == 2 and not hasattr(red, "c"):
        c, w = red
        return int(c), np.ascontiguousarray(w, dtype=np.int32)
    c = int(red.c)
    w = red.weights
    if isinstance(w, np.ndarray):
        return c, np.ascontiguousarray(w, dtype=np.int32)
    return c, np.asarray(w, dtype=np.int64).astype(np.int32)


def reduce_packing_arrays(weights: np.ndarray, assign: np.ndarray, n_bins: int, c: int):
    """Array form of reduce_packing (instances.py:262-282) for one node:
    ``assign[i]`` is the committed bin of item i or -1 if the item is open.
    Returns the reduced weights in reference order (open items in item
    order, then the positive bin loads in bin order)."""
    weights = np.asarray(weights, dtype=np.int64)
    assign = np.asarray(assign)
    open_w = weights[assign < 0]
    loads = np.bincount(assign[assign >= 0], weights=weights[assign >= 0], minlength=n_bins).astype(np.int64)
    if (loads > c).any():
        j = int(np.argmax(loads > c))
        raise ValueError(f"bin {j} committed load {int(loads[j])} exceeds capacity {c}")
    return np.concatenate([open_w, loads[loads > 0]]).astype(np.int32)
