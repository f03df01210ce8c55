"""ctypes binding of libbplb.so (include/bplb.h).

The product path has no CPU fallback: if the shared library is missing or no
sm_100 device is visible, every bound call raises.  Build the library with
``python -c "import __graft_entry__ as g; g.build()"`` (or
``python paper_2402_14821_b200/build_native.py``).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BPLB_LIB") or os.path.join(_HERE, "libbplb.so")  # BPLB_LIB: A/B builds

NKINDS = 6
F_PHASED = 0x1
F_CANCEL = 0x2
F_TIMING = 0x4
F_NOTAB = 0x8  # batched: skip the histogram x table kernel (parity testing)
F_NOPRUNE = 0x10  # dense sweep: every lambda evaluated (no bound pruning)
F_NOTC = 0x20  # batched table path on the FP32 pipe instead of the tensor cores (parity testing)

# bplb_last_path ids (include/bplb.h)
PATHS = {0: "none", 1: "tab", 2: "tab_single", 3: "warp", 4: "node_table", 5: "node_sort", 6: "wide", 7: "prune",
         8: "tc", 9: "knap"}
KN_REACH_ONLY = 0x100  # knapsack bins: reach + tightening only
KN_NO_TIGHTEN = 0x200  # knapsack bins: filter on the input interval (knapsack_item_filter)

E_INVAL, E_RANGE, E_CUDA, E_NOMEM, E_NODEV = -1, -2, -3, -4, -5

INT64_MAX = (1 << 63) - 1
INT64_MIN = -(1 << 63)


class BplbResult(ctypes.Structure):
    _fields_ = [
        ("best", ctypes.c_int64 * NKINDS),
        ("arg_lambda", ctypes.c_int64 * NKINDS),
        ("n_lambda", ctypes.c_int64 * NKINDS),
        ("evals", ctypes.c_int64 * NKINDS),
        ("evaluated", ctypes.c_int32 * NKINDS),
        ("n_done", ctypes.c_int32),
        ("exceeded", ctypes.c_int32),
        ("lb", ctypes.c_int64),
        ("evals_total", ctypes.c_int64),
    ]


_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_vp = ctypes.c_void_p

# symbol -> (restype, argtypes); also the list the CPU test checks is exported
SIGNATURES = {
    "bplb_engine_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_vp)]),
    "bplb_engine_destroy": (ctypes.c_int, [_vp]),
    # pointers as plain addresses: this is the per-node drop-in call, and
    # ctypes' data_as/byref conversions cost microseconds each
    "bplb_check": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                  _vp, ctypes.c_int32, ctypes.c_int32, _vp]),
    "bplb_check_ranges": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                         _vp, ctypes.c_int32, ctypes.c_int32, _vp, _vp, _vp]),
    "bplb_check_multi": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                        _vp, ctypes.c_int32, ctypes.c_int32, _vp]),
    "bplb_dff_bound_batch": (ctypes.c_int, [_vp, ctypes.c_int32, _i32p, ctypes.c_int64, ctypes.c_int64,
                                            ctypes.c_int64, ctypes.c_int64, _i64p]),
    "bplb_check_batch": (ctypes.c_int, [_vp, _i32p, _i64p, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_int64, _i32p, ctypes.c_int32, ctypes.c_int32,
                                        _i64p, _u8p, _i64p, _i64p]),
    "bplb_check_batch_ex": (ctypes.c_int, [_vp, _vp, ctypes.c_int32, _vp, ctypes.c_int64,
                                           ctypes.c_int64, ctypes.c_int64, _vp, ctypes.c_int32,
                                           ctypes.c_int32, _vp, _vp, _vp, _vp]),
    "bplb_check_batch_device": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64,
                                               ctypes.c_int64, ctypes.c_int64, _i32p, ctypes.c_int32,
                                               ctypes.c_int32, _vp, _vp, _vp, _vp, _vp]),
    "bplb_check_batch_device_ex": (ctypes.c_int, [_vp, _vp, ctypes.c_int32, _vp, ctypes.c_int64,
                                                  ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _vp,
                                                  ctypes.c_int32, ctypes.c_int32, _vp, _vp, _vp, _vp, _vp]),
    "bplb_check_batch_assign": (ctypes.c_int, [_vp, _i32p, ctypes.c_int64, ctypes.c_int64, _vp, ctypes.c_int32,
                                               ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _i32p,
                                               ctypes.c_int32, ctypes.c_int32, _i64p, _u8p, _i64p, _i64p]),
    "bplb_reduce_batch": (ctypes.c_int, [_vp, _i32p, ctypes.c_int64, ctypes.c_int64, _vp, ctypes.c_int32,
                                         ctypes.c_int64, ctypes.c_int64, _i64p, _i32p]),
    "bplb_multi_create": (ctypes.c_int, [_i32p, ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)]),
    "bplb_multi_destroy": (ctypes.c_int, [_vp]),
    "bplb_multi_engine": (ctypes.c_int, [_vp, ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)]),
    "bplb_multi_last_bounds": (ctypes.c_int, [_vp, _i64p]),
    "bplb_check_batch_multi": (ctypes.c_int, [_vp, _vp, ctypes.c_int32, _vp, ctypes.c_int64,
                                              ctypes.c_int64, ctypes.c_int64, _vp, ctypes.c_int32,
                                              ctypes.c_int32, _vp, _vp, _vp, _vp]),
    "bplb_knapsack_bins": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int64, _vp, _vp, _vp, _vp, _vp,
                                          ctypes.c_int32, _vp, _vp, _vp, _vp, _vp]),
    "bplb_knapsack_bins_device": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int64, _vp, _vp, _vp, _vp, _vp,
                                                 ctypes.c_int64, ctypes.c_int32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "bplb_launch_count": (ctypes.c_int64, [_vp]),
    "bplb_last_device_ms": (ctypes.c_double, [_vp]),
    "bplb_profile_kernel": (ctypes.c_int, [_vp, ctypes.c_int]),
    "bplb_last_kernel_ms": (ctypes.c_double, [_vp]),
    "bplb_last_path": (ctypes.c_int, [_vp, _i32p]),
    "bplb_last_error": (ctypes.c_char_p, []),
    "bplb_version": (ctypes.c_char_p, []),
}

_lib = None
_lib_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load libbplb.so and declare every exported signature."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"libbplb.so not found at {path}: the CUDA engine is required (no CPU fallback). "
                "Build it with `python paper_2402_14821_b200/build_native.py`.")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


_cbyte_from_buffer = ctypes.c_byte.from_buffer
_addressof = ctypes.addressof


def _addr(a: np.ndarray) -> int:
    """Data pointer of a contiguous array as a plain int (about 2.5x cheaper
    than a.ctypes.data for writable arrays; read-only ones fall back)."""
    try:
        return _addressof(_cbyte_from_buffer(a))
    except (TypeError, ValueError, BufferError):
        return a.ctypes.data


def _raise(rc: int, what: str):
    msg = load_library().bplb_last_error().decode(errors="replace")
    text = f"{what}: {msg}"
    if rc == E_INVAL:
        raise ValueError(text)
    if rc == E_RANGE:
        raise ValueError(text + " (outside the GPU integer envelope, see DESIGN.md)")
    if rc == E_NOMEM:
        raise MemoryError(text)
    raise RuntimeError(text)


def _clamp_k(k: int) -> int:
    k = int(k)
    return INT64_MAX if k > INT64_MAX else (INT64_MIN if k < INT64_MIN else k)


def as_i32(weights) -> np.ndarray:
    """Weights as a contiguous int32 array (values outside int32 are rejected)."""
    if isinstance(weights, np.ndarray) and weights.dtype == np.int32 and weights.flags.c_contiguous:
        return weights
    a = np.asarray(weights)
    if a.dtype.kind not in "iu" and a.size:
        a = a.astype(np.int64)
    if a.size and (a.max() > 2**31 - 1 or a.min() < -(2**31)):
        raise ValueError("weight outside the GPU integer envelope (int32)")
    return np.ascontiguousarray(a, dtype=np.int32).reshape(-1)


class Engine:
    """One libbplb engine: a CUDA stream plus grow-only device/pinned buffers
    on one device.  Calls are synchronous and serialised inside the library."""

    def __init__(self, device: int = 0):
        self._lib = load_library()
        h = _vp()
        rc = self._lib.bplb_engine_create(int(device), ctypes.byref(h))
        if rc != 0:
            _raise(rc, "bplb_engine_create")
        self._h = h
        self.device = int(device)
        self._kinds_cache: dict = {}

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.bplb_engine_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        if self._h is None:
            raise RuntimeError("engine is closed")
        return self._h

    def launch_count(self) -> int:
        return int(self._lib.bplb_launch_count(self.handle))

    def last_device_ms(self) -> float:
        return float(self._lib.bplb_last_device_ms(self.handle))

    def profile_kernel(self, on: bool) -> None:
        """Bracket the dominant batched kernel with CUDA events (bench)."""
        rc = self._lib.bplb_profile_kernel(self.handle, int(bool(on)))
        if rc != 0:
            _raise(rc, "bplb_profile_kernel")

    def last_kernel_ms(self) -> float:
        return float(self._lib.bplb_last_kernel_ms(self.handle))

    def last_path(self) -> tuple[str, int]:
        """(kernel family, detail) of the last check / batch launch: which
        kernel actually served it (tests assert the intended path ran)."""
        d = ctypes.c_int32(0)
        p = self._lib.bplb_last_path(self.handle, ctypes.byref(d))
        return PATHS.get(int(p), str(p)), int(d.value)

    def check(self, w: np.ndarray, c: int, k: int, kinds, flags: int) -> BplbResult:
        w = as_i32(w)
        key = tuple(kinds)
        ks = self._kinds_cache.get(key)
        if ks is None:
            ks = self._kinds_cache[key] = (ctypes.c_int32 * len(key))(*key)
        res = BplbResult()
        rc = self._lib.bplb_check(self.handle, w.ctypes.data if len(w) else None, len(w), int(c), _clamp_k(k),
                                  ctypes.addressof(ks), len(key), int(flags), ctypes.addressof(res))
        if rc != 0:
            _raise(rc, "bplb_check")
        return res

    def check_ranges(self, w: np.ndarray, c: int, k: int, kinds, flags: int, rng_lo, rng_hi) -> BplbResult:
        """One slice of a lambda-split check: every kind restricted to
        [rng_lo[kd], rng_hi[kd]] (empty when hi < lo), full collection."""
        w = as_i32(w)
        ks = (ctypes.c_int32 * len(kinds))(*kinds)
        lo = np.ascontiguousarray(rng_lo, dtype=np.int64)
        hi = np.ascontiguousarray(rng_hi, dtype=np.int64)
        res = BplbResult()
        rc = self._lib.bplb_check_ranges(self.handle, w.ctypes.data if len(w) else None, len(w), int(c),
                                         _clamp_k(k), ctypes.addressof(ks), len(kinds), int(flags),
                                         lo.ctypes.data, hi.ctypes.data, ctypes.addressof(res))
        if rc != 0:
            _raise(rc, "bplb_check_ranges")
        return res

    def dff_bound_batch(self, kind: int, w: np.ndarray, c: int, lo: int, hi: int) -> np.ndarray:
        w = as_i32(w)
        n = max(0, int(hi) - int(lo) + 1)
        out = np.zeros(n, dtype=np.int64)
        if n == 0:
            return out
        rc = self._lib.bplb_dff_bound_batch(self.handle, int(kind), w.ctypes.data_as(_i32p), len(w), int(c),
                                            int(lo), int(hi), out.ctypes.data_as(_i64p))
        if rc != 0:
            _raise(rc, "bplb_dff_bound_batch")
        return out

    def check_batch(self, w: np.ndarray, offsets: np.ndarray, c: int, k: int, kinds, flags: int,
                    want_best: bool = False, out=None):
        """CSR batch; ``w`` may be int32, or uint16 / uint8 (compact: half /
        a quarter of the host->device bytes), used as-is when contiguous."""
        if isinstance(w, np.ndarray) and w.dtype in (np.uint16, np.uint8) and w.flags.c_contiguous:
            wbytes = w.itemsize
        else:
            w = as_i32(w)
            wbytes = 4
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        n = len(off) - 1
        key = tuple(kinds)
        ks = self._kinds_cache.get(key)
        if ks is None:
            ks = self._kinds_cache[key] = (ctypes.c_int32 * len(key))(*key)
        if out is None:
            lb = np.empty(n, dtype=np.int64)
            ex = np.empty(n, dtype=np.uint8)
        else:
            lb, ex = out
            if not (isinstance(lb, np.ndarray) and lb.dtype == np.int64 and lb.flags.c_contiguous and len(lb) >= n
                    and isinstance(ex, np.ndarray) and ex.itemsize == 1 and ex.flags.c_contiguous and len(ex) >= n):
                raise ValueError("out must be (int64[n], uint8[n]) contiguous arrays")
        best = np.empty((n, NKINDS), dtype=np.int64) if want_best else None
        arg = np.empty((n, NKINDS), dtype=np.int64) if want_best else None
        # plain ints for every pointer (ctypes pointer objects cost ~1-2 us each)
        rc = self._lib.bplb_check_batch_ex(
            self.handle, _addr(w) if w.size else None, wbytes, _addr(off), n, int(c), _clamp_k(k),
            _addressof(ks), len(key), int(flags), _addr(lb), _addr(ex),
            _addr(best) if best is not None else None, _addr(arg) if arg is not None else None)
        if rc != 0:
            _raise(rc, "bplb_check_batch")
        if want_best:
            return lb, ex.view(bool), best, arg
        return lb, ex.view(bool)

    @staticmethod
    def _assign_args(inst_w, assign):
        inst = as_i32(inst_w)
        a = np.ascontiguousarray(assign)
        if a.dtype not in (np.uint8, np.uint16):
            raise ValueError("assignments must be uint8 or uint16 (open = all ones)")
        if a.ndim != 2 or a.shape[1] != len(inst):
            raise ValueError("assignments must be [n_nodes, n_items]")
        return inst, a

    def check_batch_assign(self, inst_w, assign: np.ndarray, n_bins: int, c: int, k: int, kinds, flags: int,
                           want_best: bool = False):
        """Device-side reduce_packing + LB collection for node states given
        as bin assignments (see bplb_check_batch_assign)."""
        inst, a = self._assign_args(inst_w, assign)
        n = a.shape[0]
        ks = np.ascontiguousarray(kinds, dtype=np.int32)
        lb = np.empty(n, dtype=np.int64)
        ex = np.empty(n, dtype=np.uint8)
        best = np.empty((n, NKINDS), dtype=np.int64) if want_best else None
        arg = np.empty((n, NKINDS), dtype=np.int64) if want_best else None
        rc = self._lib.bplb_check_batch_assign(
            self.handle, inst.ctypes.data_as(_i32p), len(inst), int(n_bins), _vp(a.ctypes.data), a.itemsize, n,
            int(c), _clamp_k(k), ks.ctypes.data_as(_i32p), len(ks), int(flags), lb.ctypes.data_as(_i64p),
            ex.ctypes.data_as(_u8p), best.ctypes.data_as(_i64p) if best is not None else None,
            arg.ctypes.data_as(_i64p) if arg is not None else None)
        if rc != 0:
            _raise(rc, "bplb_check_batch_assign")
        if want_best:
            return lb, ex.view(bool), best, arg
        return lb, ex.view(bool)

    def reduce_batch(self, inst_w, assign: np.ndarray, n_bins: int, c: int):
        """Device-side reduce_packing only: the reduced CSR (int32 weights, int64 offsets)."""
        inst, a = self._assign_args(inst_w, assign)
        n = a.shape[0]
        off = np.empty(n + 1, dtype=np.int64)
        w = np.empty(max(1, n * len(inst)), dtype=np.int32)
        rc = self._lib.bplb_reduce_batch(self.handle, inst.ctypes.data_as(_i32p), len(inst), int(n_bins),
                                         _vp(a.ctypes.data), a.itemsize, n, int(c), off.ctypes.data_as(_i64p),
                                         w.ctypes.data_as(_i32p))
        if rc != 0:
            _raise(rc, "bplb_reduce_batch")
        return w[:off[-1]].copy(), off

    def check_batch_device(self, w_ptr: int, off_ptr: int, n_nodes: int, max_r: int, c: int, k: int,
                           kinds, flags: int, lb_ptr: int, ex_ptr: int, best_ptr: int = 0,
                           arg_ptr: int = 0, stream_ptr: int = 0, wbytes: int = 4) -> None:
        key = tuple(kinds)
        ks = self._kinds_cache.get(key)
        if ks is None:
            ks = self._kinds_cache[key] = (ctypes.c_int32 * len(key))(*key)
        # plain ints for every pointer: this call sits inside device-timed loops
        rc = self._lib.bplb_check_batch_device_ex(
            self.handle, w_ptr, wbytes, off_ptr, n_nodes, max_r, c, _clamp_k(k), ctypes.addressof(ks), len(key),
            flags, lb_ptr, ex_ptr, best_ptr or None, arg_ptr or None, stream_ptr or None)
        if rc != 0:
            _raise(rc, "bplb_check_batch_device")

    def knapsack_bins(self, c: int, committed, lo, hi, w, offsets, flags: int = 0, want_reach: bool = False,
                      action_out: np.ndarray | None = None):
        """bplb_knapsack_bins: (status, lo, hi, action, reach or None) per bin.
        ``action_out`` (uint8, >= total items; pinned for a direct D2H copy)
        receives the per-item actions instead of a fresh array."""
        cl, l, h = (as_i32(x) for x in (committed, lo, hi))  # values outside int32 raise
        ww = as_i32(w)
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        n = len(cl)
        if len(l) != n or len(h) != n or len(off) != n + 1:
            raise ValueError("committed / lo / hi / offsets sizes disagree")
        if n and int(off[-1]) > len(ww):
            raise ValueError("offsets run past the weights")
        st = np.empty(n, dtype=np.int32)
        lo_o = np.empty(n, dtype=np.int32)
        hi_o = np.empty(n, dtype=np.int32)
        total = int(off[-1]) if n else 0
        if action_out is not None:
            if action_out.dtype != np.uint8 or not action_out.flags.c_contiguous or len(action_out) < total:
                raise ValueError("action_out must be a contiguous uint8 array of at least the item count")
            act = action_out
        else:
            act = np.zeros(max(1, total), dtype=np.uint8)
        words = (int(c) + 32) // 32
        reach = np.zeros(max(1, n * words), dtype=np.uint32) if want_reach else None
        rc = self._lib.bplb_knapsack_bins(self.handle, int(c), n, _vp(cl.ctypes.data), _vp(l.ctypes.data),
                                          _vp(h.ctypes.data), _vp(ww.ctypes.data), _vp(off.ctypes.data), int(flags),
                                          _vp(st.ctypes.data), _vp(lo_o.ctypes.data), _vp(hi_o.ctypes.data),
                                          _vp(act.ctypes.data), _vp(reach.ctypes.data) if want_reach else None)
        if rc != 0:
            _raise(rc, "bplb_knapsack_bins")
        return st, lo_o, hi_o, act[:total], (reach[:n * words].reshape(n, words) if want_reach else None)

    def knapsack_bins_device(self, c: int, n_bins: int, cl_ptr: int, lo_ptr: int, hi_ptr: int, w_ptr: int,
                             off_ptr: int, max_items: int, flags: int, st_ptr: int, lo_out_ptr: int,
                             hi_out_ptr: int, act_ptr: int, reach_ptr: int = 0, stream_ptr: int = 0) -> None:
        rc = self._lib.bplb_knapsack_bins_device(self.handle, int(c), int(n_bins), cl_ptr, lo_ptr, hi_ptr,
                                                 w_ptr or None, off_ptr, int(max_items), int(flags), st_ptr,
                                                 lo_out_ptr, hi_out_ptr, act_ptr or None, reach_ptr or None,
                                                 stream_ptr or None)
        if rc != 0:
            _raise(rc, "bplb_knapsack_bins_device")


class MultiEngine:
    """Several engines behind one call (``bplb_multi``): a host CSR batch is
    sharded over ``devices`` (contiguous node ranges balanced by item count,
    one host thread per shard) and the verdicts land in one output array."""

    def __init__(self, devices):
        self._lib = load_library()
        self.devices = [int(d) for d in devices]
        arr = (ctypes.c_int32 * len(self.devices))(*self.devices)
        h = ctypes.c_void_p()
        rc = self._lib.bplb_multi_create(arr, len(self.devices), ctypes.byref(h))
        if rc != 0:
            _raise(rc, "bplb_multi_create")
        self._h = h
        self._kinds_cache: dict = {}

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.bplb_multi_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    def last_bounds(self) -> np.ndarray:
        b = np.empty(len(self.devices) + 1, dtype=np.int64)
        rc = self._lib.bplb_multi_last_bounds(self._h, b.ctypes.data_as(_i64p))
        if rc != 0:
            _raise(rc, "bplb_multi_last_bounds")
        return b

    def launch_count(self) -> int:
        total = 0
        for i in range(len(self.devices)):
            e = ctypes.c_void_p()
            if self._lib.bplb_multi_engine(self._h, i, ctypes.byref(e)) == 0:
                total += int(self._lib.bplb_launch_count(e))
        return total

    def check(self, w: np.ndarray, c: int, k: int, kinds, flags: int) -> BplbResult:
        """One reduced instance over every device: each kind's lambda range
        split into one contiguous slice per engine, results merged
        (``bplb_check_multi``)."""
        w = as_i32(w)
        key = tuple(kinds)
        ks = self._kinds_cache.get(key)
        if ks is None:
            ks = self._kinds_cache[key] = (ctypes.c_int32 * len(key))(*key)
        res = BplbResult()
        rc = self._lib.bplb_check_multi(self._h, w.ctypes.data if len(w) else None, len(w), int(c), _clamp_k(k),
                                        ctypes.addressof(ks), len(key), int(flags), ctypes.addressof(res))
        if rc != 0:
            _raise(rc, "bplb_check_multi")
        return res

    def check_batch(self, w: np.ndarray, offsets: np.ndarray, c: int, k: int, kinds, flags: int,
                    want_best: bool = False):
        if isinstance(w, np.ndarray) and w.dtype in (np.uint16, np.uint8) and w.flags.c_contiguous:
            wbytes = w.itemsize
        else:
            w = as_i32(w)
            wbytes = 4
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        n = len(off) - 1
        key = tuple(kinds)
        ks = self._kinds_cache.get(key)
        if ks is None:
            ks = self._kinds_cache[key] = (ctypes.c_int32 * len(key))(*key)
        lb = np.empty(n, dtype=np.int64)
        ex = np.empty(n, dtype=np.uint8)
        best = np.empty((n, NKINDS), dtype=np.int64) if want_best else None
        arg = np.empty((n, NKINDS), dtype=np.int64) if want_best else None
        rc = self._lib.bplb_check_batch_multi(
            self._h, _addr(w) if w.size else None, wbytes, _addr(off), n, int(c), _clamp_k(k),
            _addressof(ks), len(key), int(flags), _addr(lb), _addr(ex),
            _addr(best) if best is not None else None, _addr(arg) if arg is not None else None)
        if rc != 0:
            _raise(rc, "bplb_check_batch_multi")
        if want_best:
            return lb, ex.view(bool), best, arg
        return lb, ex.view(bool)


_engines: dict[int, Engine] = {}
_engines_lock = threading.Lock()


def default_engine(device: int | None = None) -> Engine:
    """Process-wide engine per device (created on first use)."""
    if device is None:
        device = int(os.environ.get("BPLB_DEVICE", "0"))
    with _engines_lock:
        eng = _engines.get(device)
        if eng is None:
            eng = Engine(device)
            _engines[device] = eng
        return eng
