// bplb_ubound.cuh -- exact per-lambda and per-range upper-bound tests of the
// bound pruning (the relaxations derived in bplb_prune.cuh's header), shared by
// the bound-pruned node kernel, the grid-wide path and the multi-CTA node
// kernel.  All tests answer "bound(l) <= B is guaranteed" (true) or "unknown".
#pragma once
#include "bplb_device.cuh"

namespace bplb {

// ---- upper-bound tests (true => bound(l) <= B is guaranteed) ----------------
// Integer envelope: c <= 2^18, r <= 2^14 (PR envelope) keeps every product
// below 2^63 (l Vs <= 2^18 * 2^14 * 2^17).
// f(c, lambda) per kind (bplb_core.h bplb_fc) with 32-bit divisions (c < 2^31).
__device__ __forceinline__ int64_t pr_fc(int kind, int64_t c, int64_t lam) {
    switch (kind) {
    case K_MT: case K_RAD2: return c;
    case K_FS1: return c * lam;
    case K_CCM1: return 2 * (int64_t)((uint32_t)c / (uint32_t)lam);
    case K_VB2: return 2 * (lam - 1);
    default: {
        const int64_t q = (int64_t)((uint32_t)c / (uint32_t)lam);
        return q * (lam - (c - q * lam));
    }
    }
}

// floor(x / c) for x < 2^64 with cinv = floor((2^64 - 1) / c): the estimate is
// low by at most one (no 64-bit division in the per-lambda tests).
__device__ __forceinline__ uint64_t pr_udiv_c(uint64_t x, uint32_t c, uint64_t cinv) {
    const uint64_t q = __umul64hi(x, cinv);
    return x - q * c >= c ? q + 1 : q;
}

__device__ __forceinline__ bool ub_le_vb2(const NodeStats& st, int64_t c, int64_t lam, int64_t B) {
    const int64_t ns = st.n_small, nm = st.n_big - st.n_full, K = (int64_t)st.n_eq + 2 * (int64_t)st.n_big;
    // c * S_hi without the floors (linear in lambda)
    const int64_t env = 2 * (lam * st.Vs - ns) - 2 * (lam * st.Vm - c * nm) + c * K * (lam - 1);
    if (env <= 2 * c * B * (lam - 1)) return true;
    const int64_t fs = (int64_t)pr_udiv_c((uint64_t)(lam * st.Vs - ns), (uint32_t)c, st.cinv);  // l Vs >= 2 ns > ns
    int64_t y = (int64_t)pr_udiv_c((uint64_t)(lam * st.Vm) + (uint64_t)c - 1, (uint32_t)c, st.cinv) - nm;
    y = y > 0 ? y : 0;
    return 2 * fs - 2 * y + K * (lam - 1) <= 2 * B * (lam - 1);
}

// (32-bit divisions in the node-kernel envelope, Vs, Vm < 2^32; WENV: the
// grid-wide path's envelope, c <= 2^20, r <= 2^17, 64-bit divisions)
template <bool WENV = false>
__device__ __forceinline__ bool ub_le_ccm1(const NodeStats& st, int64_t c, int64_t lam, int64_t B) {
    const uint32_t L = (uint32_t)lam;
    const int64_t q = (int64_t)((uint32_t)c / L);
    const int64_t K = (int64_t)st.n_eq + 2 * (int64_t)st.n_big;
    const int64_t lhs = 2 * st.Vs - 2 * st.Vm + 2 * (int64_t)st.n_big * (lam - 1);
    if (lhs <= (2 * B - K) * q * lam) return true;
    const int64_t z = st.Vm - (int64_t)st.n_big * (lam - 1);
    if (WENV) {
        const int64_t y = z > 0 ? (z + lam - 1) / lam : 0;
        return 2 * (st.Vs / lam) + K * q - 2 * y <= 2 * B * q;
    }
    const int64_t y = z > 0 ? (int64_t)(((uint32_t)z + L - 1) / L) : 0;
    return 2 * (int64_t)((uint32_t)st.Vs / L) + K * q - 2 * y <= 2 * B * q;
}

__device__ __forceinline__ bool ub_le_bj1(const NodeStats& st, int64_t c, int64_t lam, int64_t B) {
    const int64_t cm = (int64_t)((uint32_t)c % (uint32_t)lam);
    return st.W <= B * (c - cm);
}

template <bool WENV = false>
__device__ __forceinline__ bool ub_le(int kind, const NodeStats& st, int64_t c, int64_t lam, int64_t B) {
    if (B < 0) return false;
    if (kind == K_VB2) return ub_le_vb2(st, c, lam, B);
    if (kind == K_CCM1) return ub_le_ccm1<WENV>(st, c, lam, B);
    return ub_le_bj1(st, c, lam, B);
}

// Every lambda of [l1, l2] has bound <= B (relaxations monotone over ranges).
__device__ __forceinline__ bool ub_le_range(int kind, const NodeStats& st, int64_t c, int64_t l1, int64_t l2,
                                            int64_t B) {
    if (B < 0) return false;
    if (kind == K_VB2) {
        const int64_t ns = st.n_small, nm = st.n_big - st.n_full, K = (int64_t)st.n_eq + 2 * (int64_t)st.n_big;
        auto g = [&](int64_t l) {
            return 2 * (l * st.Vs - ns) - 2 * (l * st.Vm - c * nm) + c * K * (l - 1) - 2 * c * B * (l - 1);
        };
        return g(l1) <= 0 && g(l2) <= 0;
    }
    if (kind == K_CCM1) {
        const int64_t K = (int64_t)st.n_eq + 2 * (int64_t)st.n_big;
        const int64_t lhs = 2 * st.Vs - 2 * st.Vm + 2 * (int64_t)st.n_big * (l2 - 1);
        const int64_t coef = 2 * B - K;
        return coef >= 0 ? lhs <= coef * (c - l2 + 1) : lhs <= coef * c;
    }
    return c - l2 + 1 > 0 && st.W <= B * (c - l2 + 1);
}

// Pruning threshold snapshot (the shared best only grows, so a stale one is safe).
struct Thr {
    int64_t B, a_rel;
    bool has, lbmode;
};

// Key-mode threshold from a packed per-kind key (the grid-wide path).
__device__ __forceinline__ Thr thr_from_key(u64 key) {
    Thr t;
    t.lbmode = false;
    t.has = key != 0;
    t.B = (int64_t)(key >> 32);
    t.a_rel = (int64_t)(0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFu));
    return t;
}

template <bool WENV = false>
__device__ __forceinline__ bool lam_skip(const Thr& t, int kind, const NodeStats& st, int64_t c, int64_t lo,
                                         int64_t lam) {
    if (!t.has) return false;
    if (t.lbmode) return ub_le<WENV>(kind, st, c, lam, t.B);
    const int64_t rel = lam - lo;
    if (rel == t.a_rel) return true;  // the current arg itself: already evaluated
    if (rel > t.a_rel) return ub_le<WENV>(kind, st, c, lam, t.B);
    return t.B >= 1 && ub_le<WENV>(kind, st, c, lam, t.B - 1);
}

__device__ __forceinline__ bool range_skip(const Thr& t, int kind, const NodeStats& st, int64_t c, int64_t lo,
                                           int64_t l1, int64_t l2) {
    if (!t.has) return false;
    if (t.lbmode) return ub_le_range(kind, st, c, l1, l2, t.B);
    if (l1 - lo > t.a_rel) return ub_le_range(kind, st, c, l1, l2, t.B);
    return t.B >= 1 && ub_le_range(kind, st, c, l1, l2, t.B - 1);
}

}  // namespace bplb
