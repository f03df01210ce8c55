// bplb_device.cuh -- device building blocks shared by the node-resident and
// the grid-wide kernels: lookup structures, the modular (VB2/FS1) dense walk,
// the magic-division (CCM1/BJ1 small lambda) dense sums, warp reductions and
// the per-lambda "emit" that ceil-divides and max-reduces.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "bplb_core.h"

namespace bplb {

constexpr int kWarp = 32;
constexpr int LMOD = 128;   // lambdas per modular (VB2/FS1) unit
constexpr int GMOD_MAX = 16; // items per lane per modular group (max)
constexpr int LLOOK = 32;   // lambdas per lookup unit (one per lane)
constexpr int LDIV = 32;    // lambdas per division unit

enum UnitType { T_LOOKUP = 0, T_MOD = 1, T_DIV = 2 };

typedef unsigned long long u64;

// ---------------------------------------------------------------------------
// Lookup structures: n_le(x) = #{w <= x}, w_le(x) = sum of those w.
// ---------------------------------------------------------------------------
struct LkSorted {  // sorted weights + prefix sums (shared memory)
    const int* sw;
    const long long* pre;
    int r;
    int top;  // highest power of two <= r (0 if r == 0)
    __device__ __forceinline__ int64_t n_le(int64_t x) const {
        int pos = 0;
        for (int s = top; s > 0; s >>= 1) {
            int nx = pos + s;
            if (nx <= r && (int64_t)sw[nx - 1] <= x) pos = nx;
        }
        return pos;
    }
    __device__ __forceinline__ void both(int64_t x, int64_t* n, int64_t* w) const {
        int64_t k = n_le(x);
        *n = k;
        *w = pre[k];
    }
};

struct LkBucket {  // sorted weights + prefix sums + coarse value->index buckets
    const int* sw;          // sorted weights [r]
    const long long* pre;   // prefix sums [r+1]
    const int* bidx;        // bidx[b] = #{w < (b << k)}, b in [0, nb]; bidx[nb] = r
    int r;
    int k;
    int64_t c;
    __device__ __forceinline__ int64_t n_le(int64_t x) const {
        if (x < 0) return 0;
        if (x >= c) return r;
        const int b = (int)(x >> k);
        int i = bidx[b];
        const int e = bidx[b + 1];
        while (i < e && (int64_t)sw[i] <= x) ++i;
        return i;
    }
    __device__ __forceinline__ void both(int64_t x, int64_t* n, int64_t* w) const {
        int64_t kk = n_le(x);
        *n = kk;
        *w = pre[kk];
    }
};

struct LkTable {  // cumulative tables over values [-1, c] (index x+1)
    const int* cnt;
    const long long* wle;
    int64_t c;
    __device__ __forceinline__ int64_t idx(int64_t x) const {
        return (x < -1 ? -1 : (x > c ? c : x)) + 1;
    }
    __device__ __forceinline__ int64_t n_le(int64_t x) const { return cnt[idx(x)]; }
    __device__ __forceinline__ void both(int64_t x, int64_t* n, int64_t* w) const {
        int64_t i = idx(x);
        *n = cnt[i];
        *w = wle[i];
    }
};

struct LkTableG {  // same, global memory (L2-resident), one 16-byte record per value
    const ulonglong2* rec;  // {W<=(x), N<=(x)} at index x+1
    int64_t c;
    __device__ __forceinline__ int64_t idx(int64_t x) const {
        return (x < -1 ? -1 : (x > c ? c : x)) + 1;
    }
    __device__ __forceinline__ int64_t n_le(int64_t x) const { return (int64_t)__ldg(&rec[idx(x)].y); }
    __device__ __forceinline__ void both(int64_t x, int64_t* n, int64_t* w) const {
        const ulonglong2 v = __ldg(rec + idx(x));
        *n = (int64_t)v.y;
        *w = (int64_t)v.x;
    }
};

// ---------------------------------------------------------------------------
// Warp helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ u64 warp_sum_u64(u64 v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Transposed reduction of 8 per-lane values: on return, every lane holds the
// warp-wide sum of v[(lane >> 2) & 7].  9 shuffles instead of 8 x 5.
template <typename T>
__device__ __forceinline__ T reduce8_transposed(T v[8], int lane) {
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
    T a[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        T send = b4 ? v[i] : v[i + 4];
        T keep = b4 ? v[i + 4] : v[i];
        a[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    T b[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        T send = b3 ? a[i] : a[i + 2];
        T keep = b3 ? a[i + 2] : a[i];
        b[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    T send = b2 ? b[0] : b[1];
    T keep = b2 ? b[1] : b[0];
    T x = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    x += __shfl_xor_sync(0xffffffffu, x, 2);
    x += __shfl_xor_sync(0xffffffffu, x, 1);
    return x;
}

// ---------------------------------------------------------------------------
// Modular dense walk (VB2 and FS1).  For every item with weight w the state
//   s(lambda) = (w * (lambda + ofs) - delta) mod c
// (VB2: ofs = 0, delta = [2w < c];  FS1: ofs = 1, delta = 0) advances by
// s <- (s + w) mod c per lambda step: one IMAD-add plus one VIADDMNMX
// (min(s + w, s + w - c), unsigned) per (item, lambda) cell.  The warp
// accumulates, per lambda, D = sum of s (weighted by the item's count for
// distinct-value lists) into the per-warp shared array tot[0..L) (added to,
// not overwritten, so several item slices may accumulate).  FS1's
// zero-remainder term is recovered from the lookup tables (bplb_fs1_zero),
// so FS1 and VB2 share this one loop.
//
// WIDE selects 64-bit lane partials (needed when 32 * G * c >= 2^32).
// ---------------------------------------------------------------------------
template <bool WIDE, bool WEIGHTED, int GMOD>
__device__ __forceinline__ void mod_group(const int* __restrict__ items, int g, int i_end,
                                          uint32_t c, u64 cinv, int64_t lam_a, int L, u64* tot,
                                          uint32_t one, const int* __restrict__ counts, int ofs,
                                          bool vb2) {
    const int lane = threadIdx.x & 31;
    const uint32_t negc = 0u - c;
    uint32_t s[GMOD], u[GMOD], um[GMOD], cw[WEIGHTED ? GMOD : 1];
    const uint32_t mult = (uint32_t)(lam_a + ofs);
#pragma unroll
    for (int t = 0; t < GMOD; ++t) {
        const int idx = g + lane + kWarp * t;
        const uint32_t w = idx < i_end ? (uint32_t)items[idx] : 0u;
        if (WEIGHTED) cw[t] = idx < i_end ? (uint32_t)counts[idx] : 0u;
        u[t] = w;
        um[t] = w + negc;
        s[t] = w == 0 ? 0u : bplb_mulmod(w, mult, (vb2 && 2 * w < c) ? 1u : 0u, c, cinv);
    }
    typedef typename std::conditional<WIDE, u64, uint32_t>::type Acc;
    for (int sb = 0; sb < L; sb += 8) {
        Acc acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            acc[j] = 0;
#pragma unroll
            for (int t = 0; t < GMOD; ++t) {
                if (WEIGHTED) {
                    acc[j] += (Acc)s[t] * (Acc)cw[t];
                } else if (!WIDE && (t % 3) == 2) {
                    // every third accumulate on the IMAD pipe: the walk is
                    // ALU-bound (VIADDMNMX + IADD3), this balances the pipes
                    uint32_t a = (uint32_t)acc[j];
                    asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(a) : "r"(s[t]), "r"(one));
                    acc[j] = (Acc)a;
                } else {
                    acc[j] += (Acc)s[t];
                }
                // s <- min(s + w, s + w - c)  (unsigned; exactly one is < c)
                uint32_t b;
                asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(b) : "r"(s[t]), "r"(one), "r"(um[t]));
                s[t] = __viaddmin_u32(s[t], u[t], b);
            }
        }
        u64 tot_j;
        if (WIDE) {
            u64 v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = (u64)acc[j];
            tot_j = reduce8_transposed<u64>(v, lane);
        } else {
            uint32_t v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = (uint32_t)acc[j];
            tot_j = (u64)reduce8_transposed<uint32_t>(v, lane);
        }
        const int jj = sb + ((lane >> 2) & 7);
        if ((lane & 3) == 0 && jj < L) tot[jj] += tot_j;
    }
}

// Walk items [i_begin, i_end) in groups of 32 x G items (G = 16 or 8;
// 4 for weighted distinct-value lists).  ofs / vb2 select FS1 or VB2.
template <bool WIDE, bool WEIGHTED = false, int GMAX = 16>
__device__ __forceinline__ void mod_walk(const int* __restrict__ items, int i_begin, int i_end,
                                         uint32_t c, u64 cinv, int64_t lam_a, int L, u64* tot,
                                         uint32_t one, bool vb2,
                                         const int* __restrict__ counts = nullptr) {
    const int ofs = vb2 ? 0 : 1;
    int g = i_begin;
    while (g < i_end) {
        const int rem = i_end - g;
        if (WEIGHTED) {
            mod_group<WIDE, WEIGHTED, 4>(items, g, i_end, c, cinv, lam_a, L, tot, one, counts, ofs, vb2);
            g += 4 * kWarp;
        } else if (GMAX >= 16 && rem > 8 * kWarp) {
            mod_group<WIDE, WEIGHTED, 16>(items, g, i_end, c, cinv, lam_a, L, tot, one, counts, ofs, vb2);
            g += 16 * kWarp;
        } else {
            mod_group<WIDE, WEIGHTED, 8>(items, g, i_end, c, cinv, lam_a, L, tot, one, counts, ofs, vb2);
            g += 8 * kWarp;
        }
    }
}

// ---------------------------------------------------------------------------
// Division dense sums for one lambda (CCM1 / BJ1 at small lambda, where the
// harmonic lookups would cost more than a pass over the items).
// ---------------------------------------------------------------------------
// CCM1: S = 2 A_s + n_eq*cq + 2 n_big*cq - 2 A_b,  A_s = sum_small floor(w/l),
//       A_b = sum_big floor((c-w)/l)      (bounds.py:181-186, 308-311)
__device__ __forceinline__ int64_t ccm1_dense(const int* sw, const NodeStats& st, int64_t c,
                                              int64_t lam) {
    const int lane = threadIdx.x & 31;
    const Div31 dv = bplb_div31((uint32_t)lam);
    u64 as = 0, ab = 0;
    for (int i = lane; i < st.n_small; i += kWarp) as += bplb_udiv31((uint32_t)sw[i], dv);
    for (int i = st.r - st.n_big + lane; i < st.r; i += kWarp)
        ab += bplb_udiv31((uint32_t)(c - sw[i]), dv);
    int64_t A = (int64_t)warp_sum_u64(as) - (int64_t)warp_sum_u64(ab);
    int64_t cq = c / lam;
    return 2 * A + (int64_t)st.n_eq * cq + 2 * (int64_t)st.n_big * cq;
}

// CCM1 over an unsorted item array (grid-wide path): classify per item.
__device__ __forceinline__ int64_t ccm1_dense_raw(const int* w, int n, const NodeStats& st, int64_t c,
                                                  int64_t lam) {
    const int lane = threadIdx.x & 31;
    const Div31 dv = bplb_div31((uint32_t)lam);
    const uint32_t c32 = (uint32_t)c;
    long long a = 0;
    for (int i = lane; i < n; i += kWarp) {
        const uint32_t x = (uint32_t)__ldg(w + i);
        if (2ull * x < c32) a += bplb_udiv31(x, dv);
        else if (2ull * x > c32) a -= bplb_udiv31(c32 - x, dv);
    }
    const int64_t A = (int64_t)warp_sum_u64((u64)a);
    const int64_t cq = c / lam;
    return 2 * A + (int64_t)st.n_eq * cq + 2 * (int64_t)st.n_big * cq;
}

// BJ1: S = (l - cm) * sum floor(w/l) + sum max(0, w mod l - cm)
//       (bounds.py:200-206, 319-323)
__device__ __forceinline__ int64_t bj1_dense(const int* w, int n, int64_t c, int64_t lam) {
    const int lane = threadIdx.x & 31;
    const Div31 dv = bplb_div31((uint32_t)lam);
    const uint32_t cm = (uint32_t)(c % lam), l32 = (uint32_t)lam;
    u64 q_sum = 0, e_sum = 0;
    for (int i = lane; i < n; i += kWarp) {
        uint32_t x = (uint32_t)w[i];
        uint32_t q = bplb_udiv31(x, dv);
        uint32_t wm = x - q * l32;
        q_sum += q;
        e_sum += (wm > cm) ? (wm - cm) : 0u;
    }
    q_sum = warp_sum_u64(q_sum);
    e_sum = warp_sum_u64(e_sum);
    return (lam - (int64_t)cm) * (int64_t)q_sum + (int64_t)e_sum;
}

// ---------------------------------------------------------------------------
// Per-lambda emit: each lane holds (lambda, bound) or an invalid lane.
// Warp-reduces max bound / lowest lambda and folds it into *key with one
// atomicMax; optionally writes the per-lambda vector.  Returns the warp max.
// key = bound << 32 | (0xFFFFFFFF - (lambda - lo))  (lowest lambda on ties).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t emit_warp(bool valid, int64_t lam, int64_t bound, int64_t kind_lo,
                                             u64* key, int64_t* lam_out, int64_t out_lo,
                                             int64_t out_hi) {
    if (lam_out && valid && lam >= out_lo && lam <= out_hi) lam_out[lam - out_lo] = bound;
    uint32_t bv = valid ? (uint32_t)bound + 1u : 0u;
    uint32_t mx = __reduce_max_sync(0xffffffffu, bv);
    if (mx == 0) return -1;
    uint32_t rel = (valid && bv == mx) ? (uint32_t)(lam - kind_lo) : 0xFFFFFFFFu;
    uint32_t mn = __reduce_min_sync(0xffffffffu, rel);
    if ((threadIdx.x & 31) == 0) {
        u64 k = ((u64)(mx - 1u) << 32) | (u64)(0xFFFFFFFFu - mn);
        atomicMax(key, k);
    }
    return (int64_t)(mx - 1u);
}

// emit_warp with a per-warp cache of the key (lane 0's view, kc): the
// atomicMax is sent only when the warp's candidate beats what it last saw, so
// losing candidates do not queue on the key's L2 line.
__device__ __forceinline__ int64_t emit_warp_cached(bool valid, int64_t lam, int64_t bound, int64_t kind_lo,
                                                    u64* key, u64* kc, int64_t* lam_out, int64_t out_lo,
                                                    int64_t out_hi) {
    if (lam_out && valid && lam >= out_lo && lam <= out_hi) lam_out[lam - out_lo] = bound;
    uint32_t bv = valid ? (uint32_t)bound + 1u : 0u;
    uint32_t mx = __reduce_max_sync(0xffffffffu, bv);
    if (mx == 0) return -1;
    uint32_t rel = (valid && bv == mx) ? (uint32_t)(lam - kind_lo) : 0xFFFFFFFFu;
    uint32_t mn = __reduce_min_sync(0xffffffffu, rel);
    if ((threadIdx.x & 31) == 0) {
        u64 k = ((u64)(mx - 1u) << 32) | (u64)(0xFFFFFFFFu - mn);
        if (k > *kc) {
            atomicMax(key, k);
            *kc = k;
        }
    }
    return (int64_t)(mx - 1u);
}

}  // namespace bplb
