// bplb_knap.cuh -- batched exact knapsack reasoning per bin.
//
// Restates, on the GPU and for many bins in one launch, the reference's
// bitset subset-sum DP (/root/reference/pkg/src/binpack/propagator.py):
//   reachable_sums      :105-110   reach = base | subset sums of the open items, cut at c
//   knapsack_load_tightening :136-143   [lo, hi] <- [lowest, highest] reachable load inside it
//   _exclusion_sums     :171-187   per item, the subset sums of all OTHER open items
//                                   (divide and conquer: m log m shifts)
//   _use_avoid / knapsack_item_filter :146-168   per item: a load in [lo, hi] that uses it /
//                                   avoids it -> keep, remove bin, commit, or wipeout
//   _knapsack_bin       :190-227   all of the above for one bin, sharing one reach pass
//
// A bin is a bitset over loads 0..c in u32 words (bit v of word v >> 5).
// Adding an item of weight w is bits |= bits << w (a funnel shift per word),
// masked at c.  Two code paths, chosen per launch by the word count:
//   * words <= 32 (c <= 1023): one lane segment of 8 / 16 / 32 lanes per bin
//     (4 / 2 / 1 bins per warp), lane i of the segment holds word i in a
//     register; a shift is two __shfl_up_sync + a funnel shift, no shared
//     memory traffic except the divide-and-conquer stack (one word per lane
//     per level).
//   * larger c: one CTA (KN_NT threads) per bin; the stack levels are
//     shared-memory bitsets, each with a live word range [wlo, whi] (bits
//     below the committed load and above committed + the weights added so
//     far are zero, so a shift touches only the live words).
// The work is integer shift/or over shared memory or registers (no
// contraction, no HBM reuse problem): it is bound by issue / shared-memory
// bandwidth, and the bytes in / out per bin are tiny.
//
// Outputs per bin: status (0 ok, 1 wipeout: no reachable load in [lo, hi],
// -1 invalid input), the tightened lo / hi, and per open item an action
// (0 keep, 1 remove the bin: no load uses it, 2 commit: no load avoids it,
// 3 wipeout: neither).  As in _knapsack_bin, the item filter runs on the
// TIGHTENED interval and is skipped (all actions 0) when the tightened lo is
// <= the committed load (propagator.py:208-212).  KN_NO_TIGHTEN filters on
// the input interval with no skip (knapsack_item_filter's semantics).
#pragma once
#include <cstdint>
#include <cub/block/block_scan.cuh>

namespace bplb {
namespace knap {

#ifndef KN_NT_N
#define KN_NT_N 256
#endif
constexpr int KN_NT = KN_NT_N;      // threads per CTA (CTA-per-bin path)
constexpr int KN_WARP_BINS = 8;     // bins per CTA on the warp path (one per warp)
constexpr int KN_MAXD = 26;         // deepest divide-and-conquer stack (m < 2^25 items per bin)
constexpr int KN_F_REACH_ONLY = 0x100;
constexpr int KN_F_NO_TIGHTEN = 0x200;

struct KnParams {
    int32_t c, words, nbuf, flags;
    int64_t n_bins;
    const int64_t* off;          // open items of bin b: w[off[b] .. off[b + 1])
    const int32_t* committed;
    const int32_t* lo;
    const int32_t* hi;
    const int32_t* w;
    int32_t* status;
    int32_t* lo_out;
    int32_t* hi_out;
    uint8_t* action;             // per open item (same CSR positions)
    uint32_t* reach;             // optional: n_bins * words
    int* err;                    // set to 1 on invalid input
    const int32_t* order;        // bins grouped by item count (kn_order_kernel), or null
    unsigned long long* next;    // CTA path: dynamic bin counter (zeroed per launch)
};

__device__ __forceinline__ uint32_t kn_last_mask(int c) {
    const int b = (c + 1) & 31;
    return b ? (1u << b) - 1u : 0xffffffffu;
}

// bits of word i inside the load window [a, b] (a <= b)
__device__ __forceinline__ uint32_t kn_win(int i, int a, int b) {
    const int wa = a >> 5, wb = b >> 5;
    if (i < wa || i > wb) return 0u;
    uint32_t m = 0xffffffffu;
    if (i == wa) m &= 0xffffffffu << (a & 31);
    if (i == wb) m &= 0xffffffffu >> (31 - (b & 31));
    return m;
}

__device__ __forceinline__ int kn_action(bool use, bool avoid) {
    return use ? (avoid ? 0 : 2) : (avoid ? 1 : 3);
}

// depth of the divide-and-conquer recursion over m items (levels below the root)
__host__ __device__ __forceinline__ int kn_depth(int64_t m) {
    int d = 0;
    while (m > 1) { m = (m + 1) >> 1; ++d; }
    return d;
}

// ---- warp path: words <= 32 -------------------------------------------------
// SEG lanes per bin (SEG = 8 / 16 / 32 for c <= 255 / 511 / 1023): a warp
// runs 32 / SEG bins side by side, each on its own lane segment (segment
// masks on every shuffle / vote, so segments may diverge).

// bits |= bits << w on the segment's register bitset (lane sl = word sl)
template <int SEG>
__device__ __forceinline__ uint32_t kn_warp_add(uint32_t v, int w, int sl, uint32_t lmask, uint32_t smask) {
    const int ws = w >> 5, bs = w & 31;
    uint32_t h = __shfl_up_sync(smask, v, ws, SEG);
    uint32_t l = __shfl_up_sync(smask, v, (ws + 1) & (SEG - 1), SEG);
    h = sl >= ws ? h : 0u;
    l = sl >= ws + 1 ? l : 0u;
    v |= bs ? __funnelshift_l(l, h, bs) : h;
    return v & lmask;
}

// v + the subset sums of w[a .. b)
template <int SEG>
__device__ __forceinline__ uint32_t kn_warp_add_range(uint32_t v, const int32_t* w, int64_t a, int64_t b, int sl,
                                                      uint32_t lmask, uint32_t smask) {
    for (int64_t t0 = a; t0 < b; t0 += SEG) {
        const int n = (int)(b - t0 < SEG ? b - t0 : SEG);
        const int mine = sl < n ? w[t0 + sl] : 0;
        for (int j = 0; j < n; ++j)
            v = kn_warp_add<SEG>(v, __shfl_sync(smask, mine, j, SEG), sl, lmask, smask);
    }
    return v;
}

template <int SEG>
__global__ void __launch_bounds__(32 * KN_WARP_BINS) kn_warp_kernel(KnParams p) {
    constexpr int NSEG = 32 / SEG;
    extern __shared__ uint32_t kn_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int seg = lane / SEG, sl = lane % SEG;
    const uint32_t smask = SEG == 32 ? 0xffffffffu : ((1u << SEG) - 1u) << (seg * SEG);
    // recursion level d word of this lane: stack[d * SEG + sl]
    uint32_t* stack = kn_smem + ((size_t)warp * NSEG + seg) * KN_MAXD * SEG;
    const int c = p.c, words = p.words;
    const uint32_t lmask = sl < words - 1 ? 0xffffffffu : sl == words - 1 ? kn_last_mask(c) : 0u;
    const int64_t stride = (int64_t)gridDim.x * KN_WARP_BINS * NSEG;
    for (int64_t i = ((int64_t)blockIdx.x * KN_WARP_BINS + warp) * NSEG + seg; i < p.n_bins; i += stride) {
        const int64_t b = p.order ? p.order[i] : i;
        const int64_t s = p.off[b], e = p.off[b + 1];
        const int m = (int)(e - s);
        const int cl = p.committed[b];
        int lo = p.lo[b], hi = p.hi[b];
        bool bad = cl < 0 || lo < 0 || lo > hi || hi > c || m < 0 || kn_depth(m) >= KN_MAXD;
        for (int64_t t = s + sl; t < e && !bad; t += SEG) {
            const int x = p.w[t];
            if (x < 1 || x > c) bad = true;
        }
        bad = __any_sync(smask, bad);
        if (bad) {
            if (sl == 0) { p.status[b] = -1; atomicExch(p.err, 1); }
            continue;
        }
        // base: the committed load (absent when above c: such a bit can never
        // reach a window inside [0, c], propagator.py:109-110)
        const uint32_t base = (cl <= c && sl == (cl >> 5)) ? (1u << (cl & 31)) : 0u;
        const uint32_t reach = kn_warp_add_range<SEG>(base, p.w, s, e, sl, lmask, smask);
        if (p.reach && sl < words) p.reach[(size_t)b * words + sl] = reach;
        // tightening (propagator.py:201-207)
        const uint32_t inter = sl < words ? reach & kn_win(sl, lo, hi) : 0u;
        const int first = __reduce_min_sync(smask, inter ? sl * 32 + __ffs(inter) - 1 : 0x7fffffff);
        const int last = __reduce_max_sync(smask, inter ? sl * 32 + 31 - __clz(inter) : -1);
        if (last < 0) {  // Wipeout: no reachable load in the interval (actions written as 0)
            if (sl == 0) { p.status[b] = 1; p.lo_out[b] = lo; p.hi_out[b] = hi; }
            if (!(p.flags & KN_F_REACH_ONLY))
                for (int64_t t = s + sl; t < e; t += SEG) p.action[t] = 0;
            continue;
        }
        if (sl == 0) { p.status[b] = 0; p.lo_out[b] = first; p.hi_out[b] = last; }
        if (!(p.flags & KN_F_NO_TIGHTEN)) {
            lo = first;
            hi = last;
        }
        const bool skip = (p.flags & KN_F_REACH_ONLY) || (!(p.flags & KN_F_NO_TIGHTEN) && lo <= cl);
        if (skip || m == 0) {
            if (!(p.flags & KN_F_REACH_ONLY))
                for (int64_t t = s + sl; t < e; t += SEG) p.action[t] = 0;
            continue;
        }
        // exclusion sums by divide and conquer (propagator.py:171-187); the
        // stack bounds are uniform across the segment
        int slo[KN_MAXD], shi[KN_MAXD], st[KN_MAXD];
        int d = 0;
        slo[0] = 0; shi[0] = m; st[0] = 0;
        stack[sl] = base & lmask;
        while (d >= 0) {
            const int a = slo[d], z = shi[d];
            if (z - a == 1) {  // leaf: the sums without item a
                const uint32_t x = stack[d * SEG + sl];
                const int wt = p.w[s + a];
                const bool use = hi >= wt && __any_sync(smask, sl < words && (x & kn_win(sl, max(0, lo - wt), hi - wt)));
                const bool avoid = __any_sync(smask, sl < words && (x & kn_win(sl, lo, hi)));
                if (sl == 0) p.action[s + a] = (uint8_t)kn_action(use, avoid);
                --d;
                continue;
            }
            const int mid = (a + z) >> 1;
            if (st[d] == 2) { --d; continue; }
            const uint32_t v = stack[d * SEG + sl];
            uint32_t nv;
            if (st[d] == 0) {  // left half keeps the right half's weights
                nv = kn_warp_add_range<SEG>(v, p.w, s + mid, s + z, sl, lmask, smask);
                st[d] = 1;
                slo[d + 1] = a; shi[d + 1] = mid;
            } else {
                nv = kn_warp_add_range<SEG>(v, p.w, s + a, s + mid, sl, lmask, smask);
                st[d] = 2;
                slo[d + 1] = mid; shi[d + 1] = z;
            }
            ++d;
            st[d] = 0;
            stack[d * SEG + sl] = nv;
        }
    }
}

// Bins of equal item count run the same divide-and-conquer schedule, so the
// segments of a warp stay converged when they get such bins: one CTA
// counting-sorts the bin ids by item count (capped at KN_ORDER_MAXM).
constexpr int KN_ORDER_MAXM = 4095;
constexpr int KN_ORDER_NT = 1024;
__device__ __forceinline__ int kn_order_key(const int64_t* off, int64_t b) {
    const int64_t m = off[b + 1] - off[b];
    return m < KN_ORDER_MAXM ? (int)m : KN_ORDER_MAXM;
}
__global__ void __launch_bounds__(KN_ORDER_NT) kn_order_kernel(const int64_t* off, int64_t n, int32_t* order) {
    __shared__ int cnt[KN_ORDER_MAXM + 1];
    using Scan = cub::BlockScan<int, KN_ORDER_NT>;
    __shared__ typename Scan::TempStorage tmp;
    for (int i = threadIdx.x; i <= KN_ORDER_MAXM; i += KN_ORDER_NT) cnt[i] = 0;
    __syncthreads();
    for (int64_t b = threadIdx.x; b < n; b += KN_ORDER_NT)
        atomicAdd(&cnt[kn_order_key(off, b)], 1);
    __syncthreads();
    int v[4];
    for (int j = 0; j < 4; ++j) v[j] = cnt[threadIdx.x * 4 + j];
    Scan(tmp).ExclusiveSum(v, v);
    __syncthreads();
    for (int j = 0; j < 4; ++j) cnt[threadIdx.x * 4 + j] = v[j];
    __syncthreads();
    for (int64_t b = threadIdx.x; b < n; b += KN_ORDER_NT)
        order[atomicAdd(&cnt[kn_order_key(off, b)], 1)] = (int32_t)b;
}

// ---- CTA path: one bin per CTA, shared-memory bitsets ------------------------

struct KnLevel {
    int buf;       // physical buffer
    int wlo, whi;  // live words (others are zero); whi < wlo = empty
};

// dst = src | src << w over the live words; returns dst's live range
__device__ __forceinline__ void kn_cta_shift(const uint32_t* src, uint32_t* dst, int slo_, int shi_, int& dlo, int& dhi,
                                             int w, int words, uint32_t lm) {
    const int ws = w >> 5, bs = w & 31;
    dlo = slo_;
    dhi = min(words - 1, shi_ + ws + 1);
    for (int i = dlo + (int)threadIdx.x; i <= dhi; i += KN_NT) {
        uint32_t v = i <= shi_ ? src[i] : 0u;
        const int j = i - ws;
        const uint32_t h = (j >= slo_ && j <= shi_) ? src[j] : 0u;
        const uint32_t l = (j - 1 >= slo_ && j - 1 <= shi_) ? src[j - 1] : 0u;
        v |= bs ? __funnelshift_l(l, h, bs) : h;
        if (i == words - 1) v &= lm;
        dst[i] = v;
    }
    __syncthreads();
}

// level `to` = level `from` + the subset sums of w[a .. b); `spare` is a free
// buffer index, swapped with the result's buffer as needed
__device__ __forceinline__ void kn_cta_add_range(uint32_t* bufs, int words, uint32_t lm, const KnLevel& from,
                                                 KnLevel& to, int& spare, const int32_t* w, int64_t a, int64_t b) {
    int cur = from.buf, clo = from.wlo, chi = from.whi;
    int dst = to.buf, other = spare;
    if (a == b) {  // copy
        for (int i = clo + (int)threadIdx.x; i <= chi; i += KN_NT)
            bufs[(size_t)dst * words + i] = bufs[(size_t)cur * words + i];
        __syncthreads();
        to.wlo = clo; to.whi = chi;
        return;
    }
    for (int64_t t = a; t < b; ++t) {
        int nlo = clo, nhi = chi;  // an empty set stays empty (nothing written)
        if (chi >= clo)
            kn_cta_shift(bufs + (size_t)cur * words, bufs + (size_t)dst * words, clo, chi, nlo, nhi, w[t], words, lm);
        clo = nlo; chi = nhi;
        if (t == a) {
            cur = dst;
            dst = other;
        } else {
            const int tmp = cur;
            cur = dst;
            dst = tmp;
        }
    }
    // result lives in `cur`; the other of (to.buf, spare) is free
    if (cur != to.buf) { spare = to.buf; to.buf = cur; }
    to.wlo = clo; to.whi = chi;
}

__device__ __forceinline__ bool kn_cta_any(const uint32_t* x, const KnLevel& L, int a, int b) {
    bool hit = false;
    if (a <= b && L.wlo <= L.whi) {
        const int i0 = max(L.wlo, a >> 5), i1 = min(L.whi, b >> 5);
        for (int i = i0 + (int)threadIdx.x; i <= i1; i += KN_NT) hit |= (x[i] & kn_win(i, a, b)) != 0u;
    }
    return __syncthreads_or(hit) != 0;
}

__global__ void __launch_bounds__(KN_NT) kn_cta_kernel(KnParams p) {
    extern __shared__ uint32_t kn_smem[];
    __shared__ int s_bad, s_first, s_last;
    const int c = p.c, words = p.words;
    const uint32_t lm = kn_last_mask(c);
    __shared__ int64_t s_bin;
    for (;;) {
        // dynamic bins, most items first (the order is ascending by item count)
        if (threadIdx.x == 0) s_bin = (int64_t)atomicAdd(p.next, 1ull);
        __syncthreads();
        const int64_t i = s_bin;
        __syncthreads();
        if (i >= p.n_bins) break;
        const int64_t b = p.order ? p.order[p.n_bins - 1 - i] : i;
        const int64_t s = p.off[b], e = p.off[b + 1];
        const int m = (int)(e - s);
        const int cl = p.committed[b];
        int lo = p.lo[b], hi = p.hi[b];
        if (threadIdx.x == 0) {
            s_bad = cl < 0 || lo < 0 || lo > hi || hi > c || m < 0 || kn_depth(m) + 2 > p.nbuf;
            s_first = 0x7fffffff;
            s_last = -1;
        }
        __syncthreads();
        for (int64_t t = s + threadIdx.x; t < e; t += KN_NT) {
            const int x = p.w[t];
            if (x < 1 || x > c) s_bad = 1;
        }
        __syncthreads();
        if (s_bad) {
            if (threadIdx.x == 0) { p.status[b] = -1; atomicExch(p.err, 1); }
            __syncthreads();
            continue;
        }
        // level 0 = base (buffer 0), reach into buffer 1 with buffer 2 spare
        KnLevel L0{0, cl >> 5, cl >> 5};
        if (cl > c) { L0.wlo = 0; L0.whi = -1; }
        if (threadIdx.x == 0 && cl <= c) kn_smem[L0.wlo] = 1u << (cl & 31);
        __syncthreads();
        KnLevel R{1, 0, -1};
        int spare = 2;
        kn_cta_add_range(kn_smem, words, lm, L0, R, spare, p.w, s, e);
        const uint32_t* rb = kn_smem + (size_t)R.buf * words;
        if (p.reach)
            for (int i = threadIdx.x; i < words; i += KN_NT)
                p.reach[(size_t)b * words + i] = (i >= R.wlo && i <= R.whi) ? rb[i] : 0u;
        // tightening
        if (R.wlo <= R.whi) {
            const int i0 = max(R.wlo, lo >> 5), i1 = min(R.whi, hi >> 5);
            int f = 0x7fffffff, l = -1;
            for (int i = i0 + (int)threadIdx.x; i <= i1; i += KN_NT) {
                const uint32_t x = rb[i] & kn_win(i, lo, hi);
                if (x) {
                    f = min(f, i * 32 + __ffs(x) - 1);
                    l = max(l, i * 32 + 31 - __clz(x));
                }
            }
            f = __reduce_min_sync(0xffffffffu, f);
            l = __reduce_max_sync(0xffffffffu, l);
            if ((threadIdx.x & 31) == 0 && l >= 0) { atomicMin(&s_first, f); atomicMax(&s_last, l); }
        }
        __syncthreads();
        const int first = s_first, last = s_last;
        __syncthreads();  // every thread has read s_first / s_last before the next bin resets them
        if (last < 0) {
            if (threadIdx.x == 0) { p.status[b] = 1; p.lo_out[b] = lo; p.hi_out[b] = hi; }
            if (!(p.flags & KN_F_REACH_ONLY))
                for (int64_t t = s + threadIdx.x; t < e; t += KN_NT) p.action[t] = 0;
            continue;
        }
        if (threadIdx.x == 0) { p.status[b] = 0; p.lo_out[b] = first; p.hi_out[b] = last; }
        if (!(p.flags & KN_F_NO_TIGHTEN)) { lo = first; hi = last; }
        const bool skip = (p.flags & KN_F_REACH_ONLY) || (!(p.flags & KN_F_NO_TIGHTEN) && lo <= cl);
        if (skip || m == 0) {
            if (!(p.flags & KN_F_REACH_ONLY))
                for (int64_t t = s + threadIdx.x; t < e; t += KN_NT) p.action[t] = 0;
            continue;
        }
        // divide and conquer; level d lives in buffer lv[d].buf; buffers
        // 0..nbuf-1, level 0 = buffer 0 (base), one spare
        KnLevel lv[KN_MAXD];
        int slo[KN_MAXD], shi[KN_MAXD], st[KN_MAXD];
        lv[0] = L0;
        for (int i = 1; i < KN_MAXD; ++i) lv[i] = KnLevel{i < p.nbuf - 1 ? i : 0, 0, -1};
        spare = p.nbuf - 1;
        int d = 0;
        slo[0] = 0; shi[0] = m; st[0] = 0;
        while (d >= 0) {
            const int a = slo[d], z = shi[d];
            if (z - a == 1) {
                const uint32_t* x = kn_smem + (size_t)lv[d].buf * words;
                const int wt = p.w[s + a];
                const bool use = hi >= wt && kn_cta_any(x, lv[d], max(0, lo - wt), hi - wt);
                const bool avoid = kn_cta_any(x, lv[d], lo, hi);
                if (threadIdx.x == 0) p.action[s + a] = (uint8_t)kn_action(use, avoid);
                --d;
                continue;
            }
            if (st[d] == 2) { --d; continue; }
            const int mid = (a + z) >> 1;
            if (st[d] == 0) {
                kn_cta_add_range(kn_smem, words, lm, lv[d], lv[d + 1], spare, p.w, s + mid, s + z);
                st[d] = 1;
                slo[d + 1] = a; shi[d + 1] = mid;
            } else {
                kn_cta_add_range(kn_smem, words, lm, lv[d], lv[d + 1], spare, p.w, s + a, s + mid);
                st[d] = 2;
                slo[d + 1] = mid; shi[d + 1] = z;
            }
            ++d;
            st[d] = 0;
        }
        __syncthreads();
    }
}

}  // namespace knap
}  // namespace bplb
