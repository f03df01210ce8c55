// bplb_prune.cuh -- bound-pruned lambda sweep: one CTA per reduced instance
// (persistent over a batch of search-node states), for 2 <= c <= PR_MAX_C.
//
// The reference evaluates every grid point (kind, lambda) of the collection
// (bounds.py:463-527).  Most of them cannot matter for the answer, and that
// can be proven per lambda from O(1) node statistics, exactly:
//
//   VB2  (bounds.py:189-197, 410-438): piece(v) = floor((v l - 1)/c) lies in
//        [(v l - c)/c, (v l - 1)/c], so the per-lambda sum S(l) is at most
//        S_hi(l) = 2 floor((l Vs - ns)/c) - 2 max(0, ceil(l Vm/c) - nm)
//                  + (n_eq + 2 n_big)(l - 1)
//        (Vs / Vm: sums of small / mirrored values), and its relaxation
//        without the floors is LINEAR in l.
//   CCM1 (bounds.py:181-186, 390-407): floor(v/l) in [(v-l+1)/l, v/l] gives
//        S_hi(l) = 2 floor(Vs/l) + (n_eq + 2 n_big) q
//                  - 2 max(0, ceil((Vm - n_big (l-1))/l)),  q = floor(c/l).
//   BJ1  (bounds.py:200-206, 441-460): with cm = c mod l, every transformed
//        item obeys f(w) <= w (l - cm)/l, so the bound is at most
//        ceil(W / (c - cm)).
//   (all three checked against the oracle on 1e8 (instance, kind, l) points)
//
// A lambda is skipped when its upper bound cannot beat what the sweep
// already holds:
//   lb mode  (only lb / exceeded requested): UB(l) <= best bound of ANY kind;
//   key mode (per-kind best + lowest arg lambda requested): (UB(l), l) cannot
//            beat the kind's (best, lowest lambda) key -- UB < best, or
//            UB == best at a higher lambda.
// Skipped lambdas provably cannot change the outputs, so lb, exceeded,
// per-kind best and arg lambda are bit-exact with the full sweep.
//
// MT and RAD2 (bounds.py:155-170, 373-387) are piecewise constant in lambda:
// their lookups N(l-1), N(c-l), N(c-2l), N(2l-1), W(.) change only at
// l = w+1, c-w+1, floor((c-w)/2)+1, floor((w+2)/2).  The maximum and its
// lowest lambda are therefore attained at the range start or at one of
// those candidates, which are the only lambdas evaluated when they are
// fewer than the range (the reference's own l2 sweep uses the same fact,
// bounds.py:139-152).
//
// Lookups: a presence bitmask over the values [0, c] with per-word rank
// prefixes (one LDS.64 + POPC) indexes cumulative count / weight tables over
// the distinct values, so N(x) and W(x) cost two shared loads for any x.
#pragma once
#include "bplb_node.cuh"

namespace bplb {

#ifndef PR_PNT
#define PR_PNT 256  // threads per CTA (one node per CTA at a time)
#endif
#ifndef PR_PNT_LB
#define PR_PNT_LB 384  // threads per CTA of the lb-mode full-collection instantiation (FAST = 1)
#endif
constexpr int PNT = PR_PNT;
constexpr int PNT_LB = PR_PNT_LB;
constexpr int PNW = (PNT > PNT_LB ? PNT : PNT_LB) / 32;  // per-warp arrays sized for the larger CTA
__host__ __device__ constexpr int prune_threads(int fast) { return fast == 1 ? PNT_LB : PNT; }
constexpr int64_t PR_MAX_C = 1 << 18;  // presence bitmask: c/32 8-byte words in smem
constexpr int PR_SUPER = 256;          // lambdas per prune unit (8 sub-blocks of 32)
#ifndef PR_QMAX_N
#define PR_QMAX_N 32
#endif
#ifndef PR_QMAX_BJ1_N
#define PR_QMAX_BJ1_N 32
#endif
#ifndef PR_QMAX_CCM1_N
#define PR_QMAX_CCM1_N 96  // cfg5: 96 / 64 / 48 / 32 -> lb 0.606 / 0.607 / 0.605 / 0.616 us/node, key 0.892 /
                           // 0.900 / 0.910 / 0.947 (160: 0.613 / 0.899)
#endif
constexpr int PR_QMAX = PR_QMAX_N;          // block bounds where floor(c / lambda) <= PR_QMAX (grid-wide path)
constexpr int PR_QMAX_CCM1 = PR_QMAX_CCM1_N;  // prune_kernel: CCM1 block units where floor(c / lambda) <= this
                                              // (its block bound costs O(c / lambda) lookups, no q-envelope)
constexpr int PR_QMAX_BJ1 = PR_QMAX_BJ1_N;  // ... and for BJ1 (its block bound costs O(q) lookups per q-piece)
#ifndef PR_QMAX_BJ1_LB_N
#define PR_QMAX_BJ1_LB_N 20  // lb-mode units (cross-kind threshold): cfg5 lb 32 / 24 / 20 / 16 / 12 ->
                             // 0.546 / 0.512 / 0.496 / 0.497 / 0.513 us/node (key mode keeps 32: 0.790 vs 0.803)
#endif
constexpr int PR_QMAX_BJ1_LB = PR_QMAX_BJ1_LB_N;
constexpr int PR_BLK_UNIT = 32 * 256;     // lambdas per block unit: 32 blocks of 256, one per lane (lb mode)
constexpr int PR_BLK_UNIT_KEY = 8 * 256;  // ... key mode: per-kind thresholds prune less, shorter units balance
                                          // better (cfg5 1.22 vs 1.34 us/node; lb mode 0.77 vs 0.86)
#ifndef PR_MINB
#define PR_MINB 2  // resident CTAs per SM the register budget is sized for (2 x 256 threads measured
                   // 0.639 vs 0.724 us/node at 3 x 256 on cfg5 lb mode, key mode 0.948 vs 1.145)
#endif
#ifndef PR_P1_ORDER
#define PR_P1_ORDER 0  // unit order of the pruned remainder (phase 1)
#endif
// Cost model of the exact per-lambda sums in the drain: weight of one
// harmonic lookup term against the per-lambda overhead (24) of the
// warp-split loop and the dense division pass.  26 / 40 (CCM1 / BJ1) until
// session 4; at 2 CTAs/SM lane-per-lambda lookups win almost everywhere:
// cfg5 lb / key 0.605 / 0.893 -> 0.546 / 0.790 us/node with 1 / 1 (0 / 0 picks
// lane lookups even at the smallest lambdas: key mode 2.3 us/node); uniform
// c = 1e5 batches 2.57 -> 2.06 (lb), 6.87 -> 5.96 (key); cfg2-shaped nodes
// unchanged (scripts/prune_shapes.py).
#ifndef PR_T_CCM1
#define PR_T_CCM1 1
#endif
#ifndef PR_T_BJ1
#define PR_T_BJ1 1
#endif
#ifndef PR_T_DENSE
#define PR_T_DENSE 10  // ... per item of a dense division pass
#endif
#ifndef PR_OVH
#define PR_OVH 24  // ... per-lambda overhead of the warp-split loop / dense pass
#endif
#ifndef PR_SEED_DIV
#define PR_SEED_DIV 4  // CCM1 / BJ1 seed window at c / PR_SEED_DIV + 1
#endif
#ifndef PR_QCAP_N
#define PR_QCAP_N 2048
#endif
constexpr int PR_QCAP = PR_QCAP_N;  // CTA queue: CCM1/BJ1 256-lambda blocks and 32-lambda sub-ranges left to evaluate
constexpr unsigned PR_QEMPTY = 0x7FFFFFFFu;  // a reserved queue slot with nothing to do
constexpr int PR_MAX_SEGS = 20;

enum { PU_CAND = 0, PU_LOOK = 1, PU_WALK = 2, PU_PRUNE = 3, PU_BLK = 4 };

struct LkRank {
    const uint2* rk;        // [c/32 + 1]: {presence mask of 32i..32i+31, #distinct values < 32i}
    const int* cn;          // [d + 1]: cn[j] = #{w <= j-th smallest distinct value}, cn[0] = 0
    const long long* cw;    // [d + 1]: the matching weight sums
    int r, d;
    int64_t c;
    __device__ __forceinline__ int rank(int64_t x) const {  // #distinct values <= x, clamped
        // branch-free: no weight is 0, so rank(x <= 0) = 0, and rank(x >= c) = d
        const int xi = (int)(x < 0 ? 0 : (x > c ? c : x));
        const uint2 e = rk[xi >> 5];
        return (int)e.y + __popc(e.x & (0xFFFFFFFFu >> (31 - (xi & 31))));
    }
    __device__ __forceinline__ int64_t n_le(int64_t x) const { return cn[rank(x)]; }
    __device__ __forceinline__ void both(int64_t x, int64_t* n, int64_t* w) const {
        const int j = rank(x);
        *n = cn[j];
        *w = cw[j];
    }
};

struct PSeg {
    int kind, type;
    int64_t lo, hi;   // inclusive lambda range
    int chunk;        // lambdas (or items, PU_CAND) per unit
    int first, count; // unit index range
};

struct PruneCtl {
    NodeStats st;
    int64_t lo[K_COUNT], hi[K_COUNT];
    PSeg segs[PR_MAX_SEGS];
    int nseg, nunits;
    int kseg_first[K_COUNT], kseg_count[K_COUNT];
    u64 key[K_COUNT];
    unsigned long long evals[K_COUNT];
    int evaluated[K_COUNT];
    int lb;
    int unit_next, unit_end;
    int n_vb2, d;
    int n_done, bad, skip;
    int q_n, q_next;           // block queue: entries pushed / taken
    unsigned blkq[PR_QCAP];    // kind << 28 | first lambda of the block
    long long wsum[PNW], wsum2[PNW];
};

struct PruneMem {
    int* sw;          // raw weights [r]
    int* vb2;         // VB2 walk items (2w != c, w < c)
    uint2* rk;        // presence words
    int* cn;          // cumulative counts by distinct rank
    long long* cw;    // cumulative weights by distinct rank
    u64* tot;         // per-warp walk accumulators [PNW][32]
};

#ifdef PRUNE_TRACE
// Per-unit cycle trace of the first CTAs (development builds only:
// scripts/prune_trace.py builds libbplb_trace.so with -DPRUNE_TRACE).
constexpr int PRUNE_TRACE_CTAS = 8;
constexpr int PRUNE_TRACE_CAP = 1 << 16;
__device__ longlong4 g_prune_trace[PRUNE_TRACE_CAP];
__device__ int g_prune_trace_n;
__device__ __forceinline__ void prune_trace_rec(const PruneCtl& ctl, int cta, int u, int si, long long t0) {
    if ((threadIdx.x & 31) || cta >= PRUNE_TRACE_CTAS) return;
    const int i = atomicAdd(&g_prune_trace_n, 1);
    if (i >= PRUNE_TRACE_CAP) return;
    const PSeg& sg = ctl.segs[si];
    g_prune_trace[i] = make_longlong4(((long long)cta << 32) | ((long long)u << 8) | (threadIdx.x >> 5),
                                      ((long long)sg.kind << 8) | sg.type, t0, clock64());
}
#endif

__host__ __device__ inline int prune_rcap(int64_t max_r) { return (int)((max_r + 3) & ~3ll) + 4; }

__host__ __device__ inline size_t prune_smem_bytes(int rcap, int64_t c) {
    size_t s = (size_t)PNW * 32 * 8;            // tot
    s += (size_t)(rcap + 2) * 8;                // cw
    s += (size_t)((c >> 5) + 2) * 8;            // rk
    s += (size_t)(rcap + 2) * 4;                // cn
    s += (size_t)rcap * 4 * 2;                  // sw, vb2
    return s + 64;
}

// ---- block upper bounds (true => bound(l) <= B for EVERY l in [l1, l2]) -------
// The per-lambda relaxations above drop each floor separately; over a block of
// lambdas the exact step functions can be bounded by evaluating them at the
// block ends instead (the same O(1)-lookup sums as the exact sweep), which is
// tight wherever no item crosses a step inside the block.
//
// CCM1 (bounds.py:181-186, 390-407): S(l) = 2 Sm(l) + K floor(c/l) - 2 Bg(l),
// Sm(l) = sum over small w of floor(w/l) and Bg(l) = sum over mirrored
// v = c - w of floor(v/l) are non-increasing in l, F(l) = 2 floor(c/l) > 0, so
// on [l1, l2]:  S(l) <= 2 Sm(l1) + K floor(c/l1) - 2 Bg(l2),  F(l) >= 2 floor(c/l2).
template <class LK>
__device__ __forceinline__ bool ccm1_blk_le(const LK& lk, const NodeStats& st, int64_t c, int64_t l1,
                                            int64_t l2, int64_t B) {
    const int hs = (int)((c - 1) / 2);
    const int L1 = (int)l1, L2 = (int)l2;
    int sm = 0, bg = 0;
    const int nbase = st.r - st.n_big;  // #{w : 2w <= c}
    for (int x = L1; x <= hs; x += L1) sm += st.n_small - (int)lk.n_le(x - 1);
    for (int x = L2; x <= hs; x += L2) bg += (int)lk.n_le(c - x) - nbase;
    const int64_t K = (int64_t)st.n_eq + 2 * (int64_t)st.n_big;
    const int64_t q1 = (int64_t)((uint32_t)c / (uint32_t)L1), q2 = (int64_t)((uint32_t)c / (uint32_t)L2);
    return 2 * (int64_t)sm + K * q1 - 2 * (int64_t)bg <= B * 2 * q2;
}

// sum over items w in [lo, hi] with w > T of (w - T)
template <class LK>
__device__ __forceinline__ int64_t lk_excess(const LK& lk, int64_t lo, int64_t hi, int64_t T) {
    if (lo < T + 1) lo = T + 1;
    if (hi < lo) return 0;
    int64_t n1, w1, n0, w0;
    lk.both(hi, &n1, &w1);
    lk.both(lo - 1, &n0, &w0);
    return (w1 - w0) - T * (n1 - n0);
}

// BJ1 (bounds.py:200-206, 441-460) on [l1, l2] inside one q-interval
// (floor(c/l) = q for every l): with cm = c - q l and P(l) = l - cm =
// (q+1) l - c > 0, f(c) = q P and every item contributes
//   f(w)/f(c) = (a + theta)/q,  a = floor(w/l),
//   theta = max(0, w - a l - cm) / P = max(0, w - c + (q - a) l) / ((q+1) l - c) in [0, 1).
// An item whose a is constant on the block (w in [t l2, (t+1) l1 - 1]) has a
// linear-fractional theta, monotone in l: increasing iff w < c (t+1)/(q+1),
// so its maximum sits at l2 (below the pivot) or l1 (above).  An item that
// crosses a step (w in [t l1, t l2 - 1]) contributes < t + 1.  Summing
// (W / N lookups per bucket):  sum f(w)/f(c) <= (I + X2/P(l2) + X1/P(l1)) / q.
// Integer envelope: c <= 2^20, r <= 2^17, q <= PR_QMAX (the final comparison in 128 bits).
template <class LK, bool WENV>
__device__ __forceinline__ bool bj1_blk_q_le(const LK& lk, const NodeStats& st, int64_t c, int64_t q,
                                             int64_t l1, int64_t l2, int64_t B) {
    const int64_t P1 = (q + 1) * l1 - c, P2 = (q + 1) * l2 - c;
    int64_t I = 0, X1 = 0, X2 = 0;
    const int tmax = (int)((uint32_t)st.maxw / (uint32_t)l1);
    for (int t = 0; t <= tmax; ++t) {
        const int64_t lo = (int64_t)t * l2, hi = (int64_t)(t + 1) * l1 - 1;
        if (hi >= lo) {
            int64_t nh, wh, nl, wl;
            lk.both(hi, &nh, &wh);
            lk.both(lo - 1, &nl, &wl);
            I += (int64_t)t * (nh - nl);
            if (t < q) {
                const int64_t pv = (int64_t)(((uint32_t)c * (uint32_t)(t + 1) + (uint32_t)q) / (uint32_t)(q + 1));
                X2 += lk_excess(lk, lo, min(hi, pv - 1), c - (q - t) * l2);
                X1 += lk_excess(lk, max(lo, pv), hi, c - (q - t) * l1);
            }
        }
        if (t >= 1 && l2 > l1) I += (int64_t)(t + 1) * (lk.n_le((int64_t)t * l2 - 1) - lk.n_le((int64_t)t * l1 - 1));
    }
    // node kernel envelope (c <= 2^18, r <= 2^14): every product < 2^60; the
    // grid-wide path (c <= 2^20, r <= 2^17) compares in 128 bits
    if (!WENV) return I * P1 * P2 + X2 * P1 + X1 * P2 <= B * q * P1 * P2;
    const __int128 P12 = (__int128)P1 * P2;
    return (__int128)I * P12 + (__int128)X2 * P1 + (__int128)X1 * P2 <= (__int128)B * q * P12;
}

// BJ1 on any [l1, l2]: split at the q-interval ends (at most 8 pieces).
template <class LK, bool WENV>
__device__ __forceinline__ bool bj1_blk_le(const LK& lk, const NodeStats& st, int64_t c, int64_t l1,
                                           int64_t l2, int64_t B) {
    int64_t a = l1;
    for (int piece = 0; piece < 8 && a <= l2; ++piece) {
        const int64_t q = (int64_t)((uint32_t)c / (uint32_t)a);
        const int64_t e = min(l2, (int64_t)((uint32_t)c / (uint32_t)q));
        if (!bj1_blk_q_le<LK, WENV>(lk, st, c, q, a, e, B)) return false;
        a = e + 1;
    }
    return a > l2;
}

// Out of line (like the other heavy helpers below): prune_kernel inlined
// everything into ~640 KB of SASS, and instruction-fetch stalls led its
// warp-state samples; one copy of each loop keeps the hot code in cache.
template <class LK, bool WENV>
__device__ __noinline__ bool blk_ub_le(int kind, const LK lk, const NodeStats& st, int64_t c, int64_t l1,
                                       int64_t l2, int64_t B) {
    if (B < 0) return false;
    return kind == K_CCM1 ? ccm1_blk_le(lk, st, c, l1, l2, B) : bj1_blk_le<LK, WENV>(lk, st, c, l1, l2, B);
}

// Exact per-lambda sums through the lookup structure, one out-of-line copy.
__device__ __noinline__ int64_t pr_lookup_sum(int kind, const LkRank lk, const NodeStats& st, int64_t c,
                                              int64_t lam) {
    switch (kind) {
    case K_MT: return bplb_mt_sum(lk, c, st.r, lam);
    case K_RAD2: return bplb_rad2_sum(lk, c, st.r, lam);
    case K_CCM1: return bplb_ccm1_sum(lk, st, c, lam);
    default: return bplb_bj1_sum(lk, st, c, lam);
    }
}

// The modular walk (FS1 / VB2 states over a 32-lambda window), one copy.
__device__ __noinline__ void pr_walk(const int* items, int n, uint32_t c32, u64 cinv, int64_t lam_a, int L,
                                     u64* t, uint32_t one, bool vb2) {
    mod_walk<false, false, 8>(items, 0, n, c32, cinv, lam_a, L, t, one, vb2);
}

// One lambda of CCM1 / BJ1 by the whole warp: a dense pass over the items
// (small lambda) or the harmonic lookups split over the lanes; one copy.
__device__ int64_t ccm1_dense_smem(const int* w, int n, const NodeStats& st, int64_t c, int64_t lam);
__device__ __noinline__ int64_t pr_warp_sum(int kind, bool dense, const LkRank lk, const NodeStats& st,
                                            const int* sw, int64_t c, int64_t lj) {
    const int lane = threadIdx.x & 31;
    if (kind == K_CCM1) {
        if (dense) return ccm1_dense_smem(sw, st.r, st, c, lj);
        int64_t part = bplb_ccm1_part(lk, st, c, lj, 1 + lane, 32);
        part = (int64_t)warp_sum_u64((u64)part);
        return bplb_ccm1_from_part(st, c, lj, part);
    }
    if (dense) return bj1_dense(sw, st.r, c, lj);
    int64_t fl, rem;
    bplb_bj1_part(lk, st, c, lj, lane, 32, &fl, &rem);
    fl = (int64_t)warp_sum_u64((u64)fl);
    rem = (int64_t)warp_sum_u64((u64)rem);
    return bplb_bj1_from_parts(c, lj, fl, rem);
}

__device__ __forceinline__ Thr read_thr(const PruneCtl& ctl, int kind, bool lbmode) {
    Thr t;
    t.lbmode = lbmode;
    if (lbmode) {
        t.B = *(volatile const int*)&ctl.lb;
        t.has = true;
        t.a_rel = 0;
    } else {
        const u64 key = *(volatile const u64*)&ctl.key[kind];
        t.has = key != 0;
        t.B = (int64_t)(key >> 32);
        t.a_rel = (int64_t)(0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFu));
    }
    return t;
}

template <class LK, bool WENV = false>
__device__ __forceinline__ bool blk_skip(const Thr& t, int kind, const LK& lk, const NodeStats& st, int64_t c,
                                         int64_t lo, int64_t l1, int64_t l2) {
    if (!t.has) return false;
    if (t.lbmode) return blk_ub_le<LK, WENV>(kind, lk, st, c, l1, l2, t.B);
    if (l1 - lo > t.a_rel) return blk_ub_le<LK, WENV>(kind, lk, st, c, l1, l2, t.B);
    return t.B >= 1 && blk_ub_le<LK, WENV>(kind, lk, st, c, l1, l2, t.B - 1);
}

// CCM1 dense sum over an unsorted item array in shared memory (the
// global-memory ccm1_dense_raw reads through __ldg).
__device__ int64_t ccm1_dense_smem(const int* w, int n, const NodeStats& st, int64_t c, int64_t lam) {
    const int lane = threadIdx.x & 31;
    const Div31 dv = bplb_div31((uint32_t)lam);
    const uint32_t c32 = (uint32_t)c;
    long long a = 0;
    for (int i = lane; i < n; i += kWarp) {
        const uint32_t x = (uint32_t)w[i];
        if (2ull * x < c32) a += bplb_udiv31(x, dv);
        else if (2ull * x > c32) a -= bplb_udiv31(c32 - x, dv);
    }
    const int64_t A = (int64_t)warp_sum_u64((u64)a);
    const int64_t cq = c / lam;
    return 2 * A + (int64_t)st.n_eq * cq + 2 * (int64_t)st.n_big * cq;
}

// ---- segments ------------------------------------------------------------------
// phase 0: exact seeds (MT / RAD2 candidates, FS1, the first VB2 window, a
// CCM1 / BJ1 window at c/4+1 where their maxima sit on typical nodes);
// phase 1: the pruned remainder of VB2, CCM1, BJ1.
template <int blk_unit>
__device__ void prune_add_kind(PruneCtl& ctl, int kind, int phase, int64_t c, int r) {
    const int64_t lo = ctl.lo[kind], hi = ctl.hi[kind];
    if (hi < lo) return;
    auto push = [&](int type, int64_t a, int64_t b, int chunk, int count) {
        if (b < a || count <= 0) return;
        PSeg& s = ctl.segs[ctl.nseg++];
        s.kind = kind;
        s.type = type;
        s.lo = a;
        s.hi = b;
        s.chunk = chunk;
        s.first = ctl.nunits;
        s.count = count;
        ctl.nunits += count;
        ctl.kseg_count[kind]++;
    };
    auto pushr = [&](int type, int64_t a, int64_t b, int chunk) {
        if (b >= a) push(type, a, b, chunk, (int)((b - a + chunk) / chunk));
    };
    const int64_t n = hi - lo + 1;
    switch (kind) {
    case K_MT: case K_RAD2:
        if (phase == 0) {
            const int64_t ncand = (kind == K_MT ? 2 : 4) * (int64_t)r + 1;
            if (n > ncand) push(PU_CAND, lo, hi, 32, (r + 31) / 32 > 0 ? (r + 31) / 32 : 1);
            else pushr(PU_LOOK, lo, hi, 32);
        }
        break;
    case K_FS1:
        if (phase == 0) pushr(PU_WALK, lo, hi, 32);
        break;
    case K_VB2:
        if (phase == 0) pushr(PU_WALK, lo, min(hi, lo + 31), 32);
        else pushr(PU_PRUNE, lo + 32, hi, blk_unit);
        break;
    default: {  // CCM1, BJ1
        int64_t s0 = c / PR_SEED_DIV + 1;
        s0 = s0 < lo ? lo : (s0 > hi ? hi : s0);
        const int64_t s1 = min(hi, s0 + 31);
        if (phase == 0) pushr(PU_LOOK, s0, s1, 32);
        else {
            // block bounds where floor(c / l) <= PR_QMAX (l >= bl), per-lambda
            // relaxations below (tight there: the dropped floors are small
            // against c / l)
            const int qbj = blk_unit == PR_BLK_UNIT_KEY ? PR_QMAX_BJ1 : PR_QMAX_BJ1_LB;
            const int64_t bl = max(lo, c / ((kind == K_BJ1 ? qbj : PR_QMAX_CCM1) + 1) + 1);
            auto region = [&](int64_t a, int64_t b) {  // [a, b] outside the seed window
                if (b < a) return;
                if (a < bl) pushr(PU_PRUNE, a, min(b, bl - 1), blk_unit);
                if (b >= bl) pushr(PU_BLK, max(a, bl), b, blk_unit);
            };
#if PR_P1_ORDER
            region(lo, s0 - 1);  // the costly block tests near bl first (shorter tail before the drain)
            region(s1 + 1, hi);
#else
            region(s1 + 1, hi);
            region(lo, s0 - 1);
#endif
        }
    }
    }
}

// ---- block unit: CCM1 / BJ1 over up to 32 x 256 lambdas --------------------------
// level 1: lane j bounds the 256-lambda block j; level 2: every surviving
// block is re-bounded as 32 sub-blocks of 8 lambdas (one per lane); level 3:
// the lambdas of surviving sub-blocks (4 sub-blocks per warp pass) get the
// per-lambda relaxation and, if still live, the exact sum (harmonic lookups,
// bounds.py:390-407 / 441-460).  Returns the best bound the warp evaluated.
// Level 2 + 3 of one 256-lambda block [base, top] of CCM1 / BJ1: 32 sub-blocks
// of 8 lambdas (one per lane) re-bounded, then the lambdas of the surviving
// sub-blocks (4 sub-blocks per warp pass) get the per-lambda relaxation and,
// if still live, the exact sum (harmonic lookups, bounds.py:390-407 /
// 441-460).  Returns the best bound the warp evaluated (-1: none).
template <class LK>
__device__ int64_t blk_block(const KParams& p, PruneCtl& ctl, const LK& lk, int kind, int64_t base, int64_t top,
                             bool lbmode) {
    const int lane = threadIdx.x & 31;
    const int64_t c = p.c, lo_k = ctl.lo[kind];
    const NodeStats& st = ctl.st;
    u64* key = &ctl.key[kind];
    int64_t wmax = -1;
    const int64_t s2 = base + 8 * (int64_t)lane;
    bool live2 = s2 <= top;
    if (live2) live2 = !blk_skip(read_thr(ctl, kind, lbmode), kind, lk, st, c, lo_k, s2, min(top, s2 + 7));
    unsigned m2 = __ballot_sync(0xffffffffu, live2);
    while (m2) {
        unsigned mm = m2;
        for (int g = 0; g < (lane >> 3); ++g) mm &= mm - 1;  // this lane's sub-block: the (lane/8)-th set bit
        const bool hb = mm != 0;
        const int64_t lam = hb ? base + 8 * (int64_t)(__ffs(mm) - 1) + (lane & 7) : 0;
        for (int g = 0; g < 4; ++g) m2 &= m2 - 1;
        const bool in = hb && lam <= top;
        const Thr th = read_thr(ctl, kind, lbmode);
        const bool keep = in && !lam_skip(th, kind, st, c, lo_k, lam);
        int64_t b = 0;
        if (keep) {
            const int64_t S = pr_lookup_sum(kind, lk, st, c, lam);
            b = bplb_bound(S, pr_fc(kind, c, lam));
        }
        const int64_t mx = emit_warp(keep, lam, b, lo_k, key, nullptr, 0, 0);
        if (mx > wmax) {
            wmax = mx;
            if (lane == 0) atomicMax(&ctl.lb, (int)mx);  // tighten the threshold now
        }
    }
    return wmax;
}

// Level 1 of a block unit (CCM1 / BJ1, up to 32 x 256 lambdas): lane j bounds
// the 256-lambda block j; the surviving blocks go to the CTA queue, drained by
// every warp after the unit sweep (so one unit's survivors do not serialise on
// one warp); blocks that do not fit in the queue are processed here.
template <class LK>
__device__ int64_t blk_unit(const KParams& p, PruneCtl& ctl, const LK& lk, int kind, int64_t lam_a, int64_t lam_b,
                            bool lbmode) {
    const int lane = threadIdx.x & 31;
    const int64_t c = p.c, lo_k = ctl.lo[kind];
    const NodeStats& st = ctl.st;
    const int64_t s1 = lam_a + 256 * (int64_t)lane;
    bool live = s1 <= lam_b;
    if (live) live = !blk_skip(read_thr(ctl, kind, lbmode), kind, lk, st, c, lo_k, s1, min(lam_b, s1 + 255));
    unsigned m1 = __ballot_sync(0xffffffffu, live);
    if (!m1) return -1;
    int q0 = 0;
    if (lane == 0) q0 = atomicAdd(&ctl.q_n, __popc(m1));
    q0 = __shfl_sync(0xffffffffu, q0, 0);
    const int pos = q0 + __popc(m1 & ((1u << lane) - 1u));
    if (live && pos < PR_QCAP) ctl.blkq[pos] = ((unsigned)kind << 28) | (unsigned)s1;
    int64_t wmax = -1;
    if (q0 + __popc(m1) > PR_QCAP) {  // overflow: the blocks past the queue's end, inline
        unsigned mo = __ballot_sync(0xffffffffu, live && pos >= PR_QCAP);
        while (mo) {
            const int j = __ffs(mo) - 1;
            mo &= mo - 1;
            const int64_t base = lam_a + 256 * (int64_t)j;
            wmax = max(wmax, blk_block(p, ctl, lk, kind, base, min(lam_b, base + 255), lbmode));
        }
    }
    return wmax;
}

// One 32-lambda sub-range [sub, sub_b] of a PU_PRUNE segment (VB2, or CCM1 /
// BJ1 below the block-bound region): the per-lambda relaxation, then the
// exact sums of the lambdas it keeps -- the VB2 walk over the window (or one
// warp pass per lambda when only a few survive), CCM1 / BJ1 by harmonic
// lookups per lane, split over the warp, or a dense pass over the items,
// whichever is cheapest.  Returns the best bound evaluated (-1: none).
template <class LK>
__device__ int64_t prune_sub(const KParams& p, PruneCtl& ctl, const LK& lk, const PruneMem& m, int kind,
                             int64_t sub, int64_t sub_b, bool lbmode) {
    const int lane = threadIdx.x & 31;
    const int64_t c = p.c, lo_k = ctl.lo[kind];
    const NodeStats& st = ctl.st;
    u64* key = &ctl.key[kind];
    const uint32_t c32 = (uint32_t)c;
    const u64 cinv = st.cinv;
                const int64_t lam = sub + lane;
                const bool in = lam <= sub_b;
                const Thr th = read_thr(ctl, kind, lbmode);
                const bool keep = in && !lam_skip(th, kind, st, c, lo_k, lam);
                const unsigned mask = __ballot_sync(0xffffffffu, keep);
                if (!mask) return -1;
                const int n = __popc(mask);
                bool have = false;
                int64_t b = 0;
                if (kind == K_VB2) {
                    if (n >= 6) {  // dense cluster: walk the 32-lambda window
                        u64* tt = m.tot + (threadIdx.x >> 5) * 32;
                        tt[lane] = 0;
                        __syncwarp();
                        pr_walk(m.vb2, ctl.n_vb2, c32, cinv, sub, (int)(sub_b - sub + 1), tt,
                                                  p.one, true);
                        __syncwarp();
                        if (in) {
                            have = true;
                            b = bplb_bound(bplb_vb2_sum(st, c, lam, tt[lane]), 2 * (lam - 1));
                        }
                    } else {  // a few lambdas: one warp pass over the items each
                        unsigned mm = mask;
                        while (mm) {
                            const int j = __ffs(mm) - 1;
                            mm &= mm - 1;
                            const int64_t lj = sub + j;
                            u64 D = 0;
                            for (int i = lane; i < ctl.n_vb2; i += 32) {
                                const uint32_t x = (uint32_t)m.vb2[i];
                                D += bplb_mulmod(x, (uint32_t)lj, 2 * x < c32 ? 1u : 0u, c32, cinv);
                            }
                            D = warp_sum_u64(D);
                            if (lane == j) {
                                have = true;
                                b = bplb_bound(bplb_vb2_sum(st, c, lj, D), 2 * (lj - 1));
                            }
                        }
                    }
                } else {  // CCM1 / BJ1: harmonic lookups or a dense item pass
                    const int64_t span = kind == K_CCM1 ? (c - 1) / 2 : (int64_t)st.maxw;
                    const int64_t tmax = (int64_t)((uint32_t)span / (uint32_t)sub);
                    const int64_t T = kind == K_CCM1 ? PR_T_CCM1 : PR_T_BJ1;
                    const int64_t cost_lane = T * (tmax + 1);
                    const int64_t cost_coop = n * (T * ((tmax + 32) / 32) + PR_OVH);
                    const int64_t cost_dense = n * (PR_T_DENSE * (((int64_t)st.r + 31) / 32) + PR_OVH);
                    if (cost_lane <= cost_coop && cost_lane <= cost_dense) {
                        if (in) {
                            have = true;
                            const int64_t S = pr_lookup_sum(kind, lk, st, c, lam);
                            b = bplb_bound(S, pr_fc(kind, c, lam));
                        }
                    } else {
                        const bool dense = cost_dense < cost_coop;
                        unsigned mm = mask;
                        while (mm) {
                            const int j = __ffs(mm) - 1;
                            mm &= mm - 1;
                            const int64_t lj = sub + j;
                            const int64_t S = pr_warp_sum(kind, dense, lk, st, m.sw, c, lj);
                            if (lane == j) {
                                have = true;
                                b = bplb_bound(S, pr_fc(kind, c, lj));
                            }
                        }
                    }
                }
                return emit_warp(have, lam, b, lo_k, key, nullptr, 0, 0);
}

// One 256-lambda block of a PU_PRUNE segment: its 32-lambda sub-ranges.
template <class LK>
__device__ int64_t prune_block(const KParams& p, PruneCtl& ctl, const LK& lk, const PruneMem& m, int kind,
                               int64_t base, int64_t top, bool lbmode) {
    int64_t wmax = -1;
    for (int64_t sub = base; sub <= top; sub += 32) {
        const int64_t mx = prune_sub(p, ctl, lk, m, kind, sub, min(top, sub + 31), lbmode);
        if (mx > wmax) {
            wmax = mx;
            if ((threadIdx.x & 31) == 0) atomicMax(&ctl.lb, (int)mx);  // tighten the threshold now
        }
    }
    return wmax;
}

// Drain the CTA queue (all warps; after the barrier that ends the unit sweep):
// 256-lambda blocks of CCM1 / BJ1 (levels 2 + 3) and 32-lambda sub-ranges of
// PU_PRUNE segments.
template <class LK>
__device__ void blk_drain(const KParams& p, PruneCtl& ctl, const LK& lk, const PruneMem& m, bool lbmode,
                          bool cancel) {
    const int lane = threadIdx.x & 31;
    const int n = min(*(volatile int*)&ctl.q_n, PR_QCAP);
    for (;;) {
        int i = 0;
        if (lane == 0) i = atomicAdd(&ctl.q_next, 1);
        i = __shfl_sync(0xffffffffu, i, 0);
        if (i >= n) break;
        if (cancel && (int64_t)(*(volatile int*)&ctl.lb) > p.k) continue;  // Alg. 4 guard
        const unsigned e = ctl.blkq[i];
        if (e == PR_QEMPTY) continue;
        const int kind = (int)((e >> 28) & 7u);
        const int64_t base = (int64_t)(e & 0x0FFFFFFFu);
#ifdef PRUNE_TRACE
        const long long t0 = clock64();
#endif
        const int64_t wm = (e & 0x80000000u)
                               ? prune_sub(p, ctl, lk, m, kind, base, min(ctl.hi[kind], base + 31), lbmode)
                               : blk_block(p, ctl, lk, kind, base, min(ctl.hi[kind], base + 255), lbmode);
        if (lane == 0 && wm >= 0) atomicMax(&ctl.lb, (int)wm);
#ifdef PRUNE_TRACE
        if (lane == 0 && blockIdx.x < PRUNE_TRACE_CTAS) {
            const int ti = atomicAdd(&g_prune_trace_n, 1);
            if (ti < PRUNE_TRACE_CAP)
                g_prune_trace[ti] = make_longlong4(((long long)blockIdx.x << 32) | 0xFFFE0000ll | (threadIdx.x >> 5),
                                                   ((long long)kind << 8) | ((e & 0x80000000u) ? 3 : 4) |
                                                       ((long long)base << 16), t0, clock64());
        }
#endif
    }
}

// ---- one unit ----------------------------------------------------------------------
template <class LK>
__device__ void prune_unit(const KParams& p, PruneCtl& ctl, const LK& lk, const PruneMem& m, int u,
                           bool lbmode, int& si) {
    const int lane = threadIdx.x & 31;
    // a warp claims increasing unit ids: its segment index only moves forward
    while (si + 1 < ctl.nseg && ctl.segs[si + 1].first <= u) ++si;
    const PSeg sg = ctl.segs[si];
    const int kind = sg.kind;
    const int64_t c = p.c;
    const int64_t lo_k = ctl.lo[kind];
    const NodeStats& st = ctl.st;
    u64* key = &ctl.key[kind];
    int64_t wmax = -1;
    int64_t nev = 0;
    if (sg.type == PU_CAND) {
        const int i = (u - sg.first) * 32 + lane;
        const bool vi = i < st.r;
        const int64_t w = vi ? m.sw[i] : 0;
        if (u == sg.first) {  // the range start (first segment of the staircase)
            const int64_t lam = sg.lo;
            int64_t b = 0;
            if (lane == 0) {
                const int64_t S = pr_lookup_sum(kind, lk, st, c, lam);
                b = bplb_bound(S, c);
            }
            wmax = max(wmax, emit_warp(lane == 0, lam, b, lo_k, key, nullptr, 0, 0));
            nev = sg.hi - sg.lo + 1;
        }
        const int nc = kind == K_MT ? 2 : 4;
#pragma unroll 1
        for (int j = 0; j < nc; ++j) {
            int64_t lam;
            if (kind == K_MT) lam = j == 0 ? w + 1 : c - w + 1;
            else lam = j == 0 ? w + 1 : (j == 1 ? (c - w) / 2 + 1 : (j == 2 ? (w + 2) / 2 : c - w + 1));
            const bool v = vi && lam >= sg.lo && lam <= sg.hi;
            int64_t b = 0;
            if (v) {
                const int64_t S = pr_lookup_sum(kind, lk, st, c, lam);
                b = bplb_bound(S, c);
            }
            wmax = max(wmax, emit_warp(v, lam, b, lo_k, key, nullptr, 0, 0));
        }
    } else if (sg.type == PU_LOOK) {
        const int64_t lam_a = sg.lo + (int64_t)(u - sg.first) * sg.chunk;
        const int64_t lam_b = min(sg.hi, lam_a + sg.chunk - 1);
        const int64_t lam = lam_a + lane;
        const bool valid = lam <= lam_b;
        int64_t S = 0;
        if (valid) {
            S = pr_lookup_sum(kind, lk, st, c, lam);
        }
        const int64_t b = valid ? bplb_bound(S, pr_fc(kind, c, lam)) : 0;
        wmax = emit_warp(valid, lam, b, lo_k, key, nullptr, 0, 0);
        nev = lam_b - lam_a + 1;
    } else if (sg.type == PU_WALK) {
        const int64_t lam_a = sg.lo + (int64_t)(u - sg.first) * sg.chunk;
        const int64_t lam_b = min(sg.hi, lam_a + sg.chunk - 1);
        const int L = (int)(lam_b - lam_a + 1);
        u64* t = m.tot + (threadIdx.x >> 5) * 32;
        t[lane] = 0;
        __syncwarp();
        const uint32_t c32 = (uint32_t)c;
        const u64 cinv = bplb_cinv(c32);
        if (kind == K_VB2) pr_walk(m.vb2, ctl.n_vb2, c32, cinv, lam_a, L, t, p.one, true);
        else pr_walk(m.sw, st.r, c32, cinv, lam_a, L, t, p.one, false);
        __syncwarp();
        const int64_t lam = lam_a + lane;
        const bool valid = lane < L;
        int64_t S = 0;
        if (valid)
            S = kind == K_VB2 ? bplb_vb2_sum(st, c, lam, t[lane])
                              : bplb_fs1_sum(st, lam, t[lane], (uint64_t)bplb_fs1_zero(lk, c, st.maxw, lam));
        const int64_t b = valid ? bplb_bound(S, pr_fc(kind, c, lam)) : 0;
        wmax = emit_warp(valid, lam, b, lo_k, key, nullptr, 0, 0);
        nev = L;
    } else if (sg.type == PU_BLK) {
        const int64_t lam_a = sg.lo + (int64_t)(u - sg.first) * sg.chunk;
        const int64_t lam_b = min(sg.hi, lam_a + sg.chunk - 1);
        nev = lam_b - lam_a + 1;
        wmax = blk_unit(p, ctl, lk, kind, lam_a, lam_b, lbmode);
    } else {  // PU_PRUNE: up to 32 x 256 lambdas; the surviving 32-lambda sub-ranges go to the CTA queue
        const int64_t lam_a = sg.lo + (int64_t)(u - sg.first) * sg.chunk;
        const int64_t lam_b = min(sg.hi, lam_a + sg.chunk - 1);
        nev = lam_b - lam_a + 1;
        // level 1: lane j tests the 256-lambda block j with the range relaxation
        const int64_t s1 = lam_a + 256 * (int64_t)lane;
        const bool l1 = s1 <= lam_b &&
                        !range_skip(read_thr(ctl, kind, lbmode), kind, st, c, lo_k, s1, min(lam_b, s1 + 255));
        unsigned m1 = __ballot_sync(0xffffffffu, l1);
        if (lbmode) {
            // lb mode: every sub-range of a surviving block goes to the CTA queue; its
            // per-lambda tests run in the drain, balanced over the warps and against
            // the threshold the seeds and the units have raised by then
            if (m1) {
                int q0 = 0;
                if (lane == 0) q0 = atomicAdd(&ctl.q_n, 8 * __popc(m1));
                q0 = __shfl_sync(0xffffffffu, q0, 0);
                const int pos = q0 + 8 * __popc(m1 & ((1u << lane) - 1u));
                if (l1 && pos < PR_QCAP)  // a block straddling the end: its slots become empty entries
                    for (int j = 0; j < 8 && pos + j < PR_QCAP; ++j)
                        ctl.blkq[pos + j] = pos + 8 <= PR_QCAP
                                                ? 0x80000000u | ((unsigned)kind << 28) | (unsigned)(s1 + 32 * j)
                                                : PR_QEMPTY;
                unsigned mo = __ballot_sync(0xffffffffu, l1 && pos + 8 > PR_QCAP);
                while (mo) {  // queue overflow: inline
                    const int j = __ffs(mo) - 1;
                    mo &= mo - 1;
                    const int64_t base = lam_a + 256 * (int64_t)j;
                    wmax = max(wmax, prune_block(p, ctl, lk, m, kind, base, min(lam_b, base + 255), lbmode));
                }
            }
            m1 = 0;
        }
        while (m1) {  // surviving 256-lambda blocks: per-lambda tests here (cheap), the
                      // 32-lambda sub-ranges that keep a lambda go to the CTA queue
            const int j1 = __ffs(m1) - 1;
            m1 &= m1 - 1;
            const int64_t base = lam_a + 256 * (int64_t)j1, top = min(lam_b, base + 255);
            const Thr t0 = read_thr(ctl, kind, lbmode);
            unsigned live = 0;  // bit j: sub-range j keeps a lambda
            for (int64_t sub = base, j = 0; sub <= top; sub += 32, ++j) {
                const int64_t lam = sub + lane;
                const bool keep = lam <= top && !lam_skip(t0, kind, st, c, lo_k, lam);
                if (__ballot_sync(0xffffffffu, keep)) live |= 1u << j;
            }
            const bool mine = lane < 8 && (live >> lane & 1u);
            const unsigned mm = __ballot_sync(0xffffffffu, mine);
            if (!mm) continue;
            int q0 = 0;
            if (lane == 0) q0 = atomicAdd(&ctl.q_n, __popc(mm));
            q0 = __shfl_sync(0xffffffffu, q0, 0);
            const int pos = q0 + __popc(mm & ((1u << lane) - 1u));
            if (mine && pos < PR_QCAP)
                ctl.blkq[pos] = 0x80000000u | ((unsigned)kind << 28) | (unsigned)(base + 32 * lane);
            unsigned mo = __ballot_sync(0xffffffffu, mine && pos >= PR_QCAP);
            while (mo) {  // queue overflow: inline
                const int j = __ffs(mo) - 1;
                mo &= mo - 1;
                const int64_t sub = base + 32 * (int64_t)j;
                wmax = max(wmax, prune_sub(p, ctl, lk, m, kind, sub, min(top, sub + 31), lbmode));
            }
        }
    }
    if (lane == 0) {
        if (nev) atomicAdd(&ctl.evals[kind], (unsigned long long)nev);
        ctl.evaluated[kind] = 1;
        if (wmax >= 0) atomicMax(&ctl.lb, (int)wmax);
    }
}


template <class LK>
__device__ void prune_run(const KParams& p, PruneCtl& ctl, const LK& lk, const PruneMem& m, bool lbmode,
                          bool cancel) {
    const int lane = threadIdx.x & 31;
    int si = 0;
    for (;;) {
        int u = 0;
        if (lane == 0) u = atomicAdd(&ctl.unit_next, 1);
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= ctl.unit_end) break;
        if (cancel && (int64_t)(*(volatile int*)&ctl.lb) > p.k) continue;  // Alg. 4 guard
#ifdef PRUNE_TRACE
        const long long t0 = clock64();
#endif
        prune_unit(p, ctl, lk, m, u, lbmode, si);
#ifdef PRUNE_TRACE
        prune_trace_rec(ctl, blockIdx.x, u, si, t0);
#endif
    }
    __syncthreads();  // every unit done: the block queue is complete
#ifdef PRUNE_TRACE
    const long long td = clock64();
#endif
    blk_drain(p, ctl, lk, m, lbmode, cancel);
#ifdef PRUNE_TRACE
    if ((threadIdx.x & 31) == 0 && blockIdx.x < PRUNE_TRACE_CTAS) {
        const int i = atomicAdd(&g_prune_trace_n, 1);
        if (i < PRUNE_TRACE_CAP) {
            g_prune_trace[i] = make_longlong4(((long long)blockIdx.x << 32) | 0xFFFF0000ll | (threadIdx.x >> 5),
                                              ctl.q_n, td, clock64());
        }
    }
#endif
}

// lbmode: only lb / exceeded are produced (cross-kind pruning).
// FAST = 1: lb mode with neither PHASED nor CANCEL (the full-collection batch,
// the bench); FAST = 2: key mode, neither PHASED nor CANCEL; every mode test a
// compile-time constant there -- half the code for a kernel whose warps stall
// on instruction fetch (lb mode 0.751 -> 0.712 us/node); FAST = 0: any mode.
template <int FAST>
__global__ void __launch_bounds__(prune_threads(FAST), PR_MINB) prune_kernel(KParams p, int rcap, int lbmode) {
    constexpr int KNT = prune_threads(FAST);
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ PruneCtl ctl;
    const int64_t c = p.c;
    const int nwords = (int)(c >> 5) + 1;
    PruneMem m;
    {
        unsigned char* q = smem;
        m.tot = (u64*)q; q += PNW * 32 * 8;
        m.cw = (long long*)q; q += (size_t)(rcap + 2) * 8;
        m.rk = (uint2*)q; q += (size_t)(nwords + 1) * 8;
        m.cn = (int*)q; q += (size_t)(rcap + 2) * 4;
        m.sw = (int*)q; q += (size_t)rcap * 4;
        m.vb2 = (int*)q;
    }
    const bool phased = FAST ? false : (p.flags & BPLB_F_PHASED) != 0;
    const bool cancel = FAST ? false : (p.flags & BPLB_F_CANCEL) && !phased;
    const bool lbm = FAST == 1 ? true : (FAST == 2 ? false : lbmode && !phased);
    for (int64_t node = p.node0 + blockIdx.x; node < p.node0 + p.n_nodes; node += gridDim.x) {
        const int64_t base = p.off[node];
        const int r = (int)(p.off[node + 1] - base);
        if (threadIdx.x == 0) {
            NodeStats& st = ctl.st;
            st.r = r; st.maxw = 0; st.n_small = st.n_eq = st.n_big = st.n_full = 0;
            st.W = st.Vs = st.Vm = 0;
            for (int i = 0; i < K_COUNT; ++i) {
                ctl.key[i] = 0; ctl.evals[i] = 0; ctl.evaluated[i] = 0;
                ctl.kseg_count[i] = 0; ctl.kseg_first[i] = 0;
            }
            ctl.lb = 0; ctl.n_vb2 = 0; ctl.nseg = 0; ctl.nunits = 0; ctl.n_done = 0; ctl.bad = 0;
        }
        for (int i = threadIdx.x; i <= nwords; i += KNT) m.rk[i] = make_uint2(0u, 0u);
        for (int i = threadIdx.x; i < r + 2; i += KNT) { m.cn[i] = 0; m.cw[i] = 0; }
        for (int i = threadIdx.x; i < r; i += KNT) m.sw[i] = load_w(p, base + i);
        __syncthreads();
        // ---- statistics, presence bits, VB2 item list --------------------------
        {
            int l_max = 0, l_bad = 0, l_s = 0, l_e = 0, l_b = 0, l_f = 0;
            long long l_W = 0, l_Vs = 0, l_Vm = 0;
            for (int i = threadIdx.x; i < r; i += KNT) {
                const int x = m.sw[i];
                if (x < 1 || (int64_t)x > c) { l_bad = 1; continue; }
                l_max = max(l_max, x);
                l_W += x;
                if (2 * (int64_t)x < c) { l_s++; l_Vs += x; }
                else if (2 * (int64_t)x == c) l_e++;
                else { l_b++; l_Vm += c - x; if (x == c) l_f++; }
                atomicOr(&m.rk[x >> 5].x, 1u << (x & 31));
                if (2 * (int64_t)x != c && (int64_t)x < c) m.vb2[atomicAdd(&ctl.n_vb2, 1)] = x;
            }
            l_max = __reduce_max_sync(0xffffffffu, (unsigned)l_max);
            l_bad = (int)__reduce_or_sync(0xffffffffu, (unsigned)l_bad);
            l_s = __reduce_add_sync(0xffffffffu, l_s);
            l_e = __reduce_add_sync(0xffffffffu, l_e);
            l_b = __reduce_add_sync(0xffffffffu, l_b);
            l_f = __reduce_add_sync(0xffffffffu, l_f);
            l_W = (long long)warp_sum_u64((u64)l_W);
            l_Vs = (long long)warp_sum_u64((u64)l_Vs);
            l_Vm = (long long)warp_sum_u64((u64)l_Vm);
            if ((threadIdx.x & 31) == 0) {
                atomicMax(&ctl.st.maxw, l_max);
                if (l_bad) ctl.bad = 1;
                atomicAdd(&ctl.st.n_small, l_s);
                atomicAdd(&ctl.st.n_eq, l_e);
                atomicAdd(&ctl.st.n_big, l_b);
                atomicAdd(&ctl.st.n_full, l_f);
                atomicAdd((unsigned long long*)&ctl.st.W, (unsigned long long)l_W);
                atomicAdd((unsigned long long*)&ctl.st.Vs, (unsigned long long)l_Vs);
                atomicAdd((unsigned long long*)&ctl.st.Vm, (unsigned long long)l_Vm);
            }
        }
        __syncthreads();
        const bool bad = ctl.bad;
        if (!bad) {
            // rank prefixes over the presence words (contiguous range per thread)
            const int per = (nwords + KNT - 1) / KNT;
            const int b0 = threadIdx.x * per, b1 = min(nwords, b0 + per);
            long long s = 0;
            for (int i = b0; i < b1; ++i) s += __popc(m.rk[i].x);
            long long run = block_excl_scan<KNT / 32>(s, ctl.wsum);
            for (int i = b0; i < b1; ++i) {
                m.rk[i].y = (unsigned)run;
                run += __popc(m.rk[i].x);
            }
            if (threadIdx.x == KNT - 1) ctl.d = (int)run;
            __syncthreads();
            // counts / weights per distinct value (index = its 1-based rank)
            for (int i = threadIdx.x; i < r; i += KNT) {
                const int x = m.sw[i];
                const uint2 e = m.rk[x >> 5];
                const int j = (int)e.y + __popc(e.x & (0xFFFFFFFFu >> (31 - (x & 31))));
                atomicAdd(&m.cn[j], 1);
                atomicAdd((unsigned long long*)&m.cw[j], (unsigned long long)x);
            }
            __syncthreads();
            // inclusive scan of cn / cw over [0, d]
            const int nd = ctl.d + 1;
            const int pe = (nd + KNT - 1) / KNT;
            const int e0 = threadIdx.x * pe, e1 = min(nd, e0 + pe);
            long long sc = 0, sw = 0;
            for (int i = e0; i < e1; ++i) { sc += m.cn[i]; sw += m.cw[i]; }
            long long rc = block_excl_scan<KNT / 32>(sc, ctl.wsum);
            long long rw = block_excl_scan<KNT / 32>(sw, ctl.wsum2);
            for (int i = e0; i < e1; ++i) {
                rc += m.cn[i];
                rw += m.cw[i];
                m.cn[i] = (int)rc;
                m.cw[i] = rw;
            }
        }
        if (threadIdx.x == 0) {
            bplb_stats_finish(&ctl.st, c);
            for (int kd = 0; kd < K_COUNT; ++kd) {
                int64_t lo, hi;
                bplb_domain(kd, c, &lo, &hi);
                if (kd == K_VB2) hi = bplb_vb2_hi(c, r, ctl.st.maxw);
                if (!kind_in(p, kd)) hi = lo - 1;
                ctl.lo[kd] = lo; ctl.hi[kd] = hi;
            }
            if (!bad) {
                if (phased) {
                    for (int i = 0; i < p.nk; ++i) {
                        const int kd = p.kinds[i];
                        ctl.kseg_first[kd] = ctl.nunits;
                        prune_add_kind<PR_BLK_UNIT>(ctl, kd, 0, c, r);
                        prune_add_kind<PR_BLK_UNIT>(ctl, kd, 1, c, r);
                        ctl.kseg_count[kd] = ctl.nunits - ctl.kseg_first[kd];  // units of the kind
                    }
                } else {
                    for (int ph = 0; ph < 2; ++ph)
                        for (int ii = 0; ii < p.nk; ++ii) {
#if PR_P1_ORDER
                            const int i = ph ? p.nk - 1 - ii : ii;  // phase 1: BJ1 / VB2 / CCM1 units first
#else
                            const int i = ii;
#endif
                            // (compile-time unit sizes: a runtime one cost lb mode 1.3 %)
                            if (lbm) prune_add_kind<PR_BLK_UNIT>(ctl, p.kinds[i], ph, c, r);
                            else prune_add_kind<PR_BLK_UNIT_KEY>(ctl, p.kinds[i], ph, c, r);
                        }
                }
            }
        }
        __syncthreads();
        // ---- sweep ---------------------------------------------------------------------
        LkRank lk{m.rk, m.cn, m.cw, r, ctl.d, c};
        if (!bad) {
            if (phased) {
                for (int i = 0; i < p.nk; ++i) {
                    const int kd = p.kinds[i];
                    if (threadIdx.x == 0) {
                        ctl.unit_next = ctl.kseg_first[kd];
                        ctl.q_n = 0;
                        ctl.q_next = 0;
                        ctl.unit_end = ctl.kseg_first[kd] + ctl.kseg_count[kd];
                        ctl.n_done = i + 1;
                    }
                    __syncthreads();
                    prune_run(p, ctl, lk, m, false, false);
                    __syncthreads();
                    if ((int64_t)ctl.lb > p.k) break;
                }
            } else {
                if (threadIdx.x == 0) {
                    ctl.unit_next = 0; ctl.unit_end = ctl.nunits; ctl.n_done = p.nk;
                    ctl.q_n = 0; ctl.q_next = 0;
                }
                __syncthreads();
                prune_run(p, ctl, lk, m, lbm, cancel);
            }
        }
        __syncthreads();
        // ---- outputs (as node_kernel) ----------------------------------------------
        if (threadIdx.x == 0) {
            if (bad && p.err_out) atomicExch(p.err_out, 1);
            int64_t lb = lbm ? (int64_t)ctl.lb : 0;
            bplb_result res;
            for (int kd = 0; kd < K_COUNT; ++kd) {
                const u64 key = ctl.key[kd];
                const bool ev = ctl.evaluated[kd] && kind_in(p, kd);
                res.best[kd] = ev ? (int64_t)(key >> 32) : 0;
                res.arg_lambda[kd] = ev && key ? ctl.lo[kd] + (int64_t)(0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFu))
                                               : ctl.lo[kd];
                res.n_lambda[kd] = ctl.hi[kd] >= ctl.lo[kd] ? ctl.hi[kd] - ctl.lo[kd] + 1 : 0;
                res.evals[kd] = (int64_t)ctl.evals[kd];
                res.evaluated[kd] = ev;
                if (!lbm && ev && res.best[kd] > lb) lb = res.best[kd];
            }
            res.lb = lb;
            res.exceeded = lb > p.k;
            res.n_done = ctl.n_done;
            int64_t et = 0;
            for (int kd = 0; kd < K_COUNT; ++kd) et += res.evals[kd];
            res.evals_total = et;
            if (p.res_out) p.res_out[node] = res;
            if (p.lb_out) p.lb_out[node] = lb;
            if (p.ex_out) p.ex_out[node] = (uint8_t)(lb > p.k);
            if (p.best_out)
                for (int kd = 0; kd < K_COUNT; ++kd) p.best_out[node * K_COUNT + kd] = res.best[kd];
            if (p.arg_out)
                for (int kd = 0; kd < K_COUNT; ++kd) p.arg_out[node * K_COUNT + kd] = res.arg_lambda[kd];
        }
        __syncthreads();
    }
}

}  // namespace bplb
