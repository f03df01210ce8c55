// bplb_node.cuh -- node-resident kernel: one CTA evaluates the full LB
// collection of one reduced instance at a time (persistent over a batch of
// search nodes).  The instance lives in shared memory for the whole sweep,
// as in the paper's calcDffLowerBound, but one launch covers
// all six families, every lambda and every node of the batch.
//
// Two shared-memory layouts, chosen per batch by capacity:
//   TABLE (c <= TABLE_MAX_C): cumulative count / weight tables over the
//     values [-1, c] (O(1) lookups) and the multiset compressed to distinct
//     (value, count) pairs for the VB2/FS1 modular walks.
//   SORT  (larger c): sorted weights + prefix sums + a coarse value->index
//     bucket table (lookups = one bucket read + a ~1-item scan).
//
// Work inside a CTA is cut into "units" pulled from a shared counter:
//   T_LOOKUP  32 lambdas, one per lane, analytic sweep (MT, RAD2, CCM1/BJ1)
//   T_WLOOK   one lambda per warp, harmonic loop split across lanes
//   T_MOD     up to LMOD lambdas x all VB2 (or FS1) items, modular walk
//   T_DIV     LDIV lambdas, warp-cooperative item pass (CCM1/BJ1 small lambda)
#pragma once
#include <climits>
#include "bplb_device.cuh"
#include "bplb_ubound.cuh"
#include "../../include/bplb.h"

namespace bplb {

constexpr int NT = 256;
constexpr int NW = NT / 32;
constexpr int TABLE_MAX_C = 2046;   // node kernel uses cumulative tables when c <= this
constexpr int NBMAX = 4096;         // SORT-mode bucket table entries
constexpr int MAX_SEGS = 3 * K_COUNT;

enum { T_WLOOK = 3 };

struct Seg {
    int kind, type;
    int64_t lo, hi;   // inclusive lambda range of the segment
    int chunk;        // lambdas per unit
    int first, count; // unit index range
};

// Cross-CTA state of the multi-CTA mode (one node, many CTAs): zeroed by the
// host before the launch.
struct MultiState {
    u64 key[K_COUNT];
    int kmax[K_COUNT];     // per-kind running max (PHASED guard at kind boundaries)
    unsigned long long evals[K_COUNT];
    int evaluated[K_COUNT];
    int lb;
    int ctas_done;
    // the per-unit counters on their own L2 lines
    alignas(256) int unit_next;
    alignas(256) int units_done;
    alignas(256) u64 live[K_COUNT];  // VB2 pruning: the best key any CTA has published
};

struct KParams {
    MultiState* ms;        // non-null: every CTA works on node node0 (single check)
    const int* w;          // CSR weights (int32; reinterpreted per wbytes)
    int wbytes;            // 4 (int32), 2 (uint16) or 1 (uint8) bytes per weight
    const int64_t* off;    // CSR offsets (global node index)
    int64_t node0;         // first node of this launch
    int64_t n_nodes;       // nodes [node0, node0 + n_nodes)
    int64_t c;
    int64_t k;
    int kinds[K_COUNT];
    int nk;
    int flags;
    uint32_t one;          // == 1 (kept opaque to ptxas so adds land on the IMAD pipe)
    int64_t* lb_out;       // [n] or null
    uint8_t* ex_out;       // [n] or null
    int64_t* best_out;     // [n*6] or null
    int64_t* arg_out;      // [n*6] or null
    bplb_result* res_out;  // [n] or null
    int* err_out;          // set to 1 if a weight is outside [1, c]
    // single-node per-lambda output (dff_bound_batch): kinds = {kind}
    int64_t* lam_out;
    int64_t out_lo, out_hi;
    int use_range;
    int64_t rng_lo[K_COUNT], rng_hi[K_COUNT];
};

struct NodeCtl {
    NodeStats st;
    int64_t lo[K_COUNT], hi[K_COUNT];
    Seg segs[MAX_SEGS];
    int nseg, nunits;
    int kind_seg_first[K_COUNT], kind_seg_count[K_COUNT];
    u64 key[K_COUNT];
    unsigned long long evals[K_COUNT];
    int evaluated[K_COUNT];
    int unit_next;
    int unit_end;
    int lb;
    int n_vb2;     // SORT: VB2 item count; TABLE: distinct VB2 values
    int n_dist;    // TABLE: distinct values
    int n_done;
    int bad;
    int skip;
    int vprune_seg;  // multi-CTA full check: the VB2 rest segment, pruned against ms->live (-1: none)
    u64 pub[K_COUNT];  // ... the keys this CTA has published to ms->live
    long long wsum[NW];
    long long wsum2[NW];
};

struct NodeMem {  // shared-memory views of one node
    int* sw;          // SORT: sorted weights (padded); TABLE: raw weights
    long long* pre;   // SORT: prefix [r+1];  TABLE: W<=(x) table [c+2]
    int* cnt;         // TABLE: N<=(x) table [c+2]
    int* bidx;        // SORT: bucket index [NBMAX+1]
    int* vb2;         // SORT: VB2 items; TABLE: distinct VB2 values
    int* vb2c;        // TABLE: their counts
    int* dval;        // TABLE: distinct values
    int* dcnt;        // TABLE: their counts
    u64* tot;
    int bk;           // SORT: bucket shift
};

// Weight i of the CSR batch in its storage dtype (uniform branch).
__device__ __forceinline__ int load_w(const KParams& p, int64_t i) {
    if (p.wbytes == 2) return (int)__ldg((const unsigned short*)p.w + i);
    if (p.wbytes == 1) return (int)__ldg((const unsigned char*)p.w + i);
    return __ldg(p.w + i);
}

__device__ __forceinline__ bool kind_in(const KParams& p, int kind) {
    for (int i = 0; i < p.nk; ++i)
        if (p.kinds[i] == kind) return true;
    return false;
}

// Threshold below which CCM1/BJ1 lambdas are summed densely (SORT mode) --
// harmonic lookups cost ~2 * 8 instructions per term, a dense pass ~3 (CCM1)
// or ~5 (BJ1) per item.
#ifndef NODE_DS_CCM1
#define NODE_DS_CCM1 16
#endif
#ifndef NODE_DS_BJ1
#define NODE_DS_BJ1 4
#endif
__device__ __forceinline__ int64_t div_split(int kind, const NodeStats& st, int64_t c) {
    const int64_t n = st.r > 0 ? st.r : 1;
    if (kind == K_CCM1) {
        const int64_t hs = (c - 1) / 2;
        return (NODE_DS_CCM1 * hs) / (3 * n + 30) + 1;
    }
    return (NODE_DS_BJ1 * (int64_t)st.maxw) / n + 1;
}

#ifdef NODE_TRACE
// phase stamps of every CTA (development builds: scripts/node_trace.py)
__device__ unsigned long long g_node_trace[1024][8];
#define NODE_STAMP(i)                                                               \
    do {                                                                            \
        if (threadIdx.x == 0 && blockIdx.x < 1024) {                                \
            unsigned long long t_;                                                  \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                  \
            g_node_trace[blockIdx.x][i] = t_;                                       \
        }                                                                           \
    } while (0)
#else
#define NODE_STAMP(i) do {} while (0)
#endif

// Build the unit segments of one kind (thread 0).
__device__ void add_kind_segs(NodeCtl& ctl, int kind, bool table, int64_t c, int ldiv = LDIV) {
    const int64_t lo = ctl.lo[kind], hi = ctl.hi[kind];
    ctl.kind_seg_first[kind] = ctl.nseg;
    ctl.kind_seg_count[kind] = 0;
    if (hi < lo) return;
    auto push = [&](int type, int64_t a, int64_t b, int chunk) {
        if (b < a) return;
        Seg& s = ctl.segs[ctl.nseg++];
        s.kind = kind;
        s.type = type;
        s.lo = a;
        s.hi = b;
        s.chunk = chunk;
        s.first = ctl.nunits;
        s.count = (int)((uint32_t)(b - a + chunk) / (uint32_t)chunk);  // (32-bit: c <= 2^30; thread 0 plans
        ctl.nunits += s.count;                                           // while the CTA waits)
        ctl.kind_seg_count[kind]++;
    };
    switch (kind) {
    case K_MT: case K_RAD2: push(T_LOOKUP, lo, hi, LLOOK); break;
    case K_FS1: case K_VB2: {
        // enough units to keep all warps busy on small nodes
        int64_t ch = (hi - lo + 1 + 2 * NW - 1) / (2 * NW);
        ch = (ch + 7) & ~7ll;
        ch = ch < 32 ? 32 : (ch > LMOD ? LMOD : ch);
        push(T_MOD, lo, hi, (int)ch);
        break;
    }
    default: {  // CCM1, BJ1
        const int64_t span = kind == K_CCM1 ? (c - 1) / 2 : (int64_t)ctl.st.maxw;
        int64_t sp = lo;
        if (!table) {
            sp = div_split(kind, ctl.st, c);
            if (sp < lo) sp = lo;
            if (sp > hi + 1) sp = hi + 1;
            push(T_DIV, lo, sp - 1, ldiv);
        }
        int64_t sw = span / 64 + 1;  // one warp per lambda while the loop is long
        if (sw < sp) sw = sp;
        if (sw > hi + 1) sw = hi + 1;
        push(T_WLOOK, sp, sw - 1, 1);
        push(T_LOOKUP, sw, hi, LLOOK);
    }
    }
}

template <bool TABLE, bool WIDE, class LK>
__device__ void run_unit(const KParams& p, NodeCtl& ctl, const LK& lk, const NodeMem& m, int u,
                         bool single) {
    const int lane = threadIdx.x & 31;
    int si = 0;
    while (si + 1 < ctl.nseg && ctl.segs[si + 1].first <= u) ++si;
    const Seg sg = ctl.segs[si];
    const int kind = sg.kind;
    const int64_t c = p.c;
    const int64_t lam_a = sg.lo + (int64_t)(u - sg.first) * sg.chunk;
    const int64_t lam_b = min(sg.hi, lam_a + sg.chunk - 1);
    int64_t* lam_out = single ? p.lam_out : nullptr;
    const NodeStats& st = ctl.st;
    int64_t wmax;
    if (sg.type == T_LOOKUP) {
        const int64_t lam = lam_a + lane;
        const bool valid = lam <= lam_b;
        int64_t S = 0;
        if (valid) {
            switch (kind) {
            case K_MT: S = bplb_mt_sum(lk, c, st.r, lam); break;
            case K_RAD2: S = bplb_rad2_sum(lk, c, st.r, lam); break;
            case K_CCM1: S = bplb_ccm1_sum(lk, st, c, lam); break;
            default: S = bplb_bj1_sum(lk, st, c, lam); break;
            }
        }
        int64_t b = valid ? bplb_bound(S, bplb_fc(kind, c, lam)) : 0;
        wmax = emit_warp(valid, lam, b, ctl.lo[kind], &ctl.key[kind], lam_out, p.out_lo, p.out_hi);
    } else if (sg.type == T_WLOOK) {
        const int64_t lam = lam_a;
        int64_t S;
        if (kind == K_CCM1) {
            int64_t part = bplb_ccm1_part(lk, st, c, lam, 1 + lane, 32);
            part = (int64_t)warp_sum_u64((u64)part);
            S = bplb_ccm1_from_part(st, c, lam, part);
        } else {
            int64_t fl, rem;
            bplb_bj1_part(lk, st, c, lam, lane, 32, &fl, &rem);
            fl = (int64_t)warp_sum_u64((u64)fl);
            rem = (int64_t)warp_sum_u64((u64)rem);
            S = bplb_bj1_from_parts(c, lam, fl, rem);
        }
        int64_t b = bplb_bound(S, bplb_fc(kind, c, lam));
        wmax = emit_warp(lane == 0, lam, b, ctl.lo[kind], &ctl.key[kind], lam_out, p.out_lo, p.out_hi);
    } else if (sg.type == T_DIV) {
        int64_t mine = 0;
        for (int64_t lam = lam_a; lam <= lam_b; ++lam) {
            int64_t S = (kind == K_CCM1) ? ccm1_dense(m.sw, st, c, lam) : bj1_dense(m.sw, st.r, c, lam);
            if (lam - lam_a == lane) mine = S;
        }
        const int64_t lam = lam_a + lane;
        const bool valid = lam <= lam_b;
        int64_t b = valid ? bplb_bound(mine, bplb_fc(kind, c, lam)) : 0;
        wmax = emit_warp(valid, lam, b, ctl.lo[kind], &ctl.key[kind], lam_out, p.out_lo, p.out_hi);
    } else if (si == ctl.vprune_seg &&
               range_skip(thr_from_key(*(volatile u64*)&p.ms->live[K_VB2]), K_VB2, st, c, ctl.lo[K_VB2], lam_a,
                          lam_b)) {
        // the whole chunk provably cannot beat the best VB2 key published so
        // far (bplb_prune.cuh relaxation; skipped lambdas count as evaluated)
        wmax = -1;
    } else {
        const int warp = threadIdx.x >> 5;
        u64* t = m.tot + warp * LMOD;
        const int L = (int)(lam_b - lam_a + 1);
        for (int j = lane; j < L; j += kWarp) t[j] = 0;
        __syncwarp();
        const uint32_t c32 = (uint32_t)c;
        const u64 cinv = bplb_cinv(c32);
        if (TABLE) {  // distinct values x counts (c small: never wide)
            if (kind == K_VB2) mod_walk<false, true>(m.vb2, 0, ctl.n_vb2, c32, cinv, lam_a, L, t, p.one, true, m.vb2c);
            else mod_walk<false, true>(m.dval, 0, ctl.n_dist, c32, cinv, lam_a, L, t, p.one, false, m.dcnt);
        } else {
            if (kind == K_VB2) mod_walk<WIDE>(m.vb2, 0, ctl.n_vb2, c32, cinv, lam_a, L, t, p.one, true);
            else mod_walk<WIDE>(m.sw, 0, st.r, c32, cinv, lam_a, L, t, p.one, false);
        }
        __syncwarp();
        wmax = -1;
        for (int j0 = 0; j0 < L; j0 += kWarp) {
            const int j = j0 + lane;
            const bool valid = j < L;
            const int64_t lam = lam_a + j;
            int64_t S = 0;
            if (valid)
                S = (kind == K_VB2) ? bplb_vb2_sum(st, c, lam, t[j])
                                    : bplb_fs1_sum(st, lam, t[j], (uint64_t)bplb_fs1_zero(lk, c, st.maxw, lam));
            int64_t b = valid ? bplb_bound(S, bplb_fc(kind, c, lam)) : 0;
            int64_t mm = emit_warp(valid, lam, b, ctl.lo[kind], &ctl.key[kind], lam_out, p.out_lo, p.out_hi);
            wmax = mm > wmax ? mm : wmax;
        }
    }
    if (lane == 0) {
        atomicAdd(&ctl.evals[kind], (unsigned long long)(lam_b - lam_a + 1));
        ctl.evaluated[kind] = 1;
        if (wmax >= 0) {
            atomicMax(&ctl.lb, (int)wmax);
            if (ctl.vprune_seg >= 0 && kind == K_VB2) {
                const u64 kk = *(volatile u64*)&ctl.key[kind];
                if (kk > ctl.pub[kind]) {  // publish only what improved (one L2 line for every CTA)
                    ctl.pub[kind] = kk;
                    atomicMax(&p.ms->live[kind], kk);
                }
            }
            // the cross-CTA running maxima only feed the PHASED / CANCEL guards
            if (p.ms && (p.flags & (BPLB_F_PHASED | BPLB_F_CANCEL))) {
                atomicMax(&p.ms->lb, (int)wmax);
                atomicMax(&p.ms->kmax[kind], (int)wmax);
            }
        }
    }
}

// Multi-CTA sweep of one node: units come from a global counter in kind
// order.  PHASED / CANCEL: before the first unit of a later kind, wait until
// every earlier unit has completed, then apply the guard lb <= k (a skipped
// unit still counts as completed).  No CTA waits while holding an unfinished
// unit (one unit per warp at a time) and the grid is co-resident, so the
// waits cannot deadlock.
template <bool TABLE, bool WIDE, class LK>
__device__ void sweep_multi(const KParams& p, NodeCtl& ctl, const LK& lk, const NodeMem& m,
                            bool single, bool guard, bool phased) {
    const int lane = threadIdx.x & 31;
    MultiState* ms = p.ms;
    for (;;) {
        int u = 0;
        if (lane == 0) u = atomicAdd(&ms->unit_next, 1);
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= ctl.nunits) break;
        bool skip = false;
        if (guard) {
            int si = 0;
            while (si + 1 < ctl.nseg && ctl.segs[si + 1].first <= u) ++si;
            const int kd = ctl.segs[si].kind;
            const int first = ctl.segs[ctl.kind_seg_first[kd]].first;  // first unit of this kind
            if (lane == 0) {
                while (*(volatile int*)&ms->units_done < first) __nanosleep(200);
            }
            __syncwarp();
            __threadfence();
            if (phased) {
                // Alg. 2: a kind runs to completion; stop at the first kind
                // boundary where the earlier kinds' max exceeds k
                // (the first kind in the order always runs: no earlier kind)
                int prev = 0;
                bool has_prev = false;
                for (int i = 0; i < p.nk && p.kinds[i] != kd; ++i) {
                    prev = max(prev, *(volatile int*)&ms->kmax[p.kinds[i]]);
                    has_prev = true;
                }
                skip = has_prev && (int64_t)prev > p.k;
            } else {
                skip = (int64_t)(*(volatile int*)&ms->lb) > p.k;  // Alg. 4 guard
            }
        }
        if (!skip) run_unit<TABLE, WIDE>(p, ctl, lk, m, u, single);
        __syncwarp();
        if (guard && lane == 0) {  // completion count: only the guards wait on it
            __threadfence();
            atomicAdd(&ms->units_done, 1);
        }
    }
}

// Process units [ctl.unit_next, ctl.unit_end) with all warps.
template <bool TABLE, bool WIDE, class LK>
__device__ void run_units(const KParams& p, NodeCtl& ctl, const LK& lk, const NodeMem& m,
                          bool single, bool cancel) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        int u = 0;
        if (lane == 0) u = atomicAdd(&ctl.unit_next, 1);
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= ctl.unit_end) break;
        if (cancel) {
            int cur = *(volatile int*)&ctl.lb;
            if ((int64_t)cur > p.k) continue;  // Alg. 4 guard
        }
        run_unit<TABLE, WIDE>(p, ctl, lk, m, u, single);
    }
}

// Kinds in order, one phase per kind (PHASED: stop after the first kind whose
// best exceeds k -- bounds.py:523-525; CANCEL: skip later kinds once lb > k,
// the Alg. 3/4 per-launch guard, and skip units inside a kind too).  Without
// either flag all units of all kinds are pulled from one counter.
template <bool TABLE, bool WIDE, class LK>
__device__ void sweep_node(const KParams& p, NodeCtl& ctl, const LK& lk, const NodeMem& m,
                           bool single, bool phased, bool cancel) {
    if (phased || cancel) {
        for (int i = 0; i < p.nk; ++i) {
            const int kd = p.kinds[i];
            if (threadIdx.x == 0) {
                const int f = ctl.kind_seg_first[kd], n = ctl.kind_seg_count[kd];
                ctl.unit_next = n ? ctl.segs[f].first : 0;
                ctl.unit_end = n ? ctl.segs[f + n - 1].first + ctl.segs[f + n - 1].count : 0;
                ctl.skip = cancel && (int64_t)ctl.lb > p.k;
                if (!ctl.skip) ctl.n_done = i + 1;
            }
            __syncthreads();
            if (!ctl.skip) run_units<TABLE, WIDE>(p, ctl, lk, m, single, cancel);
            __syncthreads();
            if (phased && (int64_t)ctl.lb > p.k) break;
        }
    } else {
        if (threadIdx.x == 0) { ctl.unit_next = 0; ctl.unit_end = ctl.nunits; ctl.n_done = p.nk; }
        __syncthreads();
        run_units<TABLE, WIDE>(p, ctl, lk, m, single, false);
    }
}

__device__ __forceinline__ void block_sort(int* a, int n) {  // bitonic, n power of two
    for (int k = 2; k <= n; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n; i += NT) {
                int ixj = i ^ j;
                if (ixj > i) {
                    int x = a[i], y = a[ixj];
                    bool up = (i & k) == 0;
                    if ((x > y) == up) { a[i] = y; a[ixj] = x; }
                }
            }
            __syncthreads();
        }
    }
}

// Exclusive block-wide scan of one value per thread (warp shuffles + one
// shared word per warp).  Returns the sum of v over threads < threadIdx.x.
template <int NWARPS = NW>
__device__ __forceinline__ long long block_excl_scan(long long v, long long* wsum) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        long long t = lane < NWARPS ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < NWARPS; o <<= 1) {
            long long y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < NWARPS) wsum[lane] = t;
    }
    __syncthreads();
    long long res = (warp ? wsum[warp - 1] : 0) + x - v;
    __syncthreads();
    return res;
}

// pre[0] = 0, pre[i+1] = pre[i] + v[i] over n elements.
__device__ __forceinline__ void block_prefix_i64(const int* v, long long* pre, int n, long long* wsum) {
    const int per = (n + NT - 1) / NT;
    const int b = threadIdx.x * per, e = min(n, b + per);
    long long s = 0;
    for (int i = b; i < e; ++i) s += v[i];
    long long run = block_excl_scan(s, wsum);
    if (threadIdx.x == 0) pre[0] = 0;
    for (int i = b; i < e; ++i) { run += v[i]; pre[i + 1] = run; }
    __syncthreads();
}

// cnt[i] holds the histogram count of value i-1 (i in [0, c+1]); converts in
// place to cnt[i] = #{w <= i-1} and fills wle[i] = sum{w <= i-1}.
__device__ __forceinline__ void block_table_scan(int* cnt, long long* wle, int n, long long* wsum,
                                                 long long* wsum2) {
    const int per = (n + NT - 1) / NT;
    const int b = threadIdx.x * per, e = min(n, b + per);
    long long sc = 0, sw = 0;
    for (int i = b; i < e; ++i) { sc += cnt[i]; sw += (long long)cnt[i] * (i - 1); }
    long long rc = block_excl_scan(sc, wsum);
    long long rw = block_excl_scan(sw, wsum2);
    for (int i = b; i < e; ++i) {
        int x = cnt[i];
        rc += x;
        rw += (long long)x * (i - 1);
        cnt[i] = (int)rc;
        wle[i] = rw;
    }
    __syncthreads();
}

// Sort the r weights of sw by a counting sort on their bucket (v >> bk),
// producing the bucket index bidx[b] = #{w < b << bk} (bidx[nb] = r) on the
// way; tmp holds rcap ints.  Buckets hold few weights on typical inputs (insertion sort per
// bucket); returns false (sw / bidx unspecified, tmp clobbered) when a
// bucket exceeds 32 weights -- the caller then falls back to block_sort.
__device__ __forceinline__ bool block_bucket_sort(int* sw, int* tmp, int* bidx, int r, int nb, int bk,
                                                  int* s_maxb, long long* wsum) {
    for (int b = threadIdx.x; b <= nb; b += NT) bidx[b] = 0;
    if (threadIdx.x == 0) *s_maxb = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < r; i += NT) {
        const int n = atomicAdd(&bidx[sw[i] >> bk], 1);
        if (n >= 32) atomicMax(s_maxb, n + 1);
    }
    __syncthreads();
    if (*s_maxb > 32) return false;
    // exclusive scan of the nb + 1 bucket counts (bidx[nb] = 0 -> r)
    {
        const int per = (nb + 1 + NT - 1) / NT, b0 = threadIdx.x * per, b1 = min(nb + 1, b0 + per);
        int s = 0;
        for (int b = b0; b < b1; ++b) s += bidx[b];
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        int x = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        long long off = 0;
        for (int w = 0; w < warp; ++w) off += wsum[w];
        int run = (int)off + x - s;  // inclusive scan: bidx[b] = end of bucket b
        for (int b = b0; b < b1; ++b) {
            run += bidx[b];
            bidx[b] = run;
        }
    }
    __syncthreads();
    // scatter from each bucket's end (bidx moves back to the bucket's start)
    for (int i = threadIdx.x; i < r; i += NT) {
        const int v = sw[i];
        tmp[atomicSub(&bidx[v >> bk], 1) - 1] = v;
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += NT) {
        const int s0 = bidx[b], e = bidx[b + 1];
        for (int i = s0; i < e; ++i) {  // insertion sort of the bucket into sw
            const int v = tmp[i];
            int j = i;
            while (j > s0 && sw[j - 1] > v) { sw[j] = sw[j - 1]; --j; }
            sw[j] = v;
        }
    }
    __syncthreads();
    return true;
}

__host__ __device__ inline int node_bucket_shift(int64_t c) {
    int k = 0;
    while ((c >> k) + 2 > NBMAX) ++k;
    return k;
}

// Dynamic shared memory size of the node kernel.
__host__ __device__ inline size_t node_smem_bytes(bool table, int rcap, int64_t c) {
    size_t s = 0;
    s += (size_t)NW * LMOD * 8;            // tot
    s += (size_t)rcap * 4;                 // sw
    if (table) {
        const size_t dc = (size_t)(rcap < c + 1 ? rcap : c + 1);
        s += (size_t)(c + 2) * 8;          // wle
        s += (size_t)(c + 2) * 4;          // cnt
        s += dc * 4 * 4;                   // dval, dcnt, vb2, vb2c
    } else {
        s += (size_t)(rcap + 1) * 8;       // pre
        s += (size_t)rcap * 4;             // vb2
        s += (size_t)(NBMAX + 1) * 4;      // bidx
    }
    return s + 64;
}

// WIDE: 64-bit lane partials in the modular walk, needed when c >= 2^23.
template <bool TABLE, bool WIDE>
#ifndef NODE_MINB
#define NODE_MINB 2  // resident node_kernel CTAs per SM the register budget is sized for
#endif
__global__ void __launch_bounds__(NT, NODE_MINB) node_kernel(KParams p, int rcap) {
    extern __shared__ __align__(16) unsigned char smem[];
    NODE_STAMP(0);
    __shared__ NodeCtl ctl;
    const int64_t c = p.c;
    NodeMem m;
    {
        unsigned char* q = smem;
        m.tot = (u64*)q; q += NW * LMOD * 8;
        if (TABLE) {
            const int dc = (int)(rcap < c + 1 ? rcap : c + 1);
            m.pre = (long long*)q; q += (c + 2) * 8;
            m.cnt = (int*)q; q += (c + 2) * 4;
            m.sw = (int*)q; q += (size_t)rcap * 4;
            m.dval = (int*)q; q += dc * 4;
            m.dcnt = (int*)q; q += dc * 4;
            m.vb2 = (int*)q; q += dc * 4;
            m.vb2c = (int*)q; q += dc * 4;
            m.bidx = nullptr;
        } else {
            m.pre = (long long*)q; q += (size_t)(rcap + 1) * 8;
            m.sw = (int*)q; q += (size_t)rcap * 4;
            m.vb2 = (int*)q; q += (size_t)rcap * 4;
            m.bidx = (int*)q;
            m.cnt = m.dval = m.dcnt = m.vb2c = nullptr;
        }
        m.bk = TABLE ? 0 : node_bucket_shift(c);
    }
    const bool single = p.lam_out != nullptr;
    const bool phased = p.flags & BPLB_F_PHASED;
    const bool cancel = (p.flags & BPLB_F_CANCEL) && !phased;

    const bool multi = p.ms != nullptr;
    for (int64_t node = p.node0 + (multi ? 0 : blockIdx.x); node < p.node0 + p.n_nodes;
         node += (multi ? p.n_nodes : gridDim.x)) {
        const int64_t base = p.off[node];
        const int r = (int)(p.off[node + 1] - base);
        if (threadIdx.x == 0) {
            NodeStats& st = ctl.st;
            st.r = r; st.maxw = 0; st.n_small = st.n_eq = st.n_big = st.n_full = 0;
            st.W = st.Vs = st.Vm = 0;
            for (int i = 0; i < K_COUNT; ++i) {
                ctl.key[i] = 0; ctl.evals[i] = 0; ctl.evaluated[i] = 0;
            }
            ctl.lb = 0; ctl.n_vb2 = 0; ctl.n_dist = 0; ctl.nseg = 0; ctl.nunits = 0; ctl.n_done = 0;
            ctl.bad = 0;
        }
        // ---- stage weights -------------------------------------------------
        int pw = 1;
        while (pw < r) pw <<= 1;
        if (TABLE) {
            for (int i = threadIdx.x; i < c + 2; i += NT) m.cnt[i] = 0;
        }
        for (int i = threadIdx.x; i < (TABLE ? r : pw); i += NT)
            m.sw[i] = i < r ? load_w(p, base + i) : INT_MAX;
        __syncthreads();
        NODE_STAMP(1);
        // ---- statistics ------------------------------------------------------
        {
            int l_max = 0, l_bad = 0, l_s = 0, l_e = 0, l_b = 0, l_f = 0;
            long long l_W = 0, l_Vs = 0, l_Vm = 0;
            for (int i = threadIdx.x; i < r; i += NT) {
                const int x = m.sw[i];
                if (x < 1 || (int64_t)x > c) { l_bad = 1; continue; }
                l_max = max(l_max, x);
                l_W += x;
                if (2 * (int64_t)x < c) { l_s++; l_Vs += x; }
                else if (2 * (int64_t)x == c) l_e++;
                else { l_b++; l_Vm += c - x; if (x == c) l_f++; }
                if (TABLE) atomicAdd(&m.cnt[x + 1], 1);
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
        NODE_STAMP(2);
        // ---- lookup structure -----------------------------------------------
        if (TABLE) {
            // distinct (value, count) pairs for the modular walks (G11: order free)
            for (int v = threadIdx.x + 1; v <= c; v += NT) {
                const int n = m.cnt[v + 1];
                if (n) {
                    const int i = atomicAdd(&ctl.n_dist, 1);
                    m.dval[i] = v;
                    m.dcnt[i] = n;
                    if (2 * (int64_t)v != c && v < c) {
                        const int j = atomicAdd(&ctl.n_vb2, 1);
                        m.vb2[j] = v;
                        m.vb2c[j] = n;
                    }
                }
            }
            __syncthreads();
            block_table_scan(m.cnt, m.pre, (int)(c + 2), ctl.wsum, ctl.wsum2);
        } else {
            // sorted weights + bucket index bidx[b] = #{w < b << k}: counting
            // sort by bucket (O(r + nb)); bitonic sort when a bucket is crowded
            const int nb = (int)(c >> m.bk) + 1;
            __shared__ int s_maxb;
            const bool bucketed = !ctl.bad && block_bucket_sort(m.sw, m.vb2, m.bidx, r, nb, m.bk, &s_maxb, ctl.wsum);
            if (!bucketed) {
                for (int i = threadIdx.x; i < pw; i += NT) m.sw[i] = i < r ? load_w(p, base + i) : INT_MAX;
                __syncthreads();
                block_sort(m.sw, pw);
            }
            NODE_STAMP(5);
            block_prefix_i64(m.sw, m.pre, r, ctl.wsum);
            const NodeStats& st = ctl.st;
            const int nm = st.n_big - st.n_full;
            for (int i = threadIdx.x; i < st.n_small + nm; i += NT)
                m.vb2[i] = i < st.n_small ? m.sw[i] : m.sw[i + st.n_eq];
            if (!bucketed) {
                for (int b = threadIdx.x; b <= nb; b += NT) {
                    const int64_t v = (int64_t)b << m.bk;
                    int lo = 0, hi = r;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if ((int64_t)m.sw[mid] < v) lo = mid + 1; else hi = mid;
                    }
                    m.bidx[b] = b == nb ? r : lo;
                }
            }
            if (threadIdx.x == 0) ctl.n_vb2 = st.n_small + nm;
            NODE_STAMP(6);
        }
        if (threadIdx.x == 0) {
            bplb_stats_finish(&ctl.st, c);
            for (int kd = 0; kd < K_COUNT; ++kd) {
                int64_t lo, hi;
                if (p.use_range) { lo = p.rng_lo[kd]; hi = p.rng_hi[kd]; }
                else {
                    bplb_domain(kd, c, &lo, &hi);
                    if (kd == K_VB2) hi = bplb_vb2_hi(c, r, ctl.st.maxw);
                }
                if (!kind_in(p, kd)) hi = lo - 1;
                ctl.lo[kd] = lo; ctl.hi[kd] = hi;
            }
            // multi-CTA full checks inside the pruning envelope: VB2 as a
            // 32-lambda seed unit first, the other kinds, then the VB2 rest,
            // whose chunks are tested against the best published VB2 key
            const bool vprune = multi && !single && !(p.flags & (BPLB_F_PHASED | BPLB_F_CANCEL | BPLB_F_NOPRUNE)) &&
                                c <= ((int64_t)1 << 20) && kind_in(p, K_VB2) &&
                                ctl.hi[K_VB2] >= ctl.lo[K_VB2] + 32 + LMOD;
            ctl.vprune_seg = -1;
            for (int kd = 0; kd < K_COUNT; ++kd) ctl.pub[kd] = 0;
            if (vprune) {
                const int64_t vlo = ctl.lo[K_VB2], vhi = ctl.hi[K_VB2];
                auto pushv = [&](int64_t a, int64_t b, int chunk) {
                    Seg& g = ctl.segs[ctl.nseg++];
                    g.kind = K_VB2; g.type = T_MOD; g.lo = a; g.hi = b; g.chunk = chunk;
                    g.first = ctl.nunits;
                    g.count = (int)((uint32_t)(b - a + chunk) / (uint32_t)chunk);
                    ctl.nunits += g.count;
                };
                pushv(vlo, vlo + 31, 32);
                // (dense-division units of 4 lambdas: 32 of them, a pass over
                // the items each, made one unit the whole sweep's tail)
                for (int i = 0; i < p.nk; ++i)
                    if (p.kinds[i] != K_VB2) add_kind_segs(ctl, p.kinds[i], TABLE, c, 4);
                ctl.vprune_seg = ctl.nseg;
                pushv(vlo + 32, vhi, 32);  // short chunks: a surviving one must not become the tail
                ctl.kind_seg_first[K_VB2] = 0;
                ctl.kind_seg_count[K_VB2] = 2;  // (kind bookkeeping: only the guards use it)
            } else {
                for (int i = 0; i < p.nk; ++i) add_kind_segs(ctl, p.kinds[i], TABLE, c, multi ? 4 : LDIV);
            }
            if (ctl.bad) {
                ctl.nunits = 0; ctl.nseg = 0;
                for (int kd = 0; kd < K_COUNT; ++kd) ctl.kind_seg_count[kd] = 0;
            }
        }
        __syncthreads();
        NODE_STAMP(3);
        // ---- sweep -------------------------------------------------------------
        if (TABLE) {
            LkTable lk{m.cnt, m.pre, c};
            if (multi) sweep_multi<TABLE, WIDE>(p, ctl, lk, m, single, phased || (p.flags & BPLB_F_CANCEL), phased);
            else sweep_node<TABLE, WIDE>(p, ctl, lk, m, single, phased, cancel);
        } else {
            LkBucket lk{m.sw, m.pre, m.bidx, r, m.bk, c};
            if (multi) sweep_multi<TABLE, WIDE>(p, ctl, lk, m, single, phased || (p.flags & BPLB_F_CANCEL), phased);
            else sweep_node<TABLE, WIDE>(p, ctl, lk, m, single, phased, cancel);
        }
        __syncthreads();
        NODE_STAMP(4);
        // ---- outputs ----------------------------------------------------------
        if (multi) {
            __shared__ int last;
            if (threadIdx.x == 0) {
                MultiState* ms = p.ms;
                for (int kd = 0; kd < K_COUNT; ++kd) {
                    if (ctl.evaluated[kd]) {
                        atomicMax(&ms->key[kd], ctl.key[kd]);
                        atomicAdd(&ms->evals[kd], ctl.evals[kd]);
                        atomicOr(&ms->evaluated[kd], 1);
                    }
                }
                __threadfence();
                last = atomicAdd(&ms->ctas_done, 1) == (int)gridDim.x - 1;
                if (last) {
                    __threadfence();
                    for (int kd = 0; kd < K_COUNT; ++kd) {
                        ctl.key[kd] = *(volatile u64*)&ms->key[kd];
                        ctl.evals[kd] = *(volatile unsigned long long*)&ms->evals[kd];
                        ctl.evaluated[kd] = *(volatile int*)&ms->evaluated[kd];
                    }
                    // kinds processed in order until the running max exceeds k
                    int nd = p.nk;
                    if (phased) {
                        int64_t run = 0;
                        for (int i = 0; i < p.nk; ++i) {
                            const int kd = p.kinds[i];
                            if (ctl.evaluated[kd]) run = max(run, (int64_t)(ctl.key[kd] >> 32));
                            if (run > p.k) { nd = i + 1; break; }
                        }
                    }
                    ctl.n_done = nd;
                    // every other CTA is past its last access: leave the
                    // cross-CTA state zeroed for the next check
                    for (int kd = 0; kd < K_COUNT; ++kd) {
                        ms->key[kd] = 0; ms->kmax[kd] = 0; ms->evals[kd] = 0; ms->evaluated[kd] = 0;
                        ms->live[kd] = 0;
                    }
                    ms->lb = 0; ms->ctas_done = 0; ms->unit_next = 0; ms->units_done = 0;
                }
            }
            __syncthreads();
            if (!last) break;
        }
        if (threadIdx.x == 0) {
            if (p.err_out) {
                if (multi) *p.err_out = ctl.bad ? 1 : 0;  // (written every check: no host memset)
                else if (ctl.bad) atomicExch(p.err_out, 1);
            }
            int64_t lb = 0;
            bplb_result res;
            for (int kd = 0; kd < K_COUNT; ++kd) {
                const u64 key = ctl.key[kd];
                const bool ev = ctl.evaluated[kd];
                res.best[kd] = ev ? (int64_t)(key >> 32) : 0;
                res.arg_lambda[kd] = ev ? ctl.lo[kd] + (int64_t)(0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFu))
                                        : ctl.lo[kd];
                res.n_lambda[kd] = ctl.hi[kd] >= ctl.lo[kd] ? ctl.hi[kd] - ctl.lo[kd] + 1 : 0;
                res.evals[kd] = (int64_t)ctl.evals[kd];
                res.evaluated[kd] = ev;
                if (ev && res.best[kd] > lb) lb = res.best[kd];
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
