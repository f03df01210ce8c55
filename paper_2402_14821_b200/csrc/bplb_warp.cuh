// bplb_warp.cuh -- warp-per-node kernel for batches of small-capacity search
// nodes (cfg2: c = 150, r ~ 400, 1e4 nodes).  Each warp owns one reduced
// instance at a time: a histogram of its weights over [0, c] in the warp's
// slice of shared memory, the cumulative count / weight tables (warp scan),
// the multiset compressed to distinct (value, count) pairs, then every kind
// in order -- lookups one lambda per lane, VB2/FS1 as the weighted modular
// walk.  No block barriers; per-node fixed cost is a few hundred
// instructions instead of a CTA-wide setup.
#pragma once
#include "bplb_node.cuh"

namespace bplb {

constexpr int WNT = 256;                 // threads per CTA
constexpr int WNW = WNT / 32;            // warps (= nodes in flight) per CTA
constexpr int WARP_MAX_C = 1024;         // capacity limit of the warp kernel

// Per-warp shared-memory slice (bytes), 16-byte aligned.
__host__ __device__ inline size_t al16(size_t b) { return (b + 15) & ~(size_t)15; }
// CTA-wide tables for the FS1 zero-remainder term (shared by all warps):
// divisors of c (<= 32 for c <= 1024), the divisor index of m_v = c/gcd(c,v)
// for every value v, and for every FS1 lambda the mask of divisors m | lambda+1.
__host__ __device__ inline size_t warp_cta_bytes(int64_t c) {
    return al16(32 * 4) + al16(100 * 4) + al16((size_t)(c + 1));
}
__host__ __device__ inline size_t warp_slice_bytes(int64_t c) {
    const size_t n = (size_t)(c + 2), d = (size_t)(c + 1);
    return al16(n * 8) + al16(n * 4) + 4 * al16(d * 4) + al16(d * 8) + al16(32 * 8) + 256;
}

// lane-local running best for one kind: higher bound wins, lower lambda on ties
struct Best {
    int64_t b;
    int64_t lam;
    __device__ __forceinline__ void offer(int64_t bd, int64_t l) {
        if (bd > b || (bd == b && l < lam)) { b = bd; lam = l; }
    }
};

__device__ __forceinline__ Best warp_best(Best x) {
    const uint32_t bv = x.b >= 0 ? (uint32_t)x.b + 1u : 0u;
    const uint32_t mx = __reduce_max_sync(0xffffffffu, bv);
    const uint32_t lr = (bv == mx && mx) ? (uint32_t)x.lam : 0xFFFFFFFFu;
    const uint32_t mn = __reduce_min_sync(0xffffffffu, lr);
    Best r;
    r.b = mx ? (int64_t)(mx - 1u) : -1;
    r.lam = mx ? (int64_t)mn : -1;
    return r;
}

// 32-bit table lookups for c <= WARP_MAX_C (index x+1 for x in [-1, c]).
struct Lk32 {
    const int* cnt;
    const long long* wle;
    int c;
    __device__ __forceinline__ int ix(int x) const { return (x < -1 ? -1 : (x > c ? c : x)) + 1; }
    __device__ __forceinline__ int n(int x) const { return cnt[ix(x)]; }
    __device__ __forceinline__ void both(int x, int* nn, long long* w) const {
        const int i = ix(x);
        *nn = cnt[i];
        *w = wle[i];
    }
};

// Partial transformed sums of the lookup kinds over a strided subset of the
// harmonic terms t = t0, t0+dt, ... (MT / RAD2 have a single term, t0 == 0).
// One out-of-line copy serves the lane-per-lambda and the warp-per-lambda
// loops (keeps the warp kernel small enough for the instruction cache).
//   MT   _sweep_mt   bounds.py:373-376    p1 = S
//   RAD2 _sweep_rad2 bounds.py:379-387    p1 = S
//   CCM1 _sweep_ccm1 bounds.py:390-407    p1 = sum_t (n_small - N(t l - 1)) - (N(c - t l) - (r - n_big))
//   BJ1  _sweep_bj1  bounds.py:441-460    p1 = floor_sum part, p2 = rem_sum part
__device__ __noinline__ void lookup_part(int kd, const Lk32& lk, const NodeStats& st, int c, int r, int lam,
                                         int t0, int dt, long long* p1, long long* p2) {
    long long a = 0, b = 0;
    if (kd == K_MT) {
        if (t0 == 0) {
            int n1, n0;
            long long w1, w0;
            lk.both(c - lam, &n1, &w1);
            lk.both(lam - 1, &n0, &w0);
            a = (long long)c * (r - n1) + w1 - w0;
        }
    } else if (kd == K_RAD2) {
        if (t0 == 0) {
            const int third = c / 3, half = c / 2;
            const int ia = lk.n(lam - 1), ib = lk.n(c - 2 * lam), id = lk.n(2 * lam - 1), ie = lk.n(c - lam);
            a = (long long)(ib - ia) * third + (long long)(id - ib) * half + (long long)(ie - id) * (c - third) +
                (long long)(r - ie) * c;
        }
    } else if (kd == K_CCM1) {
        const int tmax = ((c - 1) / 2) / lam;
        const int base = st.n_small + st.r - st.n_big;
        for (int t = t0 + 1; t <= tmax; t += dt) a += base - lk.n(t * lam - 1) - lk.n(c - t * lam);
    } else {
        const int cm = c % lam, tmax = st.maxw / lam;
        for (int t = t0; t <= tmax; t += dt) {
            const int lo_v = lam * t + cm, hi_v = lam * (t + 1) - 1;
            int nl, nh;
            long long wl, wh;
            lk.both(lo_v, &nl, &wl);
            lk.both(hi_v, &nh, &wh);
            b += (wh - wl) - (long long)lo_v * (nh - nl);
            if (t < tmax) a += st.r - nh;
        }
    }
    *p1 = a;
    *p2 = b;
}

// Bound of one lookup-kind lambda from its partial sums, 32-bit divisions
// only (c <= WARP_MAX_C): bounds.py:376, 387, 407, 460 for F.
__device__ __forceinline__ int64_t lookup_bound32(int kd, const NodeStats& st, int c, int lam,
                                                  long long p1, long long p2) {
    long long S, F;
    if (kd == K_CCM1) {
        const int cq = c / lam;
        S = 2 * p1 + (long long)st.n_eq * cq + 2ll * st.n_big * cq;
        F = 2ll * cq;
    } else if (kd == K_BJ1) {
        const int cq = c / lam, cm = c - cq * lam;
        S = (long long)(lam - cm) * p1 + p2;
        F = (long long)cq * (lam - cm);
    } else {
        S = p1;
        F = c;
    }
    return bplb_bound(S, F);
}

__device__ __forceinline__ u64 fs1_z(const u64* zacc, unsigned int mask) {
    u64 z = 0;
    while (mask) {
        z += zacc[__ffs(mask) - 1];
        mask &= mask - 1;
    }
    return z;
}

__device__ __forceinline__ void warp_kind_range(const KParams& p, int kd, int64_t c, int r, int maxw,
                                                int64_t* lo, int64_t* hi) {
    bplb_domain(kd, c, lo, hi);
    if (kd == K_VB2) *hi = bplb_vb2_hi(c, r, maxw);
    if (!kind_in(p, kd)) *hi = *lo - 1;
}

__global__ void __launch_bounds__(WNT, 3) warp_node_kernel(KParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t c = p.c;
    const int n2 = (int)c + 2, d1 = (int)c + 1;
    int* divs = (int*)smem;
    unsigned int* dmask = (unsigned int*)(smem + al16(32 * 4));
    unsigned char* mdiv = smem + al16(32 * 4) + al16(100 * 4);
    {
        __shared__ int n_div;
        if (threadIdx.x == 0) {
            int nd = 0;
            for (int d = 1; d <= (int)c && nd < 32; ++d)
                if ((int)c % d == 0) divs[nd++] = d;
            n_div = nd;
        }
        __syncthreads();
        const int ndv = n_div;
        for (int v = threadIdx.x; v <= (int)c; v += blockDim.x) {
            int a = (int)c, b = v;
            while (b) { const int t = a % b; a = b; b = t; }
            const int m = (int)c / a;
            int i = 0;
            while (i < ndv && divs[i] != m) ++i;
            mdiv[v] = (unsigned char)i;
        }
        for (int l = threadIdx.x; l < 100; l += blockDim.x) {
            unsigned int mk = 0;
            for (int i = 0; i < ndv; ++i)
                if ((l + 2) % divs[i] == 0) mk |= 1u << i;  // lambda = l + 1 -> lambda + 1 = l + 2
            dmask[l] = mk;
        }
        __syncthreads();
    }
    unsigned char* q = smem + warp_cta_bytes(c) + warp_slice_bytes(c) * warp;
    long long* wle = (long long*)q; q += al16((size_t)n2 * 8);
    int* cnt = (int*)q; q += al16((size_t)n2 * 4);
    int* dval = (int*)q; q += al16((size_t)d1 * 4);
    int* dcnt = (int*)q; q += al16((size_t)d1 * 4);
    int* vval = (int*)q; q += al16((size_t)d1 * 4);
    int* vcnt = (int*)q; q += al16((size_t)d1 * 4);
    u64* tot = (u64*)q; q += al16((size_t)d1 * 8);
    u64* zacc = (u64*)q; q += al16(32 * 8);  // FS1: sum of v*count per divisor class
    long long* kres = (long long*)q;  // per-kind best / arg (lane 0)
    const bool phased = p.flags & BPLB_F_PHASED;
    const bool cancel = (p.flags & BPLB_F_CANCEL) && !phased;
    const uint32_t c32 = (uint32_t)c;
    const u64 cinv = bplb_cinv(c32);
    const uint32_t lt_mask = (1u << lane) - 1u;

    for (int64_t node = p.node0 + (int64_t)blockIdx.x * WNW + warp; node < p.node0 + p.n_nodes;
         node += (int64_t)gridDim.x * WNW) {
        const int64_t base = p.off[node];
        const int r = (int)(p.off[node + 1] - base);
        for (int i = lane; i < n2; i += 32) cnt[i] = 0;
        __syncwarp();
        // ---- histogram + statistics ---------------------------------------
        int l_max = 0, l_bad = 0, l_s = 0, l_e = 0, l_b = 0, l_f = 0;
        long long l_W = 0, l_Vs = 0, l_Vm = 0;
        for (int i = lane; i < r; i += 32) {
            const int x = load_w(p, base + i);
            if (x < 1 || (int64_t)x > c) { l_bad = 1; continue; }
            l_max = max(l_max, x);
            l_W += x;
            if (2 * x < c) { l_s++; l_Vs += x; }
            else if (2 * x == c) l_e++;
            else { l_b++; l_Vm += c - x; if (x == c) l_f++; }
            atomicAdd(&cnt[x + 1], 1);
        }
        NodeStats st;
        st.r = r;
        st.maxw = (int32_t)__reduce_max_sync(0xffffffffu, (unsigned)l_max);
        const bool bad = __reduce_or_sync(0xffffffffu, (unsigned)l_bad) != 0;
        st.n_small = __reduce_add_sync(0xffffffffu, l_s);
        st.n_eq = __reduce_add_sync(0xffffffffu, l_e);
        st.n_big = __reduce_add_sync(0xffffffffu, l_b);
        st.n_full = __reduce_add_sync(0xffffffffu, l_f);
        st.W = (int64_t)warp_sum_u64((u64)l_W);
        st.Vs = (int64_t)warp_sum_u64((u64)l_Vs);
        st.Vm = (int64_t)warp_sum_u64((u64)l_Vm);
        bplb_stats_finish(&st, c);
        __syncwarp();
        // ---- distinct (value, count) lists (ballot compaction) --------------
        int nd = 0, nv = 0;
        for (int v0 = 1; v0 <= c; v0 += 32) {
            const int v = v0 + lane;
            const int n = v <= c ? cnt[v + 1] : 0;
            const uint32_t m1 = __ballot_sync(0xffffffffu, n > 0);
            const bool isv = n > 0 && 2 * v != c && v < c;
            const uint32_t m2 = __ballot_sync(0xffffffffu, isv);
            if (n > 0) { const int pos = nd + __popc(m1 & lt_mask); dval[pos] = v; dcnt[pos] = n; }
            if (isv) { const int pos = nv + __popc(m2 & lt_mask); vval[pos] = v; vcnt[pos] = n; }
            nd += __popc(m1);
            nv += __popc(m2);
        }
        // ---- cumulative tables (warp scan, index x+1 for x in [-1, c]) -------
        {
            long long rc = 0, rw = 0;
            for (int i0 = 0; i0 < n2; i0 += 32) {
                const int i = i0 + lane;
                long long x = i < n2 ? cnt[i] : 0;
                long long y = x * (i - 1);
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const long long xo = __shfl_up_sync(0xffffffffu, x, o);
                    const long long yo = __shfl_up_sync(0xffffffffu, y, o);
                    if (lane >= o) { x += xo; y += yo; }
                }
                __syncwarp();
                if (i < n2) { cnt[i] = (int)(rc + x); wle[i] = rw + y; }
                rc += __shfl_sync(0xffffffffu, x, 31);
                rw += __shfl_sync(0xffffffffu, y, 31);
            }
        }
        __syncwarp();
        const Lk32 lk{cnt, wle, (int)c};
        const int ci = (int)c;
        // ---- kinds in order --------------------------------------------------
        long long* kbest = kres;          // per kind (lane-0 copies; all lanes read)
        long long* karg = kres + K_COUNT;
        int* keval = (int*)(kres + 2 * K_COUNT);
        if (lane < K_COUNT) {
            int64_t lo, hi;
            warp_kind_range(p, lane, c, r, st.maxw, &lo, &hi);
            kbest[lane] = 0;
            karg[lane] = lo;
            keval[lane] = 0;
        }
        __syncwarp();
        int64_t lb = 0;
        int n_done = 0;
        for (int i = 0; i < p.nk && !bad; ++i) {
            const int kd = p.kinds[i];
            if (cancel && lb > p.k) continue;  // Alg. 3/4 guard: later kinds skip
            n_done = i + 1;
            int64_t lo, hi;
            warp_kind_range(p, kd, c, r, st.maxw, &lo, &hi);
            if (hi < lo) {
                if (phased && lb > p.k) break;
                continue;
            }
            Best bl{-1, 0};
            if (kd == K_VB2 || kd == K_FS1) {
                const bool isv = kd == K_VB2;
                if (!isv) {
                    // Z(lambda) = sum of w with c | w(lambda+1) = sum over the
                    // divisor classes m = c/gcd(c, v) with m | lambda+1
                    zacc[lane] = 0;
                    __syncwarp();
                    for (int i = lane; i < nd; i += 32) {
                        const int v = dval[i];
                        atomicAdd(&zacc[mdiv[v]], (u64)v * (u64)dcnt[i]);
                    }
                    __syncwarp();
                }
                for (int64_t la = lo; la <= hi; la += d1) {
                    const int L = (int)min((int64_t)d1, hi - la + 1);
                    for (int j = lane; j < L; j += 32) tot[j] = 0;
                    __syncwarp();
                    mod_walk<false, true>(isv ? vval : dval, 0, isv ? nv : nd, c32, cinv, la, L, tot, p.one,
                                          isv, isv ? vcnt : dcnt);
                    __syncwarp();
                    for (int j = lane; j < L; j += 32) {
                        const int lam = (int)la + j;
                        const int64_t S = isv ? bplb_vb2_sum(st, c, lam, tot[j])
                                              : bplb_fs1_sum(st, lam, tot[j], fs1_z(zacc, dmask[lam - 1]));
                        bl.offer(bplb_bound(S, isv ? 2ll * (lam - 1) : (long long)ci * lam), lam);
                    }
                    __syncwarp();
                }
            } else {
                // small lambda with a long harmonic loop: one lambda per warp,
                // the t-loop split across lanes; afterwards one lambda per lane
                const int span = kd == K_CCM1 ? (ci - 1) / 2 : (kd == K_BJ1 ? st.maxw : 0);
                const int lw = min((int)hi + 1, span / 16 + 1);
                int lam = (int)lo;
                bool coop = lam < lw;
                while (true) {
                    const int my = coop ? lam : lam + lane;
                    long long p1 = 0, p2 = 0;
                    if (my <= (int)hi) lookup_part(kd, lk, st, ci, r, my, coop ? lane : 0, coop ? 32 : 1, &p1, &p2);
                    if (coop) {
                        p1 = (long long)warp_sum_u64((u64)p1);
                        p2 = (long long)warp_sum_u64((u64)p2);
                    }
                    if ((!coop || lane == 0) && my <= (int)hi)
                        bl.offer(lookup_bound32(kd, st, ci, my, p1, p2), my);
                    lam += coop ? 1 : 32;
                    if (lam > (int)hi) break;
                    coop = lam < lw;
                }
            }
            const Best wb = warp_best(bl);
            if (lane == 0) { kbest[kd] = wb.b; karg[kd] = wb.lam; keval[kd] = 1; }
            if (wb.b > lb) lb = wb.b;
            if (phased && lb > p.k) break;
        }
        __syncwarp();
        if (lane == 0) {
            if (bad && p.err_out) atomicExch(p.err_out, 1);
            if (p.lb_out) p.lb_out[node] = lb;
            if (p.ex_out) p.ex_out[node] = (uint8_t)(lb > p.k);
            if (p.best_out)
                for (int kd = 0; kd < K_COUNT; ++kd) p.best_out[node * K_COUNT + kd] = keval[kd] ? kbest[kd] : 0;
            if (p.arg_out)
                for (int kd = 0; kd < K_COUNT; ++kd) p.arg_out[node * K_COUNT + kd] = karg[kd];
            if (p.res_out) {
                bplb_result res;
                int64_t et = 0;
                for (int kd = 0; kd < K_COUNT; ++kd) {
                    int64_t lo, hi;
                    warp_kind_range(p, kd, c, r, st.maxw, &lo, &hi);
                    const int64_t nl = hi >= lo ? hi - lo + 1 : 0;
                    res.best[kd] = keval[kd] ? kbest[kd] : 0;
                    res.arg_lambda[kd] = karg[kd];
                    res.n_lambda[kd] = nl;
                    res.evals[kd] = keval[kd] ? nl : 0;
                    res.evaluated[kd] = keval[kd];
                    et += res.evals[kd];
                }
                res.lb = lb;
                res.exceeded = lb > p.k;
                res.n_done = n_done;
                res.evals_total = et;
                p.res_out[node] = res;
            }
        }
        __syncwarp();
    }
}

}  // namespace bplb
