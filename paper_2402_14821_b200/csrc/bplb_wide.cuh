// bplb_wide.cuh -- grid-wide path for one large reduced instance (cfg3-style
// c = 1e5 single checks, cfg4-style r = 1e5 / c = 1e6 checks, and
// dff_bound_batch).  The instance is described by global cumulative tables
// over the weight values (L2-resident: 12 bytes per value), every SM pulls
// warp units from one global counter, and the VB2/FS1 modular walk is cut
// into (lambda chunk x item slice) tiles whose partial sums meet in a global
// per-lambda accumulator.
//
// Launch sequence (one stream, no host round trip):
//   wide_init     zero state, tables and accumulators (one kernel)
//   wide_stats    per-item statistics, histogram, VB2 item compaction
//   wide_scan_*   3-phase scan of the histogram into N<=(x), W<=(x) tables,
//                 last block computes lambda ranges and the unit plan
//   wide_units    all warp units (one launch per kind in PHASED mode:
//                 the Alg. 3/4 "one launch per DFF, guard lb <= k" shape)
//   wide_final    per-lambda bounds of the sliced accumulators (item-sliced
//                 VB2/FS1 walks, term-sliced CCM1/BJ1 harmonic sums)
//   wide_finish   one warp writes the bplb_result / batch outputs
// With bound pruning (full-collection checks) the units run in two launches:
// the exact seeds, then wide_prefilter (threshold snapshot, VB2 walk chunks
// tested once and compacted into a list) and the pruned rest.
//
// The lookups into the {W, N} records are L2 reads (16 MB at c = 1e6); every
// harmonic loop issues HB iterations' loads before consuming any, so a lane
// keeps 2 HB independent requests in flight instead of one dependent chain.
#pragma once
#include <algorithm>
#include <string>
#include "bplb_node.cuh"
#include "bplb_prune.cuh"

namespace bplb {

constexpr int WT = 256;              // threads per CTA (wide kernels)
constexpr int ISLICE = 1024;         // items per modular tile (2 x 16 per lane)
constexpr int ISLICE_SEED = 256;     // ... for the pruning seeds (short units: they gate the rest)
constexpr int LLW = 128;             // lambdas per lane-lookup unit, MT / RAD2 (4 x 32)
constexpr int LLW_H = 32;            // ... CCM1 / BJ1 (harmonic loop per lane)
constexpr int HSL_TS = 2048;         // harmonic terms per sliced CCM1 / BJ1 unit (64 per lane)
constexpr int WIDE_MAX_SEGS = 64;
enum { T_HSL = 4 };                  // CCM1 / BJ1 lambda with more than HSL_TS terms: term slices
// Bound pruning on the grid-wide path (full-collection checks only): the
// integer envelope of the bplb_prune.cuh upper bounds.
constexpr int64_t WIDE_PRUNE_MAX_C = (int64_t)1 << 20;
constexpr int64_t WIDE_PRUNE_MAX_R = (int64_t)1 << 17;
constexpr int64_t WIDE_MAX_C = (int64_t)1 << 27;
constexpr int SCAN_TILE_MIN = 512;  // entries per scan block (at least)
// Scan tile for n entries: >= 512 and a multiple of WT, with at most ~512
// blocks, so every SM gets work and each block's prefix over the block
// sums before it stays short.
inline int64_t scan_tile(int64_t n) {
    const int64_t t = ((n + 511) / 512 + WT - 1) / WT * WT;
    return t < SCAN_TILE_MIN ? SCAN_TILE_MIN : t;
}


struct WSeg {
    int kind, type;
    int64_t lo, hi;
    int chunk;
    int nslice;       // T_MOD: item slices per lambda chunk; T_HSL: term slices per lambda
    int islice;       // T_MOD: items per slice
    long long first, count;
};

struct WideState {
    NodeStats st;
    int bad;
    int fin_fs1, fin_vb2[3];  // wide_final work: FS1 item-sliced; VB2 item-sliced per part (0, 1, 2)
    int64_t lo[K_COUNT], hi[K_COUNT];
    WSeg segs[WIDE_MAX_SEGS];
    int nseg;
    long long nunits;
    int kind_seg_first[K_COUNT], kind_seg_count[K_COUNT];
    // the fields every warp updates live on their own L2 lines (one line
    // taking every unit's atomics queued the table lookups behind it)
    alignas(256) u64 key[K_COUNT];
    alignas(256) unsigned long long evals[K_COUNT];
    int evaluated[K_COUNT];
    alignas(256) int lb;
    int stop;              // PHASED: set when a completed kind exceeded k
    int n_done;
    alignas(256) long long unit_next;
    alignas(256) int n_vb2;
    alignas(256) int nvlist;  // pruning: surviving VB2 walk chunks
    alignas(256) long long unit_end;
    int scan_blocks_done;
    int prune;             // bound pruning: seeds (units [0, nA)) then the pruned rest
    long long nA;
    u64 thr[K_COUNT];      // per-kind keys after the seeds (VB2 chunk / sliced-lambda decisions)
    int vb2_seg;           // pruning: the VB2 rest segment, enumerated through vlist (-1: none)
    int64_t hsl_hi[K_COUNT];  // CCM1 / BJ1: lambdas [lo, hsl_hi] are term-sliced (T_HSL)
};

struct WideBufs {
    WideState* state;
    ulonglong2* rec;            // [c+2] {W<=(x), N<=(x)} at index x+1 (one 16-byte load)
    unsigned long long* bsum;   // [2 * nblocks] block sums for the scan
    int* vb2;                   // [r]
    unsigned* cnt;              // [c+2] histogram counts (index x+1): zero between checks -- the
                                // scan that consumes them clears them (no 16 MB zeroing pass)
    unsigned long long* acc;    // [c+1] VB2 per-lambda D (indexed by lambda)
    unsigned long long* pz;     // [2*101] FS1 P and Z (indexed by lambda)
    int* vlist;                 // [c/LMOD + 2] pruning: surviving VB2 walk chunks (index from lo)
    unsigned long long* hacc;   // [3 * hn] T_HSL partial sums: CCM1 part, BJ1 floor, BJ1 rem (by lambda)
    int64_t hn;                 // c / HSL_TS + 2
    int64_t tile;               // scan tile (scan_tile(c + 2))
};

inline size_t wide_bytes(int64_t r, int64_t c, int64_t* nblocks_out) {
    int64_t n = c + 2;
    int64_t nb = (n + scan_tile(n) - 1) / scan_tile(n);
    *nblocks_out = nb;
    size_t b = 0;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    b += al(sizeof(WideState));
    b += al((size_t)n * 4);
    b += al((size_t)n * 16);
    b += al((size_t)nb * 16);
    b += al((size_t)std::max<int64_t>(r, 1) * 4);
    b += al((size_t)(c + 1) * 8);
    b += al((size_t)2 * 101 * 8);
    b += al((size_t)(c / LMOD + 2) * 4);
    b += al((size_t)3 * (c / HSL_TS + 2) * 8);
    return b;
}

inline WideBufs wide_carve(void* base, int64_t r, int64_t c) {
    int64_t n = c + 2, nb = (n + scan_tile(n) - 1) / scan_tile(n);
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    char* p = (char*)base;
    WideBufs w;
    w.tile = scan_tile(n);
    w.state = (WideState*)p; p += al(sizeof(WideState));
    w.cnt = (unsigned*)p; p += al((size_t)n * 4);  // right after the state: a fixed offset for every c
    w.rec = (ulonglong2*)p; p += al((size_t)n * 16);
    w.bsum = (unsigned long long*)p; p += al((size_t)nb * 16);
    w.vb2 = (int*)p; p += al((size_t)std::max<int64_t>(r, 1) * 4);
    w.acc = (unsigned long long*)p; p += al((size_t)(c + 1) * 8);
    w.pz = (unsigned long long*)p; p += al((size_t)2 * 101 * 8);
    w.vlist = (int*)p; p += al((size_t)(c / LMOD + 2) * 4);
    w.hn = c / HSL_TS + 2;
    w.hacc = (unsigned long long*)p;
    return w;
}

// -------------------------------------------------------------------------
// acc[acc_lo, acc_lo + acc_n): VB2 accumulators to clear (all of them without
// pruning; with it the seed chunk only -- the prefilter clears the surviving chunks)
__global__ void wide_init(WideBufs b, int64_t c, int64_t acc_lo, int64_t acc_n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t i = i0; i < acc_n; i += stride) b.acc[acc_lo + i] = 0;
    for (int64_t i = i0; i < 2 * 101; i += stride) b.pz[i] = 0;
    for (int64_t i = i0; i < 3 * b.hn; i += stride) b.hacc[i] = 0;
    unsigned int* st = (unsigned int*)b.state;  // zero the state word by word
    for (int64_t i = i0; i < (int64_t)(sizeof(WideState) / 4); i += stride) st[i] = 0u;
}

__global__ void __launch_bounds__(WT) wide_stats(WideBufs b, const int* __restrict__ w, int64_t r,
                                                 int64_t c) {
    int l_max = 0, l_bad = 0, l_s = 0, l_e = 0, l_b = 0, l_f = 0;
    long long l_W = 0, l_Vs = 0, l_Vm = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    // warp-uniform trip count: the VB2 item list is appended one warp
    // allocation at a time (one counter atomic per warp, not per item)
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); i0 < r; i0 += stride) {
        const int64_t i = i0 + lane;
        const int x = i < r ? w[i] : 1;
        const bool ok = i < r && x >= 1 && (int64_t)x <= c;
        if (i < r && !ok) l_bad = 1;
        bool isv = false;
        if (ok) {
            l_max = max(l_max, x);
            l_W += x;
            if (2 * (int64_t)x < c) { l_s++; l_Vs += x; }
            else if (2 * (int64_t)x == c) l_e++;
            else { l_b++; l_Vm += c - x; if (x == c) l_f++; }
            atomicAdd(&b.cnt[x + 1], 1u);
            isv = 2 * (int64_t)x != c && x < c;
        }
        const unsigned m = __ballot_sync(0xffffffffu, isv);
        int pos0 = 0;
        if (lane == 0 && m) pos0 = atomicAdd(&b.state->n_vb2, __popc(m));
        pos0 = __shfl_sync(0xffffffffu, pos0, 0);
        if (isv) b.vb2[pos0 + __popc(m & ((1u << lane) - 1u))] = x;
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
    // block-level reduction first: one set of global atomics per block
    __shared__ int s_i[6];
    __shared__ unsigned long long s_l[3];
    if (threadIdx.x < 6) s_i[threadIdx.x] = 0;
    if (threadIdx.x < 3) s_l[threadIdx.x] = 0;
    __syncthreads();
    if (lane == 0) {
        atomicMax(&s_i[0], l_max);
        atomicOr(&s_i[1], l_bad);
        atomicAdd(&s_i[2], l_s);
        atomicAdd(&s_i[3], l_e);
        atomicAdd(&s_i[4], l_b);
        atomicAdd(&s_i[5], l_f);
        atomicAdd(&s_l[0], (unsigned long long)l_W);
        atomicAdd(&s_l[1], (unsigned long long)l_Vs);
        atomicAdd(&s_l[2], (unsigned long long)l_Vm);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        NodeStats* st = &b.state->st;
        atomicMax(&st->maxw, s_i[0]);
        if (s_i[1]) atomicExch(&b.state->bad, 1);
        if (s_i[2]) atomicAdd(&st->n_small, s_i[2]);
        if (s_i[3]) atomicAdd(&st->n_eq, s_i[3]);
        if (s_i[4]) atomicAdd(&st->n_big, s_i[4]);
        if (s_i[5]) atomicAdd(&st->n_full, s_i[5]);
        atomicAdd((unsigned long long*)&st->W, s_l[0]);
        atomicAdd((unsigned long long*)&st->Vs, s_l[1]);
        atomicAdd((unsigned long long*)&st->Vm, s_l[2]);
    }
}

// Block-level sums of (count, count*(i-1)) over one scan tile.
__device__ __forceinline__ void tile_sums(const unsigned* cnt, int64_t n, int64_t t0, int64_t tile,
                                          unsigned long long* sc, unsigned long long* sw) {
    unsigned long long a = 0, bw = 0;
    for (int64_t i = t0 + threadIdx.x; i < min(n, t0 + tile); i += WT) {
        unsigned long long x = cnt[i];
        a += x;
        bw += x * (unsigned long long)(i - 1);
    }
    *sc = a;
    *sw = bw;
}

__device__ __forceinline__ unsigned long long block_sum_u64(unsigned long long v, unsigned long long* red) {
    v = warp_sum_u64(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    unsigned long long t = 0;
    if (threadIdx.x < 32) {
        t = threadIdx.x < (WT / 32) ? red[threadIdx.x] : 0;
        t = warp_sum_u64(t);
    }
    __syncthreads();
    return t;  // valid in warp 0
}

__global__ void __launch_bounds__(WT) wide_scan_reduce(WideBufs b, int64_t c) {
    __shared__ unsigned long long red[WT / 32];
    const int64_t n = c + 2;
    unsigned long long sc, sw;
    tile_sums(b.cnt, n, (int64_t)blockIdx.x * b.tile, b.tile, &sc, &sw);
    unsigned long long tc = block_sum_u64(sc, red);
    unsigned long long tw = block_sum_u64(sw, red);
    if (threadIdx.x == 0) {
        b.bsum[2 * blockIdx.x] = tc;
        b.bsum[2 * blockIdx.x + 1] = tw;
    }
}

// Every block sums the block totals before it (<= ~512, in parallel), then
// writes its tile with a warp-level scan.
__global__ void __launch_bounds__(WT) wide_scan_apply(WideBufs b, int64_t c) {
    __shared__ unsigned long long carry_c[WT / 32 + 1], carry_w[WT / 32 + 1];
    __shared__ unsigned long long base_c, base_w, red[WT / 32];
    const int64_t n = c + 2;
    {
        unsigned long long a = 0, bw = 0;
        for (int j = threadIdx.x; j < (int)blockIdx.x; j += WT) { a += b.bsum[2 * j]; bw += b.bsum[2 * j + 1]; }
        a = block_sum_u64(a, red);
        bw = block_sum_u64(bw, red);
        if (threadIdx.x == 0) { base_c = a; base_w = bw; }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long rc = base_c, rw = base_w;
    const int64_t t0 = (int64_t)blockIdx.x * b.tile;
    const int64_t t1 = min(n, t0 + b.tile);
    for (int64_t s = t0; s < t1; s += WT) {
        const int64_t i = s + threadIdx.x;
        unsigned long long x = 0;
        if (i < t1) {
            x = b.cnt[i];
            b.cnt[i] = 0u;  // consumed: zero for the next check
        }
        unsigned long long y = x * (unsigned long long)(i - 1);
        // inclusive warp scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long xo = __shfl_up_sync(0xffffffffu, x, o);
            unsigned long long yo = __shfl_up_sync(0xffffffffu, y, o);
            if (lane >= o) { x += xo; y += yo; }
        }
        if (lane == 31) { carry_c[warp + 1] = x; carry_w[warp + 1] = y; }
        __syncthreads();
        if (threadIdx.x == 0) {
            carry_c[0] = 0; carry_w[0] = 0;
            for (int j = 1; j <= WT / 32; ++j) { carry_c[j] += carry_c[j - 1]; carry_w[j] += carry_w[j - 1]; }
        }
        __syncthreads();
        if (i < t1) b.rec[i] = make_ulonglong2(rw + carry_w[warp] + y, rc + carry_c[warp] + x);
        rc += carry_c[WT / 32];
        rw += carry_w[WT / 32];
        __syncthreads();
    }
}

// Lambda ranges and the unit plan (one thread, on a shared-memory copy of
// the state: the plan's read-modify-write chains through global memory were
// dependent L2 round trips).
struct KRange {  // per-kind lambda ranges when use_range (dff_bound_batch; lambda-split checks)
    int64_t lo[K_COUNT], hi[K_COUNT];
};

__device__ void plan_body(WideState* s, int64_t c, int nk, const int* kinds, int use_range, const KRange& rg,
                          int phased, int prune) {
    bplb_stats_finish(&s->st, c);
    s->st.r = s->st.n_small + s->st.n_eq + s->st.n_big;
    for (int kd = 0; kd < K_COUNT; ++kd) {
        int64_t lo, hi;
        bplb_domain(kd, c, &lo, &hi);
        if (kd == K_VB2) hi = bplb_vb2_hi(c, s->st.r, s->st.maxw);
        bool in = false;
        for (int i = 0; i < nk; ++i) in |= kinds[i] == kd;
        if (use_range) { lo = rg.lo[kd]; hi = rg.hi[kd]; }
        if (!in) hi = lo - 1;
        s->lo[kd] = lo;
        s->hi[kd] = hi;
        s->kind_seg_count[kd] = 0;
        s->kind_seg_first[kd] = 0;
        s->hsl_hi[kd] = lo - 1;
    }
    s->nseg = 0;
    s->nunits = 0;
    s->vb2_seg = -1;
    s->nvlist = 0;
    s->fin_fs1 = 0;
    s->fin_vb2[0] = s->fin_vb2[1] = s->fin_vb2[2] = 0;
    if (s->bad) return;
    const NodeStats& st = s->st;
    auto push = [&](int kind, int type, int64_t a, int64_t z, int chunk, int nslice, int islice = 0) {
        if (z < a) return;
        WSeg& g = s->segs[s->nseg++];
        g.kind = kind; g.type = type; g.lo = a; g.hi = z; g.chunk = chunk; g.nslice = nslice; g.islice = islice;
        g.first = s->nunits;
        // 32-bit divisions throughout the plan (lambda ranges <= c <= 2^27,
        // item counts < 2^31): the 64-bit ones were most of its 17 us
        g.count = (long long)((uint32_t)(z - a + chunk) / (uint32_t)chunk) * nslice;
        s->nunits += g.count;
        s->kind_seg_count[kind]++;
    };
    s->prune = prune;
    s->nA = 0;
    // CCM1 / BJ1 segments over [a, z] by the length of the harmonic loop
    // (span / lambda terms, one or two L2 lookups each): term slices of
    // HSL_TS spread over many warps where it is longer than HSL_TS (partial
    // sums per lambda, finished in wide_final), one warp per lambda while it
    // is longer than 64, one lane per lambda after.  The sliced lambdas come
    // in doubling groups so every lambda of a group needs about the group's
    // slice count (the surplus slices of its upper lambdas are empty).
    // types: bit 0 T_HSL, bit 1 T_WLOOK, bit 2 T_LOOKUP (segment order control).
    auto push_div_look = [&](int kd, int64_t a, int64_t z, int types) {
        if (z < a) return;
        const int64_t span = kd == K_CCM1 ? (c - 1) / 2 : (int64_t)st.maxw;
        int64_t sh = span / HSL_TS + 1;
        if (sh < a) sh = a;
        if (sh > z + 1) sh = z + 1;
        int64_t sp = span / 64 + 1;
        if (sp < sh) sp = sh;
        if (sp > z + 1) sp = z + 1;
        if (types & 1) {
            for (int64_t x = a; x < sh;) {
                const int64_t y = min(sh - 1, 2 * x - 1);
                push(kd, T_HSL, x, y, 1, (int)((uint32_t)span / (uint32_t)x / HSL_TS + 1));
                x = y + 1;
            }
            if (sh > a) s->hsl_hi[kd] = sh - 1;
        }
        if (types & 2) push(kd, T_WLOOK, sh, sp - 1, 1, 1);
        if (types & 4) push(kd, T_LOOKUP, sp, z, LLW_H, 1);
    };
    auto push_mod = [&](int kd, int64_t a, int64_t z, int islice) {
        const int64_t items = kd == K_VB2 ? s->n_vb2 : st.r;
        int nsl = (int)((uint32_t)(items + islice - 1) / (uint32_t)islice);
        if (nsl < 1) nsl = 1;
        push(kd, T_MOD, a, z, LMOD, nsl, islice);
        return nsl > 1;
    };
    if (prune) {
        // seeds (units [0, nA)): MT, RAD2 and FS1 complete, VB2's first walk
        // chunk, a CCM1 / BJ1 window at c/4 + 1; then every other lambda,
        // tested against the seeds' keys (bplb_prune.cuh bounds).  The seed
        // walks are cut finer (they gate the rest).
        int64_t w0[K_COUNT], w1[K_COUNT];
        for (int i = 0; i < nk; ++i) {
            const int kd = kinds[i];
            const int64_t lo = s->lo[kd], hi = s->hi[kd];
            s->kind_seg_first[kd] = s->nseg;
            w0[kd] = hi + 1; w1[kd] = hi;
            if (hi < lo) continue;
            switch (kd) {
            case K_MT: case K_RAD2: push(kd, T_LOOKUP, lo, hi, LLW, 1); break;
            case K_FS1: s->fin_fs1 = push_mod(kd, lo, hi, ISLICE_SEED); break;
            case K_VB2: s->fin_vb2[1] = push_mod(kd, lo, min(hi, lo + LMOD - 1), ISLICE_SEED); break;
            default: {
                int64_t a = c / 4 + 1;
                a = a < lo ? lo : (a > hi ? hi : a);
                w0[kd] = a; w1[kd] = min(hi, a + 31);
                push(kd, T_LOOKUP, w0[kd], w1[kd], LLW_H, 1);
            }
            }
        }
        s->nA = s->nunits;
        // the rest, longest units first (claims follow segment order): the
        // VB2 walk chunks, the long per-lane CCM1 / BJ1 loops below the seed
        // window, the term slices, the short loops above it, one warp per
        // lambda last
        for (int pass = 0; pass < 4; ++pass)
            for (int i = 0; i < nk; ++i) {
                const int kd = kinds[i];
                const int64_t lo = s->lo[kd], hi = s->hi[kd];
                if (hi < lo) continue;
                if (kd == K_VB2 && pass == 0 && hi >= lo + LMOD) {
                    s->vb2_seg = s->nseg;  // enumerated through the prefilter's chunk list
                    s->fin_vb2[2] = push_mod(kd, lo + LMOD, hi, ISLICE);
                }
                if (kd == K_CCM1 || kd == K_BJ1) {
                    if (pass == 0) push_div_look(kd, lo, w0[kd] - 1, 4);
                    if (pass == 1) push_div_look(kd, lo, w0[kd] - 1, 1);
                    if (pass == 2) push_div_look(kd, w1[kd] + 1, hi, 7);
                    if (pass == 3) push_div_look(kd, lo, w0[kd] - 1, 2);
                }
            }
        return;
    }
    // Heavy modular units first in concurrent mode (longest-processing-time
    // order); kind order in PHASED / CANCEL mode so cheap early kinds can
    // raise lb before later units start.
    int order[K_COUNT];
    int no = 0;
    if (!phased) {
        for (int i = 0; i < nk; ++i) if (kinds[i] == K_VB2 || kinds[i] == K_FS1) order[no++] = kinds[i];
        for (int i = 0; i < nk; ++i) if (!(kinds[i] == K_VB2 || kinds[i] == K_FS1)) order[no++] = kinds[i];
    } else {
        for (int i = 0; i < nk; ++i) order[no++] = kinds[i];
    }
    for (int i = 0; i < no; ++i) {
        const int kd = order[i];
        const int64_t lo = s->lo[kd], hi = s->hi[kd];
        s->kind_seg_first[kd] = s->nseg;
        if (hi < lo) continue;
        switch (kd) {
        case K_MT: case K_RAD2: push(kd, T_LOOKUP, lo, hi, LLW, 1); break;
        case K_FS1: s->fin_fs1 = push_mod(kd, lo, hi, ISLICE); break;
        case K_VB2: s->fin_vb2[0] = push_mod(kd, lo, hi, ISLICE); break;
        default: push_div_look(kd, lo, hi, 7);
        }
    }
}

constexpr int PLAN_T = 512;  // (the copy in is ~1500 words: a few loads in flight per thread)
__global__ void __launch_bounds__(PLAN_T) wide_plan(WideBufs b, int64_t c, int nk, int use_range, KRange rg,
                                                    int kinds0, int kinds1, int kinds2, int kinds3,
                                                    int kinds4, int kinds5, int phased, int prune) {
    __shared__ WideState ls;
    static_assert(sizeof(WideState) % 4 == 0, "word copy");
    const int nw = (int)(sizeof(WideState) / 4);
    unsigned* g = (unsigned*)b.state;
    unsigned* l = (unsigned*)&ls;
#pragma unroll 4
    for (int i = threadIdx.x; i < nw; i += PLAN_T) l[i] = g[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        const int kinds[K_COUNT] = {kinds0, kinds1, kinds2, kinds3, kinds4, kinds5};
        plan_body(&ls, c, nk, kinds, use_range, rg, phased, prune);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nw; i += PLAN_T) g[i] = l[i];
}

// ---- batched harmonic loops over the global records (LkTableG layout) -------
// rec[x + 1] = {W<=(x), N<=(x)}, rec[0] = {0, 0}; 32-bit value indices
// (c <= WIDE_MAX_C = 2^27, every t * lambda below 2c).  HB iterations' loads
// are issued before any is consumed; lanes past t_end load rec[0].
constexpr int HB_CCM1 = 8;
constexpr int HB_BJ1 = 4;

// CCM1 (bounds.py:390-407): sum over t = t0, t0 + dt, ... <= t_end of
//   base - N(t lam - 1) - N(c - t lam),  base = n_small + r - n_big
// (bplb_ccm1_part with the loads batched).
__device__ __forceinline__ int64_t ccm1_part_g(const ulonglong2* __restrict__ rec, int c, int lam, int t0,
                                               int dt, int t_end, int64_t base) {
    int64_t acc = 0;
    for (int t = t0; t <= t_end; t += HB_CCM1 * dt) {
        unsigned long long a[HB_CCM1], b[HB_CCM1];
#pragma unroll
        for (int j = 0; j < HB_CCM1; ++j) {
            const int tt = t + j * dt;
            const int x = tt <= t_end ? tt * lam : 0;
            a[j] = __ldg(&rec[x].y);                      // N(t lam - 1)
            b[j] = __ldg(&rec[x ? c - x + 1 : 0].y);      // N(c - t lam)
        }
#pragma unroll
        for (int j = 0; j < HB_CCM1; ++j)
            if (t + j * dt <= t_end) acc += base - (int64_t)a[j] - (int64_t)b[j];
    }
    return acc;
}

// BJ1 (bounds.py:441-460): buckets t = t0, t0 + dt, ... <= t_end of
//   rem += W(hi) - W(lo) - lo (N(hi) - N(lo)),  lo = t lam + cm, hi = (t+1) lam - 1
//   fl  += r - N(hi)  for t < tmax
// (bplb_bj1_part with the loads batched; values clamped to c).
__device__ __forceinline__ void bj1_part_g(const ulonglong2* __restrict__ rec, int c, int lam, int cm, int r,
                                           int t0, int dt, int t_end, int tmax, int64_t* fl_out,
                                           int64_t* rem_out) {
    int64_t fl = 0, rem = 0;
    for (int t = t0; t <= t_end; t += HB_BJ1 * dt) {
        ulonglong2 L[HB_BJ1], H[HB_BJ1];
#pragma unroll
        for (int j = 0; j < HB_BJ1; ++j) {
            const int tt = t + j * dt;
            const bool ok = tt <= t_end;
            const int tc = ok ? tt : 0;
            const int lo = tc * lam + cm, hi = (tc + 1) * lam - 1;
            L[j] = __ldg(&rec[ok ? min(lo, c) + 1 : 0]);
            H[j] = __ldg(&rec[ok ? min(hi, c) + 1 : 0]);
        }
#pragma unroll
        for (int j = 0; j < HB_BJ1; ++j) {
            const int tt = t + j * dt;
            if (tt <= t_end) {
                const int64_t lo = (int64_t)tt * lam + cm;
                rem += (int64_t)(H[j].x - L[j].x) - lo * (int64_t)(H[j].y - L[j].y);
                if (tt < tmax) fl += (int64_t)r - (int64_t)H[j].y;
            }
        }
    }
    *fl_out = fl;
    *rem_out = rem;
}

__device__ __forceinline__ int64_t ccm1_sum_g(const ulonglong2* rec, const NodeStats& st, int64_t c, int64_t lam) {
    const int64_t base = (int64_t)st.n_small + st.r - st.n_big;
    const int tmax = (int)(((c - 1) / 2) / lam);
    return bplb_ccm1_from_part(st, c, lam, ccm1_part_g(rec, (int)c, (int)lam, 1, 1, tmax, base));
}

__device__ __forceinline__ int64_t bj1_sum_g(const ulonglong2* rec, const NodeStats& st, int64_t c, int64_t lam) {
    const int L = (int)lam, tmax = st.maxw / L;
    int64_t fl, rem;
    bj1_part_g(rec, (int)c, L, (int)(c % lam), st.r, 0, 1, tmax, tmax, &fl, &rem);
    return bplb_bj1_from_parts(c, lam, fl, rem);
}

// Read-only state of a wide_units launch, copied to shared memory once per
// CTA (the per-unit reads of the global WideState were L2 round trips).
struct WideRO {
    NodeStats st;
    int64_t lo[K_COUNT], hi[K_COUNT], hsl_hi[K_COUNT];
    u64 thr[K_COUNT];
    long long nA;
    int prune, vb2_seg, n_vb2;
};

// One warp unit of the wide path.  segs / si: the block's shared copy of the
// segment table and the warp's forward-only cursor (a warp claims increasing
// unit ids).  cancel_now: the Alg. 4 guard has fired -- unsliced units are
// skipped, sliced ones (partial sums per lambda) still run so no lambda is
// finished from an incomplete sum.
// WarpAcc: the warp's own evals / evaluated / lb / key views (lane 0),
// flushed to the state at the end of the launch.
struct WarpAcc {
    unsigned long long ev[K_COUNT];
    u64 kc[K_COUNT];
    int evd, lb_sent;
};

template <bool WIDE>
__device__ void wide_unit(const KParams& p, WideBufs& b, WideState* s, const WideRO& ro, const LkTableG& lk,
                          const WSeg* segs, int nseg, int& si, long long u, u64* tot, bool cancel_now,
                          WarpAcc& wa) {
    const int lane = threadIdx.x & 31;
    while (si + 1 < nseg && segs[si + 1].first <= u) ++si;
    const WSeg& sg = segs[si];
    if (cancel_now && !(sg.type == T_HSL || (sg.type == T_MOD && sg.nslice > 1))) return;
    const int kind = sg.kind;
    const int64_t c = p.c;
    const NodeStats& st = ro.st;
    const long long rel = u - sg.first;
    int64_t* lam_out = p.lam_out;
    int64_t wmax = -1;
    int64_t n_eval = 0;
    // pruned group (bplb_prune.cuh bounds against the live per-kind keys, read
    // once per unit): skipped lambdas still count as evaluated (they provably
    // cannot change the outputs)
    const bool pruned = ro.prune && u >= ro.nA;
    const int64_t lo_k = ro.lo[kind];
    do {
        if (sg.type == T_LOOKUP) {
            const int64_t lam_a = sg.lo + rel * sg.chunk;
            const int64_t lam_b = min(sg.hi, lam_a + sg.chunk - 1);
            n_eval = lam_b - lam_a + 1;
            bool skip_unit = false;
            Thr th{};
            if (pruned) {
                const u64 kv = *(volatile u64*)&s->key[kind];
                if (lane == 0 && kv > wa.kc[kind]) wa.kc[kind] = kv;
                th = thr_from_key(kv);
                skip_unit = (c / lam_a <= PR_QMAX) ? blk_skip<LkTableG, true>(th, kind, lk, st, c, lo_k, lam_a, lam_b)
                                                   : range_skip(th, kind, st, c, lo_k, lam_a, lam_b);
            }
            for (int64_t l0 = lam_a; l0 <= lam_b && !skip_unit; l0 += 32) {
                const int64_t lam = l0 + lane;
                bool valid = lam <= lam_b;
                if (pruned && valid) valid = !lam_skip<true>(th, kind, st, c, lo_k, lam);
                if (pruned && !__ballot_sync(0xffffffffu, valid)) continue;
                int64_t S = 0;
                if (valid) {
                    switch (kind) {
                    case K_MT: S = bplb_mt_sum(lk, c, st.r, lam); break;
                    case K_RAD2: S = bplb_rad2_sum(lk, c, st.r, lam); break;
                    case K_CCM1: S = ccm1_sum_g(b.rec, st, c, lam); break;
                    default: S = bj1_sum_g(b.rec, st, c, lam); break;
                    }
                }
                int64_t bd = valid ? bplb_bound(S, bplb_fc(kind, c, lam)) : 0;
                int64_t m = emit_warp_cached(valid, lam, bd, lo_k, &s->key[kind], &wa.kc[kind], lam_out, p.out_lo, p.out_hi);
                wmax = m > wmax ? m : wmax;
            }
        } else if (sg.type == T_WLOOK) {
            const int64_t lam = sg.lo + rel;
            n_eval = 1;
            if (pruned && lam_skip<true>(thr_from_key(*(volatile u64*)&s->key[kind]), kind, st, c, lo_k, lam)) break;
            const int L = (int)lam;
            int64_t S;
            if (kind == K_CCM1) {
                const int64_t base = (int64_t)st.n_small + st.r - st.n_big;
                int64_t part = ccm1_part_g(b.rec, (int)c, L, 1 + lane, 32, (int)(((c - 1) / 2) / lam), base);
                part = (int64_t)warp_sum_u64((u64)part);
                S = bplb_ccm1_from_part(st, c, lam, part);
            } else {
                const int tmax = st.maxw / L;
                int64_t fl, rem;
                bj1_part_g(b.rec, (int)c, L, (int)(c % lam), st.r, lane, 32, tmax, tmax, &fl, &rem);
                fl = (int64_t)warp_sum_u64((u64)fl);
                rem = (int64_t)warp_sum_u64((u64)rem);
                S = bplb_bj1_from_parts(c, lam, fl, rem);
            }
            const int64_t bd = bplb_bound(S, bplb_fc(kind, c, lam));
            wmax = emit_warp_cached(lane == 0, lam, bd, lo_k, &s->key[kind], &wa.kc[kind], lam_out, p.out_lo, p.out_hi);
        } else if (sg.type == T_HSL) {
            // one term slice of one lambda: partial sums into hacc (wide_final);
            // with pruning the decision uses the post-seed snapshot, identical
            // in every slice and in wide_final
            const int64_t lam = sg.lo + rel / sg.nslice;
            const int slice = (int)(rel % sg.nslice);
            n_eval = slice == 0 ? 1 : 0;
            if (ro.prune && lam_skip<true>(thr_from_key(ro.thr[kind]), kind, st, c, lo_k, lam)) break;
            const int L = (int)lam;
            if (kind == K_CCM1) {
                const int tmax = (int)(((c - 1) / 2) / lam);
                const int ta = 1 + slice * HSL_TS, tb = min(tmax, ta + HSL_TS - 1);
                if (ta > tb) break;
                const int64_t base = (int64_t)st.n_small + st.r - st.n_big;
                const u64 part = warp_sum_u64((u64)ccm1_part_g(b.rec, (int)c, L, ta + lane, 32, tb, base));
                if (lane == 0) atomicAdd(&b.hacc[lam], part);
            } else {
                const int tmax = st.maxw / L;
                const int ta = slice * HSL_TS, tb = min(tmax, ta + HSL_TS - 1);
                if (ta > tb) break;
                int64_t fl, rem;
                bj1_part_g(b.rec, (int)c, L, (int)(c % lam), st.r, ta + lane, 32, tb, tmax, &fl, &rem);
                const u64 f = warp_sum_u64((u64)fl), m = warp_sum_u64((u64)rem);
                if (lane == 0) {
                    atomicAdd(&b.hacc[b.hn + lam], f);
                    atomicAdd(&b.hacc[2 * b.hn + lam], m);
                }
            }
        } else {  // T_MOD
            const long long chunk = rel / sg.nslice;
            const int slice = (int)(rel % sg.nslice);
            // the pruned VB2 rest: only the chunks the prefilter kept (its evals
            // were counted there)
            const bool listed = ro.prune && si == ro.vb2_seg;
            const int64_t lam_a = listed ? lo_k + (int64_t)b.vlist[chunk] * LMOD : sg.lo + chunk * sg.chunk;
            const int64_t lam_b = min(sg.hi, lam_a + sg.chunk - 1);
            const int L = (int)(lam_b - lam_a + 1);
            const int n_items = kind == K_VB2 ? ro.n_vb2 : st.r;
            const int* items = kind == K_VB2 ? b.vb2 : p.w;
            const int i0 = slice * sg.islice, i1 = min(n_items, i0 + sg.islice);
            const int warp = threadIdx.x >> 5;
            u64* t = tot + warp * LMOD;
            for (int j = lane; j < LMOD; j += kWarp) t[j] = 0;
            __syncwarp();
            const uint32_t c32 = (uint32_t)c;
            const u64 cinv = bplb_cinv(c32);
            mod_walk<WIDE>(items, i0, i1, c32, cinv, lam_a, L, t, p.one, kind == K_VB2);
            __syncwarp();
            if (sg.nslice > 1) {
                for (int j = lane; j < L; j += kWarp) {
                    if (kind == K_VB2) atomicAdd(&b.acc[lam_a + j], t[j]);
                    else atomicAdd(&b.pz[lam_a + j], t[j]);
                }
                n_eval = (slice == 0 && !listed) ? L : 0;  // count each lambda once
            } else {
                n_eval = listed ? 0 : L;
                for (int j0 = 0; j0 < L; j0 += kWarp) {
                    const int j = j0 + lane;
                    const bool valid = j < L;
                    const int64_t lam = lam_a + j;
                    int64_t S = 0;
                    if (valid)
                        S = (kind == K_VB2) ? bplb_vb2_sum(st, c, lam, t[j])
                                            : bplb_fs1_sum(st, lam, t[j], (uint64_t)bplb_fs1_zero(lk, c, st.maxw, lam));
                    int64_t bd = valid ? bplb_bound(S, bplb_fc(kind, c, lam)) : 0;
                    int64_t m = emit_warp_cached(valid, lam, bd, lo_k, &s->key[kind], &wa.kc[kind], lam_out, p.out_lo, p.out_hi);
                    wmax = m > wmax ? m : wmax;
                }
            }
        }
    } while (0);
    if (lane == 0) {
        wa.ev[kind] += (unsigned long long)n_eval;
        wa.evd |= 1 << kind;
        if (wmax > wa.lb_sent) {  // lb: the Alg. 4 guard reads it live
            atomicMax(&s->lb, (int)wmax);
            wa.lb_sent = (int)wmax;
        }
    }
}

#ifdef WIDE_TRACE
// Per-unit trace (development builds only: scripts/wide_trace.py builds
// libbplb_wtrace.so with -DWIDE_TRACE):
// {seg | part << 8 | smid << 16 | kind << 32 | type << 40, unit - seg.first, t0, t1}.
constexpr int WIDE_TRACE_CAP = 1 << 18;
__device__ longlong4 g_wide_trace[WIDE_TRACE_CAP];
__device__ int g_wide_trace_n;
#endif

// Persistent warp-unit kernel.  phase_kind >= 0 restricts to that kind's
// segments (PHASED mode) and applies the Alg. 4 entry guard lb <= k.
#ifndef WIDE_MINB
#define WIDE_MINB 3  // resident wide_units CTAs per SM the register budget is sized for
#endif
template <bool WIDE>
__global__ void __launch_bounds__(WT, WIDE_MINB) wide_units(KParams p, WideBufs b, int phase_kind, int part) {
    __shared__ u64 tot[(WT / 32) * LMOD];
    __shared__ WSeg segs[WIDE_MAX_SEGS];
    __shared__ WideRO ro;
    __shared__ WarpAcc wacc[WT / 32];
    __shared__ long long u_begin, u_end;
    __shared__ int skip, nseg;
    WideState* s = b.state;
    if (threadIdx.x == 0) {
        skip = 0;
        nseg = s->nseg;
        ro.st = s->st;
        for (int kd = 0; kd < K_COUNT; ++kd) {
            ro.lo[kd] = s->lo[kd];
            ro.hi[kd] = s->hi[kd];
            ro.hsl_hi[kd] = s->hsl_hi[kd];
            ro.thr[kd] = s->thr[kd];
        }
        ro.nA = s->nA;
        ro.prune = s->prune;
        ro.vb2_seg = s->vb2_seg;
        ro.n_vb2 = s->n_vb2;
        if (s->bad) skip = 1;
        if (phase_kind >= 0) {
            if (s->stop) skip = 1;
            const int f = s->kind_seg_first[phase_kind], n = s->kind_seg_count[phase_kind];
            u_begin = n ? s->segs[f].first : 0;
            u_end = n ? s->segs[f + n - 1].first + s->segs[f + n - 1].count : 0;
        } else if (part == 1) {  // pruning: the seeds
            u_begin = 0;
            u_end = s->nA;
        } else if (part == 2) {  // pruning: the rest
            u_begin = s->nA;
            u_end = s->nunits;
        } else {
            u_begin = 0;
            u_end = s->nunits;
        }
    }
    __syncthreads();
    if (skip) return;
    for (int i = threadIdx.x; i < nseg; i += WT) segs[i] = s->segs[i];
    __syncthreads();
    if (part == 2 && threadIdx.x == 0 && ro.vb2_seg >= 0) {  // the pruned VB2 rest: the prefilter's list
        const int v = ro.vb2_seg;
        segs[v].count = (long long)s->nvlist * segs[v].nslice;
        for (int j = v + 1; j < nseg; ++j) segs[j].first = segs[j - 1].first + segs[j - 1].count;
        u_end = segs[nseg - 1].first + segs[nseg - 1].count;
    }
    __syncthreads();
    const LkTableG lk{b.rec, p.c};
    const bool cancel = (p.flags & BPLB_F_CANCEL) && phase_kind < 0;
    const int lane = threadIdx.x & 31;
    int si = 0;
    WarpAcc& wa = wacc[threadIdx.x >> 5];
    if (lane < K_COUNT) {
        wa.ev[lane] = 0;
        wa.kc[lane] = 0;
    }
    if (lane == 0) {
        wa.evd = 0;
        wa.lb_sent = -1;
    }
    __syncwarp();
    // unit claims one ahead: the next claim's atomic is in flight while the
    // current unit runs (a warp's claims still increase)
    long long u_nx = 0;
    if (lane == 0) u_nx = u_begin + atomicAdd((unsigned long long*)&s->unit_next, 1ull);
    for (;;) {
        const long long u = __shfl_sync(0xffffffffu, u_nx, 0);
        if (u >= u_end) break;
        if (lane == 0) u_nx = u_begin + atomicAdd((unsigned long long*)&s->unit_next, 1ull);
        const bool cancel_now = cancel && (int64_t)(*(volatile int*)&s->lb) > p.k;  // Alg. 4 guard
#ifdef WIDE_TRACE
        long long t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#endif
        wide_unit<WIDE>(p, b, s, ro, lk, segs, nseg, si, u, tot, cancel_now, wa);
        __syncwarp();
#ifdef WIDE_TRACE
        if (lane == 0) {
            long long t1;
            unsigned sm;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            const int i = atomicAdd(&g_wide_trace_n, 1);
            if (i < WIDE_TRACE_CAP)
                g_wide_trace[i] = make_longlong4((long long)si | ((long long)part << 8) | ((long long)sm << 16) |
                                                     ((long long)segs[si].kind << 32) |
                                                     ((long long)segs[si].type << 40),
                                                 u - segs[si].first, t0, t1);
        }
        __syncwarp();
#endif
    }
    __syncwarp();
    if (lane < K_COUNT) {
        if (wa.ev[lane]) atomicAdd(&s->evals[lane], wa.ev[lane]);
        if (wa.evd >> lane & 1) s->evaluated[lane] = 1;
    }
}

// Pruning, between the seeds and the rest: snapshot the per-kind keys, reset
// the unit counter, test every VB2 walk chunk of the rest once against the
// keys (the range relaxation the units used to apply per slice) and append
// the survivors to vlist (any order); each wide_units CTA of the rest then
// resizes the VB2 segment to the list in its shared copy of the plan.
constexpr int PF_T = 256;
__global__ void __launch_bounds__(PF_T) wide_prefilter(KParams p, WideBufs b) {
    WideState* s = b.state;
    const int si = s->vb2_seg;
    if (blockIdx.x == 0) {
        if (threadIdx.x < K_COUNT) s->thr[threadIdx.x] = s->key[threadIdx.x];
        if (threadIdx.x == 0) s->unit_next = 0;
    }
    if (s->bad || si < 0) return;
    const WSeg g = s->segs[si];
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // every lambda of the rest is accounted here
        atomicAdd(&s->evals[K_VB2], (unsigned long long)(g.hi - g.lo + 1));
        s->evaluated[K_VB2] = 1;
    }
    const int64_t c = p.c, lo_k = s->lo[K_VB2];
    const Thr th = thr_from_key(s->key[K_VB2]);  // no unit runs now: the keys are final for this step
    const NodeStats st = s->st;
    const int64_t nch = (g.hi - g.lo + LMOD) / LMOD;
    const int64_t first = (g.lo - lo_k) / LMOD;
    const int lane = threadIdx.x & 31;
    for (int64_t c0 = (int64_t)blockIdx.x * PF_T + (threadIdx.x & ~31); c0 < nch; c0 += (int64_t)gridDim.x * PF_T) {
        const int64_t ch = c0 + lane;
        const int64_t la = g.lo + ch * LMOD;
        const bool keep = ch < nch && !range_skip(th, K_VB2, st, c, lo_k, la, min(g.hi, la + LMOD - 1));
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        int pos = 0;
        if (lane == 0 && m) pos = atomicAdd(&s->nvlist, __popc(m));
        pos = __shfl_sync(0xffffffffu, pos, 0);
        if (keep) {
            b.vlist[pos + __popc(m & ((1u << lane) - 1u))] = (int)(first + ch);
            for (int j = 0; j < LMOD && la + j <= g.hi; ++j) b.acc[la + j] = 0;  // (wide_init: the seed chunk only)
        }
    }
}

// Reset the unit counter between phased launches and record the kind.
__global__ void wide_phase_begin(WideBufs b, int idx) {
    WideState* s = b.state;
    s->unit_next = 0;
    if (!s->stop) s->n_done = idx + 1;
}

// Per-lambda bounds of the sliced accumulators: FS1 / VB2 walks cut into
// item slices (acc / pz) and CCM1 / BJ1 harmonic sums cut into term slices
// (hacc).  part 0: no pruning (everything); part 1: after the seeds (FS1,
// the first VB2 chunk); part 2: after the pruned rest (the listed VB2
// chunks, the sliced CCM1 / BJ1 lambdas the snapshot did not skip).
__global__ void __launch_bounds__(WT) wide_final(KParams p, WideBufs b, int only_kind, int part) {
    WideState* s = b.state;
    if (s->bad) return;
    if (only_kind >= 0 && s->stop) return;
    __shared__ NodeStats sst;
    if (threadIdx.x == 0) sst = s->st;
    __syncthreads();
    const int64_t c = p.c;
    const NodeStats& st = sst;
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t j_first = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31);
    int64_t wmax = -1;
    // one warp-uniform sweep over n lambdas: lam(j) (-1: not evaluated), sum(lam)
    auto sweep = [&](int kd, int64_t n, auto lam_of, auto sum_of) {
        for (int64_t j0 = j_first; j0 < n; j0 += stride) {
            const int64_t j = j0 + lane;
            const int64_t lam = j < n ? lam_of(j) : -1;
            const bool valid = lam >= 0;
            const int64_t S = valid ? sum_of(lam) : 0;
            const int64_t bd = valid ? bplb_bound(S, bplb_fc(kd, c, lam)) : 0;
            const int64_t m = emit_warp(valid, lam, bd, s->lo[kd], &s->key[kd], p.lam_out, p.out_lo, p.out_hi);
            wmax = m > wmax ? m : wmax;
        }
    };
    auto want = [&](int kd) { return (only_kind < 0 || only_kind == kd) && s->hi[kd] >= s->lo[kd]; };
    if (want(K_FS1) && part != 2 && s->fin_fs1) {
        // one warp per lambda: Z = sum over the multiples v of m = c / gcd(c,
        // lambda + 1) of W(v) - W(v-1), split over the lanes (<= maxw / m terms)
        const int64_t lo = s->lo[K_FS1], n = s->hi[K_FS1] - lo + 1;
        const int64_t nwarps = stride / 32;
        for (int64_t j = j_first / 32; j < n; j += nwarps) {
            const int64_t lam = lo + j;
            const int64_t m = c / bplb_gcd(c, lam + 1);
            long long z = 0;
            for (int64_t v = m * (1 + lane); v <= st.maxw; v += 32 * m) {
                const ulonglong2 h = __ldg(&b.rec[v + 1]), l = __ldg(&b.rec[v]);
                z += (long long)(h.x - l.x);
            }
            z = (long long)warp_sum_u64((u64)z);
            const int64_t S = bplb_fs1_sum(st, lam, b.pz[lam], (uint64_t)z);
            const int64_t bd = bplb_bound(S, bplb_fc(K_FS1, c, lam));
            const int64_t mm = emit_warp(lane == 0, lam, bd, lo, &s->key[K_FS1], p.lam_out, p.out_lo, p.out_hi);
            wmax = mm > wmax ? mm : wmax;
        }
    }
    if (want(K_VB2) && s->fin_vb2[part]) {
        const int64_t lo = s->lo[K_VB2], hi = s->hi[K_VB2];
        auto vsum = [&](int64_t lam) { return bplb_vb2_sum(st, c, lam, b.acc[lam]); };
        if (part == 0) sweep(K_VB2, hi - lo + 1, [&](int64_t j) { return lo + j; }, vsum);
        else if (part == 1) sweep(K_VB2, min(hi, lo + LMOD - 1) - lo + 1, [&](int64_t j) { return lo + j; }, vsum);
        else
            sweep(K_VB2, (int64_t)s->nvlist * LMOD,
                  [&](int64_t j) {
                      const int64_t lam = lo + (int64_t)b.vlist[j / LMOD] * LMOD + j % LMOD;
                      return lam <= hi ? lam : (int64_t)-1;
                  },
                  vsum);
    }
    if (part != 1) {
        const int hk[2] = {K_CCM1, K_BJ1};
        for (int i = 0; i < 2; ++i) {
            const int kd = hk[i];
            if (!want(kd) || s->hsl_hi[kd] < s->lo[kd]) continue;
            const int64_t lo = s->lo[kd];
            const Thr th = thr_from_key(s->thr[kd]);
            sweep(kd, s->hsl_hi[kd] - lo + 1,
                  [&](int64_t j) {
                      const int64_t lam = lo + j;
                      return (s->prune && lam_skip<true>(th, kd, st, c, lo, lam)) ? (int64_t)-1 : lam;
                  },
                  [&](int64_t lam) {
                      return kd == K_CCM1
                                 ? bplb_ccm1_from_part(st, c, lam, (int64_t)b.hacc[lam])
                                 : bplb_bj1_from_parts(c, lam, (int64_t)b.hacc[b.hn + lam],
                                                       (int64_t)b.hacc[2 * b.hn + lam]);
                  });
        }
    }
    if (lane == 0 && wmax >= 0) atomicMax(&s->lb, (int)wmax);
}

// After each phased kind: stop further kinds once lb > k (bounds.py:523-525).
__global__ void wide_phase_end(WideBufs b, int64_t k) {
    WideState* s = b.state;
    if ((int64_t)s->lb > k) s->stop = 1;
}

__global__ void wide_finish(KParams p, WideBufs b, int phased) {
    if (threadIdx.x != 0) return;
    WideState* s = b.state;
    if (s->bad && p.err_out) atomicExch(p.err_out, 1);
    bplb_result res;
    int64_t lb = 0;
    for (int kd = 0; kd < K_COUNT; ++kd) {
        const u64 key = s->key[kd];
        const bool ev = s->evaluated[kd];
        res.best[kd] = ev ? (int64_t)(key >> 32) : 0;
        res.arg_lambda[kd] = ev ? s->lo[kd] + (int64_t)(0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFu)) : s->lo[kd];
        res.n_lambda[kd] = s->hi[kd] >= s->lo[kd] ? s->hi[kd] - s->lo[kd] + 1 : 0;
        res.evals[kd] = (int64_t)s->evals[kd];
        res.evaluated[kd] = ev;
        if (ev && res.best[kd] > lb) lb = res.best[kd];
    }
    res.lb = lb;
    res.exceeded = lb > p.k;
    res.n_done = phased ? s->n_done : p.nk;
    int64_t et = 0;
    for (int kd = 0; kd < K_COUNT; ++kd) et += res.evals[kd];
    res.evals_total = et;
    if (p.res_out) p.res_out[0] = res;
    if (p.lb_out) p.lb_out[0] = lb;
    if (p.ex_out) p.ex_out[0] = (uint8_t)(lb > p.k);
    if (p.best_out) for (int kd = 0; kd < K_COUNT; ++kd) p.best_out[kd] = res.best[kd];
    if (p.arg_out) for (int kd = 0; kd < K_COUNT; ++kd) p.arg_out[kd] = res.arg_lambda[kd];
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
inline std::string& wide_err_ref() {
    static thread_local std::string e;
    return e;
}
inline const std::string& wide_error() { return wide_err_ref(); }

// Work heuristic: the grid-wide path pays ~8 launches; use it when the node
// does not fit the node-resident kernel or when one CTA would take longer
// than a few tens of microseconds (canonical cells > ~2e6).
inline bool wide_preferred(int64_t r, int64_t c) {
    const bool table = c <= TABLE_MAX_C;
    if (r > (table ? 16384 : 8192)) return true;
    const int64_t cells = r * (3 * c);  // ~ sum of lambda ranges x items
    return cells > 2000000 && c <= WIDE_MAX_C;
}

// cnt_zero: how many leading histogram counts of *buf are known to be zero
// (the engine's; the scan keeps [0, c + 2) zero after every check).
inline int wide_check(cudaStream_t st, int num_sms, void** buf, size_t* cap, int64_t* launches,
                      const KParams& p0, int64_t r, int64_t* cnt_zero) {
    KParams p = p0;
    const int64_t c = p.c;
    if (c > WIDE_MAX_C) {
        wide_err_ref() = "capacity above the grid-wide envelope (2^27) for this instance size";
        return BPLB_ERANGE;
    }
    int64_t nb;
    const size_t need = wide_bytes(r, c, &nb);
    if (need > *cap) {
        if (*buf) cudaFree(*buf);
        *buf = nullptr;
        *cap = 0;
        if (cudaMalloc(buf, need) != cudaSuccess) {
            wide_err_ref() = "cudaMalloc failed (wide path)";
            return BPLB_ENOMEM;
        }
        *cap = need;
        *cnt_zero = 0;
    }
    WideBufs b = wide_carve(*buf, r, c);
    if (*cnt_zero < c + 2 &&
        cudaMemsetAsync(b.cnt + *cnt_zero, 0, (size_t)(c + 2 - *cnt_zero) * 4, st) != cudaSuccess) {
        wide_err_ref() = "cudaMemsetAsync failed (wide path)";
        return BPLB_ECUDA;
    }
    *cnt_zero = c + 2;  // (the bytes past it may hold other arrays of this layout)
    const bool phased = p.flags & BPLB_F_PHASED;
    int ks[K_COUNT] = {0, 0, 0, 0, 0, 0};
    for (int i = 0; i < p.nk; ++i) ks[i] = p.kinds[i];
    KRange rg;
    for (int kd = 0; kd < K_COUNT; ++kd) {
        rg.lo[kd] = p.use_range ? p.rng_lo[kd] : 0;
        rg.hi[kd] = p.use_range ? p.rng_hi[kd] : -1;
    }
    // bound pruning: full-collection checks (no per-lambda output) inside the
    // integer envelope of the bplb_prune.cuh bounds
    // (per-kind ranges without per-lambda output -- a lambda-split slice -- prune too)
    const bool prune = !phased && !(p.flags & (BPLB_F_CANCEL | BPLB_F_NOPRUNE)) && !p.lam_out &&
                       c <= WIDE_PRUNE_MAX_C && r <= WIDE_PRUNE_MAX_R;
    const int64_t acc_lo = prune ? std::min<int64_t>(std::max<int64_t>(rg.lo[K_VB2], 0), c) : 0;
    const int64_t acc_n = prune ? std::min<int64_t>(c + 1 - acc_lo, LMOD + 2) : c + 1;
    const int g_init = (int)std::min<int64_t>((acc_n + WT - 1) / WT, (int64_t)num_sms * 8);
    wide_init<<<std::max(g_init, 1), WT, 0, st>>>(b, c, acc_lo, acc_n);
    const int g_stats = (int)std::max<int64_t>(1, std::min<int64_t>((r + WT - 1) / WT, (int64_t)num_sms * 4));
    wide_stats<<<g_stats, WT, 0, st>>>(b, p.w, r, c);
    wide_scan_reduce<<<(unsigned)nb, WT, 0, st>>>(b, c);
    wide_scan_apply<<<(unsigned)nb, WT, 0, st>>>(b, c);
    wide_plan<<<1, PLAN_T, 0, st>>>(b, c, p.nk, p.use_range, rg, ks[0], ks[1], ks[2], ks[3], ks[4], ks[5],
                                    (phased || (p.flags & BPLB_F_CANCEL)) ? 1 : 0, prune ? 1 : 0);
    *launches += 5;
    int per_sm = 0;
    const bool wide = c >= (1 << 23);
    auto units = wide ? wide_units<true> : wide_units<false>;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, units, WT, 0);
    if (per_sm < 1) per_sm = 1;
    const int grid = per_sm * num_sms;
    const int g_fin = num_sms * 2;
    if (prune) {
        units<<<grid, WT, 0, st>>>(p, b, -1, 1);
        wide_final<<<g_fin, WT, 0, st>>>(p, b, -1, 1);
        wide_prefilter<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((c / LMOD + PF_T) / PF_T, num_sms)), PF_T, 0,
                         st>>>(p, b);
        units<<<grid, WT, 0, st>>>(p, b, -1, 2);
        wide_final<<<g_fin, WT, 0, st>>>(p, b, -1, 2);
        *launches += 5;
    } else if (phased) {
        for (int i = 0; i < p.nk; ++i) {
            wide_phase_begin<<<1, 1, 0, st>>>(b, i);
            units<<<grid, WT, 0, st>>>(p, b, p.kinds[i], 0);
            wide_final<<<g_fin, WT, 0, st>>>(p, b, p.kinds[i], 0);
            wide_phase_end<<<1, 1, 0, st>>>(b, p.k);
            *launches += 4;
        }
    } else {
        units<<<grid, WT, 0, st>>>(p, b, -1, 0);
        wide_final<<<g_fin, WT, 0, st>>>(p, b, -1, 0);
        *launches += 2;
    }
    wide_finish<<<1, 32, 0, st>>>(p, b, phased ? 1 : 0);
    *launches += 1;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        wide_err_ref() = std::string("wide path launch: ") + cudaGetErrorString(e);
        return BPLB_ECUDA;
    }
    return 0;
}

}  // namespace bplb
