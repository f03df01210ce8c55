// bplb_tc.cuh -- the batched small-capacity contraction on the 5th-generation
// tensor cores (tcgen05, kind::i8, accumulators in TMEM).
//
// The table path (bplb_tab.cuh) evaluates, for every search node and every
// (kind, lambda) column of the collection, S = sum_w hist[w] * T[col][w] with
// T[col][w] = f_kind(w, c, lambda) (bounds.py:155-206, 276-290, 463-501).
// Here one CTA owns 128 nodes (the MMA M dimension) and produces their whole
// result in one launch:
//   1. the nodes' weight histograms are counted in shared memory (u32) and
//      split into two unsigned byte planes, A_lo = count & 255 and
//      A_hi = count >> 8, stored K-major in the UMMA core-matrix layout
//      (8 rows x 16 bytes per core matrix; LBO = 128 B along K, SBO = KT/16 x
//      128 B between 8-row groups, no swizzle);
//   2. the cached table is laid out the same way per N-tile of 144 columns in
//      two byte planes T_lo, T_hi (T <= 101c < 2^16), one bulk copy per tile;
//   3. one thread issues, per 32-wide K step, four tcgen05.mma.kind::i8 (u8 x
//      u8 -> s32) into three TMEM accumulators: D1 = A_lo T_lo,
//      D2 = A_lo T_hi + A_hi T_lo, D3 = A_hi T_hi, so
//      S = D1 + 256 D2 + 65536 D3 exactly (integer MMA: no rounding at all);
//      a slice whose counts are all < 256 (A_hi = 0) issues only the two
//      A_lo products;
//   4. every thread reads its node's row of D1..D3 (tcgen05.ld, TMEM lane =
//      node), applies the exact ceil-div / key epilogue of the table path
//      (key = bound << 9 | 511 - lambda) and keeps the per-kind maxima in
//      registers; after the last N-tile it writes the node's outputs with the
//      table path's mode replay (tab_node_emit: full / PHASED / CANCEL).
// TMEM: 512 columns (3 x 144 used) per CTA, one CTA per SM (shared memory).
#pragma once
#include "bplb_tab.cuh"

namespace bplb {

constexpr int TC_M = 128;         // nodes per CTA (MMA M, TMEM lanes)
constexpr int TC_NT = 144;        // table columns per N-tile (MMA N)
constexpr int TC_THREADS = 512;   // 16 warps: warp w reads TMEM lanes 32(w%4).. and column group w/4
constexpr int TC_CG = TC_NT / 4;  // epilogue columns per warp (36 = 9 x 4)
constexpr uint32_t TC_TMEM_COLS = 512;

struct TcDev {
    const uint8_t* B;    // [nnt][2 planes][TC_NT x KT] core-matrix layout
    const int4* meta;    // [nnt][TC_NT] epilogue constants (TabDev meta; padding kind 6)
    int KT;              // K extent: c rounded up to 32
    int nnt;             // N-tiles
    int rows;            // nodes per CTA (<= TC_M; the batch spread over every SM)
};

__host__ __device__ inline size_t tc_a_bytes(int KT) { return (size_t)2 * TC_M * KT; }
__host__ __device__ inline size_t tc_b_bytes(int KT) { return (size_t)2 * TC_NT * KT; }
// counts rows padded to KT + 1 words: the conversion reads a column of rows
// (stride KT + 1, odd) without bank conflicts
__host__ __device__ inline size_t tc_cnt_bytes(int KT) { return (size_t)TC_M * (KT + 1) * 4; }
// dynamic smem: A planes | max(counts, B planes + meta) | barriers
__host__ __device__ inline size_t tc_smem_bytes(int KT) {
    size_t x = tc_cnt_bytes(KT), y = tc_b_bytes(KT) + (size_t)TC_NT * 16;
    return tc_a_bytes(KT) + (x > y ? x : y) + 64;
}

// byte offset of (row, k) in a K-major u8 operand with KT columns
__host__ __device__ inline uint32_t tc_core_off(int row, int k, int KT) {
    return (uint32_t)((row >> 3) * (KT / 16) * 128 + (k >> 4) * 128 + (row & 7) * 16 + (k & 15));
}

// Table planes from the cached fp32 table (exact integers < 2^16).
__global__ void tc_build_kernel(uint8_t* Bq, int4* metaq, const float* T, const int4* meta, int KV, int nsub,
                                int KT, int nnt, int c) {
    const int ncols = nsub * TAB_SUB;
    const int64_t n = (int64_t)nnt * TC_NT * KT;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(i % KT);
        const int64_t rj = i / KT;
        const int row = (int)(rj % TC_NT);
        const int nt = (int)(rj / TC_NT);
        const int j = nt * TC_NT + row;
        int v = 0;
        if (j < ncols && k < c) v = (int)T[(size_t)(j / TAB_SUB) * (KV + 2) * TAB_SUB + (size_t)k * TAB_SUB + (j % TAB_SUB)];
        uint8_t* base = Bq + (size_t)nt * 2 * TC_NT * KT;
        const uint32_t off = tc_core_off(row, k, KT);
        base[off] = (uint8_t)(v & 255);
        base[(size_t)TC_NT * KT + off] = (uint8_t)(v >> 8);
        if (k == 0)
            metaq[nt * TC_NT + row] = j < ncols ? meta[j]
                                                : int4{(int)0x80000000u, (int)(0u - 0x96000000u), 0, K_COUNT << 16};
    }
}

__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr, int KT) {
    const uint32_t lbo = 128, sbo = (uint32_t)(KT / 16) * 128;
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version 1 (sm_100); base offset 0, SWIZZLE_NONE
    return d;
}

// kind::i8 instruction descriptor: D s32, A / B unsigned 8-bit, both K-major
__host__ __device__ constexpr uint32_t tc_idesc(int M, int N) {
    return (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void tc_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}

__device__ __forceinline__ void tc_ld4(uint32_t taddr, uint32_t (&v)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(taddr));
}

template <int WB>
__device__ __forceinline__ int tc_load_w(const void* w, int64_t i) {
    if (WB == 1) return (int)__ldg((const uint8_t*)w + i);
    if (WB == 2) return (int)__ldg((const uint16_t*)w + i);
    return __ldg((const int*)w + i);
}

#ifdef TC_TRACE
__device__ unsigned long long g_tc_trace[64];  // CTA 0: globaltimer at the phase boundaries
__device__ unsigned long long g_tc_cta[256][3];  // every CTA: start, histogram done, end
#define TC_CTA(i)                                                                              \
    do {                                                                                       \
        if (threadIdx.x == 0 && blockIdx.x < 256) {                                            \
            unsigned long long t_;                                                             \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                             \
            g_tc_cta[blockIdx.x][i] = t_;                                                      \
        }                                                                                      \
    } while (0)
#define TC_STAMP(i)                                                                            \
    do {                                                                                       \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                                             \
            unsigned long long t_;                                                             \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                             \
            g_tc_trace[i] = t_;                                                                \
        }                                                                                      \
    } while (0)
#else
#define TC_STAMP(i) do {} while (0)
#define TC_CTA(i) do {} while (0)
#endif

// Shared memory: A planes | X = counts, then B buffer 0 + meta 0 | (DB) B
// buffer 1 + meta 1 | barriers.  DB (double-buffered table tiles) when it fits.
__host__ __device__ inline size_t tc_bm_bytes(int KT) { return tc_b_bytes(KT) + (size_t)TC_NT * 16; }
__host__ __device__ inline size_t tc_x_bytes(int KT) {
    return tc_cnt_bytes(KT) > tc_bm_bytes(KT) ? tc_cnt_bytes(KT) : tc_bm_bytes(KT);
}
__host__ __device__ inline size_t tc_smem_bytes_db(int KT, bool db) {
    return tc_a_bytes(KT) + tc_x_bytes(KT) + (db ? tc_bm_bytes(KT) : 0) + 64;
}

// One thread: both bulk copies of N-tile nt (planes + column constants) into
// buffer (B, M), completing on bar.
__device__ __forceinline__ void tc_load_tile(const TcDev& t, int nt, uint8_t* B, int4* M, unsigned long long* bar) {
    const unsigned bb = (unsigned)tc_b_bytes(t.KT);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tab_smem_addr(bar)),
                 "r"(bb + (unsigned)(TC_NT * 16))
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     tab_smem_addr(B)),
                 "l"(t.B + (size_t)nt * bb), "r"(bb), "r"(tab_smem_addr(bar))
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     tab_smem_addr(M)),
                 "l"(t.meta + (size_t)nt * TC_NT), "r"((unsigned)(TC_NT * 16)), "r"(tab_smem_addr(bar))
                 : "memory");
}

// One CTA per SM-sized slice of the batch (t.rows <= 128 nodes: the MMA's
// M = 128 rows, the rows past the slice are zero): the histograms -- the
// part bound by shared-memory atomics -- spread over every SM.
template <int WB, bool DB>
__global__ void __launch_bounds__(TC_THREADS, 1) tc_kernel(KParams p, TcDev t) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint32_t s_tmem;
    __shared__ int s_bad, s_hi;
    __shared__ unsigned kbest[TC_M][K_COUNT];  // per-node per-kind best keys
    constexpr int rank = 0, nstep = 1;  // every N-tile in this CTA
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int KT = t.KT;
    uint8_t* As = smem;                                  // [2][TC_M x KT]
    unsigned char* X = smem + tc_a_bytes(KT);            // counts, then B buffer 0
    uint32_t* cnt = (uint32_t*)X;                        // [TC_M][KT + 1]
    const int KP = KT + 1;
    uint8_t* Bbuf[2];
    int4* Mbuf[2];
    Bbuf[0] = X;
    Mbuf[0] = (int4*)(X + tc_b_bytes(KT));
    Bbuf[1] = DB ? X + tc_x_bytes(KT) : Bbuf[0];
    Mbuf[1] = DB ? (int4*)(Bbuf[1] + tc_b_bytes(KT)) : Mbuf[0];
    unsigned long long* bars = (unsigned long long*)(X + tc_x_bytes(KT) + (DB ? tc_bm_bytes(KT) : 0));
    // bars: [0], [1] tile buffer landed, [2] MMAs done
    const int64_t n0 = p.node0 + (int64_t)blockIdx.x * t.rows;
    const int64_t rem = p.node0 + p.n_nodes - n0;
    const int nn = (int)(rem < t.rows ? rem : t.rows);
    const int c = (int)p.c;
    TC_STAMP(0);
    TC_CTA(0);

    if (tid == 0) {
        s_bad = 0;
        s_hi = 0;
        tab_bar_init(&bars[0]);
        tab_bar_init(&bars[1]);
        tab_bar_init(&bars[2]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {  // TMEM: 512 columns (the CTA owns the SM)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tab_smem_addr(&s_tmem)),
                     "n"(TC_TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // ---- 1. histograms (u32 counts), validated weights ------------------------
    for (int i = tid; i < TC_M * KP; i += TC_THREADS) cnt[i] = 0u;
    for (int i = tid; i < TC_M * K_COUNT; i += TC_THREADS) (&kbest[0][0])[i] = 0u;
    __syncthreads();
    // the second tile of this CTA lands in buffer 1 while the histograms are counted
    if (DB && tid == 0 && rank + nstep < t.nnt) tc_load_tile(t, rank + nstep, Bbuf[1], Mbuf[1], &bars[1]);
    bool bad = false;
    if (WB == 1) {
        // groups of four nodes per warp: each lane loads four aligned 4-byte
        // words of each node (16 loads in flight), then counts the bytes
        // inside the node's range
        const uint32_t* w32 = (const uint32_t*)p.w;
        for (int g0 = warp; g0 < nn; g0 += 4 * (TC_THREADS / 32)) {
            int64_t a[4], b[4], wa[4], wb[4];
            int64_t words = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int r = g0 + q * (TC_THREADS / 32);
                const bool v = r < nn;
                a[q] = v ? p.off[n0 + r] : 0;
                b[q] = v ? p.off[n0 + r + 1] : 0;
                wa[q] = a[q] >> 2;
                wb[q] = b[q] > a[q] ? (b[q] + 3) >> 2 : wa[q];
                words = max(words, wb[q] - wa[q]);
            }
            for (int64_t j0 = 0; j0 < words; j0 += 4 * 32) {
                uint32_t v[4][4];
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int64_t j = wa[q] + j0 + u * 32 + lane;
                        v[q][u] = j < wb[q] ? __ldg(w32 + j) : 0u;
                    }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    uint32_t* row = cnt + (g0 + q * (TC_THREADS / 32)) * KP;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int64_t j = wa[q] + j0 + u * 32 + lane;
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int64_t i = 4 * j + e;
                            if (i < a[q] || i >= b[q]) continue;
                            const int x = (int)((v[q][u] >> (8 * e)) & 255u);
                            if (x < 1 || x > c) { bad = true; continue; }
                            atomicAdd(row + x - 1, 1u);
                        }
                    }
                }
            }
        }
    } else {
        for (int r = warp; r < nn; r += TC_THREADS / 32) {
            const int64_t a = p.off[n0 + r], b = p.off[n0 + r + 1];
            uint32_t* row = cnt + r * KP;
            for (int64_t i0 = a; i0 < b; i0 += 4 * 32) {  // four loads in flight per lane
                int x[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int64_t i = i0 + u * 32 + lane;
                    x[u] = i < b ? tc_load_w<WB>(p.w, i) : -1;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (x[u] == -1) continue;
                    if (x[u] < 1 || x[u] > c) { bad = true; continue; }
                    atomicAdd(row + x[u] - 1, 1u);
                }
            }
        }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) s_bad = 1;
    __syncthreads();
    TC_STAMP(1);
    TC_CTA(1);
    // ---- A planes: row tid % 128, a quarter of its 16-byte core rows -----------
    {
        const int arow = tid & (TC_M - 1), part = tid >> 7;
        const uint32_t* row = cnt + arow * KP;
        for (int kc = part; kc < KT / 16; kc += TC_THREADS / TC_M) {
            uint32_t lo[4], hi[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t l = 0, h = 0;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const uint32_t v = row[kc * 16 + q * 4 + e];  // < 2^16 (r <= 65535)
                    l |= (v & 255u) << (8 * e);
                    h |= (v >> 8) << (8 * e);
                }
                lo[q] = l;
                hi[q] = h;
            }
            const uint32_t off = tc_core_off(arow, kc * 16, KT);
            *(uint4*)(As + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
            *(uint4*)(As + (size_t)TC_M * KT + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
            if (hi[0] | hi[1] | hi[2] | hi[3]) s_hi = 1;  // a count >= 256 somewhere
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // A planes -> tensor core (async proxy)
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();  // the counts are consumed: buffer 0 may be overwritten
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (tid == 0 && rank < t.nnt) tc_load_tile(t, rank, Bbuf[0], Mbuf[0], &bars[0]);
    TC_STAMP(2);
    const uint32_t tmem = s_tmem;
    const uint32_t idesc = tc_idesc(TC_M, TC_NT);
    const uint32_t a_lo = tab_smem_addr(As), a_hi = tab_smem_addr(As + (size_t)TC_M * KT);
    const bool hiA = s_hi != 0;  // uniform: read after the barrier that follows the conversion
    unsigned best[K_COUNT] = {0u, 0u, 0u, 0u, 0u, 0u};
    int it = 0;
    for (int nt = rank; nt < t.nnt; nt += nstep, ++it) {
        const int bi = DB ? (it & 1) : 0;
        uint8_t* Bs = Bbuf[bi];
        int4* Ms = Mbuf[bi];
        if (!DB && it > 0 && tid == 0) tc_load_tile(t, nt, Bs, Ms, &bars[0]);
        // ---- 2. this tile's planes in smem -----------------------------------------
        tab_bar_wait(&bars[bi], DB ? ((it >> 1) & 1) : (it & 1));
        TC_STAMP(3 + 4 * it);
        // ---- 3. MMAs (one thread) -----------------------------------------------
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t b_lo = tab_smem_addr(Bs), b_hi = tab_smem_addr(Bs + (size_t)TC_NT * KT);
            for (int ks = 0; ks < KT / 32; ++ks) {
                const uint32_t ko = (uint32_t)ks * 256;  // two 16-byte core matrices along K
                const uint64_t dAl = tc_desc(a_lo + ko, KT), dAh = tc_desc(a_hi + ko, KT);
                const uint64_t dBl = tc_desc(b_lo + ko, KT), dBh = tc_desc(b_hi + ko, KT);
                tc_mma(tmem, dAl, dBl, idesc, ks > 0);
                tc_mma(tmem + TC_NT, dAl, dBh, idesc, ks > 0);
                if (hiA) {  // counts >= 256 in this slice: the A_hi plane's two products
                    tc_mma(tmem + TC_NT, dAh, dBl, idesc, 1);
                    tc_mma(tmem + 2 * TC_NT, dAh, dBh, idesc, ks > 0);
                }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             tab_smem_addr(&bars[2]))
                         : "memory");
        }
        tab_bar_wait(&bars[2], it & 1);
        TC_STAMP(4 + 4 * it);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // ---- 4. epilogue: warp w: rows 32(w%4).., columns [36 (w/4), +36) --------
        const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        const int cg0 = (warp >> 2) * TC_CG;
        if ((warp & 3) * 32 < nn) {  // a warp whose 32 TMEM lanes hold no node skips
        // three rounds (16 + 16 + 4 columns), one tcgen05.wait::ld each; the
        // per-kind maxima through a running (kind, max) flushed at kind changes
        int cur_kind = -1;
        unsigned cur = 0u;
        auto fold = [&](const uint32_t* d1, const uint32_t* d2, const uint32_t* d3, int c0, int ncol) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                if (j >= ncol) break;
                const int4 m = Ms[c0 + j];
                const unsigned S = d1[j] + (d2[j] << 8) + (d3[j] << 16);        // exact, < 2^23
                const unsigned n2 = 2u * S + (unsigned)m.y + 2u * 0x4B000000u;  // 2 (S + F - 1)
                const unsigned q = __umulhi(n2, (unsigned)m.x) >> m.z;
                const unsigned key = (q << 9) | (unsigned)(m.w & 0xffff);
                const int kind = m.w >> 16;
                if (kind != cur_kind) {
#pragma unroll
                    for (int x = 0; x < K_COUNT; ++x)
                        if (x == cur_kind) best[x] = max(best[x], cur);
                    cur_kind = kind;
                    cur = 0u;
                }
                cur = max(cur, key);
            }
        };
#pragma unroll 1
        for (int r = 0; r < 2; ++r) {
            uint32_t d1[16], d2[16], d3[16];
            const int c0 = cg0 + 16 * r;
            tc_ld16(lane_base + c0, d1);
            tc_ld16(lane_base + TC_NT + c0, d2);
            if (hiA) tc_ld16(lane_base + 2 * TC_NT + c0, d3);
            else
#pragma unroll
                for (int j = 0; j < 16; ++j) d3[j] = 0u;
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            fold(d1, d2, d3, c0, 16);
        }
        {
            uint32_t d1[4], d2[4], d3[4];
            const int c0 = cg0 + 32;
            tc_ld4(lane_base + c0, d1);
            tc_ld4(lane_base + TC_NT + c0, d2);
            if (hiA) tc_ld4(lane_base + 2 * TC_NT + c0, d3);
            else
#pragma unroll
                for (int j = 0; j < 4; ++j) d3[j] = 0u;
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            uint32_t e1[16], e2[16], e3[16];
#pragma unroll
            for (int j = 0; j < 4; ++j) { e1[j] = d1[j]; e2[j] = d2[j]; e3[j] = d3[j]; }
            fold(e1, e2, e3, c0, 4);
        }
#pragma unroll
        for (int x = 0; x < K_COUNT; ++x)
            if (x == cur_kind) best[x] = max(best[x], cur);
        }
        // the next tile's MMAs overwrite TMEM (and, single-buffered, its copy Bs / Ms)
        TC_STAMP(5 + 4 * it);
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        TC_STAMP(6 + 4 * it);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // the MMAs and the epilogue are done with this buffer (planes and column
        // constants): the tile after next lands in it during the next tile
        if (DB && tid == 0 && nt + 2 * nstep < t.nnt) tc_load_tile(t, nt + 2 * nstep, Bs, Ms, &bars[bi]);
    }
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TC_TMEM_COLS));
    {
        const int row = (warp & 3) * 32 + lane;
#pragma unroll
        for (int x = 0; x < K_COUNT; ++x)
            if (best[x]) atomicMax(&kbest[row][x], best[x]);
    }
    __syncthreads();
    TC_STAMP(40);
    if (s_bad && tid == 0 && p.err_out) atomicExch(p.err_out, 1);
    if (tid < nn) {
        unsigned kk[K_COUNT];
#pragma unroll
        for (int x = 0; x < K_COUNT; ++x) kk[x] = kbest[tid][x];
        tab_node_emit(p, kk, n0 + tid);
    }
    TC_STAMP(41);
    TC_CTA(2);
}

}  // namespace bplb
