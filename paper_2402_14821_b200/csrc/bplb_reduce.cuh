// bplb_reduce.cuh -- device-side reduction of search-node states (SURVEY.md
// 8(f)1): the reference's reduce_packing (instances.py:262-282) for a whole
// batch of partial packings at once.
//
// A node state is the bin assignment of every item of the instance,
// assign[node][i] = committed bin of item i, or OPEN (all ones of the
// element type) while the item's domain still has several bins.  The
// reduced instance keeps the open items' weights in item order, then one
// virtual item per bin with a positive committed load, in bin order; a load
// above the capacity fails the reduction (ValueError).  Three launches:
//   reduce_count_kernel  one warp per node: bin loads in smem, r = #open +
//                        #positive bins, validation
//   reduce_scan_kernel   offsets = exclusive prefix sum of r (one CTA)
//   reduce_write_kernel  one warp per node: order-preserving compaction of
//                        the open weights (ballot/popc), then the loads
// The CSR it writes (uint8 / uint16 / int32 weights by capacity) feeds the
// batched bound kernels unchanged.
#pragma once
#include <cstdint>

namespace bplb {

constexpr int RED_NT = 256;          // 8 warps, one node each
constexpr int RED_MAX_BINS = 2048;   // smem loads per warp (u64): 8 x 16 KB

struct ReduceArgs {
    const int* w;            // instance weights [n_items]
    const void* assign;      // [n_nodes][n_items], element abytes (1 or 2), OPEN = all ones
    int abytes;
    int64_t n_items, n_bins, n_nodes;
    int64_t c;
    int64_t* r;              // [n_nodes] reduced sizes (count pass) / offsets [n_nodes + 1] (scan)
    void* out_w;             // reduced weights, element obytes
    int obytes;
    int* err;                // 1: load > c, 2: bin id out of range
    unsigned long long* max_r;
};

__device__ __forceinline__ unsigned red_assign(const ReduceArgs& a, int64_t idx) {
    return a.abytes == 1 ? (unsigned)__ldg((const unsigned char*)a.assign + idx)
                         : (unsigned)__ldg((const unsigned short*)a.assign + idx);
}

// Bin loads of one node into the warp's smem slice; returns #open items.
__device__ __forceinline__ int red_loads(const ReduceArgs& a, int64_t node, unsigned long long* loads, int* bad) {
    const int lane = threadIdx.x & 31;
    const unsigned open = a.abytes == 1 ? 0xffu : 0xffffu;
    const int nb = (int)a.n_bins;
    for (int j = lane; j < nb; j += 32) loads[j] = 0ull;
    __syncwarp();
    int n_open = 0;
    const int64_t base = node * a.n_items;
    for (int64_t i = lane; i < a.n_items; i += 32) {
        const unsigned b = red_assign(a, base + i);
        if (b == open) ++n_open;
        else if (b >= (unsigned)nb) *bad |= 2;
        else atomicAdd(&loads[b], (unsigned long long)__ldg(a.w + i));
    }
    __syncwarp();
    return n_open;
}

__global__ void __launch_bounds__(RED_NT) reduce_count_kernel(ReduceArgs a) {
    extern __shared__ unsigned long long red_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long* loads = red_smem + warp * a.n_bins;
    for (int64_t node = (int64_t)blockIdx.x * (RED_NT / 32) + warp; node < a.n_nodes;
         node += (int64_t)gridDim.x * (RED_NT / 32)) {
        int bad = 0;
        int cnt = red_loads(a, node, loads, &bad);
        for (int j = lane; j < (int)a.n_bins; j += 32) {
            const unsigned long long ld = loads[j];
            if (ld > (unsigned long long)a.c) bad |= 1;  // reduce_packing: committed load exceeds capacity
            cnt += ld > 0ull;
        }
        cnt = __reduce_add_sync(0xffffffffu, cnt);
        bad = (int)__reduce_or_sync(0xffffffffu, (unsigned)bad);
        if (lane == 0) {
            a.r[node] = cnt;
            atomicMax(a.max_r, (unsigned long long)cnt);
            if (bad) atomicOr(a.err, bad);
        }
        __syncwarp();
    }
}

// In place: r[0..n) -> offsets[0..n] (offsets[n] = total), one CTA of 1024.
__global__ void __launch_bounds__(1024) reduce_scan_kernel(int64_t* r, int64_t n) {
    __shared__ int64_t part[1024];
    const int t = threadIdx.x;
    const int64_t per = (n + 1023) / 1024;
    const int64_t lo = min(n, t * per), hi = min(n, lo + per);
    int64_t s = 0;
    for (int64_t i = lo; i < hi; ++i) s += r[i];
    part[t] = s;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {  // Hillis-Steele inclusive scan
        const int64_t v = t >= o ? part[t - o] : 0;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    int64_t run = part[t] - s;  // exclusive prefix of this segment
    for (int64_t i = lo; i < hi; ++i) {
        const int64_t x = r[i];
        r[i] = run;
        run += x;
    }
    if (t == 1023) r[n] = part[1023];
}

__device__ __forceinline__ void red_store(const ReduceArgs& a, int64_t idx, unsigned v) {
    if (a.obytes == 1) ((unsigned char*)a.out_w)[idx] = (unsigned char)v;
    else if (a.obytes == 2) ((unsigned short*)a.out_w)[idx] = (unsigned short)v;
    else ((int*)a.out_w)[idx] = (int)v;
}

__global__ void __launch_bounds__(RED_NT) reduce_write_kernel(ReduceArgs a) {
    extern __shared__ unsigned long long red_smem[];
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned open = a.abytes == 1 ? 0xffu : 0xffffu;
    unsigned long long* loads = red_smem + warp * a.n_bins;
    for (int64_t node = (int64_t)blockIdx.x * (RED_NT / 32) + warp; node < a.n_nodes;
         node += (int64_t)gridDim.x * (RED_NT / 32)) {
        int bad = 0;
        red_loads(a, node, loads, &bad);
        int64_t pos = a.r[node];
        const int64_t base = node * a.n_items;
        // open items, in item order
        for (int64_t i0 = 0; i0 < a.n_items; i0 += 32) {
            const int64_t i = i0 + lane;
            const bool take = i < a.n_items && red_assign(a, base + i) == open;
            const unsigned m = __ballot_sync(FULL, take);
            if (take) red_store(a, pos + __popc(m & lt), (unsigned)__ldg(a.w + i));
            pos += __popc(m);
        }
        // positive committed loads, in bin order
        for (int j0 = 0; j0 < (int)a.n_bins; j0 += 32) {
            const int j = j0 + lane;
            const unsigned long long ld = j < (int)a.n_bins ? loads[j] : 0ull;  // <= c (checked)
            const unsigned m = __ballot_sync(FULL, ld > 0ull);
            if (ld > 0ull) red_store(a, pos + __popc(m & lt), (unsigned)ld);
            pos += __popc(m);
        }
        __syncwarp();
    }
}

}  // namespace bplb
