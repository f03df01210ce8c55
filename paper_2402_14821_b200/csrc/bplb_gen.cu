// bplb_gen.cu -- synthetic search-node generator (workload data, NOT the
// bound path): libbplb_gen.so.  The same generator runs on the host (for the
// CPU oracle / baselines and golden fixtures) and on the device (for the
// 10^6-node batches of BASELINE cfg5), producing identical nodes.
//
// Node g of stream `seed` (SURVEY.md 8(d), cfg2 / cfg5 "search-node states"):
//   draw depth d ~ U{0..n}; the d heaviest items (stable by index) are each
//   committed to a uniformly random bin among those with load + w <= c, or
//   stay open when no bin fits; the reduced instance is the open weights in
//   item order followed by the positive bin loads in bin order -- the layout
//   of reduce_packing (reference instances.py:262-282).
// Randomness: a splitmix64 stream per node keyed by (seed, g), so any node
// range is generated independently (ranks generate only their own shard).
#include <cuda_runtime.h>
#include <stdint.h>
#include <cub/cub.cuh>
#include <algorithm>
#include <thread>
#include <vector>

#define GEN_API extern "C" __attribute__((visibility("default")))
#define GEN_HD __host__ __device__ __forceinline__

namespace {

constexpr int GEN_MAX_BINS = 1024;
constexpr int GEN_MAX_ITEMS = 2048;
constexpr int GEN_WARPS = 4;  // nodes per CTA on the device (one warp each)

GEN_HD uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
struct Rng {
    uint64_t s;
    GEN_HD explicit Rng(uint64_t seed, int64_t node)
        : s(mix64(seed * 0x632BE59BD9B4E019ull + 0x9E3779B97F4A7C15ull) ^ mix64((uint64_t)node + 0x5851F42D4C957F2Dull)) {}
    GEN_HD uint32_t next() {
        s += 0x9E3779B97F4A7C15ull;
        return (uint32_t)(mix64(s) >> 32);
    }
    GEN_HD uint32_t below(uint32_t m) { return (uint32_t)(((uint64_t)next() * m) >> 32); }  // U{0..m-1}
};

// Host reference of one node: returns r; writes weights / assignment when given.
int gen_node_host(const int32_t* w, int n, const int32_t* order, int64_t c, int k, uint64_t seed, int64_t g,
                  int32_t* out, uint16_t* assign, std::vector<int64_t>& load, std::vector<int32_t>& bin) {
    Rng rng(seed, g);
    const int d = (int)rng.below((uint32_t)n + 1);
    std::fill(load.begin(), load.begin() + k, 0);
    std::fill(bin.begin(), bin.begin() + n, -1);
    for (int i = 0; i < d; ++i) {
        const int it = order[i];
        const int64_t wi = w[it];
        int cnt = 0;
        for (int j = 0; j < k; ++j) cnt += load[j] + wi <= c;
        const uint32_t pick = rng.below((uint32_t)(cnt > 0 ? cnt : 1));
        if (cnt == 0) continue;
        int seen = 0;
        for (int j = 0; j < k; ++j) {
            if (load[j] + wi <= c) {
                if ((uint32_t)seen == pick) { load[j] += wi; bin[it] = j; break; }
                ++seen;
            }
        }
    }
    int r = 0;
    for (int i = 0; i < n; ++i)
        if (bin[i] < 0) { if (out) out[r] = w[i]; ++r; }
    for (int j = 0; j < k; ++j)
        if (load[j] > 0) { if (out) out[r] = (int32_t)load[j]; ++r; }
    if (assign)
        for (int i = 0; i < n; ++i) assign[i] = bin[i] < 0 ? 0xFFFF : (uint16_t)bin[i];
    return r;
}

// Device: one warp per node; bin loads and item->bin in shared memory.
// fill == false: r per node into off[g + 1]; fill == true: weights at off[g].
template <bool FILL>
__global__ void __launch_bounds__(GEN_WARPS * 32) gen_kernel(const int32_t* __restrict__ w, int n,
                                                             const int32_t* __restrict__ order, int64_t c, int k,
                                                             uint64_t seed, int64_t node0, int64_t n_nodes,
                                                             int64_t* off, int32_t* wout, uint16_t* assign) {
    __shared__ int32_t s_load[GEN_WARPS][GEN_MAX_BINS];  // loads <= c < 2^31
    __shared__ int16_t s_bin[GEN_WARPS][GEN_MAX_ITEMS];
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    int32_t* load = s_load[wp];
    int16_t* bin = s_bin[wp];
    for (int64_t g = (int64_t)blockIdx.x * GEN_WARPS + wp; g < n_nodes; g += (int64_t)gridDim.x * GEN_WARPS) {
        Rng rng(seed, node0 + g);
        const int d = (int)rng.below((uint32_t)n + 1);
        for (int j = lane; j < k; j += 32) load[j] = 0;
        for (int i = lane; i < n; i += 32) bin[i] = -1;
        __syncwarp();
        for (int i = 0; i < d; ++i) {
            const int it = __ldg(order + i);
            const int64_t wi = __ldg(w + it);
            int cnt = 0;
            for (int j0 = 0; j0 < k; j0 += 32) {
                const int j = j0 + lane;
                cnt += __popc(__ballot_sync(0xffffffffu, j < k && (int64_t)load[j] + wi <= c));
            }
            const uint32_t pick = rng.below((uint32_t)(cnt > 0 ? cnt : 1));
            if (cnt == 0) continue;
            int seen = 0;
            for (int j0 = 0; j0 < k; j0 += 32) {
                const int j = j0 + lane;
                const unsigned m = __ballot_sync(0xffffffffu, j < k && (int64_t)load[j] + wi <= c);
                const int pc = __popc(m);
                if ((uint32_t)(seen + pc) > pick) {
                    const int b = j0 + __fns(m, 0, (int)(pick - seen) + 1);
                    if (lane == 0) { load[b] += (int32_t)wi; bin[it] = (int16_t)b; }
                    break;
                }
                seen += pc;
            }
            __syncwarp();
        }
        // reduced instance: open items in item order, then positive loads in bin order
        int base = 0;
        int64_t o = FILL ? off[g] : 0;
        for (int i0 = 0; i0 < n; i0 += 32) {
            const int i = i0 + lane;
            const bool open = i < n && bin[i] < 0;
            const unsigned m = __ballot_sync(0xffffffffu, open);
            if (FILL && open) wout[o + base + __popc(m & ((1u << lane) - 1))] = __ldg(w + i);
            if (FILL && assign && i < n) assign[g * n + i] = bin[i] < 0 ? 0xFFFF : (uint16_t)bin[i];
            base += __popc(m);
        }
        for (int j0 = 0; j0 < k; j0 += 32) {
            const int j = j0 + lane;
            const bool pos = j < k && load[j] > 0;
            const unsigned m = __ballot_sync(0xffffffffu, pos);
            if (FILL && pos) wout[o + base + __popc(m & ((1u << lane) - 1))] = (int32_t)load[j];
            base += __popc(m);
        }
        if (!FILL && lane == 0) off[g + 1] = base;
        __syncwarp();
    }
}

}  // namespace

// Host generation of nodes [node0, node0 + n_nodes): off_out[n_nodes + 1]
// always; w_out (sized off_out[n_nodes]) and assign_out (n_nodes * n uint16,
// 0xFFFF = open) when non-null.  order = item indices by weight descending,
// stable.  Returns 0, or -1 on bad arguments.
GEN_API int bplbgen_nodes_host(const int32_t* w, int32_t n, const int32_t* order, int64_t c, int32_t k,
                               uint64_t seed, int64_t node0, int64_t n_nodes, int64_t* off_out, int32_t* w_out,
                               uint16_t* assign_out, int32_t nthreads) {
    if (n < 0 || n > GEN_MAX_ITEMS || k < 1 || k > GEN_MAX_BINS || n_nodes < 0 || !off_out) return -1;
    if (nthreads < 1) nthreads = 1;
    off_out[0] = 0;
    auto run = [&](bool fill) {
        std::vector<std::thread> th;
        for (int t = 0; t < nthreads; ++t)
            th.emplace_back([&, t] {
                std::vector<int64_t> load(k);
                std::vector<int32_t> bin(std::max(n, 1));
                for (int64_t g = t; g < n_nodes; g += nthreads) {
                    if (!fill) off_out[g + 1] = gen_node_host(w, n, order, c, k, seed, node0 + g, nullptr, nullptr, load, bin);
                    else gen_node_host(w, n, order, c, k, seed, node0 + g, w_out + off_out[g],
                                       assign_out ? assign_out + g * (int64_t)n : nullptr, load, bin);
                }
            });
        for (auto& x : th) x.join();
    };
    run(false);
    for (int64_t g = 0; g < n_nodes; ++g) off_out[g + 1] += off_out[g];
    if (w_out || assign_out) {
        if (!w_out) return -1;
        run(true);
    }
    return 0;
}

// Device generation, step 1: d_off[n_nodes + 1] (inclusive prefix of r,
// d_off[0] = 0).  Step 2 (bplbgen_fill_device): weights into d_wout (sized
// d_off[n_nodes]) and optionally the assignments.  d_w / d_order are device
// arrays.  Asynchronous on `stream`; returns 0 or a cudaError_t.
GEN_API int bplbgen_sizes_device(const int32_t* d_w, int32_t n, const int32_t* d_order, int64_t c, int32_t k,
                                 uint64_t seed, int64_t node0, int64_t n_nodes, int64_t* d_off, void* stream) {
    if (n < 0 || n > GEN_MAX_ITEMS || k < 1 || k > GEN_MAX_BINS || n_nodes < 0) return -1;
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(d_off, 0, 8, s);
    if (n_nodes == 0) return (int)cudaGetLastError();
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)std::min<int64_t>((n_nodes + GEN_WARPS - 1) / GEN_WARPS, (int64_t)sms * 16);
    gen_kernel<false><<<grid, GEN_WARPS * 32, 0, s>>>(d_w, n, d_order, c, k, seed, node0, n_nodes, d_off, nullptr,
                                                      nullptr);
    size_t tmp = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tmp, d_off + 1, d_off + 1, n_nodes, s);
    void* d_tmp = nullptr;
    if (cudaMallocAsync(&d_tmp, tmp, s) != cudaSuccess) return (int)cudaGetLastError();
    cub::DeviceScan::InclusiveSum(d_tmp, tmp, d_off + 1, d_off + 1, n_nodes, s);
    cudaFreeAsync(d_tmp, s);
    return (int)cudaGetLastError();
}

GEN_API int bplbgen_fill_device(const int32_t* d_w, int32_t n, const int32_t* d_order, int64_t c, int32_t k,
                                uint64_t seed, int64_t node0, int64_t n_nodes, const int64_t* d_off,
                                int32_t* d_wout, uint16_t* d_assign, void* stream) {
    if (n < 0 || n > GEN_MAX_ITEMS || k < 1 || k > GEN_MAX_BINS || n_nodes < 0) return -1;
    if (n_nodes == 0) return 0;
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)std::min<int64_t>((n_nodes + GEN_WARPS - 1) / GEN_WARPS, (int64_t)sms * 16);
    gen_kernel<true><<<grid, GEN_WARPS * 32, 0, s>>>(d_w, n, d_order, c, k, seed, node0, n_nodes,
                                                     const_cast<int64_t*>(d_off), d_wout, d_assign);
    return (int)cudaGetLastError();
}
