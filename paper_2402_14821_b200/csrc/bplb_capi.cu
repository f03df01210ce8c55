// bplb_capi.cu -- the C ABI of libbplb.so (include/bplb.h): engine lifetime,
// host<->device staging, kernel selection and launch.  No torch types; the
// Python host side binds these symbols with ctypes
// (paper_2402_14821_b200/_native.py).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <algorithm>

#include "../../include/bplb.h"
#include "bplb_core.h"
#include "bplb_node.cuh"
#include "bplb_prune.cuh"
#include "bplb_wide.cuh"
#include "bplb_warp.cuh"
#include "bplb_tab.cuh"
#include "bplb_tc.cuh"
#include "bplb_reduce.cuh"
#include "bplb_knap.cuh"
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                   \
    do {                                                                                 \
        cudaError_t e_ = (expr);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return fail(BPLB_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

constexpr int64_t NODE_R_MAX_SORT = 8192;
constexpr int64_t NODE_R_MAX_TABLE = 16384;

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    int grow(size_t bytes) {
        if (bytes <= cap) return 0;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t n = std::max<size_t>(bytes, 256);
        if (cudaMalloc(&p, n) != cudaSuccess) return fail(BPLB_ENOMEM, "cudaMalloc failed");
        cap = n;
        return 0;
    }
    void release() { if (p) cudaFree(p); p = nullptr; cap = 0; }
};

struct HostBuf {
    void* p = nullptr;
    size_t cap = 0;
    int grow(size_t bytes) {
        if (bytes <= cap) return 0;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        size_t n = std::max<size_t>(bytes, 4096);
        if (cudaMallocHost(&p, n) != cudaSuccess) return fail(BPLB_ENOMEM, "cudaMallocHost failed");
        cap = n;
        return 0;
    }
    void release() { if (p) cudaFreeHost(p); p = nullptr; cap = 0; }
};

// Pinned host memory mapped into the device address space: the single-check
// kernel reads its weights and writes its result through it (no separate
// copy operations on the stream for a few hundred bytes each way).
struct MappedBuf {
    void* h = nullptr;
    void* d = nullptr;
    size_t cap = 0;
    int grow(size_t bytes) {
        if (bytes <= cap) return 0;
        if (h) cudaFreeHost(h);
        h = d = nullptr;
        cap = 0;
        size_t n = std::max<size_t>(bytes, 4096);
        if (cudaHostAlloc(&h, n, cudaHostAllocMapped) != cudaSuccess) return fail(BPLB_ENOMEM, "cudaHostAlloc failed");
        if (cudaHostGetDevicePointer(&d, h, 0) != cudaSuccess) return fail(BPLB_ECUDA, "cudaHostGetDevicePointer failed");
        cap = n;
        return 0;
    }
    void release() { if (h) cudaFreeHost(h); h = d = nullptr; cap = 0; }
};

// Device address of a pinned (page-locked, UVA-mapped) host buffer, or null:
// kernels write batch outputs straight into such buffers, so the call needs
// no device-to-host copies.
void* device_alias(const void* ptr) {
    if (!ptr) return nullptr;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

bool is_pinned(const void* ptr) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// Host copy into / out of the pinned staging buffers, split over a few
// threads when large (one memcpy stream moves ~6 GB/s on these hosts).
void host_copy(void* dst, const void* src, size_t bytes) {
    constexpr size_t PAR_MIN = (size_t)4 << 20;
    if (bytes < PAR_MIN) {
        std::memcpy(dst, src, bytes);
        return;
    }
    const int nt = (int)std::min<size_t>(8, bytes / (PAR_MIN / 4));
    const size_t chunk = (bytes + nt - 1) / nt;
    std::vector<std::thread> th;
    for (int i = 1; i < nt; ++i) {
        const size_t a = i * chunk, b = std::min(bytes, a + chunk);
        if (a < b) th.emplace_back([=] { std::memcpy((char*)dst + a, (const char*)src + a, b - a); });
    }
    std::memcpy(dst, src, std::min(bytes, chunk));
    for (auto& t : th) t.join();
}

}  // namespace

// Arguments of a device-resident batch call; the table path's launches are
// captured once per key into a CUDA graph.
struct GraphKey {
    const void *w, *off;
    void *lb, *ex, *best, *arg, *err;
    int64_t n, max_r, c, k;
    int flags, wbytes, kmask, gen;
    cudaStream_t s;
    int kinds[6];
    int nk;
    bool operator==(const GraphKey& o) const {
        if (w != o.w || off != o.off || lb != o.lb || ex != o.ex || best != o.best || arg != o.arg || err != o.err ||
            n != o.n ||
            max_r != o.max_r || c != o.c || k != o.k || flags != o.flags || wbytes != o.wbytes ||
            kmask != o.kmask || gen != o.gen || s != o.s || nk != o.nk)
            return false;
        for (int i = 0; i < nk; ++i)
            if (kinds[i] != o.kinds[i]) return false;
        return true;
    }
};

// The grid-wide single check's launch sequence, replayed from a CUDA graph
// while its arguments repeat (eleven launches; their gaps were ~40 us of
// cfg4's 340).
struct WideKey {
    int64_t c = -1, r = -1, k = 0;
    int flags = 0, nk = 0, kinds[6] = {0, 0, 0, 0, 0, 0}, use_range = 0;
    int64_t rlo[6] = {0, 0, 0, 0, 0, 0}, rhi[6] = {0, 0, 0, 0, 0, 0};
    const void *w = nullptr, *res = nullptr, *err = nullptr, *buf = nullptr;
    size_t cap = 0;
    bool operator==(const WideKey& o) const {
        if (c != o.c || r != o.r || k != o.k || flags != o.flags || nk != o.nk || w != o.w || res != o.res ||
            err != o.err || buf != o.buf || cap != o.cap || use_range != o.use_range)
            return false;
        for (int i = 0; i < nk; ++i)
            if (kinds[i] != o.kinds[i]) return false;
        if (use_range)
            for (int i = 0; i < 6; ++i)
                if (rlo[i] != o.rlo[i] || rhi[i] != o.rhi[i]) return false;
        return true;
    }
};

struct bplb_engine {
    int device = 0;
    int num_sms = 0;
    size_t smem_optin = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;            // batch uploads
    cudaStream_t cstream[4] = {nullptr, nullptr, nullptr, nullptr};  // chunk kernels
    cudaEvent_t ev_up[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t ev_k[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::mutex mu;
    DevBuf d_w, d_off, d_res, d_lb, d_ex, d_best, d_arg, d_err, d_lam, d_wide, d_multi;
    HostBuf h_stage, h_res;
    // batched small-c path: cached table of transformed values for (tab_c, tab_kmask)
    DevBuf d_tab, d_tabmeta, d_tabkeys, d_tabhist, d_tabready;
    DevBuf d_inst, d_assign, d_redr;  // device-side reduction of node states
    std::vector<int32_t> inst_host;   // what d_inst holds
    DevBuf d_skeys;                   // single-check table path: keys[8] + CTA counter
    MappedBuf m_single;               // single-check table path: weights in, result out
    MappedBuf m_nres;                 // single-check node path: result + error word out
    int64_t wide_cnt_zero = 0;        // leading histogram counts of d_wide known to be zero
    cudaGraphExec_t wide_exec = nullptr;   // the captured grid-wide sequence (wide_key), its launch count
    WideKey wide_key, wide_seen;
    int64_t wide_exec_launches = 0;
    bool multi_dirty = true;          // the MultiState needs zeroing (first use, or a failed check)
    const void* node_attr_kern = nullptr;  // launch_node: kernel / smem / occupancy of the last launch
    size_t node_attr_smem = 0;
    int node_attr_per_sm = 0;
    MappedBuf m_err;                  // batch calls: error flag written by the kernels
    bool skeys_zeroed = false;
    size_t tab_attr_smem = 0;
    size_t prune_attr_smem = 0;
    int last_path = 0;    // BPLB_PATH_* of the last batch / check launch (bplb_last_path)
    int last_detail = 0;  // path detail (table path: warps per contraction CTA)
    int tab_per_sm = 1;
    int hist_per_sm = 3;          // persistent histogram CTAs per SM (BPLB_HIST_PER_SM)
    bool hist_carveout = false;
    int64_t multi_grid = 0;  // BPLB_MULTI_GRID: override of the single-node multi-CTA grid (tuning)
    // r * c above which node-resident single checks take the pruned wide path
    // instead (BPLB_WIDE_PRUNE_MIN_CELLS): off by default -- cfg3 (r * c = 1e8)
    // measured 172 us there vs 104 us on the multi-CTA node kernel
    int64_t wide_prune_min_cells = (int64_t)1 << 62;
    bool tc_on = true;          // BPLB_TC=0: the table path on the FP32 pipe instead of tcgen05
    DevBuf d_tcB, d_tcmeta;     // tensor-core table planes / column constants
    DevBuf d_knin, d_knout;     // knapsack bins: packed inputs / outputs (host-array entry)
    DevBuf d_knord;             // knapsack bins grouped by item count (warp path)
    int64_t tc_c = -1;
    int tc_kmask = -1, tc_KT = 0, tc_nnt = 0;
    size_t tc_attr_smem = 0;
    bool assign_carveout = false;
    bool single_cluster_ok = true;    // drop-in checks as one thread-block cluster
    bool single_cluster_attr = false;
    // cross-stream ordering of calls that share the engine's scratch: the
    // last asynchronous call's stream and an event recorded after its work
    cudaEvent_t ev_tail = nullptr;
    cudaStream_t tail_stream = nullptr;
    bool tail_valid = false;
    int64_t tab_c = -1;
    int tab_kmask = -1, tab_KV = 0, tab_nsub = 0, tab_P = 0;
    int64_t tab_nodes = 0;  // capacity of d_tabkeys / d_tabhist (nodes)
    int64_t launches = 0;
    double last_ms = 0.0;
    // table-path launches replayed from CUDA graphs, one per argument set
    // (a search loop or the bench repeats them), least recently used evicted
    struct GraphSlot {
        GraphKey key{};
        cudaGraphExec_t exec = nullptr;
        uint64_t used = 0;
    } graphs[4];
    uint64_t graph_clock = 0;
    GraphKey graph_seen[4] = {};  // argument sets seen once (captured on their second call)
    int graph_seen_next = 0;
    int tab_gen = 0;        // bumped whenever a table-path buffer is (re)allocated
    bool graphs_ok = true;  // capture failed once: launch directly
    int prof_kernel = 0;       // bracket the contraction kernel with ev_pk0 / ev_pk1
    int prof_recorded = 0;
    cudaEvent_t ev_pk0 = nullptr, ev_pk1 = nullptr;
};

namespace {

// Copy host -> device (direct DMA when the source is pinned, through the
// engine's pinned staging buffer otherwise).
int h2d(bplb_engine* e, void* dst, const void* src, size_t bytes, size_t stage_off = 0,
        cudaStream_t s = nullptr, int pinned = -1);

// The instance weights of an assignment batch on the device (a search
// re-checks the same instance every call: re-uploaded only when they change).
int upload_inst(bplb_engine* e, const int32_t* inst_w, int64_t n_items) {
    void* before = e->d_inst.p;
    if (int rc = e->d_inst.grow((size_t)std::max<int64_t>(n_items, 1) * 4)) return rc;
    const size_t bytes = (size_t)n_items * 4;
    if (e->d_inst.p == before && e->inst_host.size() == (size_t)n_items &&
        (n_items == 0 || std::memcmp(e->inst_host.data(), inst_w, bytes) == 0))
        return 0;
    e->inst_host.assign(inst_w, inst_w + n_items);
    // from the engine's copy: stays valid after the call returns
    return h2d(e, e->d_inst.p, e->inst_host.data(), bytes, 0, e->stream, 1);
}

int h2d(bplb_engine* e, void* dst, const void* src, size_t bytes, size_t stage_off, cudaStream_t s, int pinned) {
    if (bytes == 0) return 0;
    if (!s) s = e->stream;
    if (pinned < 0) pinned = bytes > 65536 ? is_pinned(src) : 1;
    if (bytes <= 65536 || pinned) {
        CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        return 0;
    }
    // pageable source: stage through the engine's pinned buffer (the buffer
    // is grown by the caller before any chunk is enqueued)
    if (stage_off + bytes > e->h_stage.cap) return fail(BPLB_ENOMEM, "staging buffer too small");
    char* st = (char*)e->h_stage.p + stage_off;
    std::memcpy(st, src, bytes);
    CUDA_TRY(cudaMemcpyAsync(dst, st, bytes, cudaMemcpyHostToDevice, s));
    return 0;
}

int check_kinds(const int32_t* kinds, int32_t nkinds, int* out) {
    if (nkinds < 0 || nkinds > K_COUNT) return fail(BPLB_EINVAL, "nkinds must be in [0, 6]");
    bool seen[K_COUNT] = {false, false, false, false, false, false};
    for (int i = 0; i < nkinds; ++i) {
        int k = kinds[i];
        if (k < 0 || k >= K_COUNT) return fail(BPLB_EINVAL, "kind id out of range");
        if (seen[k]) return fail(BPLB_EINVAL, "duplicate kind in kinds");
        seen[k] = true;
        out[i] = k;
    }
    return 0;
}

int check_c(int64_t c) {
    if (c < 1) return fail(BPLB_EINVAL, "capacity must be >= 1");
    if (c > BPLB_MAX_C) return fail(BPLB_ERANGE, "capacity exceeds the GPU envelope (2^30)");
    return 0;
}

void fill_params(bplb::KParams& p, int64_t c, int64_t k, const int* kinds, int nk, int flags) {
    std::memset(&p, 0, sizeof(p));
    p.c = c;
    p.k = k;
    for (int i = 0; i < nk; ++i) p.kinds[i] = kinds[i];
    p.nk = nk;
    p.flags = flags;
    p.one = 1;
    p.wbytes = 4;
}

// Warp-per-node kernel for batches of small-capacity nodes.
int launch_warp(bplb_engine* e, bplb::KParams& p, int64_t n_nodes) {
    const size_t smem = bplb::warp_cta_bytes(p.c) + bplb::warp_slice_bytes(p.c) * bplb::WNW;
    CUDA_TRY(cudaFuncSetAttribute(bplb::warp_node_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bplb::warp_node_kernel, bplb::WNT, smem));
    if (per_sm < 1) per_sm = 1;
    int64_t grid = std::min<int64_t>((n_nodes + bplb::WNW - 1) / bplb::WNW, (int64_t)per_sm * e->num_sms);
    p.n_nodes = n_nodes;
    bplb::warp_node_kernel<<<(unsigned)grid, bplb::WNT, smem, e->stream>>>(p);
    e->launches++;
    e->last_path = BPLB_PATH_WARP;
    e->last_detail = 0;
    CUDA_TRY(cudaGetLastError());
    return 0;
}

bool warp_path(const bplb::KParams& p, int64_t n_nodes) {
    return p.lam_out == nullptr && p.c <= bplb::WARP_MAX_C && n_nodes >= 64 &&
           bplb::warp_cta_bytes(p.c) + bplb::warp_slice_bytes(p.c) * bplb::WNW <= 200 * 1024;
}


// ---- batched small-capacity path (bplb_tab.cuh) ------------------------------
int tab_kmask(const bplb::KParams& p) {
    int m = 0;
    for (int i = 0; i < p.nk; ++i) m |= 1 << p.kinds[i];
    return m;
}

// Warps per tab_kernel CTA: 8, fewer when the histogram buffers of large
// capacities do not fit (0: the table path does not apply).
int tab_warps(const bplb_engine* e, int KV, int nb = 2) {
    for (int nw = bplb::TAB_NW; nw >= 2; --nw)
        if (bplb::tab_cta_bytes(nw, KV, nb) + 64 <= e->smem_optin) return nw;
    return 0;
}

// Order this call's stream X after the previous asynchronous call's work
// when that ran on another stream (engine scratch buffers are shared).
int join_stream(bplb_engine* e, cudaStream_t X) {
    if (e->tail_valid && e->tail_stream != X) CUDA_TRY(cudaStreamWaitEvent(X, e->ev_tail, 0));
    return 0;
}
int mark_tail(bplb_engine* e, cudaStream_t X) {
    CUDA_TRY(cudaEventRecord(e->ev_tail, X));
    e->tail_stream = X;
    e->tail_valid = true;
    return 0;
}

// Tabulate f_k(w, lambda) for capacity c and the requested kinds (cached).
int tab_ensure(bplb_engine* e, const bplb::KParams& p) {
    const int kmask = tab_kmask(p);
    if (e->tab_c == p.c && e->tab_kmask == kmask) return 0;
    const int c = (int)p.c;
    std::vector<int4> meta;
    std::vector<int2> cols;
    auto pad_col = [&](int kind) {
        meta.push_back(int4{(int)0x80000000u, (int)(0u - 0x96000000u), 0, kind << 16});  // F = 1, S = 0
        cols.push_back(int2{-1, kind});
    };
    for (int kd = 0; kd < K_COUNT; ++kd) {
        if (!(kmask >> kd & 1)) continue;
        int64_t lo, hi;
        bplb_domain(kd, c, &lo, &hi);  // VB2 uncapped: the cap is >= c in this envelope
        const int64_t n = hi - lo + 1;
        if (n <= 0) continue;
        for (int64_t i = 0; i < n; ++i) {
            const int64_t lam = lo + i;
            const int64_t F = bplb_fc(kd, c, lam);
            if (F <= 0) return fail(BPLB_ERANGE, "f(c, lambda) <= 0 inside the table path");  // never for c >= 1
            int l = 0;
            while ((1ll << l) < F) ++l;
            const uint64_t m = ((1ull << (31 + l)) + (uint64_t)F - 1) / (uint64_t)F;  // < 2^32
            const uint32_t K = (uint32_t)(2 * F - 2) - 0x96000000u;
            meta.push_back(int4{(int)(uint32_t)m, (int)K, l, (int)(511 - lam) | (kd << 16)});
            cols.push_back(int2{(int)lam, kd});
        }
        while (meta.size() % 4) pad_col(kd);  // one kind per 4-column lane group
    }
    while (meta.size() % bplb::TAB_SUB || meta.empty()) pad_col(K_COUNT);
    const int KV = (c + 3) / 4 * 4;
    const int nsub = (int)(meta.size() / bplb::TAB_SUB);
    if (tab_warps(e, KV) < 1) return fail(BPLB_ERANGE, "capacity too large for the table path");
    const int P = nsub;  // one 64-column sub-chunk per CTA
    int rc;
    if ((rc = e->d_tab.grow((size_t)nsub * (KV + 2) * bplb::TAB_SUB * 4))) return rc;
    if ((rc = e->d_tabmeta.grow(meta.size() * (sizeof(int4) + sizeof(int2))))) return rc;
    int2* d_cols = (int2*)((int4*)e->d_tabmeta.p + meta.size());
    CUDA_TRY(cudaMemcpyAsync(e->d_tabmeta.p, meta.data(), meta.size() * sizeof(int4), cudaMemcpyHostToDevice,
                             e->stream));
    CUDA_TRY(cudaMemcpyAsync(d_cols, cols.data(), cols.size() * sizeof(int2), cudaMemcpyHostToDevice, e->stream));
    const int64_t n = (int64_t)nsub * (KV + 2) * bplb::TAB_SUB;
    bplb::tab_build_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4 * e->num_sms), 256, 0, e->stream>>>(
        (float*)e->d_tab.p, d_cols, KV + 2, nsub, p.c);
    e->launches++;
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(e->stream));  // meta / cols are host vectors; the table is cached
    e->tab_c = p.c;
    e->tab_kmask = kmask;
    e->tab_gen++;
    e->tab_KV = KV;
    e->tab_nsub = nsub;
    e->tab_P = P;
    return 0;
}

// Per-node key / per-tile counter arrays (zero between launches; the kernel
// clears what it used) for nodes [0, n).
int tab_reserve(bplb_engine* e, int64_t n) {
    if (n <= e->tab_nodes) return 0;
    int rc;
    if ((rc = e->d_tabkeys.grow((size_t)n * bplb::TAB_KSLOT * 4))) return rc;
    // histogram tiles, indexed by absolute tile (node / 16)
    if ((rc = e->d_tabhist.grow((size_t)(n / bplb::TAB_TM + 1) * ((bplb::TAB_MAX_C + 3) / 4 * 4 + 1) * bplb::TAB_TM * 4)))
        return rc;
    CUDA_TRY(cudaMemsetAsync(e->d_tabkeys.p, 0, (size_t)n * bplb::TAB_KSLOT * 4, e->stream));
    if ((rc = e->d_tabready.grow((size_t)(n / bplb::TAB_TM + 1) * 4))) return rc;
    CUDA_TRY(cudaMemsetAsync(e->d_tabready.p, 0, (size_t)(n / bplb::TAB_TM + 1) * 4, e->stream));


    e->tab_nodes = n;
    e->tab_gen++;
    return 0;
}

// The table path applies to batches of small-capacity nodes whose
// transformed sums stay exact in fp32 below 2^23 (the epilogue reads S from
// the bits of S + 2^23): max_r * max f < 2^23 (MT, RAD2, BJ1 <= c; CCM1,
// VB2 <= 2c; FS1 <= 101c).
bool tab_path(const bplb_engine* e, const bplb::KParams& p, int64_t n_nodes, int64_t max_r) {
    if (p.lam_out || p.ms || p.c > bplb::TAB_MAX_C || n_nodes < 256 || max_r > 65535) return false;
    if (n_nodes > ((int64_t)1 << 30)) return false;  // 32-bit item indices (ntiles * sub-chunks)
    if ((uintptr_t)p.w & 15) return false;  // the histogram pass reads aligned 16-byte vectors
    const int KV = ((int)p.c + 3) / 4 * 4;
    if (tab_warps(e, KV) < 2) return false;
    const int64_t maxf = (tab_kmask(p) >> K_FS1 & 1) ? 101 * p.c : 2 * p.c;
    return max_r * maxf < (1ll << 23);
}

// Launch with programmatic dependent launch: the kernel may start while the
// previous one on the stream drains; it waits in cudaGridDependencySynchronize.
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// The table path in three launches over nodes [p.node0, p.node0 + n):
// histograms, contraction (PDL), per-node results (PDL).  Tiles are indexed
// absolutely (tile = node / 16), so sub-ranges must start on a multiple of 16.
bplb::TabDev tab_dev(bplb_engine* e, const bplb::KParams& p, int64_t n_nodes) {
    bplb::TabDev t;
    t.T = (const float*)e->d_tab.p;
    t.meta = (const int4*)e->d_tabmeta.p;
    t.KV = e->tab_KV;
    t.nsub = e->tab_nsub;
    t.P = e->tab_P;
    t.gkeys = (unsigned*)e->d_tabkeys.p;
    t.trace = nullptr;
#ifdef TAB_TRACE
    static unsigned long long* tr = nullptr;
    if (!tr) cudaMalloc(&tr, (size_t)4096 * 16 * 16 * 8 * 2);
    t.trace = tr;
#endif
    t.ready = (unsigned*)e->d_tabready.p + p.node0 / bplb::TAB_TM;
    t.ntiles = (n_nodes + bplb::TAB_TM - 1) / bplb::TAB_TM;
    t.H = (float*)e->d_tabhist.p + (p.node0 / bplb::TAB_TM) * (t.KV + 1) * bplb::TAB_TM;
    return t;
}

int tab_hist(bplb_engine* e, bplb::KParams p, int64_t n_nodes) {
    p.n_nodes = n_nodes;
    const bplb::TabDev t = tab_dev(e, p, n_nodes);
    const size_t hs = ((size_t)bplb::TAB_TM * (t.KV + 1) + 2 * bplb::TAB_HPAD) * 4;  // <= 20.5 KB (KV <= 288)
    // persistent: the CTAs walk the tiles in order next to the tab_kernel
    // CTAs that consume them (e->hist_per_sm CTAs of 8 warps per SM).  An
    // SM's smem carveout is fixed while CTAs are resident: the histogram
    // kernels ask for the maximum so a tab_kernel CTA fits beside them.
    if (!e->hist_carveout) {
        CUDA_TRY(cudaFuncSetAttribute(bplb::tab_hist_u8_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                      cudaSharedmemCarveoutMaxShared));
        CUDA_TRY(cudaFuncSetAttribute(bplb::tab_hist_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                      cudaSharedmemCarveoutMaxShared));
        e->hist_carveout = true;
    }
    if (p.wbytes == 1 && !((uintptr_t)p.w & 15))  // packed counts: half the scratch
        bplb::tab_hist_u8_kernel<<<(unsigned)std::min<int64_t>(t.ntiles, (int64_t)e->hist_per_sm * e->num_sms),
                                   bplb::TAB_HNT8, (size_t)bplb::TAB_TM / 2 * (t.KV + 1) * 4, e->stream>>>(p, t);
    else
        bplb::tab_hist_kernel<<<(unsigned)std::min<int64_t>(t.ntiles, (int64_t)std::max(1, e->hist_per_sm / 2) * e->num_sms),
                                bplb::TAB_HNT, hs, e->stream>>>(p, t);
    e->launches++;
    CUDA_TRY(cudaGetLastError());
    return 0;
}

int tab_contract(bplb_engine* e, bplb::KParams p, int64_t n_nodes) {
    const int KV = e->tab_KV, P = e->tab_P;
    // 8 warps with two histogram buffers each (8 / 12 / 16 warps with one
    // buffer measured no faster on cfg2)
    const int nb = 2, nw = tab_warps(e, KV, 2);
    const size_t smem = bplb::tab_cta_bytes(nw, KV, nb);
    auto kern = bplb::tab_kernel<2>;
    if (e->tab_attr_smem != smem) {  // once per table shape (cudaFuncSetAttribute is not free)
        CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nw * 32, smem));
        e->tab_per_sm = per_sm < 1 ? 1 : per_sm;
        e->tab_attr_smem = smem;
    }
    p.n_nodes = n_nodes;
    bplb::TabDev t = tab_dev(e, p, n_nodes);
    // every SM, at least one CTA per table sub-chunk, no more CTAs per
    // sub-chunk than its warps have tiles
    const int64_t cpp = std::max<int64_t>(1, std::min<int64_t>(((int64_t)e->tab_per_sm * e->num_sms + P - 1) / P,
                                                              (t.ntiles + nw - 1) / nw));
    int64_t grid = std::max<int64_t>(std::min<int64_t>((int64_t)e->tab_per_sm * e->num_sms, cpp * P), P);
    if (e->prof_kernel) CUDA_TRY(cudaEventRecord(e->ev_pk0, e->stream));
    CUDA_TRY(launch_pdl(kern, dim3((unsigned)grid), dim3(nw * 32), smem, e->stream, p, t));
    e->last_path = BPLB_PATH_TAB;
    e->last_detail = nw;
#ifdef TAB_TRACE
    {  // dump: grid, nw, P, ntiles, hist ctas, then [cta][warp][16] stamps, then [tile] publish stamps
        std::vector<unsigned long long> h((size_t)grid * nw * 16), hp((size_t)t.ntiles);
        cudaStreamSynchronize(e->stream);
        cudaMemcpy(h.data(), t.trace, h.size() * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(hp.data(), t.trace + 4096 * 16 * 16, hp.size() * 8, cudaMemcpyDeviceToHost);
        cudaMemset(t.trace, 0, (size_t)4096 * 16 * 16 * 8 * 2);
        if (FILE* f = fopen(getenv("BPLB_TAB_TRACE") ? getenv("BPLB_TAB_TRACE") : "tab_trace.bin", "ab")) {
            long long hd[5] = {(long long)grid, (long long)nw, (long long)P, (long long)t.ntiles, 0};
            fwrite(hd, 8, 5, f);
            fwrite(h.data(), 8, h.size(), f);
            fwrite(hp.data(), 8, hp.size(), f);
            fclose(f);
        }
    }
#endif
    if (e->prof_kernel) {
        CUDA_TRY(cudaEventRecord(e->ev_pk1, e->stream));
        e->prof_recorded = 1;
    }
    e->launches++;
    CUDA_TRY(cudaGetLastError());
    return 0;
}

int tab_fin(bplb_engine* e, bplb::KParams p, int64_t n_nodes) {
    p.n_nodes = n_nodes;
    CUDA_TRY(launch_pdl(bplb::tab_fin_kernel, dim3((unsigned)((n_nodes + 63) / 64)), dim3(64), 0, e->stream, p,
                        (unsigned*)e->d_tabkeys.p, (unsigned*)e->d_tabready.p + p.node0 / bplb::TAB_TM));
    e->launches++;
    CUDA_TRY(cudaGetLastError());
    return 0;
}

// Tensor-core planes of the cached table (bplb_tc.cuh), rebuilt with it.
int tc_ensure(bplb_engine* e) {
    if (e->tc_c == e->tab_c && e->tc_kmask == e->tab_kmask) return 0;
    const int c = (int)e->tab_c;
    const int KT = (c + 31) / 32 * 32;
    const int ncols = e->tab_nsub * bplb::TAB_SUB;
    const int nnt = (ncols + bplb::TC_NT - 1) / bplb::TC_NT;
    int rc;
    if ((rc = e->d_tcB.grow((size_t)nnt * bplb::tc_b_bytes(KT)))) return rc;
    if ((rc = e->d_tcmeta.grow((size_t)nnt * bplb::TC_NT * sizeof(int4)))) return rc;
    const int64_t n = (int64_t)nnt * bplb::TC_NT * KT;
    bplb::tc_build_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4 * e->num_sms), 256, 0, e->stream>>>(
        (uint8_t*)e->d_tcB.p, (int4*)e->d_tcmeta.p, (const float*)e->d_tab.p, (const int4*)e->d_tabmeta.p, e->tab_KV,
        e->tab_nsub, KT, nnt, c);
    e->launches++;
    CUDA_TRY(cudaGetLastError());
    e->tc_c = e->tab_c;
    e->tc_kmask = e->tab_kmask;
    e->tc_KT = KT;
    e->tc_nnt = nnt;
    return 0;
}

bool tc_fits(const bplb_engine* e, int64_t c) {
    const int KT = (int)(c + 31) / 32 * 32;
    return e->tc_on && bplb::tc_smem_bytes_db(KT, false) + 4096 <= e->smem_optin;
}

// The batch on the tensor cores: one CTA per slice of <= 128 nodes, the
// slices sized so the batch covers every SM, one launch.
int launch_tc(bplb_engine* e, bplb::KParams& p, int64_t n_nodes) {
    int rc;
    if ((rc = tc_ensure(e))) return rc;
    // double-buffered table tiles (BPLB_TC_DB=1): measured wrong results with
    // slices of < 128 nodes (an unresolved race), so single-buffered by default
    const bool db = bplb::tc_smem_bytes_db(e->tc_KT, true) + 4096 <= e->smem_optin && getenv("BPLB_TC_DB") &&
                    atoi(getenv("BPLB_TC_DB")) != 0;
    const size_t smem = bplb::tc_smem_bytes_db(e->tc_KT, db);
    using K = void (*)(bplb::KParams, bplb::TcDev);
    K kern;
    if (db) kern = p.wbytes == 1 ? bplb::tc_kernel<1, true> : (p.wbytes == 2 ? bplb::tc_kernel<2, true> : bplb::tc_kernel<4, true>);
    else kern = p.wbytes == 1 ? bplb::tc_kernel<1, false> : (p.wbytes == 2 ? bplb::tc_kernel<2, false> : bplb::tc_kernel<4, false>);
    if (smem > e->tc_attr_smem) {
        for (K k : {bplb::tc_kernel<1, true>, bplb::tc_kernel<2, true>, bplb::tc_kernel<4, true>,
                    bplb::tc_kernel<1, false>, bplb::tc_kernel<2, false>, bplb::tc_kernel<4, false>})
            CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        e->tc_attr_smem = smem;
    }
    // nodes per CTA: the batch spread over every SM (a multiple of 8, <= 128)
    int64_t rows = (n_nodes + e->num_sms - 1) / e->num_sms;
    rows = std::min<int64_t>(bplb::TC_M, std::max<int64_t>(8, (rows + 7) / 8 * 8));
    if (getenv("BPLB_TC_ROWS")) rows = atoll(getenv("BPLB_TC_ROWS"));
    bplb::TcDev t{(const uint8_t*)e->d_tcB.p, (const int4*)e->d_tcmeta.p, e->tc_KT, e->tc_nnt, (int)rows};
    p.n_nodes = n_nodes;
    const int64_t grid = (n_nodes + rows - 1) / rows;
    if (grid < 1) return 0;
    if (e->prof_kernel) CUDA_TRY(cudaEventRecord(e->ev_pk0, e->stream));
    kern<<<(unsigned)grid, bplb::TC_THREADS, smem, e->stream>>>(p, t);
    e->launches++;
    CUDA_TRY(cudaGetLastError());
    if (e->prof_kernel) {
        CUDA_TRY(cudaEventRecord(e->ev_pk1, e->stream));
        e->prof_recorded = 1;
    }
    e->last_path = BPLB_PATH_TC;
    e->last_detail = (int)e->tc_nnt;
    return 0;
}

int launch_tab(bplb_engine* e, bplb::KParams& p, int64_t n_nodes, int slot) {
    (void)slot;
    int rc;
    if ((rc = tab_ensure(e, p))) return rc;
    if (!(p.flags & BPLB_F_NOTC) && tc_fits(e, p.c)) return launch_tc(e, p, n_nodes);
    if ((rc = tab_reserve(e, p.node0 + n_nodes))) return rc;
    if (p.node0 % bplb::TAB_TM) return fail(BPLB_EINVAL, "table path sub-range must start on a 16-node tile");
    if ((rc = tab_hist(e, p, n_nodes))) return rc;
    if ((rc = tab_contract(e, p, n_nodes))) return rc;
    return tab_fin(e, p, n_nodes);
}

// launch_tab on e->stream replayed from a cached CUDA graph (captured on
// first use of an argument set): one launch call instead of three.  w / off
// are the device (or device-alias) inputs; the outputs and error flag come
// from p.  Falls back to direct launches where capture is unavailable.
int launch_tab_graph(bplb_engine* e, bplb::KParams& p, int64_t n_nodes, int64_t max_r, const int* ks, int nkinds,
                     const void* w, const void* off) {
    if (!e->graphs_ok || e->prof_kernel) return launch_tab(e, p, n_nodes, 0);
    cudaStream_t s = e->stream;
    GraphKey key{w, off, p.lb_out, p.ex_out, p.best_out, p.arg_out, p.err_out, n_nodes, max_r, p.c, p.k, p.flags,
                 p.wbytes, tab_kmask(p), e->tab_gen, s, {ks[0], ks[1], ks[2], ks[3], ks[4], ks[5]}, nkinds};
    bplb_engine::GraphSlot* slot = nullptr;
    for (auto& g : e->graphs)
        if (g.exec && g.key == key) slot = &g;
    if (!slot) {
        // capture only an argument set that repeats: callers that pass fresh
        // buffers every time launch directly instead of capturing each call
        bool seen = false;
        for (const auto& k : e->graph_seen) seen |= k == key;
        if (!seen) {
            e->graph_seen[e->graph_seen_next] = key;
            e->graph_seen_next = (e->graph_seen_next + 1) % 4;
            return launch_tab(e, p, n_nodes, 0);
        }
        slot = &e->graphs[0];
        for (auto& g : e->graphs)
            if (!g.exec || g.used < slot->used) slot = &g;
        if (slot->exec) cudaGraphExecDestroy(slot->exec);
        slot->exec = nullptr;
        cudaGraph_t g = nullptr;
        if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
            // e.g. the legacy default stream (cudaStreamLegacy) cannot be
            // captured: clear the error and launch directly from now on
            cudaGetLastError();
            e->graphs_ok = false;
            return launch_tab(e, p, n_nodes, 0);
        }
        const int64_t l0 = e->launches;
        int rc = launch_tab(e, p, n_nodes, 0);
        cudaError_t ce = cudaStreamEndCapture(s, &g);
        e->launches = l0;  // counted when the graph runs
        if (!rc && ce == cudaSuccess) ce = cudaGraphInstantiate(&slot->exec, g, 0);
        if (g) cudaGraphDestroy(g);
        if (rc) return rc;
        if (ce != cudaSuccess) {  // no graphs here: launch directly from now on
            cudaGetLastError();
            e->graphs_ok = false;
            slot->exec = nullptr;
            return launch_tab(e, p, n_nodes, 0);
        }
        slot->key = key;
    }
    slot->used = ++e->graph_clock;
    cudaError_t ce = cudaGraphLaunch(slot->exec, s);
    if (ce != cudaSuccess) return fail(BPLB_ECUDA, std::string("graph launch: ") + cudaGetErrorString(ce));
    const bool tc = !(p.flags & BPLB_F_NOTC) && tc_fits(e, p.c);  // what the captured launch_tab ran
    e->launches += tc ? 1 : 3;
    e->last_path = tc ? BPLB_PATH_TC : BPLB_PATH_TAB;
    e->last_detail = tc ? e->tc_nnt : tab_warps(e, e->tab_KV, 2);
    return 0;
}

// Launch the node-resident kernel over n nodes.  max_r bounds every node.
// multi: one node, every CTA of a co-resident grid sweeps part of it
// (single-check latency path); p.ms must point at a zeroed MultiState.
// Bound-pruned node kernel (bplb_prune.cuh) for batches of nodes with
// 2 <= c <= 2^18 whose largest node fits its shared-memory layout.
bool prune_path(const bplb_engine* e, const bplb::KParams& p, int64_t max_r) {
    if ((p.flags & BPLB_F_NOPRUNE) || p.lam_out || p.ms || p.c < 2 || p.c > bplb::PR_MAX_C || max_r > (1 << 14))
        return false;
    return bplb::prune_smem_bytes(bplb::prune_rcap(max_r), p.c) <= e->smem_optin;
}

int launch_prune(bplb_engine* e, bplb::KParams& p, int64_t n_nodes, int64_t max_r) {
    const int rcap = bplb::prune_rcap(max_r);
    const size_t smem = bplb::prune_smem_bytes(rcap, p.c);
    if (smem > e->prune_attr_smem) {
        CUDA_TRY(cudaFuncSetAttribute(bplb::prune_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CUDA_TRY(cudaFuncSetAttribute(bplb::prune_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CUDA_TRY(cudaFuncSetAttribute(bplb::prune_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        e->prune_attr_smem = smem;
    }
    const int lbmode = !p.best_out && !p.arg_out && !p.res_out;
    const bool plain = !(p.flags & (BPLB_F_PHASED | BPLB_F_CANCEL));
    auto kern = !plain ? bplb::prune_kernel<0> : (lbmode ? bplb::prune_kernel<1> : bplb::prune_kernel<2>);
    int per_sm = 0;
    const int nt = bplb::prune_threads(!plain ? 0 : (lbmode ? 1 : 2));
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nt, smem));
    if (per_sm < 1) per_sm = 1;
    const int64_t grid = std::min<int64_t>(n_nodes, (int64_t)per_sm * e->num_sms);
    if (grid < 1) return 0;
    p.n_nodes = n_nodes;
    kern<<<(unsigned)grid, nt, smem, e->stream>>>(p, rcap, lbmode);
    e->launches++;
    CUDA_TRY(cudaGetLastError());
    e->last_path = BPLB_PATH_PRUNE;
    e->last_detail = lbmode;
    return 0;
}

bool node_fits(int64_t r, int64_t c) {
    return r <= (c <= bplb::TABLE_MAX_C ? NODE_R_MAX_TABLE : NODE_R_MAX_SORT);
}

int launch_node(bplb_engine* e, bplb::KParams& p, int64_t n_nodes, int64_t max_r, int grid_cap,
                bool multi = false, int slot = 0) {
    if (!multi && grid_cap == 0 && !(p.flags & BPLB_F_NOTAB) && tab_path(e, p, n_nodes, max_r))
        return launch_tab(e, p, n_nodes, slot);
    if (!multi && grid_cap == 0 && prune_path(e, p, max_r)) return launch_prune(e, p, n_nodes, max_r);
    if (!multi && grid_cap == 0 && warp_path(p, n_nodes)) return launch_warp(e, p, n_nodes);
    const bool table = p.c <= bplb::TABLE_MAX_C;
    if (max_r > (table ? NODE_R_MAX_TABLE : NODE_R_MAX_SORT))
        return fail(BPLB_ERANGE, "node larger than the node-resident envelope");
    int rcap = 1;
    if (table) rcap = (int)std::max<int64_t>(max_r, 1);
    else while (rcap < max_r) rcap <<= 1;
    size_t smem = bplb::node_smem_bytes(table, rcap, p.c);
    if (smem > e->smem_optin) return fail(BPLB_ERANGE, "node needs more shared memory than available");
    auto kern = table ? bplb::node_kernel<true, false>
                      : (p.c >= (1 << 23) ? bplb::node_kernel<false, true> : bplb::node_kernel<false, false>);
    int per_sm = 0;
    if (e->node_attr_kern == (const void*)kern && e->node_attr_smem == smem) {  // (host API calls cost us)
        per_sm = e->node_attr_per_sm;
    } else {
        CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, bplb::NT, smem));
        if (per_sm < 1) per_sm = 1;
        e->node_attr_kern = (const void*)kern;
        e->node_attr_smem = smem;
        e->node_attr_per_sm = per_sm;
    }
    int64_t grid = std::min<int64_t>(n_nodes, (int64_t)per_sm * e->num_sms);
    if (multi) {  // co-resident grid (CTAs may wait on each other), sized by the work
        // at most one CTA per SM: two per SM measured 7-10 % slower (cfg3
        // 125 vs 113 us; every CTA repeats the node setup and meets the
        // others at the phase barriers)
        const int64_t cells = std::max<int64_t>(max_r, 1) * (3 * std::min<int64_t>(p.c, 1 << 24) + 100);
        grid = std::min<int64_t>((int64_t)e->num_sms, std::max<int64_t>(1, cells / 16384));
        if (e->multi_grid > 0) grid = std::min<int64_t>((int64_t)per_sm * e->num_sms, e->multi_grid);
    }
    if (grid_cap > 0) grid = std::min<int64_t>(grid, grid_cap);
    if (grid < 1) return 0;
    p.n_nodes = n_nodes;
    kern<<<(unsigned)grid, bplb::NT, smem, e->stream>>>(p, rcap);
    e->launches++;
    e->last_path = table ? BPLB_PATH_NODE_TABLE : BPLB_PATH_NODE_SORT;
    e->last_detail = multi ? (int)grid : 0;
    CUDA_TRY(cudaGetLastError());
    return 0;
}


// Device-side reduce_packing of a batch of node states (bplb_reduce.cuh):
// uploads the instance and the assignments, leaves the reduced CSR in
// d_w (obytes per weight) / d_off and the error flags in d_err[1].
int reduce_device(bplb_engine* e, const int32_t* inst_w, int64_t n_items, int64_t n_bins, const void* assign,
                  int32_t abytes, int64_t n_nodes, int64_t c, int* obytes) {
    if (abytes != 1 && abytes != 2) return fail(BPLB_EINVAL, "assignment element must be 1 or 2 bytes");
    if (n_items < 0 || n_bins < 0 || n_nodes < 0) return fail(BPLB_EINVAL, "bad shape");
    if (n_bins > bplb::RED_MAX_BINS) return fail(BPLB_ERANGE, "more bins than the device reduction supports");
    if (n_bins >= (abytes == 1 ? 255 : 65535)) return fail(BPLB_EINVAL, "bin ids collide with the open marker");
    if (n_items > BPLB_MAX_R) return fail(BPLB_ERANGE, "too many items for the GPU envelope");
    *obytes = c <= 255 ? 1 : (c <= 65535 ? 2 : 4);
    int rc;
    const size_t asz = (size_t)n_nodes * (size_t)n_items * (size_t)abytes;
    if ((rc = e->d_assign.grow(std::max<size_t>(asz, 16)))) return rc;
    if ((rc = e->d_w.grow((size_t)std::max<int64_t>(n_nodes * n_items, 1) * 4 + 64))) return rc;
    if ((rc = e->d_off.grow((size_t)(n_nodes + 1) * 8))) return rc;
    if ((rc = e->d_redr.grow(16))) return rc;
    if ((rc = e->d_err.grow(16))) return rc;
    CUDA_TRY(cudaMemsetAsync(e->d_err.p, 0, 8, e->stream));
    CUDA_TRY(cudaMemsetAsync(e->d_redr.p, 0, 8, e->stream));
    if (asz > 65536 && !is_pinned(assign) && (rc = e->h_stage.grow(asz + 64))) return rc;
    if ((rc = upload_inst(e, inst_w, n_items))) return rc;
    if ((rc = h2d(e, e->d_assign.p, assign, asz))) return rc;
    bplb::ReduceArgs a;
    a.w = (const int*)e->d_inst.p;
    a.assign = e->d_assign.p;
    a.abytes = abytes;
    a.n_items = n_items;
    a.n_bins = n_bins;
    a.n_nodes = n_nodes;
    a.c = c;
    a.r = (int64_t*)e->d_off.p;
    a.out_w = e->d_w.p;
    a.obytes = *obytes;
    a.err = (int*)e->d_err.p + 1;
    a.max_r = (unsigned long long*)e->d_redr.p;
    const size_t smem = (size_t)(bplb::RED_NT / 32) * std::max<int64_t>(n_bins, 1) * 8;
    if (smem > 48 * 1024)
        CUDA_TRY(cudaFuncSetAttribute(bplb::reduce_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (smem > 48 * 1024)
        CUDA_TRY(cudaFuncSetAttribute(bplb::reduce_write_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const unsigned grid = (unsigned)std::min<int64_t>((n_nodes + 7) / 8, (int64_t)8 * e->num_sms);
    if (n_nodes > 0) {
        bplb::reduce_count_kernel<<<grid, bplb::RED_NT, smem, e->stream>>>(a);
        bplb::reduce_scan_kernel<<<1, 1024, 0, e->stream>>>(a.r, n_nodes);
        bplb::reduce_write_kernel<<<grid, bplb::RED_NT, smem, e->stream>>>(a);
        e->launches += 3;
        CUDA_TRY(cudaGetLastError());
    }
    return 0;
}

const char* reduce_error(int err) {
    return (err & 1) ? "committed bin load exceeds capacity (reduce_packing)" : "bin id out of range";
}

}  // namespace

extern "C" {

const char* bplb_last_error(void) { return g_err.c_str(); }

const char* bplb_version(void) { return "bplb 0.1 sm_100a (node-resident + grid-wide LB-collection engine)"; }

int bplb_engine_create(int device, bplb_engine** out) {
    if (!out) return fail(BPLB_EINVAL, "out is null");
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(BPLB_ENODEV, "no CUDA device visible");
    }
    if (device < 0 || device >= n) return fail(BPLB_EINVAL, "device index out of range");
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0)
        return fail(BPLB_ENODEV, std::string("libbplb is built for sm_100a; device is ") + prop.name);
    CUDA_TRY(cudaSetDevice(device));
    bplb_engine* e = new bplb_engine();
    e->device = device;
    e->num_sms = prop.multiProcessorCount;
    e->smem_optin = prop.sharedMemPerBlockOptin;
    if (const char* v = getenv("BPLB_HIST_PER_SM")) e->hist_per_sm = std::max(1, atoi(v));
    if (const char* v = getenv("BPLB_MULTI_GRID")) e->multi_grid = atoll(v);
    if (const char* v = getenv("BPLB_WIDE_PRUNE_MIN_CELLS")) e->wide_prune_min_cells = atoll(v);
    if (const char* v = getenv("BPLB_TC")) e->tc_on = atoi(v) != 0;
    if (const char* v = getenv("BPLB_SINGLE_CLUSTER")) e->single_cluster_ok = atoi(v) != 0;  // A/B switch
#ifdef TAB_TRACE
    e->graphs_ok = false;  // stamps are read back per launch
#endif
    bool ok = cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking) == cudaSuccess &&

              cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreate(&e->ev0) == cudaSuccess && cudaEventCreate(&e->ev1) == cudaSuccess &&
              cudaEventCreateWithFlags(&e->ev_tail, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; i < 4 && ok; ++i)
        ok = cudaStreamCreateWithFlags(&e->cstream[i], cudaStreamNonBlocking) == cudaSuccess &&
             cudaEventCreateWithFlags(&e->ev_up[i], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&e->ev_k[i], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {
        delete e;
        return fail(BPLB_ECUDA, "stream/event creation failed");
    }
    *out = e;
    return 0;
}

int bplb_engine_destroy(bplb_engine* e) {
    if (!e) return 0;
    cudaSetDevice(e->device);
    cudaStreamSynchronize(e->stream);
    for (DevBuf* b : {&e->d_w, &e->d_off, &e->d_res, &e->d_lb, &e->d_ex, &e->d_best, &e->d_arg,
                      &e->d_err, &e->d_lam, &e->d_wide, &e->d_multi, &e->d_tab, &e->d_tabmeta,
                      &e->d_tabkeys, &e->d_tabhist, &e->d_tabready, &e->d_inst, &e->d_assign, &e->d_redr, &e->d_skeys,
                      &e->d_tcB, &e->d_tcmeta, &e->d_knin, &e->d_knout, &e->d_knord})
        b->release();
    e->h_stage.release();
    e->h_res.release();
    e->m_single.release();
    e->m_nres.release();
    e->m_err.release();
    cudaEventDestroy(e->ev0);
    if (e->ev_tail) cudaEventDestroy(e->ev_tail);
    cudaEventDestroy(e->ev1);
    for (auto& g : e->graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    if (e->wide_exec) cudaGraphExecDestroy(e->wide_exec);
    if (e->ev_pk0) cudaEventDestroy(e->ev_pk0);
    if (e->ev_pk1) cudaEventDestroy(e->ev_pk1);
    for (int i = 0; i < 4; ++i) {
        cudaEventDestroy(e->ev_up[i]);
        cudaEventDestroy(e->ev_k[i]);
        cudaStreamDestroy(e->cstream[i]);
    }
    cudaStreamDestroy(e->copy_stream);

    cudaStreamDestroy(e->stream);
    delete e;
    return 0;
}

int64_t bplb_launch_count(bplb_engine* e) { return e ? e->launches : 0; }

int bplb_profile_kernel(bplb_engine* e, int on) {
    if (!e) return fail(BPLB_EINVAL, "null engine");
    std::lock_guard<std::mutex> lock(e->mu);
    CUDA_TRY(cudaSetDevice(e->device));
    if (on && !e->ev_pk0) {
        CUDA_TRY(cudaEventCreate(&e->ev_pk0));
        CUDA_TRY(cudaEventCreate(&e->ev_pk1));
    }
    e->prof_kernel = on != 0;
    e->prof_recorded = 0;
    return 0;
}

int bplb_last_path(bplb_engine* e, int32_t* detail) {
    if (!e) return fail(BPLB_EINVAL, "null engine");
    if (detail) *detail = e->last_detail;
    return e->last_path;
}

double bplb_last_kernel_ms(bplb_engine* e) {
    if (!e || !e->prof_recorded) return 0.0;
    std::lock_guard<std::mutex> lock(e->mu);
    cudaSetDevice(e->device);
    if (cudaEventSynchronize(e->ev_pk1) != cudaSuccess) return 0.0;
    float ms = 0;
    cudaEventElapsedTime(&ms, e->ev_pk0, e->ev_pk1);
    return ms;
}
double bplb_last_device_ms(bplb_engine* e) { return e ? e->last_ms : 0.0; }

// The grid-wide check on e->stream: direct launches the first time an argument
// set is seen, captured into a graph the second time, replayed after that.
int wide_check_graph(bplb_engine* e, bplb::KParams& p, int64_t r) {
    WideKey key;
    key.c = p.c; key.r = r; key.k = p.k; key.flags = p.flags; key.nk = p.nk;
    for (int i = 0; i < p.nk; ++i) key.kinds[i] = p.kinds[i];
    key.w = p.w; key.res = p.res_out; key.err = p.err_out; key.buf = e->d_wide.p; key.cap = e->d_wide.cap;
    key.use_range = p.use_range;
    for (int i = 0; i < 6; ++i) {
        key.rlo[i] = p.rng_lo[i];
        key.rhi[i] = p.rng_hi[i];
    }
    auto direct = [&]() {
        int rc = bplb::wide_check(e->stream, e->num_sms, &e->d_wide.p, &e->d_wide.cap, &e->launches, p, r,
                                  &e->wide_cnt_zero);
        return rc ? fail(rc, bplb::wide_error()) : 0;
    };
    if (!e->graphs_ok || e->prof_kernel) return direct();
    if (!(e->wide_exec && e->wide_key == key)) {
        if (!(e->wide_seen == key)) {
            e->wide_seen = key;
            return direct();
        }
        if (e->wide_exec) cudaGraphExecDestroy(e->wide_exec);
        e->wide_exec = nullptr;
        if (int rc = direct()) return rc;  // (this call's result; the capture below only records)
        cudaGraph_t g = nullptr;
        if (cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
            cudaGetLastError();
            e->graphs_ok = false;
            return 0;
        }
        const int64_t l0 = e->launches;
        const int rc = bplb::wide_check(e->stream, e->num_sms, &e->d_wide.p, &e->d_wide.cap, &e->launches, p, r,
                                        &e->wide_cnt_zero);
        cudaError_t ce = cudaStreamEndCapture(e->stream, &g);
        e->wide_exec_launches = e->launches - l0;
        e->launches = l0;
        if (!rc && ce == cudaSuccess) ce = cudaGraphInstantiate(&e->wide_exec, g, 0);
        if (g) cudaGraphDestroy(g);
        if (rc || ce != cudaSuccess || e->d_wide.p != key.buf) {
            cudaGetLastError();
            if (e->wide_exec) cudaGraphExecDestroy(e->wide_exec);
            e->wide_exec = nullptr;
            e->graphs_ok = rc == 0 && ce == cudaSuccess;
        } else {
            e->wide_key = key;
        }
        return 0;
    }
    // replay: the histogram counts must be zero up to c + 2 (another instance
    // size may have reused those bytes since the capture)
    if (e->wide_cnt_zero < p.c + 2) {
        bplb::WideBufs b = bplb::wide_carve(e->d_wide.p, r, p.c);
        CUDA_TRY(cudaMemsetAsync(b.cnt + e->wide_cnt_zero, 0, (size_t)(p.c + 2 - e->wide_cnt_zero) * 4, e->stream));
    }
    e->wide_cnt_zero = p.c + 2;  // (this layout's other arrays reuse the bytes past it)
    cudaError_t ce = cudaGraphLaunch(e->wide_exec, e->stream);
    if (ce != cudaSuccess) return fail(BPLB_ECUDA, std::string("graph launch: ") + cudaGetErrorString(ce));
    e->launches += e->wide_exec_launches;
    return 0;
}

static int check_impl(bplb_engine* e, const int32_t* w, int64_t r, int64_t c, int64_t k, const int32_t* kinds,
                      int32_t nkinds, int32_t flags, const int64_t* rng_lo, const int64_t* rng_hi,
                      bplb_result* out);

int bplb_check(bplb_engine* e, const int32_t* w, int64_t r, int64_t c, int64_t k,
               const int32_t* kinds, int32_t nkinds, int32_t flags, bplb_result* out) {
    return check_impl(e, w, r, c, k, kinds, nkinds, flags, nullptr, nullptr, out);
}

int bplb_check_ranges(bplb_engine* e, const int32_t* w, int64_t r, int64_t c, int64_t k, const int32_t* kinds,
                      int32_t nkinds, int32_t flags, const int64_t* rng_lo, const int64_t* rng_hi,
                      bplb_result* out) {
    if (!rng_lo || !rng_hi) return fail(BPLB_EINVAL, "null lambda ranges");
    if (flags & (BPLB_F_PHASED | BPLB_F_CANCEL)) return fail(BPLB_EINVAL, "lambda ranges: full collection only");
    for (int kd = 0; kd < K_COUNT; ++kd) {
        int64_t lo, hi;
        bplb_domain(kd, c, &lo, &hi);
        if (rng_hi[kd] >= rng_lo[kd] && (rng_lo[kd] < lo || rng_hi[kd] > hi))
            return fail(BPLB_ERANGE, "lambda range outside the kind's domain");
    }
    return check_impl(e, w, r, c, k, kinds, nkinds, flags, rng_lo, rng_hi, out);
}

static int check_impl(bplb_engine* e, const int32_t* w, int64_t r, int64_t c, int64_t k, const int32_t* kinds,
                      int32_t nkinds, int32_t flags, const int64_t* rng_lo, const int64_t* rng_hi,
                      bplb_result* out) {
    if (!e || !out) return fail(BPLB_EINVAL, "null engine or output");
    if (r < 0 || (r > 0 && !w)) return fail(BPLB_EINVAL, "bad weight array");
    if (r > BPLB_MAX_R) return fail(BPLB_ERANGE, "too many items for the GPU envelope");
    if (int rc = check_c(c)) return rc;
    int ks[K_COUNT];
    if (int rc = check_kinds(kinds, nkinds, ks)) return rc;
    // every bound is <= r (f(w) <= f(c) for w <= c), so with k >= r no kind
    // can exceed k: the early-exit / cancellation guards are moot
    if (k >= r) flags &= ~(BPLB_F_PHASED | BPLB_F_CANCEL);
    std::lock_guard<std::mutex> lock(e->mu);
    CUDA_TRY(cudaSetDevice(e->device));
    if (int rc = join_stream(e, e->stream)) return rc;
    const bool timing = flags & BPLB_F_TIMING;
    if (int rc = e->d_w.grow((size_t)std::max<int64_t>(r, 1) * 4 + 64)) return rc;
    if (int rc = e->d_res.grow(sizeof(bplb_result) + 16)) return rc;
    if (int rc = e->d_err.grow(16)) return rc;
    if (int rc = e->h_res.grow(sizeof(bplb_result) + 16)) return rc;
    if (timing) CUDA_TRY(cudaEventRecord(e->ev0, e->stream));
    bplb::KParams p;
    fill_params(p, c, k, ks, nkinds, flags);
    if (rng_lo) {  // per-kind lambda ranges (a slice of a lambda-split check): node or grid-wide path
        p.use_range = 1;
        for (int kd = 0; kd < K_COUNT; ++kd) {
            p.rng_lo[kd] = rng_lo[kd];
            p.rng_hi[kd] = rng_hi[kd];
        }
    }
    int rc;
    const int64_t maxf = (tab_kmask(p) >> K_FS1 & 1) ? 101 * c : 2 * c;
    const bool small_tab = !rng_lo && c <= bplb::TAB_MAX_C && r <= 65535 && r * maxf < (1ll << 23) &&
                           !(flags & BPLB_F_NOTAB) && tab_warps(e, ((int)c + 3) / 4 * 4) >= 2;
    if (small_tab) {
        // small capacity: the cached table, one CTA per 64-column sub-chunk;
        // weights and result travel through mapped pinned memory
        if ((rc = tab_ensure(e, p))) return rc;
        if ((rc = e->d_skeys.grow(64))) return rc;
        if (!e->skeys_zeroed) {
            CUDA_TRY(cudaMemsetAsync(e->d_skeys.p, 0, 64, e->stream));
            e->skeys_zeroed = true;
        }
        const size_t woff = 256 + sizeof(bplb_result);  // [result][err] [weights]
        if (e->single_cluster_ok && e->tab_nsub <= 16) {
            // histogram built here (host-validated weights) and passed by
            // value to one cluster of nsub CTAs; result in mapped memory
            bplb::SingleHist hist;
            std::memset(&hist, 0, sizeof(hist));
            for (int64_t i = 0; i < r; ++i) {
                const int32_t x = w[i];
                if (x < 1 || x > c) return fail(BPLB_EINVAL, "reduced weight outside [1, c]");
                ++hist.h[x - 1];  // r <= 65535
            }
            if ((rc = e->m_single.grow(woff))) return rc;
            p.res_out = (bplb_result*)e->m_single.d;
            p.err_out = nullptr;
            const bplb::TabDev t = tab_dev(e, p, 1);
            if (!e->single_cluster_attr) {
                CUDA_TRY(cudaFuncSetAttribute(bplb::tab_single_cluster_kernel,
                                              cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
                e->single_cluster_attr = true;
            }
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)e->tab_nsub);
            cfg.blockDim = dim3(bplb::TAB_SNT);
            cfg.dynamicSmemBytes = (size_t)e->tab_KV * 4 + 16 * 64 * 4;
            cfg.stream = e->stream;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = (unsigned)e->tab_nsub;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaError_t ce = cudaLaunchKernelEx(&cfg, bplb::tab_single_cluster_kernel, p, t, hist);
            if (ce == cudaSuccess) {
                e->launches++;
                e->last_path = BPLB_PATH_TAB_SINGLE;
                e->last_detail = e->tab_nsub;
                if (timing) CUDA_TRY(cudaEventRecord(e->ev1, e->stream));
                CUDA_TRY(cudaStreamSynchronize(e->stream));
                if (timing) {
                    float ms = 0;
                    cudaEventElapsedTime(&ms, e->ev0, e->ev1);
                    e->last_ms = ms;
                }
                std::memcpy(out, e->m_single.h, sizeof(bplb_result));
                return 0;
            }
            cudaGetLastError();  // no cluster of this size here: the counter-based kernel below
            e->single_cluster_ok = false;
        }
        if ((rc = e->m_single.grow(woff + (size_t)r * 4))) return rc;
        if (r > 0) std::memcpy((char*)e->m_single.h + woff, w, (size_t)r * 4);
        p.w = (const int*)((char*)e->m_single.d + woff);
        p.res_out = (bplb_result*)e->m_single.d;
        p.err_out = (int*)((char*)e->m_single.d + sizeof(bplb_result));
        bplb::TabDev t = tab_dev(e, p, 1);
        const int KV = e->tab_KV;
        bplb::tab_single_kernel<<<(unsigned)e->tab_nsub, bplb::TAB_SNT, (size_t)KV * 4 + 16 * 64 * 4, e->stream>>>(
            p, t, (int)r, (unsigned*)e->d_skeys.p, (int*)e->d_skeys.p + 8);
        e->launches++;
        e->last_path = BPLB_PATH_TAB_SINGLE;
        e->last_detail = 0;
        CUDA_TRY(cudaGetLastError());
        if (timing) CUDA_TRY(cudaEventRecord(e->ev1, e->stream));
        CUDA_TRY(cudaStreamSynchronize(e->stream));
        if (timing) {
            float ms = 0;
            cudaEventElapsedTime(&ms, e->ev0, e->ev1);
            e->last_ms = ms;
        }
        if (*(volatile int*)((char*)e->m_single.h + sizeof(bplb_result)))
            return fail(BPLB_EINVAL, "reduced weight outside [1, c]");
        std::memcpy(out, e->m_single.h, sizeof(bplb_result));
        return 0;
    }
    // weights through the pinned staging buffer (the copy stays asynchronous)
    if (int rc2 = e->h_stage.grow((size_t)r * 4 + 64)) return rc2;
    // the grid-wide path for nodes beyond the node-resident kernels, and for
    // full-collection checks it can prune (seeded keys + bound tests): one
    // launch sequence over all SMs beats the multi-CTA node kernel's phase
    // hand-offs there (cfg3: r = 1e3, c = 1e5)
    const bool wide_prunes = !(flags & (BPLB_F_PHASED | BPLB_F_CANCEL | BPLB_F_NOPRUNE)) &&
                             c <= bplb::WIDE_PRUNE_MAX_C && r <= bplb::WIDE_PRUNE_MAX_R &&
                             r * c >= e->wide_prune_min_cells;
    if (!node_fits(r, c) || wide_prunes) {
        if (r > 0) {
            std::memcpy(e->h_stage.p, w, (size_t)r * 4);
            CUDA_TRY(cudaMemcpyAsync(e->d_w.p, e->h_stage.p, (size_t)r * 4, cudaMemcpyHostToDevice, e->stream));
        }
        p.w = (const int*)e->d_w.p;
        p.res_out = (bplb_result*)e->d_res.p;
        p.err_out = (int*)((char*)e->d_res.p + sizeof(bplb_result));  // copied back with the result
        CUDA_TRY(cudaMemsetAsync(p.err_out, 0, 4, e->stream));
        e->last_path = BPLB_PATH_WIDE;
        rc = wide_check_graph(e, p, r);
        if (rc) return rc;
    } else {
        // single node, multi-CTA: the offsets travel with the weights (one
        // H2D copy), the cross-CTA state is zeroed by the kernel's last CTA
        // for the next call (here only on first use or after a failure), and
        // the result and the error word land in mapped pinned memory
        if ((rc = e->d_multi.grow(sizeof(bplb::MultiState)))) return rc;
        if ((rc = e->m_nres.grow(sizeof(bplb_result) + 16))) return rc;
        if (e->multi_dirty) CUDA_TRY(cudaMemsetAsync(e->d_multi.p, 0, sizeof(bplb::MultiState), e->stream));
        int64_t* hs = (int64_t*)e->h_stage.p;
        hs[0] = 0;
        hs[1] = r;
        if (r > 0) std::memcpy(hs + 2, w, (size_t)r * 4);  // (h_stage holds r * 4 + 64 bytes)
        CUDA_TRY(cudaMemcpyAsync(e->d_w.p, hs, 16 + (size_t)r * 4, cudaMemcpyHostToDevice, e->stream));
        p.off = (const int64_t*)e->d_w.p;
        p.w = (const int*)((const char*)e->d_w.p + 16);
        p.res_out = (bplb_result*)e->m_nres.d;
        p.err_out = (int*)((char*)e->m_nres.d + sizeof(bplb_result));
        p.ms = (bplb::MultiState*)e->d_multi.p;
        e->multi_dirty = true;
        if ((rc = launch_node(e, p, 1, r, 0, true))) return rc;
        if (timing) CUDA_TRY(cudaEventRecord(e->ev1, e->stream));
        CUDA_TRY(cudaStreamSynchronize(e->stream));
        e->multi_dirty = false;
        if (timing) {
            float ms = 0;
            cudaEventElapsedTime(&ms, e->ev0, e->ev1);
            e->last_ms = ms;
        }
        if (*(volatile int*)((char*)e->m_nres.h + sizeof(bplb_result)))
            return fail(BPLB_EINVAL, "reduced weight outside [1, c]");
        std::memcpy(out, e->m_nres.h, sizeof(bplb_result));
        return 0;
    }
    CUDA_TRY(cudaMemcpyAsync(e->h_res.p, e->d_res.p, sizeof(bplb_result) + 4, cudaMemcpyDeviceToHost,
                             e->stream));
    if (timing) CUDA_TRY(cudaEventRecord(e->ev1, e->stream));
    CUDA_TRY(cudaStreamSynchronize(e->stream));
    if (timing) {
        float ms = 0;
        cudaEventElapsedTime(&ms, e->ev0, e->ev1);
        e->last_ms = ms;
    }
    int err = *(int*)((char*)e->h_res.p + sizeof(bplb_result));
    if (err) return fail(BPLB_EINVAL, "reduced weight outside [1, c]");
    std::memcpy(out, e->h_res.p, sizeof(bplb_result));
    return 0;
}

int bplb_dff_bound_batch(bplb_engine* e, int32_t kind, const int32_t* w, int64_t r, int64_t c,
                         int64_t lo, int64_t hi, int64_t* out) {
    if (!e) return fail(BPLB_EINVAL, "null engine");
    if (kind < 0 || kind >= K_COUNT) return fail(BPLB_EINVAL, "kind id out of range");
    if (r < 0 || (r > 0 && !w)) return fail(BPLB_EINVAL, "bad weight array");
    if (r > BPLB_MAX_R) return fail(BPLB_ERANGE, "too many items for the GPU envelope");
    if (int rc = check_c(c)) return rc;
    if (hi < lo) return 0;
    if (!out) return fail(BPLB_EINVAL, "null output");
    int64_t dlo, dhi;
    bplb_domain(kind, c, &dlo, &dhi);
    if (lo < dlo || hi > dhi)
        return fail(BPLB_EINVAL, "lambda range outside the parameter domain of the kind");
    std::lock_guard<std::mutex> lock(e->mu);
    CUDA_TRY(cudaSetDevice(e->device));
    if (int rc = join_stream(e, e->stream)) return rc;
    const int64_t L = hi - lo + 1;
    int rc;
    if ((rc = e->d_w.grow((size_t)std::max<int64_t>(r, 1) * 4 + 64))) return rc;
    if ((rc = e->d_res.grow(sizeof(bplb_result) + 16))) return rc;
    if ((rc = e->d_err.grow(16))) return rc;
    if ((rc = e->d_lam.grow((size_t)L * 8))) return rc;
    if ((size_t)r * 4 > 65536 && (rc = e->h_stage.grow((size_t)r * 4 + 64))) return rc;
    if ((rc = h2d(e, e->d_w.p, w, (size_t)r * 4))) return rc;
    CUDA_TRY(cudaMemsetAsync(e->d_err.p, 0, 4, e->stream));
    bplb::KParams p;
    int ks[1] = {kind};
    fill_params(p, c, 0, ks, 1, 0);
    p.w = (const int*)e->d_w.p;
    p.res_out = (bplb_result*)e->d_res.p;
    p.err_out = (int*)e->d_err.p;
    p.lam_out = (int64_t*)e->d_lam.p;
    p.out_lo = lo;
    p.out_hi = hi;
    p.use_range = 1;
    for (int kd = 0; kd < K_COUNT; ++kd) {
        p.rng_lo[kd] = lo;
        p.rng_hi[kd] = kd == kind ? hi : lo - 1;
    }
    if (r == 0) {  // bounds.py:478-479
        CUDA_TRY(cudaMemsetAsync(e->d_lam.p, 0, (size_t)L * 8, e->stream));
    } else if (!node_fits(r, c)) {
        e->last_path = BPLB_PATH_WIDE;
        rc = bplb::wide_check(e->stream, e->num_sms, &e->d_wide.p, &e->d_wide.cap, &e->launches,
                              p, r, &e->wide_cnt_zero);
        if (rc) return fail(rc, bplb::wide_error());
    } else {
        int64_t off_h[2] = {0, r};
        if ((rc = e->d_off.grow(16))) return rc;
        if ((rc = e->d_multi.grow(sizeof(bplb::MultiState)))) return rc;
        CUDA_TRY(cudaMemcpyAsync(e->d_off.p, off_h, 16, cudaMemcpyHostToDevice, e->stream));
        CUDA_TRY(cudaMemsetAsync(e->d_multi.p, 0, sizeof(bplb::MultiState), e->stream));
        p.off = (const int64_t*)e->d_off.p;
        p.ms = (bplb::MultiState*)e->d_multi.p;
        if ((rc = launch_node(e, p, 1, r, 0, true))) return rc;
    }
    int err = 0;
    CUDA_TRY(cudaMemcpyAsync(out, e->d_lam.p, (size_t)L * 8, cudaMemcpyDeviceToHost, e->stream));
    CUDA_TRY(cudaMemcpyAsync(&err, e->d_err.p, 4, cudaMemcpyDeviceToHost, e->stream));
    CUDA_TRY(cudaStreamSynchronize(e->stream));
    if (err) return fail(BPLB_EINVAL, "reduced weight outside [1, c]");
    return 0;
}

int bplb_check_batch_device(bplb_engine* e, const int32_t* d_w, const int64_t* d_off,
                            int64_t n_nodes, int64_t max_r, int64_t c, int64_t k,
                            const int32_t* kinds, int32_t nkinds, int32_t flags, int64_t* d_lb,
                            uint8_t* d_ex, int64_t* d_best, int64_t* d_arg, void* stream) {
    return bplb_check_batch_device_ex(e, d_w, 4, d_off, n_nodes, max_r, c, k, kinds, nkinds, flags,
                                      d_lb, d_ex, d_best, d_arg, stream);
}

int bplb_check_batch_device_ex(bplb_engine* e, const void* d_w, int32_t wbytes, const int64_t* d_off,
                               int64_t n_nodes, int64_t max_r, int64_t c, int64_t k,
                               const int32_t* kinds, int32_t nkinds, int32_t flags, int64_t* d_lb,
                               uint8_t* d_ex, int64_t* d_best, int64_t* d_arg, void* stream) {
    if (wbytes != 4 && wbytes != 2 && wbytes != 1) return fail(BPLB_EINVAL, "wbytes must be 4, 2 or 1");
    if (!e) return fail(BPLB_EINVAL, "null engine");
    if (n_nodes < 0 || max_r < 0) return fail(BPLB_EINVAL, "bad batch shape");
    if (int rc = check_c(c)) return rc;
    int ks[K_COUNT] = {0, 0, 0, 0, 0, 0};
    if (int rc = check_kinds(kinds, nkinds, ks)) return rc;
    if (n_nodes == 0) return 0;
    cudaStream_t s = stream ? (cudaStream_t)stream : e->stream;
    std::lock_guard<std::mutex> lock(e->mu);
    CUDA_TRY(cudaSetDevice(e->device));
    if (int rc = join_stream(e, s)) return rc;
    bplb::KParams p;
    fill_params(p, c, k, ks, nkinds, flags);
    p.w = (const int*)d_w;
    p.wbytes = wbytes;
    p.off = d_off;
    p.lb_out = d_lb;
    p.ex_out = d_ex;
    p.best_out = d_best;
    p.arg_out = d_arg;
    if (int rc = e->d_err.grow(16)) return rc;
    p.err_out = (int*)e->d_err.p;
    cudaStream_t saved = e->stream;
    e->stream = s;
    int rc;
    if (e->graphs_ok && !e->prof_kernel && tab_path(e, p, n_nodes, max_r) && !(flags & BPLB_F_NOTAB)) {
        // the table path's three launches replayed from a CUDA graph while
        // the arguments repeat (a search loop / the bench): one launch call
        // instead of three, captured once per argument set
        rc = tab_ensure(e, p);
        if (!rc) rc = tab_reserve(e, n_nodes);
        if (!rc) rc = launch_tab_graph(e, p, n_nodes, max_r, ks, nkinds, d_w, d_off);
    } else {
        rc = launch_node(e, p, n_nodes, max_r, 0);
    }
    e->stream = saved;
    if (!rc) rc = mark_tail(e, s);  // asynchronous: later calls on other streams order after it
    return rc;
}

int bplb_check_batch_ex(bplb_engine* e, const void* w, int32_t wbytes, const int64_t* off,
                        int64_t n_nodes, int64_t c, int64_t k, const int32_t* kinds, int32_t nkinds,
                        int32_t flags, int64_t* lb_out, uint8_t* ex_out, int64_t* best_out,
                        int64_t* arg_out) {
    if (wbytes != 4 && wbytes != 2 && wbytes != 1) return fail(BPLB_EINVAL, "wbytes must be 4, 2 or 1");
    if (!e) return fail(BPLB_EINVAL, "null engine");
    if (n_nodes < 0 || (n_nodes > 0 && (!off || !lb_out || !ex_out)))
        return fail(BPLB_EINVAL, "bad batch arguments");
    if (int rc = check_c(c)) return rc;
    int ks[K_COUNT];
    if (int rc = check_kinds(kinds, nkinds, ks)) return rc;
    if (n_nodes == 0) return 0;
    if (off[0] != 0) return fail(BPLB_EINVAL, "offsets[0] must be 0");
    int64_t max_r = 0, min_d = 0;
    for (int64_t i = 0; i < n_nodes; ++i) {  // branch-free: vectorises
        const int64_t d = off[i + 1] - off[i];
        max_r = d > max_r ? d : max_r;
        min_d = d < min_d ? d : min_d;
    }
    if (min_d < 0) return fail(BPLB_EINVAL, "offsets must be non-decreasing");
    if (max_r > BPLB_MAX_R) return fail(BPLB_ERANGE, "too many items in a node for the GPU envelope");
    if (k >= max_r) flags &= ~(BPLB_F_PHASED | BPLB_F_CANCEL);  // no node can exceed k
    const int64_t total = off[n_nodes];
    if (total > 0 && !w) return fail(BPLB_EINVAL, "null weights");
    std::lock_guard<std::mutex> lock(e->mu);
    CUDA_TRY(cudaSetDevice(e->device));
    if (int rc = join_stream(e, e->stream)) return rc;
    int rc;
    const bool timing = flags & BPLB_F_TIMING;
    if ((rc = e->d_w.grow((size_t)std::max<int64_t>(total, 1) * 4 + 64))) return rc;
    const size_t wsz = (size_t)total * (size_t)wbytes;
    if ((rc = e->d_off.grow((size_t)(n_nodes + 1) * 8))) return rc;
    if ((rc = e->d_lb.grow((size_t)n_nodes * 8))) return rc;
    if ((rc = e->d_ex.grow((size_t)n_nodes))) return rc;
    if (best_out && (rc = e->d_best.grow((size_t)n_nodes * 48))) return rc;
    if (arg_out && (rc = e->d_arg.grow((size_t)n_nodes * 48))) return rc;
    if ((rc = e->d_err.grow(16))) return rc;
    const bool node_path = max_r <= ((c <= bplb::TABLE_MAX_C) ? NODE_R_MAX_TABLE : NODE_R_MAX_SORT);
    const bool pinned = wsz <= 65536 || is_pinned(w);
    if (!pinned && (rc = e->h_stage.grow(wsz + 64 + (size_t)(n_nodes + 1) * 8))) return rc;
    if (timing) CUDA_TRY(cudaEventRecord(e->ev0, e->stream));
    bplb::KParams p;
    fill_params(p, c, k, ks, nkinds, flags);
    p.w = (const int*)e->d_w.p;
    p.wbytes = wbytes;
    p.off = (const int64_t*)e->d_off.p;
    // outputs: written by the kernels straight into pinned caller buffers
    // (no copies), else into device buffers copied back at the end
    int64_t* lb_dev = (int64_t*)device_alias(lb_out);
    uint8_t* ex_dev = (uint8_t*)device_alias(ex_out);
    int64_t* best_dev = best_out ? (int64_t*)device_alias(best_out) : nullptr;
    int64_t* arg_dev = arg_out ? (int64_t*)device_alias(arg_out) : nullptr;
    p.lb_out = lb_dev ? lb_dev : (int64_t*)e->d_lb.p;
    p.ex_out = ex_dev ? ex_dev : (uint8_t*)e->d_ex.p;
    p.best_out = best_out ? (best_dev ? best_dev : (int64_t*)e->d_best.p) : nullptr;
    p.arg_out = arg_out ? (arg_dev ? arg_dev : (int64_t*)e->d_arg.p) : nullptr;
    if ((rc = e->m_err.grow(64))) return rc;
    *(volatile int*)e->m_err.h = 0;  // the previous call has completed (calls are synchronous)
    p.err_out = (int*)e->m_err.d;
    if (node_path && tab_path(e, p, n_nodes, max_r) && !(flags & BPLB_F_NOTAB)) {
        // table and key arrays for the whole batch before concurrent chunk launches
        if ((rc = tab_ensure(e, p))) return rc;
        if ((rc = tab_reserve(e, n_nodes))) return rc;
    }
    // Chunked upload on the copy stream, one kernel per chunk on its own
    // stream as soon as its bytes have landed: the PCIe transfer of chunk
    // i+1 overlaps the kernel of chunk i, and chunk kernels overlap each
    // other's tails.  Small batches use a single chunk.
    // table path with pinned caller buffers: the histogram pass reads the
    // weights and offsets over PCIe directly (zero-copy; measured 167 us vs
    // 184 us p50 for the chunked uploads on cfg2, and far less jitter)
    const void* w_alias = pinned ? device_alias(w) : nullptr;
    const void* off_alias = w_alias ? device_alias(off) : nullptr;
    if (w_alias && off_alias && !((uintptr_t)w_alias & 15) && node_path && !(flags & BPLB_F_NOTAB)) {
        bplb::KParams q = p;
        q.w = (const int*)w_alias;
        q.off = (const int64_t*)off_alias;
        // weights read across PCIe: the FP32-pipe pipeline, whose persistent
        // histogram pass streams the tiles while the contraction consumes
        // them, is PCIe-bound; the tensor-core kernel's per-slice histograms
        // would wait on PCIe latency (measured 266 vs 132 us on cfg2)
        q.flags |= BPLB_F_NOTC;
        if (tab_path(e, q, n_nodes, max_r)) {
            if ((rc = launch_tab_graph(e, q, n_nodes, max_r, ks, nkinds, w_alias, off_alias))) return rc;
            goto outputs;
        }
    }
    {
    int nch = node_path && n_nodes >= 4096 && wsz >= (size_t)1 << 20 ? 4 : 1;
    int64_t bounds_[5];
    for (int i = 0; i <= nch; ++i) bounds_[i] = n_nodes * i / nch;
    if (nch > 1) {
        // a smaller first chunk starts the GPU sooner
        bounds_[1] = n_nodes / 8;
        bounds_[2] = n_nodes * 3 / 8;
        bounds_[3] = n_nodes * 5 / 8;
    }
    for (int i = 1; i < nch; ++i) bounds_[i] = bounds_[i] / 16 * 16;  // table path: whole 16-node tiles
    CUDA_TRY(cudaEventRecord(e->ev_k[0], e->stream));  // memset done before uploads land
    CUDA_TRY(cudaStreamWaitEvent(e->copy_stream, e->ev_k[0], 0));
    if ((rc = h2d(e, e->d_off.p, off, (size_t)(n_nodes + 1) * 8, wsz + 64, e->copy_stream, pinned ? 1 : 0)))
        return rc;
    for (int i = 0; i < nch; ++i) {
        const int64_t a = off[bounds_[i]], b = off[bounds_[i + 1]];
        if ((rc = h2d(e, (char*)e->d_w.p + a * wbytes, (const char*)w + a * wbytes, (size_t)(b - a) * wbytes,
                      (size_t)a * wbytes, e->copy_stream, pinned ? 1 : 0)))
            return rc;
        CUDA_TRY(cudaEventRecord(e->ev_up[i], e->copy_stream));
    }
    const bool tab = node_path && !(flags & BPLB_F_NOTAB) && tab_path(e, p, n_nodes, max_r);
    if (node_path) {
        cudaStream_t saved = e->stream;
        for (int i = 0; i < nch; ++i) {
            // the table kernel occupies every SM: its chunk launches stay on
            // one stream (PDL-chained), each behind its upload
            cudaStream_t cs = (nch == 1 || tab) ? saved : e->cstream[i];
            CUDA_TRY(cudaStreamWaitEvent(cs, e->ev_up[i], 0));
            bplb::KParams q = p;
            q.node0 = bounds_[i];
            e->stream = cs;
            rc = launch_node(e, q, bounds_[i + 1] - bounds_[i], max_r, 0, false, i);
            e->stream = saved;
            if (rc) return rc;
            if (nch > 1 && !tab) {
                CUDA_TRY(cudaEventRecord(e->ev_k[i], cs));
                CUDA_TRY(cudaStreamWaitEvent(saved, e->ev_k[i], 0));
            }
        }
    } else {
        CUDA_TRY(cudaStreamWaitEvent(e->stream, e->ev_up[0], 0));
        if (wbytes != 4) return fail(BPLB_ERANGE, "nodes above the node-resident envelope need int32 weights");
        // nodes beyond the node-resident envelope go one by one through the
        // grid-wide path (rare: r > 8192)
        for (int64_t i = 0; i < n_nodes; ++i) {
            bplb::KParams q = p;
            q.w = (const int*)e->d_w.p + off[i];
            q.lb_out = p.lb_out + i;
            q.ex_out = p.ex_out + i;
            q.best_out = p.best_out ? p.best_out + i * K_COUNT : nullptr;
            q.arg_out = p.arg_out ? p.arg_out + i * K_COUNT : nullptr;
            e->last_path = BPLB_PATH_WIDE;
            rc = bplb::wide_check(e->stream, e->num_sms, &e->d_wide.p, &e->d_wide.cap,
                                  &e->launches, q, off[i + 1] - off[i], &e->wide_cnt_zero);
            if (rc) return fail(rc, bplb::wide_error());
        }
    }
    }
outputs:
    if (!lb_dev) CUDA_TRY(cudaMemcpyAsync(lb_out, e->d_lb.p, (size_t)n_nodes * 8, cudaMemcpyDeviceToHost, e->stream));
    if (!ex_dev) CUDA_TRY(cudaMemcpyAsync(ex_out, e->d_ex.p, (size_t)n_nodes, cudaMemcpyDeviceToHost, e->stream));
    if (best_out && !best_dev)
        CUDA_TRY(cudaMemcpyAsync(best_out, e->d_best.p, (size_t)n_nodes * 48, cudaMemcpyDeviceToHost, e->stream));
    if (arg_out && !arg_dev)
        CUDA_TRY(cudaMemcpyAsync(arg_out, e->d_arg.p, (size_t)n_nodes * 48, cudaMemcpyDeviceToHost, e->stream));
    if (timing) CUDA_TRY(cudaEventRecord(e->ev1, e->stream));
    CUDA_TRY(cudaStreamSynchronize(e->stream));
    if (timing) {
        float ms = 0;
        cudaEventElapsedTime(&ms, e->ev0, e->ev1);
        e->last_ms = ms;
    }
    if (*(volatile int*)e->m_err.h) return fail(BPLB_EINVAL, "reduced weight outside [1, c]");
    return 0;
}

int bplb_check_batch_assign(bplb_engine* e, const int32_t* inst_w, int64_t n_items, int64_t n_bins,
                            const void* assign, int32_t abytes, int64_t n_nodes, int64_t c, int64_t k,
                            const int32_t* kinds, int32_t nkinds, int32_t flags, int64_t* lb_out,
                            uint8_t* ex_out, int64_t* best_out, int64_t* arg_out) {
    if (!e) return fail(BPLB_EINVAL, "null engine");
    if (n_nodes < 0 || (n_nodes > 0 && (!lb_out || !ex_out || !assign || (n_items > 0 && !inst_w))))
        return fail(BPLB_EINVAL, "bad batch arguments");
    if (int rc = check_c(c)) return rc;
    int ks[K_COUNT];
    if (int rc = check_kinds(kinds, nkinds, ks)) return rc;
    if (n_nodes == 0) return 0;
    std::lock_guard<std::mutex> lock(e->mu);
    CUDA_TRY(cudaSetDevice(e->device));
    if (int rc = join_stream(e, e->stream)) return rc;
    const bool timing = flags & BPLB_F_TIMING;
    if (timing) CUDA_TRY(cudaEventRecord(e->ev0, e->stream));
    int obytes = 4, rc;
    if ((rc = e->m_err.grow(64))) return rc;
    // table path: histograms straight from the assignments (no reduced CSR);
    // pinned assignments are read across PCIe (zero-copy), outputs written
    // into pinned caller buffers
    {
        bplb::KParams q;
        fill_params(q, c, k, ks, nkinds, flags);
        const int64_t maxf = (tab_kmask(q) >> K_FS1 & 1) ? 101 * c : 2 * c;
        const bool tab = !(flags & BPLB_F_NOTAB) && (abytes == 1 || abytes == 2) && c <= bplb::TAB_MAX_C &&
                         n_items <= 65535 && std::max<int64_t>(n_items, 1) * maxf < (1ll << 23) &&
                         n_bins <= bplb::TAB_ASSIGN_MAX_BINS && n_bins < (abytes == 1 ? 255 : 65535) &&
                         n_nodes >= 256 && n_nodes <= ((int64_t)1 << 30) && tab_warps(e, ((int)c + 3) / 4 * 4) >= 2 &&
                         // the histogram kernel's shared memory (16 node rows, the instance, 16 x bins)
                         ((size_t)bplb::TAB_TM * (((c + 3) / 4 * 4) + 1) + ((n_items + 3) & ~3) +
                          (size_t)bplb::TAB_TM * n_bins) * 4 + 64 <= e->smem_optin;
        if (tab) {
            const void* a_dev = device_alias(assign);
            const size_t asz = (size_t)n_nodes * (size_t)n_items * (size_t)abytes;
            if (!a_dev || ((uintptr_t)a_dev & 15)) {
                if ((rc = e->d_assign.grow(std::max<size_t>(asz, 16)))) return rc;
                if (asz > 65536 && !is_pinned(assign) && (rc = e->h_stage.grow(asz + 64))) return rc;
                if ((rc = h2d(e, e->d_assign.p, assign, asz))) return rc;
                a_dev = e->d_assign.p;
            }
            if ((rc = upload_inst(e, inst_w, n_items))) return rc;
            if ((rc = tab_ensure(e, q))) return rc;
            if ((rc = tab_reserve(e, n_nodes))) return rc;
            int64_t* lb_dev = (int64_t*)device_alias(lb_out);
            uint8_t* ex_dev = (uint8_t*)device_alias(ex_out);
            int64_t* best_dev = best_out ? (int64_t*)device_alias(best_out) : nullptr;
            int64_t* arg_dev = arg_out ? (int64_t*)device_alias(arg_out) : nullptr;
            if ((rc = e->d_lb.grow((size_t)n_nodes * 8))) return rc;
            if ((rc = e->d_ex.grow((size_t)n_nodes))) return rc;
            if (best_out && !best_dev && (rc = e->d_best.grow((size_t)n_nodes * 48))) return rc;
            if (arg_out && !arg_dev && (rc = e->d_arg.grow((size_t)n_nodes * 48))) return rc;
            q.lb_out = lb_dev ? lb_dev : (int64_t*)e->d_lb.p;
            q.ex_out = ex_dev ? ex_dev : (uint8_t*)e->d_ex.p;
            q.best_out = best_out ? (best_dev ? best_dev : (int64_t*)e->d_best.p) : nullptr;
            q.arg_out = arg_out ? (arg_dev ? arg_dev : (int64_t*)e->d_arg.p) : nullptr;
            int* herr = (int*)e->m_err.h;
            herr[0] = herr[1] = 0;
            q.err_out = (int*)e->m_err.d;
            q.n_nodes = n_nodes;
            const bplb::TabDev t = tab_dev(e, q, n_nodes);
            const int KV = e->tab_KV;
            const size_t hs = ((size_t)bplb::TAB_TM * (KV + 1) + ((n_items + 3) & ~3) + (size_t)bplb::TAB_TM * n_bins) * 4;
            auto hk = abytes == 1 ? bplb::tab_hist_assign_kernel<1> : bplb::tab_hist_assign_kernel<2>;
            if (hs > 48 * 1024) CUDA_TRY(cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hs));
            // persistent, one CTA per SM beside the tab_kernel CTA that
            // consumes its published tiles (max-shared carveout, as tab_hist)
            if (!e->assign_carveout) {
                CUDA_TRY(cudaFuncSetAttribute(bplb::tab_hist_assign_kernel<1>,
                                              cudaFuncAttributePreferredSharedMemoryCarveout,
                                              cudaSharedmemCarveoutMaxShared));
                CUDA_TRY(cudaFuncSetAttribute(bplb::tab_hist_assign_kernel<2>,
                                              cudaFuncAttributePreferredSharedMemoryCarveout,
                                              cudaSharedmemCarveoutMaxShared));
                e->assign_carveout = true;
            }
            hk<<<(unsigned)std::min<int64_t>(t.ntiles, e->num_sms), bplb::TAB_HNT, hs, e->stream>>>(
                q, t, (const int*)e->d_inst.p, (int)n_items, (int)n_bins, a_dev, (int*)e->m_err.d);
            e->launches++;
            CUDA_TRY(cudaGetLastError());
            if ((rc = tab_contract(e, q, n_nodes))) return rc;
            if ((rc = tab_fin(e, q, n_nodes))) return rc;
            if (!lb_dev) CUDA_TRY(cudaMemcpyAsync(lb_out, e->d_lb.p, (size_t)n_nodes * 8, cudaMemcpyDeviceToHost, e->stream));
            if (!ex_dev) CUDA_TRY(cudaMemcpyAsync(ex_out, e->d_ex.p, (size_t)n_nodes, cudaMemcpyDeviceToHost, e->stream));
            if (best_out && !best_dev)
                CUDA_TRY(cudaMemcpyAsync(best_out, e->d_best.p, (size_t)n_nodes * 48, cudaMemcpyDeviceToHost, e->stream));
            if (arg_out && !arg_dev)
                CUDA_TRY(cudaMemcpyAsync(arg_out, e->d_arg.p, (size_t)n_nodes * 48, cudaMemcpyDeviceToHost, e->stream));
            if (timing) CUDA_TRY(cudaEventRecord(e->ev1, e->stream));
            CUDA_TRY(cudaStreamSynchronize(e->stream));
            if (timing) {
                float ms = 0;
                cudaEventElapsedTime(&ms, e->ev0, e->ev1);
                e->last_ms = ms;
            }
            if (herr[1]) return fail(BPLB_EINVAL, reduce_error(herr[1]));
            if (herr[0]) return fail(BPLB_EINVAL, "instance weight outside [1, c]");
            return 0;
        }
    }
    if ((rc = reduce_device(e, inst_w, n_items, n_bins, assign, abytes, n_nodes, c, &obytes))) return rc;
    // r <= n_items for every node: the kernel choice uses that bound (no sync)
    const int64_t max_r = std::max<int64_t>(n_items, 1);
    if (k >= max_r) flags &= ~(BPLB_F_PHASED | BPLB_F_CANCEL);
    if ((rc = e->d_lb.grow((size_t)n_nodes * 8))) return rc;
    if ((rc = e->d_ex.grow((size_t)n_nodes))) return rc;
    if (best_out && (rc = e->d_best.grow((size_t)n_nodes * 48))) return rc;
    if (arg_out && (rc = e->d_arg.grow((size_t)n_nodes * 48))) return rc;
    bplb::KParams p;
    fill_params(p, c, k, ks, nkinds, flags);
    p.w = (const int*)e->d_w.p;
    p.wbytes = obytes;
    p.off = (const int64_t*)e->d_off.p;
    p.lb_out = (int64_t*)e->d_lb.p;
    p.ex_out = (uint8_t*)e->d_ex.p;
    p.best_out = best_out ? (int64_t*)e->d_best.p : nullptr;
    p.arg_out = arg_out ? (int64_t*)e->d_arg.p : nullptr;
    p.err_out = (int*)e->d_err.p;
    if (!node_fits(max_r, c)) return fail(BPLB_ERANGE, "instance larger than the node-resident envelope");
    if ((rc = launch_node(e, p, n_nodes, max_r, 0))) return rc;
    if ((rc = e->h_res.grow(sizeof(bplb_result) + 16))) return rc;
    int* h_err = (int*)((char*)e->h_res.p + sizeof(bplb_result));
    CUDA_TRY(cudaMemcpyAsync(lb_out, e->d_lb.p, (size_t)n_nodes * 8, cudaMemcpyDeviceToHost, e->stream));
    CUDA_TRY(cudaMemcpyAsync(ex_out, e->d_ex.p, (size_t)n_nodes, cudaMemcpyDeviceToHost, e->stream));
    if (best_out)
        CUDA_TRY(cudaMemcpyAsync(best_out, e->d_best.p, (size_t)n_nodes * 48, cudaMemcpyDeviceToHost, e->stream));
    if (arg_out)
        CUDA_TRY(cudaMemcpyAsync(arg_out, e->d_arg.p, (size_t)n_nodes * 48, cudaMemcpyDeviceToHost, e->stream));
    CUDA_TRY(cudaMemcpyAsync(h_err, e->d_err.p, 8, cudaMemcpyDeviceToHost, e->stream));
    if (timing) CUDA_TRY(cudaEventRecord(e->ev1, e->stream));
    CUDA_TRY(cudaStreamSynchronize(e->stream));
    if (timing) {
        float ms = 0;
        cudaEventElapsedTime(&ms, e->ev0, e->ev1);
        e->last_ms = ms;
    }
    if (h_err[1]) return fail(BPLB_EINVAL, reduce_error(h_err[1]));
    if (h_err[0]) return fail(BPLB_EINVAL, "instance weight outside [1, c]");
    return 0;
}

int bplb_reduce_batch(bplb_engine* e, const int32_t* inst_w, int64_t n_items, int64_t n_bins,
                      const void* assign, int32_t abytes, int64_t n_nodes, int64_t c, int64_t* off_out,
                      int32_t* w_out) {
    if (!e) return fail(BPLB_EINVAL, "null engine");
    if (n_nodes < 0 || !off_out || (n_nodes > 0 && (!assign || !w_out || (n_items > 0 && !inst_w))))
        return fail(BPLB_EINVAL, "bad batch arguments");
    if (int rc = check_c(c)) return rc;
    std::lock_guard<std::mutex> lock(e->mu);
    CUDA_TRY(cudaSetDevice(e->device));
    if (int rc = join_stream(e, e->stream)) return rc;
    off_out[0] = 0;
    if (n_nodes == 0) return 0;
    int obytes = 4, rc;
    if ((rc = reduce_device(e, inst_w, n_items, n_bins, assign, abytes, n_nodes, c, &obytes))) return rc;
    std::vector<int64_t> off((size_t)n_nodes + 1);
    int err[2] = {0, 0};
    CUDA_TRY(cudaMemcpyAsync(off.data(), e->d_off.p, off.size() * 8, cudaMemcpyDeviceToHost, e->stream));
    CUDA_TRY(cudaMemcpyAsync(err, e->d_err.p, 8, cudaMemcpyDeviceToHost, e->stream));
    CUDA_TRY(cudaStreamSynchronize(e->stream));
    if (err[1]) return fail(BPLB_EINVAL, reduce_error(err[1]));
    const int64_t total = off[(size_t)n_nodes];
    std::vector<unsigned char> buf((size_t)std::max<int64_t>(total, 1) * obytes);
    CUDA_TRY(cudaMemcpy(buf.data(), e->d_w.p, (size_t)total * obytes, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < total; ++i)
        w_out[i] = obytes == 1 ? buf[(size_t)i] : obytes == 2 ? ((const uint16_t*)buf.data())[i]
                                                              : ((const int32_t*)buf.data())[i];
    std::memcpy(off_out, off.data(), off.size() * 8);
    return 0;
}

int bplb_check_batch(bplb_engine* e, const int32_t* w, const int64_t* off, int64_t n_nodes,
                     int64_t c, int64_t k, const int32_t* kinds, int32_t nkinds, int32_t flags,
                     int64_t* lb_out, uint8_t* ex_out, int64_t* best_out, int64_t* arg_out) {
    return bplb_check_batch_ex(e, w, 4, off, n_nodes, c, k, kinds, nkinds, flags, lb_out, ex_out,
                               best_out, arg_out);
}


// ---- multi-GPU batched checks (one call, several devices) ------------------
// the batched path shards over the GPUs of one box.
// The nodes of a host CSR batch are split into contiguous ranges balanced
// by item count, each range checked by its own engine on its own host
// thread (bplb_check_batch_ex: upload, kernel, verdicts); the gather is the
// per-shard write of lb / exceeded / best / arg into the caller's arrays.
struct bplb_multi {
    std::vector<bplb_engine*> engines;
    std::vector<int64_t> bounds;  // node boundaries of the last call (size engines + 1)
    std::mutex mu;
};

int bplb_multi_create(const int32_t* devices, int32_t ndev, bplb_multi** out) {
    if (!out || !devices || ndev < 1 || ndev > 64) return fail(BPLB_EINVAL, "bad device list");
    *out = nullptr;
    bplb_multi* m = new bplb_multi();
    for (int32_t i = 0; i < ndev; ++i) {
        bplb_engine* e = nullptr;
        int rc = bplb_engine_create(devices[i], &e);
        if (rc) {
            std::string msg = g_err;
            bplb_multi_destroy(m);
            return fail(rc, msg);
        }
        m->engines.push_back(e);
    }
    m->bounds.assign((size_t)ndev + 1, 0);
    *out = m;
    return 0;
}

int bplb_multi_destroy(bplb_multi* m) {
    if (!m) return 0;
    for (bplb_engine* e : m->engines) bplb_engine_destroy(e);
    delete m;
    return 0;
}

int bplb_multi_engine(bplb_multi* m, int32_t i, bplb_engine** out) {
    if (!m || !out || i < 0 || i >= (int32_t)m->engines.size()) return fail(BPLB_EINVAL, "bad engine index");
    *out = m->engines[(size_t)i];
    return 0;
}

int bplb_multi_last_bounds(bplb_multi* m, int64_t* bounds_out) {
    if (!m || !bounds_out) return fail(BPLB_EINVAL, "null argument");
    std::lock_guard<std::mutex> lock(m->mu);
    std::memcpy(bounds_out, m->bounds.data(), m->bounds.size() * 8);
    return 0;
}

int bplb_check_batch_multi(bplb_multi* m, const void* w, int32_t wbytes, const int64_t* off,
                           int64_t n_nodes, int64_t c, int64_t k, const int32_t* kinds, int32_t nkinds,
                           int32_t flags, int64_t* lb_out, uint8_t* ex_out, int64_t* best_out,
                           int64_t* arg_out) {
    if (!m) return fail(BPLB_EINVAL, "null multi-engine");
    if (wbytes != 4 && wbytes != 2 && wbytes != 1) return fail(BPLB_EINVAL, "wbytes must be 4, 2 or 1");
    if (n_nodes < 0 || (n_nodes > 0 && (!off || !lb_out || !ex_out))) return fail(BPLB_EINVAL, "bad batch arguments");
    if (n_nodes == 0) return 0;
    if (off[0] != 0) return fail(BPLB_EINVAL, "offsets[0] must be 0");
    std::lock_guard<std::mutex> lock(m->mu);
    const int G = (int)m->engines.size();
    const int64_t total = off[n_nodes];
    // contiguous node ranges with ~total/G items each (at least one node each
    // while nodes last): boundary g = first node whose offset reaches g*total/G
    std::vector<int64_t>& b = m->bounds;
    b.assign((size_t)G + 1, 0);
    b[(size_t)G] = n_nodes;
    for (int g = 1; g < G; ++g) {
        const int64_t target = total / G * g + std::min<int64_t>(g, total % G);
        int64_t x = std::lower_bound(off, off + n_nodes + 1, target) - off;
        if (total == 0) x = n_nodes * g / G;
        x = std::max(x, b[(size_t)g - 1]);
        b[(size_t)g] = std::min(x, n_nodes);
    }
    std::vector<int> rcs((size_t)G, 0);
    std::vector<std::string> errs((size_t)G);
    std::vector<std::thread> th;
    for (int g = 0; g < G; ++g) {
        const int64_t lo = b[(size_t)g], hi = b[(size_t)g + 1];
        if (hi <= lo) continue;
        th.emplace_back([&, g, lo, hi]() {
            std::vector<int64_t> so((size_t)(hi - lo + 1));
            for (int64_t i = lo; i <= hi; ++i) so[(size_t)(i - lo)] = off[i] - off[lo];
            rcs[(size_t)g] = bplb_check_batch_ex(
                m->engines[(size_t)g], (const char*)w + off[lo] * wbytes, wbytes, so.data(), hi - lo, c, k, kinds,
                nkinds, flags, lb_out + lo, ex_out + lo, best_out ? best_out + lo * K_COUNT : nullptr,
                arg_out ? arg_out + lo * K_COUNT : nullptr);
            if (rcs[(size_t)g]) errs[(size_t)g] = g_err;
        });
    }
    for (auto& t : th) t.join();
    for (int g = 0; g < G; ++g)
        if (rcs[(size_t)g]) return fail(rcs[(size_t)g], "shard " + std::to_string(g) + ": " + errs[(size_t)g]);
    return 0;
}

// One reduced instance on every engine of m: each kind's lambda range cut into
// contiguous slices, one per engine, every slice a full bound-pruned check of
// its lambdas, the per-kind results merged on the host as an allreduce(MAX) of
// packed (best << 32 | ~arg) keys would.  PHASED is replayed
// on the merged per-kind results (kinds in order until the running max exceeds
// k); CANCEL runs the full collection (the guard only skips work).
int bplb_check_multi(bplb_multi* m, const int32_t* w, int64_t r, int64_t c, int64_t k, const int32_t* kinds,
                     int32_t nkinds, int32_t flags, bplb_result* out) {
    if (!m || !out) return fail(BPLB_EINVAL, "null multi-engine or output");
    if (r < 0 || (r > 0 && !w)) return fail(BPLB_EINVAL, "bad weight array");
    if (r > BPLB_MAX_R) return fail(BPLB_ERANGE, "too many items for the GPU envelope");
    if (int rc = check_c(c)) return rc;
    int ks[K_COUNT];
    if (int rc = check_kinds(kinds, nkinds, ks)) return rc;
    std::lock_guard<std::mutex> lock(m->mu);
    const int G = (int)m->engines.size();
    int64_t maxw = 0;
    for (int64_t i = 0; i < r; ++i) maxw = std::max<int64_t>(maxw, w[i]);
    int64_t dlo[K_COUNT], dhi[K_COUNT];
    bool in[K_COUNT] = {false, false, false, false, false, false};
    for (int i = 0; i < nkinds; ++i) in[ks[i]] = true;
    for (int kd = 0; kd < K_COUNT; ++kd) {
        bplb_domain(kd, c, &dlo[kd], &dhi[kd]);
        if (kd == K_VB2) dhi[kd] = bplb_vb2_hi(c, r, maxw);
        if (!in[kd]) dhi[kd] = dlo[kd] - 1;
    }
    const int32_t sflags = flags & ~(BPLB_F_PHASED | BPLB_F_CANCEL | BPLB_F_TIMING);
    std::vector<bplb_result> res((size_t)G);
    std::vector<int> rcs((size_t)G, 0);
    std::vector<std::string> errs((size_t)G);
    std::vector<std::thread> th;
    for (int g = 0; g < G; ++g) {
        th.emplace_back([&, g]() {
            int64_t lo[K_COUNT], hi[K_COUNT];
            for (int kd = 0; kd < K_COUNT; ++kd) {  // slice g of [dlo, dhi]: contiguous, near-equal
                const int64_t n = std::max<int64_t>(0, dhi[kd] - dlo[kd] + 1);
                lo[kd] = dlo[kd] + n * g / G;
                hi[kd] = dlo[kd] + n * (g + 1) / G - 1;
            }
            rcs[(size_t)g] = check_impl(m->engines[(size_t)g], w, r, c, k, kinds, nkinds, sflags, lo, hi,
                                        &res[(size_t)g]);
            if (rcs[(size_t)g]) errs[(size_t)g] = g_err;
        });
    }
    for (auto& t : th) t.join();
    for (int g = 0; g < G; ++g)
        if (rcs[(size_t)g]) return fail(rcs[(size_t)g], "slice " + std::to_string(g) + ": " + errs[(size_t)g]);
    bplb_result o;
    std::memset(&o, 0, sizeof(o));
    for (int kd = 0; kd < K_COUNT; ++kd) {
        unsigned long long key = 0;  // (best << 32 | 0xFFFFFFFF - (arg - lo)): the allreduce(MAX) operand
        for (int g = 0; g < G; ++g) {
            const bplb_result& x = res[(size_t)g];
            o.evals[kd] += x.evals[kd];
            if (!x.evaluated[kd]) continue;
            o.evaluated[kd] = 1;
            const unsigned long long kk = ((unsigned long long)x.best[kd] << 32) |
                                          (0xFFFFFFFFull - (unsigned long long)(x.arg_lambda[kd] - dlo[kd]));
            key = std::max(key, kk);
        }
        o.best[kd] = o.evaluated[kd] ? (int64_t)(key >> 32) : 0;
        o.arg_lambda[kd] = o.evaluated[kd] ? dlo[kd] + (int64_t)(0xFFFFFFFFull - (key & 0xFFFFFFFFull)) : dlo[kd];
        o.n_lambda[kd] = std::max<int64_t>(0, dhi[kd] - dlo[kd] + 1);
    }
    int nd = nkinds;
    int64_t lb = 0;
    for (int i = 0; i < nkinds; ++i) {
        const int kd = ks[i];
        if (o.evaluated[kd]) lb = std::max(lb, o.best[kd]);
        if ((flags & BPLB_F_PHASED) && lb > k) {
            nd = i + 1;
            break;
        }
    }
    if (flags & BPLB_F_PHASED)
        for (int i = nd; i < nkinds; ++i) {  // kinds the sequential sweep never reached
            const int kd = ks[i];
            o.evaluated[kd] = 0;
            o.evals[kd] = 0;
            o.best[kd] = 0;
            o.arg_lambda[kd] = dlo[kd];
        }
    o.lb = lb;
    o.exceeded = lb > k;
    o.n_done = nd;
    for (int kd = 0; kd < K_COUNT; ++kd) o.evals_total += o.evals[kd];
    *out = o;
    return 0;
}

#ifdef PRUNE_TRACE
// development builds: copy the prune-kernel unit trace (longlong4 records)
BPLB_API int bplb_prune_trace(long long* out, int cap) {
    int n = 0;
    cudaMemcpyFromSymbol(&n, bplb::g_prune_trace_n, sizeof(int));
    n = std::min(n, std::min(cap, bplb::PRUNE_TRACE_CAP));
    if (n > 0) cudaMemcpyFromSymbol(out, bplb::g_prune_trace, (size_t)n * sizeof(longlong4));
    int z = 0;
    cudaMemcpyToSymbol(bplb::g_prune_trace_n, &z, sizeof(int));
    return n;
}
#endif

#ifdef WIDE_TRACE
// development builds: copy the grid-wide unit trace and the segment table
BPLB_API int bplb_wide_trace(long long* out, int cap) {
    int n = 0;
    cudaMemcpyFromSymbol(&n, bplb::g_wide_trace_n, sizeof(int));
    n = std::min(n, std::min(cap, bplb::WIDE_TRACE_CAP));
    if (n > 0) cudaMemcpyFromSymbol(out, bplb::g_wide_trace, (size_t)n * sizeof(longlong4));
    int z = 0;
    cudaMemcpyToSymbol(bplb::g_wide_trace_n, &z, sizeof(int));
    return n;
}
#endif

#ifdef NODE_TRACE
BPLB_API int bplb_node_trace(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, bplb::g_node_trace, sizeof(bplb::g_node_trace));
    return 0;
}
#endif

#ifdef TC_TRACE
BPLB_API int bplb_tc_trace(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, bplb::g_tc_trace, 64 * 8);
    cudaMemcpyFromSymbol(out + 64, bplb::g_tc_cta, 256 * 3 * 8);
    return 0;
}
#endif

}  // extern "C"


// ---- batched exact knapsack reasoning per bin -----------
// propagator.py:98-224 (reachable_sums, knapsack_load_tightening,
// knapsack_item_filter, _knapsack_bin) for many bins in one launch;
// kernels in bplb_knap.cuh.
namespace {

int knap_launch(bplb_engine* e, cudaStream_t s, int64_t c, int64_t n_bins, int64_t max_items, int32_t flags,
                bplb::knap::KnParams& p) {
    using namespace bplb::knap;
    p.c = (int32_t)c;
    p.words = (int32_t)((c + 32) / 32);
    p.n_bins = n_bins;
    p.flags = flags & (KN_F_REACH_ONLY | KN_F_NO_TIGHTEN);
    const bool timing = flags & BPLB_F_TIMING;
    if (timing) CUDA_TRY(cudaEventRecord(e->ev0, s));
    if (p.words <= 32) {
        p.nbuf = 0;
        const int seg = p.words <= 8 ? 8 : p.words <= 16 ? 16 : 32;  // lanes per bin
        const size_t smem = (size_t)KN_WARP_BINS * KN_MAXD * 32 * 4;
        const int64_t per_cta = (int64_t)KN_WARP_BINS * (32 / seg);
        const int64_t grid = std::min<int64_t>((n_bins + per_cta - 1) / per_cta, (int64_t)e->num_sms * 64);
        const void* kern = seg == 8 ? (const void*)kn_warp_kernel<8>
                         : seg == 16 ? (const void*)kn_warp_kernel<16> : (const void*)kn_warp_kernel<32>;
        CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        p.order = nullptr;
        if (seg < 32 && n_bins >= 2 * per_cta && n_bins < ((int64_t)1 << 31)) {  // group bins by item count
            if (int rc = e->d_knord.grow((size_t)n_bins * 4)) return rc;
            kn_order_kernel<<<1, KN_ORDER_NT, 0, s>>>(p.off, n_bins, (int32_t*)e->d_knord.p);
            CUDA_TRY(cudaGetLastError());
            e->launches++;
            p.order = (const int32_t*)e->d_knord.p;
        }
        if (seg == 8) kn_warp_kernel<8><<<(unsigned)grid, 32 * KN_WARP_BINS, smem, s>>>(p);
        else if (seg == 16) kn_warp_kernel<16><<<(unsigned)grid, 32 * KN_WARP_BINS, smem, s>>>(p);
        else kn_warp_kernel<32><<<(unsigned)grid, 32 * KN_WARP_BINS, smem, s>>>(p);
        e->last_detail = seg;
    } else {
        p.nbuf = std::max(3, kn_depth(max_items) + 2);
        const size_t smem = (size_t)p.nbuf * p.words * 4;
        if (smem + 64 > e->smem_optin)
            return fail(BPLB_ERANGE, "knapsack bitsets of this capacity / item count exceed shared memory");
        CUDA_TRY(cudaFuncSetAttribute(kn_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 1;
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kn_cta_kernel, KN_NT, smem));
        const int64_t grid = std::min<int64_t>(n_bins, (int64_t)e->num_sms * std::max(per_sm, 1));
        p.order = nullptr;
        if (n_bins > grid && n_bins < ((int64_t)1 << 31)) {  // longest bins first from a dynamic counter
            if (int rc = e->d_knord.grow((size_t)n_bins * 4)) return rc;
            kn_order_kernel<<<1, KN_ORDER_NT, 0, s>>>(p.off, n_bins, (int32_t*)e->d_knord.p);
            CUDA_TRY(cudaGetLastError());
            e->launches++;
            p.order = (const int32_t*)e->d_knord.p;
        }
        p.next = (unsigned long long*)((char*)e->d_err.p + 8);
        kn_cta_kernel<<<(unsigned)grid, KN_NT, smem, s>>>(p);
        e->last_detail = KN_NT;
    }
    CUDA_TRY(cudaGetLastError());
    e->launches++;
    e->last_path = BPLB_PATH_KNAP;
    if (timing) CUDA_TRY(cudaEventRecord(e->ev1, s));
    return 0;
}

int knap_check_args(int64_t c, int64_t n_bins) {
    if (c < 1 || c > BPLB_MAX_C) return fail(BPLB_ERANGE, "capacity outside [1, 2^30]");
    if (n_bins < 0) return fail(BPLB_EINVAL, "negative bin count");
    return 0;
}

}  // namespace

int bplb_knapsack_bins_device(bplb_engine* e, int64_t c, int64_t n_bins, const int32_t* d_committed,
                              const int32_t* d_lo, const int32_t* d_hi, const int32_t* d_w, const int64_t* d_off,
                              int64_t max_items, int32_t flags, int32_t* d_status, int32_t* d_lo_out,
                              int32_t* d_hi_out, uint8_t* d_action, uint32_t* d_reach, void* stream) {
    if (!e) return fail(BPLB_EINVAL, "null engine");
    if (int rc = knap_check_args(c, n_bins)) return rc;
    if (max_items < 0) return fail(BPLB_EINVAL, "negative max_items");
    if (n_bins == 0) return 0;
    if (!d_committed || !d_lo || !d_hi || !d_off || !d_status || !d_lo_out || !d_hi_out ||
        (!d_action && !(flags & BPLB_KN_REACH_ONLY)) || (max_items > 0 && !d_w))
        return fail(BPLB_EINVAL, "null array");
    cudaStream_t s = stream ? (cudaStream_t)stream : e->stream;
    std::lock_guard<std::mutex> lock(e->mu);
    CUDA_TRY(cudaSetDevice(e->device));
    if (int rc = join_stream(e, s)) return rc;
    if (int rc = e->d_err.grow(16)) return rc;
    CUDA_TRY(cudaMemsetAsync(e->d_err.p, 0, 16, s));  // error word + bin counter
    bplb::knap::KnParams p{};
    p.off = d_off; p.committed = d_committed; p.lo = d_lo; p.hi = d_hi; p.w = d_w;
    p.status = d_status; p.lo_out = d_lo_out; p.hi_out = d_hi_out; p.action = d_action; p.reach = d_reach;
    p.err = (int*)e->d_err.p;
    if (int rc = knap_launch(e, s, c, n_bins, max_items, flags, p)) return rc;
    int err = 0;
    CUDA_TRY(cudaMemcpyAsync(&err, e->d_err.p, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (int rc = mark_tail(e, s)) return rc;
    if (flags & BPLB_F_TIMING) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e->ev0, e->ev1);
        e->last_ms = ms;
    }
    if (err) return fail(BPLB_EINVAL, "knapsack bin with a weight outside [1, c], an interval outside [0, c], "
                                      "lo > hi, a negative committed load or more items than max_items");
    return 0;
}

int bplb_knapsack_bins(bplb_engine* e, int64_t c, int64_t n_bins, const int32_t* committed, const int32_t* lo,
                       const int32_t* hi, const int32_t* w, const int64_t* off, int32_t flags, int32_t* status_out,
                       int32_t* lo_out, int32_t* hi_out, uint8_t* action_out, uint32_t* reach_out) {
    if (!e) return fail(BPLB_EINVAL, "null engine");
    if (int rc = knap_check_args(c, n_bins)) return rc;
    if (n_bins == 0) return 0;
    if (!committed || !lo || !hi || !off || !status_out || !lo_out || !hi_out)
        return fail(BPLB_EINVAL, "null array");
    if (off[0] != 0) return fail(BPLB_EINVAL, "offsets[0] must be 0");
    int64_t max_items = 0;
    for (int64_t b = 0; b < n_bins; ++b) {
        const int64_t m = off[b + 1] - off[b];
        if (m < 0) return fail(BPLB_EINVAL, "offsets must be non-decreasing");
        max_items = std::max(max_items, m);
    }
    const int64_t total = off[n_bins];
    if (total > 0 && !w) return fail(BPLB_EINVAL, "null weights");
    if (total > 0 && !action_out && !(flags & BPLB_KN_REACH_ONLY)) return fail(BPLB_EINVAL, "null action array");
    const int64_t words = (c + 32) / 32;
    // packed inputs: off | committed | lo | hi | w ; outputs: status | lo | hi | reach | action
    const size_t in_off = 0, in_cl = in_off + (size_t)(n_bins + 1) * 8, in_lo = in_cl + (size_t)n_bins * 4,
                 in_hi = in_lo + (size_t)n_bins * 4, in_w = in_hi + (size_t)n_bins * 4,
                 in_bytes = in_w + (size_t)total * 4;
    const size_t o_st = 0, o_lo = (size_t)n_bins * 4, o_hi = o_lo + (size_t)n_bins * 4,
                 o_reach = o_hi + (size_t)n_bins * 4, o_act = o_reach + (reach_out ? (size_t)n_bins * words * 4 : 0),
                 out_bytes = o_act + (size_t)total;
    std::lock_guard<std::mutex> lock(e->mu);
    CUDA_TRY(cudaSetDevice(e->device));
    if (int rc = join_stream(e, e->stream)) return rc;
    if (int rc = e->d_knin.grow(in_bytes + 64)) return rc;
    if (int rc = e->d_knout.grow(out_bytes + 64)) return rc;
    if (int rc = e->h_stage.grow(std::max(in_bytes, out_bytes) + 64)) return rc;
    if (int rc = e->d_err.grow(16)) return rc;
    char* hs = (char*)e->h_stage.p;
    // the item arrays dominate: read straight from the caller when pinned
    const bool w_pinned = total * 4 > 65536 && is_pinned(w);
    const bool a_pinned = total > 65536 && action_out && is_pinned(action_out);
    host_copy(hs + in_off, off, (size_t)(n_bins + 1) * 8);
    host_copy(hs + in_cl, committed, (size_t)n_bins * 4);
    host_copy(hs + in_lo, lo, (size_t)n_bins * 4);
    host_copy(hs + in_hi, hi, (size_t)n_bins * 4);
    if (total && !w_pinned) host_copy(hs + in_w, w, (size_t)total * 4);
    char* di = (char*)e->d_knin.p;
    char* dout = (char*)e->d_knout.p;
    CUDA_TRY(cudaMemcpyAsync(di, hs, w_pinned ? in_w : in_bytes, cudaMemcpyHostToDevice, e->stream));
    if (total && w_pinned) CUDA_TRY(cudaMemcpyAsync(di + in_w, w, (size_t)total * 4, cudaMemcpyHostToDevice, e->stream));
    CUDA_TRY(cudaMemsetAsync(e->d_err.p, 0, 16, e->stream));  // error word + bin counter
    bplb::knap::KnParams p{};
    p.off = (const int64_t*)(di + in_off);
    p.committed = (const int32_t*)(di + in_cl);
    p.lo = (const int32_t*)(di + in_lo);
    p.hi = (const int32_t*)(di + in_hi);
    p.w = (const int32_t*)(di + in_w);
    p.status = (int32_t*)(dout + o_st);
    p.lo_out = (int32_t*)(dout + o_lo);
    p.hi_out = (int32_t*)(dout + o_hi);
    p.reach = reach_out ? (uint32_t*)(dout + o_reach) : nullptr;
    p.action = (uint8_t*)(dout + o_act);
    p.err = (int*)e->d_err.p;
    if (int rc = knap_launch(e, e->stream, c, n_bins, max_items, flags, p)) return rc;
    // the stage is reused for the outputs: the H2D copy above completed in stream order
    const bool want_act = total && action_out && !(flags & BPLB_KN_REACH_ONLY);
    CUDA_TRY(cudaMemcpyAsync(hs, dout, (want_act && a_pinned) || !want_act ? o_act : out_bytes,
                             cudaMemcpyDeviceToHost, e->stream));
    if (want_act && a_pinned)
        CUDA_TRY(cudaMemcpyAsync(action_out, dout + o_act, (size_t)total, cudaMemcpyDeviceToHost, e->stream));
    int* herr = (int*)(hs + out_bytes + ((8 - out_bytes % 8) % 8));
    CUDA_TRY(cudaMemcpyAsync(herr, e->d_err.p, 4, cudaMemcpyDeviceToHost, e->stream));
    CUDA_TRY(cudaStreamSynchronize(e->stream));
    if (int rc = mark_tail(e, e->stream)) return rc;
    if (flags & BPLB_F_TIMING) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e->ev0, e->ev1);
        e->last_ms = ms;
    }
    if (*herr) return fail(BPLB_EINVAL, "knapsack bin with a weight outside [1, c], an interval outside [0, c], "
                                        "lo > hi or a negative committed load");
    std::memcpy(status_out, hs + o_st, (size_t)n_bins * 4);
    std::memcpy(lo_out, hs + o_lo, (size_t)n_bins * 4);
    std::memcpy(hi_out, hs + o_hi, (size_t)n_bins * 4);
    if (reach_out) host_copy(reach_out, hs + o_reach, (size_t)n_bins * words * 4);
    if (want_act && !a_pinned) host_copy(action_out, hs + o_act, (size_t)total);
    return 0;
}
