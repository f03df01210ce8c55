// bplb_peaks.cu -- measured issue-rate denominators for the roofline of the
// integer bound kernels (measurement infrastructure, not the product path;
// built as libbplb_peaks.so and called by bench.py on the GPU box).
//
// The LB-collection kernels are integer-issue bound: their
// roofline is the rate at which an SM can issue the instruction mix they
// execute.  MEASURED_PEAKS.json carries HBM and bf16 tensor figures only, so
// this library measures, on the box, with every SM busy:
//   alu   : independent integer adds (ptxas splits them between IADD3 on the
//           ALU pipe and IMAD.IADD on the FMA pipe: an issue-rate probe)
//   imad  : IMAD integer multiply-adds (FMA pipe on sm_100)
//   mix   : IADD3 and IMAD interleaved 1:1 -- both pipes, i.e. the warp
//           scheduler's issue ceiling (1 warp-instruction / clk / SMSP)
//   ffma  : FP32 FMA (FMA pipe), reported in flop/s
//   clock : the SM clock during the runs (clock64 cycles / globaltimer ns)
// Rates are warp-instructions/s (x32 for thread ops) over 148 SMs.
//   gather: independent random 16-byte loads from an L2-resident table (the
//           grid-wide path's {W, N} record lookups): 32-byte sectors / s
//           delivered L2 -> SM, 16 loads in flight per thread.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace {

constexpr int kNT = 256;   // 8 warps per CTA
constexpr int kAcc = 8;    // independent chains per thread
constexpr int kUnroll = 8; // inner unroll

template <int MODE>
__global__ void __launch_bounds__(kNT) issue_kernel(uint32_t* sink, int iters, uint32_t seed,
                                                    unsigned long long* cyc, unsigned long long* ns) {
    uint32_t a[kAcc];
    float f[kAcc];
#pragma unroll
    for (int i = 0; i < kAcc; ++i) {
        a[i] = seed * (threadIdx.x + 1) + i;
        f[i] = (float)(a[i] & 0xff) * 1e-3f;
    }
    const uint32_t s1 = seed | 1u, s2 = seed ^ 0x9e3779b9u;
    const float fm = 1.0000001f, fa = 1e-7f;
    unsigned long long c0 = clock64(), t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
#pragma unroll
            for (int i = 0; i < kAcc; ++i) {
                if (MODE == 0) {  // IADD3 (a variable operand: no constant folding of the chain)
                    asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(a[(i + 1) % kAcc]));
                } else if (MODE == 1) {  // IMAD
                    asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(s1), "r"(s2));
                } else if (MODE == 2) {  // interleaved ALU / FMA pipe
                    if (i & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(a[i - 1]), "r"(s2));
                    else asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(a[i + 1]));
                } else {  // FFMA
                    asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[i]) : "f"(fm), "f"(fa));
                }
            }
        }
    }
    unsigned long long c1 = clock64(), t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < kAcc; ++i) x ^= a[i] ^ __float_as_uint(f[i]);
    if (x == 0x12345678u) sink[0] = x;
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        *cyc = c1 - c0;
        *ns = t1 - t0;
    }
}

template <int MODE>
int run_one(int sms, int per_sm, int iters, double* rate, double* mhz) {
    uint32_t* sink;
    unsigned long long* d;
    if (cudaMalloc(&sink, 4) != cudaSuccess) return -1;
    if (cudaMalloc(&d, 16) != cudaSuccess) return -1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = sms * per_sm;
    issue_kernel<MODE><<<grid, kNT>>>(sink, 16, 7u, d, d + 1);  // warm-up
    cudaEventRecord(e0);
    issue_kernel<MODE><<<grid, kNT>>>(sink, iters, 7u, d, d + 1);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[2] = {0, 0};
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const double warp_inst = (double)grid * (kNT / 32) * (double)iters * kUnroll * kAcc;
    *rate = warp_inst / (ms * 1e-3);
    *mhz = h[1] ? (double)h[0] / (double)h[1] * 1e3 : 0.0;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    cudaFree(d);
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

constexpr int kG = 16;  // gather: loads in flight per thread

__global__ void __launch_bounds__(kNT) gather_kernel(const ulonglong2* __restrict__ tab, uint32_t mask, int iters,
                                                     unsigned long long* sink) {
    uint32_t h = (blockIdx.x * kNT + threadIdx.x) * 2654435761u + 12345u;
    unsigned long long acc = 0;
    for (int it = 0; it < iters; ++it) {
        ulonglong2 v[kG];
#pragma unroll
        for (int j = 0; j < kG; ++j) {
            h = h * 1664525u + 1013904223u;
            v[j] = __ldg(&tab[(h >> 7) & mask]);
        }
#pragma unroll
        for (int j = 0; j < kG; ++j) acc += v[j].x ^ v[j].y;
    }
    if (acc == 0x123456789ull) sink[0] = acc;
}

// L2 flush for timing harnesses: writes `bytes` with a CTA that holds
// `smem` bytes of dynamic shared memory, so the SMs keep the shared-memory
// carveout of the kernel being measured (a flush kernel without shared memory
// leaves the SMs configured for L1, and the next launch pays the switch).
__global__ void flush_kernel(uint4* p, size_t n) {
    extern __shared__ unsigned char fl_smem[];
    if (threadIdx.x == 0 && n == 0) fl_smem[0] = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4((unsigned)i, 0u, 0u, 0u);
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) int bplb_flush_l2(void* p, size_t bytes, void* stream, int smem) {
    static int attr = -1;
    if (smem > 48 * 1024 && smem != attr) {
        if (cudaFuncSetAttribute(flush_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
            return -1;
        attr = smem;
    }
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    flush_kernel<<<sms, 512, (size_t)smem, (cudaStream_t)stream>>>((uint4*)p, bytes / 16);
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// out[0]: random 16-byte gathers/s from a 16 MB L2-resident table (one
// 32-byte sector each), out[1]: the same in GB/s of sectors.  Returns 0 on success.
__attribute__((visibility("default"))) int bplb_measure_gather_peak(int device, double* out) {
    if (cudaSetDevice(device) != cudaSuccess) return -1;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const uint32_t n = 1u << 20;  // 16 MB of 16-byte records, as at c = 1e6
    ulonglong2* tab;
    unsigned long long* sink;
    if (cudaMalloc(&tab, (size_t)n * 16) != cudaSuccess) return -1;
    if (cudaMalloc(&sink, 8) != cudaSuccess) return -1;
    cudaMemset(tab, 1, (size_t)n * 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = sms * 4, iters = 256;
    gather_kernel<<<grid, kNT>>>(tab, n - 1, 16, sink);  // warm-up (table into L2)
    cudaEventRecord(e0);
    gather_kernel<<<grid, kNT>>>(tab, n - 1, iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double loads = (double)grid * kNT * iters * kG;
    out[0] = loads / (ms * 1e-3);
    out[1] = out[0] * 32 / 1e9;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(tab);
    cudaFree(sink);
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}


// out[0..3]: warp-instructions/s for alu, imad, mix, ffma; out[4..7]: the SM
// MHz seen by each run; out[8]: SM count.  Returns 0 on success.
__attribute__((visibility("default"))) int bplb_measure_issue_peaks(int device, double* out) {
    if (cudaSetDevice(device) != cudaSuccess) return -1;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int per_sm = 4;  // 32 warps per SM: 8 per scheduler
    const int iters = 4096;
    int rc = 0;
    rc |= run_one<0>(sms, per_sm, iters, &out[0], &out[4]);
    rc |= run_one<1>(sms, per_sm, iters, &out[1], &out[5]);
    rc |= run_one<2>(sms, per_sm, iters, &out[2], &out[6]);
    rc |= run_one<3>(sms, per_sm, iters, &out[3], &out[7]);
    out[8] = sms;
    return rc;
}

}  // extern "C"
