// Microbenchmark: achievable FP32 FMA rate (reg-reg-reg form) on one B200,
// with 32 independent accumulators per thread, at several warps/SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int NACC>
__global__ void k(float* out, float a0, float b0, int iters) {
    float acc[NACC];
    float a[4], b[8];
    for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x * 1e-7f + i;
    for (int i = 0; i < 4; ++i) a[i] = a0 + i * threadIdx.x;
    for (int i = 0; i < 8; ++i) b[i] = b0 - i * blockIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[(i * 4 + j) % NACC] = fmaf(b[i], a[j], acc[(i * 4 + j) % NACC]);
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = __shfl_xor_sync(0xffffffff, a[i], 1);  // keep operands live
    }
    float s = 0;
    for (int i = 0; i < NACC; ++i) s += acc[i];
    if (s == 12345.f) out[0] = s;
}
int main() {
    float* d; cudaMalloc(&d, 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int iters = 20000;
    for (int warps : {4, 8, 16, 32}) {
        int blocks = 148 * (warps / 4 > 0 ? warps / 4 : 1);
        k<32><<<blocks, 128>>>(d, 1.0f, 2.0f, 10);
        cudaEventRecord(e0);
        k<32><<<blocks, 128>>>(d, 1.0f, 2.0f, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fma = (double)blocks * 128 * iters * 32;
        printf("warps/SM=%d  %.2f TFMA/s  = %.1f FMA/clk/SM at 1.965 GHz\n", warps, fma / ms / 1e9,
               fma / (ms * 1e-3) / 148 / 1.965e9);
    }
    return 0;
}
