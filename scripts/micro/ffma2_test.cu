#include <cstdio>
#include <cuda_runtime.h>
// packed fp32x2 FMA (PTX fma.rn.f32x2, sm_100+): does it exist and what does it compile to?
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
template <int NACC>
__global__ void k2(float* out, float a0, float b0, int iters) {
    unsigned long long acc[NACC];
    unsigned long long a[2], b[8];
    for (int i = 0; i < NACC; ++i) { float2 v = make_float2(threadIdx.x * 1e-7f + i, i); acc[i] = *(unsigned long long*)&v; }
    for (int i = 0; i < 2; ++i) { float2 v = make_float2(a0 + i, a0 - i * threadIdx.x); a[i] = *(unsigned long long*)&v; }
    for (int i = 0; i < 8; ++i) { float2 v = make_float2(b0 - i * blockIdx.x, b0 - i * blockIdx.x); b[i] = *(unsigned long long*)&v; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) acc[(i * 2 + j) % NACC] = ffma2(b[i], a[j], acc[(i * 2 + j) % NACC]);
#pragma unroll
        for (int i = 0; i < 2; ++i) a[i] = __shfl_xor_sync(0xffffffff, a[i], 1);
    }
    float s = 0;
    for (int i = 0; i < NACC; ++i) { float2 v = *(float2*)&acc[i]; s += v.x + v.y; }
    if (s == 12345.f) out[0] = s;
}
__global__ void kimad(int* out, int a0, int b0, int iters) {
    int acc[32], a[4], b[8];
    for (int i = 0; i < 32; ++i) acc[i] = threadIdx.x + i;
    for (int i = 0; i < 4; ++i) a[i] = a0 + i * threadIdx.x;
    for (int i = 0; i < 8; ++i) b[i] = b0 - i * blockIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i * 4 + j] += b[i] * a[j];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = __shfl_xor_sync(0xffffffff, a[i], 1);
    }
    int s = 0;
    for (int i = 0; i < 32; ++i) s += acc[i];
    if (s == 12345) out[0] = s;
}
int main() {
    float* d; cudaMalloc(&d, 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int iters = 20000;
    for (int warps : {4, 8, 16, 32}) {
        int blocks = 148 * (warps / 4);
        k2<16><<<blocks, 128>>>(d, 1.0f, 2.0f, 10);
        cudaEventRecord(e0);
        k2<16><<<blocks, 128>>>(d, 1.0f, 2.0f, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fma = (double)blocks * 128 * iters * 32;
        printf("FFMA2 warps/SM=%d  %.1f FMA/clk/SM\n", warps, fma / (ms * 1e-3) / 148 / 1.965e9);
        kimad<<<blocks, 128>>>((int*)d, 1, 2, 10);
        cudaEventRecord(e0);
        kimad<<<blocks, 128>>>((int*)d, 1, 2, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("IMAD  warps/SM=%d  %.1f MAC/clk/SM\n", warps, fma / (ms * 1e-3) / 148 / 1.965e9);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
