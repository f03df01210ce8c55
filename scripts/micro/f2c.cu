__device__ __forceinline__ void ffma2b(unsigned long long& acc, float h, unsigned long long f) {
    asm("{\n\t.reg .b64 hh;\n\tmov.b64 hh, {%2, %2};\n\tfma.rn.f32x2 %0, hh, %1, %0;\n\t}" : "+l"(acc) : "l"(f), "r"(__float_as_uint(h)));
}
__global__ void t(float* o, const float* a, const float4* b, int n) {
    unsigned long long acc[8][2] = {};
    for (int i = 0; i < n; ++i) {
        float4 f = b[i];
        unsigned long long f01 = ((unsigned long long)__float_as_uint(f.y) << 32) | __float_as_uint(f.x);
        unsigned long long f23 = ((unsigned long long)__float_as_uint(f.w) << 32) | __float_as_uint(f.z);
        #pragma unroll
        for (int a2 = 0; a2 < 8; ++a2) { float h = a[i * 8 + a2]; ffma2b(acc[a2][0], h, f01); ffma2b(acc[a2][1], h, f23); }
    }
    float s = 0;
    for (int a2 = 0; a2 < 8; ++a2) s += __uint_as_float((unsigned)acc[a2][0]) + __uint_as_float((unsigned)(acc[a2][1] >> 32));
    o[threadIdx.x] = s;
}
