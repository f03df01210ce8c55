__global__ void t(float* o, const float* a, const float* b, int n) {
    float2 acc0 = make_float2(0,0), acc1 = make_float2(0,0);
    for (int i = 0; i < n; ++i) {
        float h = a[i];
        float2 f = ((const float2*)b)[i];
        acc0.x = fmaf(h, f.x, acc0.x); acc0.y = fmaf(h, f.y, acc0.y);
        float h2 = a[i+n];
        acc1.x = fmaf(h2, f.x, acc1.x); acc1.y = fmaf(h2, f.y, acc1.y);
    }
    o[threadIdx.x] = acc0.x + acc0.y + acc1.x + acc1.y;
}
