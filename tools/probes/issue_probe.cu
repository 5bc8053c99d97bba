// Does an FFMA2 occupy one or two issue slots?  Kernel A: 8 independent FFMA2
// chains per thread.  Kernel B: the same plus one independent IADD3 per FFMA2.
// If B runs as fast as A, the integer ops issued in the FFMA2 shadow.
#include <cstdio>
#include <cuda_runtime.h>

template <int EXTRA>
__global__ void k(float2* out, int iters, float2 w, int seed) {
    float2 acc[8];
    int ia[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { acc[j] = make_float2(threadIdx.x * 1e-3f + j, j * 0.5f); ia[j] = seed + j; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            acc[j] = __ffma2_rn(w, acc[j], acc[j]);
            if (EXTRA == 1) ia[j] ^= i;                  // LOP3 (ALU pipe)
            if (EXTRA == 2) ia[j] = ia[j] * 3 + i;       // IMAD (FMA pipe)
        }
    }
    float2 s = make_float2(0.f, 0.f);
    int t = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) { s.x += acc[j].x; s.y += acc[j].y; t ^= ia[j]; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = make_float2(s.x + (float)t, s.y);
}

int main() {
    float2* out;
    cudaMalloc(&out, 148 * 8 * 256 * sizeof(float2));
    const int iters = 4096;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float ms[3];
        for (int v = 0; v < 3; ++v) {
            cudaEventRecord(e0);
            if (v == 0) k<0><<<148 * 8, 256>>>(out, iters, make_float2(0.999f, 0.999f), 1);
            else if (v == 1) k<1><<<148 * 8, 256>>>(out, iters, make_float2(0.999f, 0.999f), 1);
            else k<2><<<148 * 8, 256>>>(out, iters, make_float2(0.999f, 0.999f), 1);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms[v], e0, e1);
        }
        const double flops = 148.0 * 8 * 256 * iters * 8 * 4;  // FFMA2 = 4 flops
        printf("FFMA2 only: %.1f TF/s   + LOP3 (ALU): %.1f TF/s   + IMAD (FMA pipe): %.1f TF/s\n",
               flops / ms[0] / 1e9, flops / ms[1] / 1e9, flops / ms[2] / 1e9);
    }
    return 0;
}
