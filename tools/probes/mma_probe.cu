// Legacy warp-level tensor-core throughput on B200 (mma.sync, compiled for
// sm_100a): tf32 m16n8k8 and bf16 m16n8k16, 8 independent accumulators per
// warp -- is a 3xTF32 column pass worth it against the 72 TF/s FFMA path?
#include <cstdio>
#include <cuda_runtime.h>

__global__ void tf32_k(float* out, int iters) {
    float acc[8][4];
    unsigned a[4], b[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
    b[0] = __float_as_uint(0.5f); b[1] = __float_as_uint(0.25f);
#pragma unroll
    for (int j = 0; j < 8; ++j) for (int i = 0; i < 4; ++i) acc[j][i] = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                         : "+f"(acc[j][0]), "+f"(acc[j][1]), "+f"(acc[j][2]), "+f"(acc[j][3])
                         : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) for (int i = 0; i < 4; ++i) s += acc[j][i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void bf16_k(float* out, int iters) {
    float acc[8][4];
    unsigned a[4], b[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = 0x3f803f80u + threadIdx.x;
    b[0] = 0x3f003f00u; b[1] = 0x3e803e80u;
#pragma unroll
    for (int j = 0; j < 8; ++j) for (int i = 0; i < 4; ++i) acc[j][i] = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                         : "+f"(acc[j][0]), "+f"(acc[j][1]), "+f"(acc[j][2]), "+f"(acc[j][3])
                         : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) for (int i = 0; i < 4; ++i) s += acc[j][i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float* out;
    cudaMalloc(&out, 148 * 16 * 256 * sizeof(float));
    const int iters = 2048;
    for (int rep = 0; rep < 3; ++rep) {
        for (int blocks_per_sm : {4, 8, 16}) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            float ms_t, ms_b;
            cudaEventRecord(e0);
            tf32_k<<<148 * blocks_per_sm, 256>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms_t, e0, e1);
            cudaEventRecord(e0);
            bf16_k<<<148 * blocks_per_sm, 256>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms_b, e0, e1);
            const double warps = 148.0 * blocks_per_sm * 8;
            const double ft = warps * iters * 8 * (2.0 * 16 * 8 * 8);
            const double fb = warps * iters * 8 * (2.0 * 16 * 8 * 16);
            printf("blocks/SM %2d: mma.sync tf32 %.1f TF/s   bf16 %.1f TF/s\n", blocks_per_sm, ft / ms_t / 1e9, fb / ms_b / 1e9);
        }
    }
    return 0;
}
