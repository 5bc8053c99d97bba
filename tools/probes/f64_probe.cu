// fp64 pipe costs that shape the IIR kernels: DFMA throughput alone, and
// with one fp32 <-> fp64 conversion per DFMA (F2F, or integer bit tricks on
// the ALU pipe).  8 independent chains per thread, 148 x 8 CTAs x 256.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/f64p tools/probes/f64_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double f2d_bits(float f) {  // normal floats and zero (-> 2^-127), no inf / NaN
    const uint32_t b = __float_as_uint(f);
    const uint32_t hi = (b & 0x80000000u) | (((b & 0x7fffffffu) >> 3) + 0x38000000u);
    return __hiloint2double((int)hi, (int)(b << 29));
}

template <int V>
__global__ void k(double* out, int iters, double w, float seedf) {
    double acc[8];
    float fv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { acc[j] = threadIdx.x * 1e-3 + j; fv[j] = seedf + j; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (V == 0) acc[j] = fma(w, acc[j], acc[j]);
            if (V == 1) { acc[j] = fma(w, acc[j], (double)fv[j]); fv[j] += 1.0f; }          // F2F.F64.F32
            if (V == 2) { acc[j] = fma(w, acc[j], acc[j]); fv[j] += (float)acc[j]; }         // F2F.F32.F64
            if (V == 3) { acc[j] = fma(w, acc[j], f2d_bits(fv[j])); fv[j] += 1.0f; }         // bit trick
        }
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += acc[j] + fv[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    double* out;
    cudaMalloc(&out, 148 * 8 * 256 * sizeof(double));
    const int iters = 2048;
    const char* names[4] = {"DFMA only", "DFMA + F2F.F64.F32", "DFMA + F2F.F32.F64", "DFMA + bit-trick f32->f64"};
    for (int rep = 0; rep < 2; ++rep) {
        for (int v = 0; v < 4; ++v) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            if (v == 0) k<0><<<148 * 8, 256>>>(out, iters, 0.999, 1.f);
            if (v == 1) k<1><<<148 * 8, 256>>>(out, iters, 0.999, 1.f);
            if (v == 2) k<2><<<148 * 8, 256>>>(out, iters, 0.999, 1.f);
            if (v == 3) k<3><<<148 * 8, 256>>>(out, iters, 0.999, 1.f);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double ops = 148.0 * 8 * 256 * iters * 8;
            if (rep == 1) printf("%-28s %7.2f G DFMA/s  (%.1f TF/s)\n", names[v], ops / ms / 1e6, 2 * ops / ms / 1e9);
        }
    }
    return 0;
}
