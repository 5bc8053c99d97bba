// K6: peak probes for the roofline denominators (MEASURED_PEAKS.json has HBM
// and bf16 tensor peaks only; the Gabor bank is FP32-pipe bound).
//   fp32: 8 independent FFMA chains per thread, all SMs, many warps.
//   fp64: same with DFMA.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"

namespace fgb {

namespace {

template <typename T>
__global__ void __launch_bounds__(256) fma_probe(T* out, int iters, T a, T b) {
    T x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = (T)(threadIdx.x + i) * (T)1e-3;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
        }
    }
    T s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == (T)12345.678) out[threadIdx.x] = s;  // keep the chains alive
}

}  // namespace

// Returns achieved FMA throughput in TFLOP/s (2 flops per FMA), best of 5.
template <typename T> double probe_fma_tflops() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    T* out = nullptr;
    if (cudaMalloc(&out, 256 * sizeof(T)) != cudaSuccess) return -1.0;
    const int blocks = sms * 8;
    const int iters = sizeof(T) == 4 ? 4096 : 1024;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    fma_probe<T><<<blocks, 256>>>(out, 64, (T)0.999, (T)1e-4);  // warm-up
    double best = 0.0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        fma_probe<T><<<blocks, 256>>>(out, iters, (T)0.999, (T)1e-4);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fmas = (double)blocks * 256 * iters * 16 * 8;
        best = std::max(best, 2.0 * fmas / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return cudaGetLastError() == cudaSuccess ? best : -1.0;
}

template double probe_fma_tflops<float>();
template double probe_fma_tflops<double>();

}  // namespace fgb
