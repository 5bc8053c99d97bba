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

// Register-operand FFMA variants: mode 1 = shared multiplier (operand reuse,
// the pattern of the FIR kernels), mode 2 = distinct multipliers (3 register
// reads per FFMA).
__constant__ float c_probe_w32[16];
__constant__ double c_probe_w64[16];
template <typename T> __device__ __forceinline__ T cw(int i);
template <> __device__ __forceinline__ float cw<float>(int i) { return c_probe_w32[i]; }
template <> __device__ __forceinline__ double cw<double>(int i) { return c_probe_w64[i]; }

template <typename T, int MODE>
__global__ void __launch_bounds__(256) fma_probe_reg(T* out, int iters, const T* wp) {
    T acc[8], v[8], w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        acc[i] = (T)(threadIdx.x + i) * (T)1e-3;
        v[i] = wp[i] + (T)threadIdx.x;
        w[i] = wp[8 + i] + (T)(threadIdx.x & 1) * (T)1e-7;  // per-thread: forces vector registers
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (MODE == 3)  // multiplier from the constant bank (compile-time offset)
                    acc[i] = fma(cw<T>(u & 7), v[(i + u) & 7], acc[i]);
                else
                    acc[i] = fma(MODE == 1 ? w[u & 7] : w[i], v[(i + u) & 7], acc[i]);
            }
        }
    }
    T s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == (T)12345.678) out[threadIdx.x] = s;
}

// Packed FP32 (sm_100 FFMA2): 8 float2 accumulators; MODE 4 = uniform (constant
// bank) float2 multiplier, MODE 5 = register multiplier.
template <int MODE>
__global__ void __launch_bounds__(256) fma2_probe(float* out, int iters, const float* wp) {
    float2 acc[8], v[8], w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        acc[i] = make_float2((threadIdx.x + i) * 1e-3f, (threadIdx.x - i) * 1e-3f);
        v[i] = make_float2(wp[i] + threadIdx.x, wp[i] - threadIdx.x);
        w[i] = make_float2(wp[8 + i] + (threadIdx.x & 1) * 1e-7f, wp[8 + i]);
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (MODE == 4) {
                    const float c = c_probe_w32[u & 7];
                    acc[i] = __ffma2_rn(make_float2(c, c), v[(i + u) & 7], acc[i]);
                } else {
                    acc[i] = __ffma2_rn(w[u & 7], v[(i + u) & 7], acc[i]);
                }
            }
        }
    }
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i].x + acc[i].y;
    if (s == 12345.678f) out[threadIdx.x] = s;
}

}  // namespace

double probe_ffma2_tflops(int mode) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    float *out = nullptr, *wp = nullptr;
    if (cudaMalloc(&out, 256 * sizeof(float)) != cudaSuccess) return -1.0;
    if (cudaMalloc(&wp, 16 * sizeof(float)) != cudaSuccess) return -1.0;
    float hw[16];
    for (int i = 0; i < 16; ++i) hw[i] = 0.5f + 0.01f * i;
    cudaMemcpy(wp, hw, sizeof(hw), cudaMemcpyHostToDevice);
    cudaMemcpyToSymbol(c_probe_w32, hw, sizeof(hw));
    auto kern = mode == 4 ? fma2_probe<4> : fma2_probe<5>;
    const int blocks = sms * 8, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<blocks, 256>>>(out, 64, wp);
    double best = 0.0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        kern<<<blocks, 256>>>(out, iters, wp);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fmas = 2.0 * (double)blocks * 256 * iters * 16 * 8;
        best = std::max(best, 2.0 * fmas / (ms * 1e-3) / 1e12);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    cudaFree(wp);
    return cudaGetLastError() == cudaSuccess ? best : -1.0;
}

template <typename T> double probe_fma_reg_tflops(int mode) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    T* out = nullptr;
    T* wp = nullptr;
    if (cudaMalloc(&out, 256 * sizeof(T)) != cudaSuccess) return -1.0;
    if (cudaMalloc(&wp, 16 * sizeof(T)) != cudaSuccess) return -1.0;
    T hw[16];
    for (int i = 0; i < 16; ++i) hw[i] = (T)(0.5 + 0.01 * i);
    cudaMemcpy(wp, hw, sizeof(hw), cudaMemcpyHostToDevice);
    const int blocks = sms * 8;
    const int iters = sizeof(T) == 4 ? 4096 : 1024;
    auto kern = mode == 1 ? fma_probe_reg<T, 1> : (mode == 2 ? fma_probe_reg<T, 2> : fma_probe_reg<T, 3>);
    if (sizeof(T) == 4) cudaMemcpyToSymbol(c_probe_w32, hw, 16 * sizeof(float));
    else cudaMemcpyToSymbol(c_probe_w64, hw, 16 * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<blocks, 256>>>(out, 64, wp);
    double best = 0.0;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        kern<<<blocks, 256>>>(out, iters, wp);
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
    cudaFree(wp);
    return cudaGetLastError() == cudaSuccess ? best : -1.0;
}
template double probe_fma_reg_tflops<float>(int);
template double probe_fma_reg_tflops<double>(int);

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
