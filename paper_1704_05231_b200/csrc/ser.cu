// Signal-to-error ratio on the device (metrics.py:63-83 of the reference):
// SER = 10 log10(sum t^2 / sum (a - t)^2) per plane, for interleaved complex
// approx / truth planes that already live in HBM -- `compare` sweeps full-size
// outputs without pulling float64 planes back to the host.
//
// Deterministic two-pass reduction in fp64: pass 1 gives each of a fixed
// number of CTAs a fixed grid-stride slice (per-thread sums, then a fixed
// shared-memory tree), pass 2 folds the per-CTA partials in index order.  No
// floating-point atomics, so the result is bit-identical run to run.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace fgb {
namespace {

constexpr int kSerThreads = 256;
constexpr int kSerBlocks = 296;  // 2 per SM

__device__ __forceinline__ void tree4(double (*sm)[kSerThreads], double v[4]) {
    const int t = threadIdx.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) sm[k][t] = v[k];
    __syncthreads();
    for (int s = kSerThreads / 2; s > 0; s >>= 1) {
        if (t < s)
#pragma unroll
            for (int k = 0; k < 4; ++k) sm[k][t] += sm[k][t + s];
        __syncthreads();
    }
}

template <typename T>
__global__ void __launch_bounds__(kSerThreads) ser_partial(const cx_t<T>* a, const cx_t<T>* t, int64_t n,
                                                           double* part) {
    __shared__ double sm[4][kSerThreads];
    double v[4] = {0.0, 0.0, 0.0, 0.0};  // signal re, error re, signal im, error im
    for (int64_t i = blockIdx.x * (int64_t)kSerThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kSerThreads) {
        const cx_t<T> x = a[i], y = t[i];
        const double tr = (double)y.x, ti = (double)y.y;
        const double er = (double)x.x - tr, ei = (double)x.y - ti;
        v[0] = fma(tr, tr, v[0]);
        v[1] = fma(er, er, v[1]);
        v[2] = fma(ti, ti, v[2]);
        v[3] = fma(ei, ei, v[3]);
    }
    tree4(sm, v);
    if (threadIdx.x < 4) part[blockIdx.x * 4 + threadIdx.x] = sm[threadIdx.x][0];
}

__global__ void __launch_bounds__(kSerThreads) ser_final(const double* part, int nb, double* out) {
    __shared__ double sm[4][kSerThreads];
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (int b = threadIdx.x; b < nb; b += kSerThreads)
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] += part[b * 4 + k];
    tree4(sm, v);
    if (threadIdx.x < 4) out[threadIdx.x] = sm[threadIdx.x][0];
}

}  // namespace

size_t ser_scratch_doubles() { return (size_t)kSerBlocks * 4 + 4; }

template <typename T>
cudaError_t launch_ser(const cx_t<T>* a, const cx_t<T>* t, int64_t n, double* scratch, cudaStream_t s) {
    const int nb = (int)std::min<int64_t>(kSerBlocks, (n + kSerThreads - 1) / kSerThreads > 0 ? (n + kSerThreads - 1) / kSerThreads : 1);
    ser_partial<T><<<nb, kSerThreads, 0, s>>>(a, t, n, scratch + 4);
    ser_final<<<1, kSerThreads, 0, s>>>(scratch + 4, nb, scratch);
    return cudaGetLastError();
}
template cudaError_t launch_ser<float>(const float2*, const float2*, int64_t, double*, cudaStream_t);
template cudaError_t launch_ser<double>(const double2*, const double2*, int64_t, double*, cudaStream_t);

}  // namespace fgb
