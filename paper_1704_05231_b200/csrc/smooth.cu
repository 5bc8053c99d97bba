// 1-D smoothing of independent lines -- the reference's smooth_lines /
// smooth_1d / smooth_pair_1d (gaussian.py:245-302) as a standalone entry
// (fgb_smooth_lines).  The bank and SDFT kernels never call these: they fold
// the smoothing into their fused stages.
//
//   FIR  (gaussian.py:231-233, correlate1d mode="nearest"): out[x] =
//        sum_t w[t] in[clamp(x + t0 + t)], taps = unit-sum sampled Gaussian.
//   Box / _AsymBox (gaussian.py:236-242): out[x] = sum_{k=lo..hi} in[x+k],
//        zero outside the line -- the same correlation with unit taps and a
//        zero boundary.
//   IIR  (gaussian.py:215-228): replicate pad P = ceil(5 sigma) + 2 (0 when
//        the caller already padded), forward then backward 3rd-order direct
//        form y = B z - a1 y1 - a2 y2 - a3 y3 with lfilter_zi steady-state
//        init (past outputs = first sample of the pass), crop.  fp64 state
//        for both precisions: the direct form's poles sit within 1e-3 of the
//        unit circle at sigma = 32 and lose ~1e-3 relative in fp32.
//
// Layout: lines are rows of a real [n_lines][pitch] array; outputs dense
// [n_lines][len].  Correlations stage a tile of TILE outputs plus the tap
// span in shared memory (coalesced clamped loads, each sample read once per
// tile); the IIR runs one thread per line with the forward sequence parked
// sample-major ([L][n_lines]) so a warp's loads and stores coalesce.
#include <cuda_runtime.h>

#include "kernels.h"

namespace fgb {
namespace {

constexpr int kLTile = 1024;   // outputs per CTA
constexpr int kLThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kLThreads) lines_corr_kernel(LinesCorrArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smraw[];
    T* tile = reinterpret_cast<T*>(smraw);
    const int64_t tiles = (a.len + kLTile - 1) / kLTile;
    const int64_t line = blockIdx.x / tiles;
    const int x0 = (int)(blockIdx.x - line * tiles) * kLTile;
    const T* src = a.in + line * a.pitch;
    const int n = kLTile + a.nt - 1;
    for (int i = threadIdx.x; i < n; i += kLThreads) {
        const int x = x0 + a.t0 + i;
        T v;
        if (x >= 0 && x < a.len) v = src[x];
        else v = a.zero_boundary ? T(0) : src[x < 0 ? 0 : a.len - 1];
        tile[i] = v;
    }
    __syncthreads();
    T* dst = a.out + line * a.out_pitch;
#pragma unroll 1
    for (int o = threadIdx.x; o < kLTile; o += kLThreads) {
        const int x = x0 + o;
        if (x >= a.len) break;
        T acc = T(0);
        for (int q = 0; q < a.nt; ++q) acc = fma(__ldg(a.w + q), tile[o + q], acc);
        dst[x] = acc;
    }
}

// Tap spans too wide for a shared tile: straight clamped global reads.
template <typename T> __global__ void lines_corr_gmem_kernel(LinesCorrArgs<T> a) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)a.n_lines * a.len) return;
    const int64_t line = i / a.len;
    const int x = (int)(i - line * a.len);
    const T* src = a.in + line * a.pitch;
    T acc = T(0);
    for (int q = 0; q < a.nt; ++q) {
        const int xx = x + a.t0 + q;
        T v;
        if (xx >= 0 && xx < a.len) v = src[xx];
        else v = a.zero_boundary ? T(0) : src[xx < 0 ? 0 : a.len - 1];
        acc = fma(a.w[q], v, acc);
    }
    a.out[line * a.out_pitch + x] = acc;
}

template <typename T> __global__ void lines_iir_kernel(LinesIirArgs<T> a) {
    const int line = blockIdx.x * blockDim.x + threadIdx.x;
    if (line >= a.n_lines) return;
    const T* src = a.in + (int64_t)line * a.pitch;
    const int L = a.len + 2 * a.P;
    const int64_t nl = a.n_lines;
    const double B = a.c.B, a1 = a.c.a1, a2 = a.c.a2, a3 = a.c.a3;
    // forward: replicate-padded input, past outputs = first padded sample (lfilter_zi * x[0])
    double y1 = (double)src[0], y2 = y1, y3 = y1;
    for (int n = 0; n < L; ++n) {
        const int x = clampi(n - a.P, 0, a.len - 1);
        const double y = B * (double)src[x] - a1 * y1 - a2 * y2 - a3 * y3;
        a.scratch[(int64_t)n * nl + line] = y;
        y3 = y2;
        y2 = y1;
        y1 = y;
    }
    // backward over the reversed forward sequence, past outputs = its first sample
    T* dst = a.out + (int64_t)line * a.out_pitch;
    y2 = y3 = y1;
    for (int n = L - 1; n >= 0; --n) {
        const double y = B * a.scratch[(int64_t)n * nl + line] - a1 * y1 - a2 * y2 - a3 * y3;
        y3 = y2;
        y2 = y1;
        y1 = y;
        const int x = n - a.P;
        if (x >= 0 && x < a.len) dst[x] = (T)y;
    }
}

}  // namespace

template <typename T> cudaError_t launch_lines_corr(const LinesCorrArgs<T>& a, cudaStream_t s) {
    if (a.n_lines == 0 || a.len == 0) return cudaSuccess;
    const size_t smem = sizeof(T) * (size_t)(kLTile + a.nt - 1);
    if (smem <= 200 * 1024) {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(lines_corr_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int64_t tiles = (a.len + kLTile - 1) / kLTile;
        lines_corr_kernel<T><<<(unsigned)(tiles * a.n_lines), kLThreads, smem, s>>>(a);
    } else {
        const int64_t n = (int64_t)a.n_lines * a.len;
        lines_corr_gmem_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(a);
    }
    return cudaGetLastError();
}

template <typename T> cudaError_t launch_lines_iir(const LinesIirArgs<T>& a, cudaStream_t s) {
    if (a.n_lines == 0 || a.len == 0) return cudaSuccess;
    lines_iir_kernel<T><<<(a.n_lines + 127) / 128, 128, 0, s>>>(a);
    return cudaGetLastError();
}

template cudaError_t launch_lines_corr<float>(const LinesCorrArgs<float>&, cudaStream_t);
template cudaError_t launch_lines_corr<double>(const LinesCorrArgs<double>&, cudaStream_t);
template cudaError_t launch_lines_iir<float>(const LinesIirArgs<float>&, cudaStream_t);
template cudaError_t launch_lines_iir<double>(const LinesIirArgs<double>&, cudaStream_t);

}  // namespace fgb
