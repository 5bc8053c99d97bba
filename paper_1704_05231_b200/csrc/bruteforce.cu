// Brute-force 2-D references on the GPU (the reference's oracle.py:33-109):
// direct tap sums of Eq. 1 (complex Gabor) and Eq. 17 (localized DFT bin),
// O(support^2) per pixel, accumulated in T (fp64 for validation runs).
//
//   fir_gabor     (oracle.py:53-66): out(y,x) = sum_{dy,dx} g(dy) g(dx)
//                 e^{i w (dx cos t + dy sin t)} f[clamp(y-dy)][clamp(x-dx)]
//   localized_dft (oracle.py:69-109): out(y,x) = sum_{dn,dm} env(dn,dm)
//                 e^{i (w0x u (Mx//2 + dm) + w0y v (My//2 + dn))} f[y+dn][x+dm]
//                 (replicate boundary for the Gaussian window, zero for box)
// The 2-D kernel is materialised once on the host (fp64) and streamed from
// shared memory; this path is independent of the separable decomposition,
// so full-size bank / SDFT outputs can be checked against it on the GPU.
#include "common.cuh"
#include "kernels.h"

namespace fgb {

namespace {

constexpr int kBfX = 32, kBfY = 8, kBfR = 4;  // CTA: 32 x 32 outputs, 4 rows per thread

// Kernel rows are processed in bands of KB so the staged input tile
// (32 rows + KB - 1) x (32 + kx - 1) fits shared memory for any support.
template <typename T>
__global__ void __launch_bounds__(kBfX * kBfY) direct2d_kernel(Direct2DArgs<T> a, int KB) {
    using C = cx_t<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int ky = a.ky, kx = a.kx;        // kernel extents
    const int oy = a.oy, ox = a.ox;        // input offset of kernel index 0 (input row = y + iy - oy)
    const int TH = kBfY * kBfR;
    const int NR = TH + KB - 1, NC = kBfX + kx - 1;
    T* tile = reinterpret_cast<T*>(smem_raw);  // [NR][NC]
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * kBfX + tx;
    const int b = blockIdx.z;
    const int x0 = blockIdx.x * kBfX, y0 = blockIdx.y * TH;
    const T* src = a.img + (size_t)b * a.img_bstride;
    T ar[kBfR], ai[kBfR];
#pragma unroll
    for (int r = 0; r < kBfR; ++r) ar[r] = ai[r] = T(0);
    for (int iy0 = 0; iy0 < ky; iy0 += KB) {
        const int kb = min(KB, ky - iy0);
        const int nr = TH + kb - 1;
        __syncthreads();
        for (int i = tid; i < nr * NC; i += kBfX * kBfY) {
            const int r = i / NC, q = i - r * NC;
            int yy = y0 + iy0 + r - oy, xx = x0 + q - ox;
            T v;
            if (a.zero_boundary) {
                v = (yy >= 0 && yy < a.H && xx >= 0 && xx < a.W) ? src[(size_t)yy * a.pitch + xx] : T(0);
            } else {
                yy = clampi(yy, 0, a.H - 1);
                xx = clampi(xx, 0, a.W - 1);
                v = src[(size_t)yy * a.pitch + xx];
            }
            tile[i] = v;
        }
        __syncthreads();
        for (int iy = 0; iy < kb; ++iy) {
            const C* krow = a.kern + (size_t)(iy0 + iy) * kx;
            const T* trow = tile + (size_t)(ty * kBfR + iy) * NC + tx;
            for (int ix = 0; ix < kx; ++ix) {
                const C k = krow[ix];
#pragma unroll
                for (int r = 0; r < kBfR; ++r) {
                    const T v = trow[(size_t)r * NC + ix];
                    ar[r] = fma(k.x, v, ar[r]);
                    ai[r] = fma(k.y, v, ai[r]);
                }
            }
        }
    }
    (void)NR;
    const int x = x0 + tx;
    if (x >= a.W) return;
#pragma unroll
    for (int r = 0; r < kBfR; ++r) {
        const int y = y0 + ty * kBfR + r;
        if (y < a.H) a.out[(size_t)b * a.out_bstride + (size_t)y * a.W + x] = mk<T>(ar[r], ai[r]);
    }
}

}  // namespace

template <typename T> size_t direct2d_smem(int kb, int kx) {
    return sizeof(T) * (size_t)(kBfY * kBfR + kb - 1) * (kBfX + kx - 1);
}

template <typename T> cudaError_t launch_direct2d(const Direct2DArgs<T>& a, cudaStream_t s) {
    int KB = a.ky;
    while (KB > 1 && direct2d_smem<T>(KB, a.kx) > 96 * 1024) KB = (KB + 1) / 2;
    const size_t smem = direct2d_smem<T>(KB, a.kx);
    if (smem > 220 * 1024) return cudaErrorInvalidConfiguration;
    auto kern = direct2d_kernel<T>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    dim3 grid((a.W + kBfX - 1) / kBfX, (a.H + kBfY * kBfR - 1) / (kBfY * kBfR), a.batch);
    kern<<<grid, dim3(kBfX, kBfY), smem, s>>>(a, KB);
    return cudaGetLastError();
}

template size_t direct2d_smem<float>(int, int);
template size_t direct2d_smem<double>(int, int);
template cudaError_t launch_direct2d<float>(const Direct2DArgs<float>&, cudaStream_t);
template cudaError_t launch_direct2d<double>(const Direct2DArgs<double>&, cudaStream_t);

}  // namespace fgb
