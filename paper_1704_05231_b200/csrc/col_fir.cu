// K2: column pass with two real kernels on a complex plane.
//
// For one source plane J and taps t0..t0+nt-1:
//     A(y) = sum_t ka[t] J[y+t],   B(y) = sum_t kb[t] J[y+t]
// then up to four outputs  out_o = phase_o * {X, Y, conj X, conj Y}
// with X = A - iB, Y = A + iB.
//
//  * Gabor vertical stage (gabor.py:135-164): ka = w cos(ws t), kb = w sin(ws t);
//    F_theta = X and F_{pi-theta} = conj(Y) -- the mirrored orientation of
//    vertical_stage_conjugate (bank.py:68-74) comes from the SAME J read and
//    the same accumulators (Eqs. 13-16 of the paper).
//  * SDFT vertical bins (sdft.py:153-166, 202-212): ka = w cos(phi t),
//    kb = w sin(phi t), phase = e^{i phi c}:  bin(u,v) = P Y,
//    bin(M-u,v) = P conj(X), and the conjugate-filled bins conj(P) conj(Y),
//    conj(P) X are written from the same registers.
//
// Layout: CTA = 32 columns x G row-groups; each thread owns one column and
// R consecutive output rows.  The (TY + nt - 1) x 32 complex tile (rows
// clamped = replicate pad, or zeroed for the box window) is staged in
// shared memory; taps run in chunks of R with a (2R-1)-deep register
// window so every J load feeds 4R FFMAs, and each (ka, kb) tap pair is one
// broadcast LDS.  REM = nt % R is a template parameter so no taps are
// padded.
#include "common.cuh"
#include "kernels.h"

namespace fgb {

namespace {

template <typename T> struct ColCfg;
template <> struct ColCfg<float> { static constexpr int R = 8; };
template <> struct ColCfg<double> { static constexpr int R = 4; };

template <typename T, int REM, bool HASB>
__global__ void __launch_bounds__(256) col_kernel(ColArgs<T> a) {
    constexpr int R = ColCfg<T>::R;
    using C = cx_t<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int G = blockDim.y;
    const int TY = G * R;
    const int nt = a.nt;
    C* wts = reinterpret_cast<C*>(smem_raw);
    C* tile = wts + ((nt + 1) & ~1);

    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * 32 + tx;
    const int job = blockIdx.z % a.njobs;
    const int b = blockIdx.z / a.njobs;
    const ColJob<T>* jb = a.jobs + job;
    const int x = blockIdx.x * 32 + tx;
    const int xc = x < a.W ? x : a.W - 1;
    const int y0 = blockIdx.y * TY;

    {
        const C* wg = a.weights + jb->wofs;
        for (int i = tid; i < nt; i += 32 * G) wts[i] = wg[i];
    }
    {
        const C* src = a.src_base + jb->src_off + (size_t)b * a.src_bstride;
        const int nrows = TY + nt - 1;
        for (int j = ty; j < nrows; j += G) {
            int yy = y0 + a.t0 + j;
            C v;
            if (a.zero_boundary && (yy < 0 || yy >= a.H)) {
                v = mk<T>(T(0), T(0));
            } else {
                yy = clampi(yy, 0, a.H - 1);
                v = __ldg(src + (size_t)yy * a.W + xc);
            }
            tile[j * 32 + tx] = v;
        }
    }
    __syncthreads();

    T Ar[R], Ai[R], Br[R], Bi[R];
#pragma unroll
    for (int r = 0; r < R; ++r) { Ar[r] = Ai[r] = Br[r] = Bi[r] = T(0); }

    const C* tb = tile + (ty * R) * 32 + tx;
    const int nfull = (nt - REM) / R;
#pragma unroll 1
    for (int c = 0; c < nfull; ++c) {
        C v[2 * R - 1];
#pragma unroll
        for (int m = 0; m < 2 * R - 1; ++m) v[m] = tb[(c * R + m) * 32];
#pragma unroll
        for (int tt = 0; tt < R; ++tt) {
            const C w = wts[c * R + tt];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                Ar[r] = fma(w.x, v[r + tt].x, Ar[r]);
                Ai[r] = fma(w.x, v[r + tt].y, Ai[r]);
                if (HASB) {
                    Br[r] = fma(w.y, v[r + tt].x, Br[r]);
                    Bi[r] = fma(w.y, v[r + tt].y, Bi[r]);
                }
            }
        }
    }
    if constexpr (REM > 0) {
        const int c = nfull;
        C v[R + REM - 1];
#pragma unroll
        for (int m = 0; m < R + REM - 1; ++m) v[m] = tb[(c * R + m) * 32];
#pragma unroll
        for (int tt = 0; tt < REM; ++tt) {
            const C w = wts[c * R + tt];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                Ar[r] = fma(w.x, v[r + tt].x, Ar[r]);
                Ai[r] = fma(w.x, v[r + tt].y, Ai[r]);
                if (HASB) {
                    Br[r] = fma(w.y, v[r + tt].x, Br[r]);
                    Bi[r] = fma(w.y, v[r + tt].y, Bi[r]);
                }
            }
        }
    }

    if (x >= a.W) return;
    const int nout = jb->nout;
    const size_t ob = (size_t)b * a.dst_bstride;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int y = y0 + ty * R + r;
        if (y >= a.H) break;
        const T xr = Ar[r] + Bi[r], xi = Ai[r] - Br[r];  // X = A - iB
        const T yr = Ar[r] - Bi[r], yi = Ai[r] + Br[r];  // Y = A + iB
        for (int o = 0; o < nout; ++o) {
            T re = jb->base[o] ? yr : xr;
            T im = jb->base[o] ? yi : xi;
            if (jb->conj[o]) im = -im;
            const T pr = jb->phase_re[o], pi = jb->phase_im[o];
            const T orr = pr * re - pi * im;
            const T oi = pr * im + pi * re;
            st_cs(a.dst_base + jb->dst_off[o] + ob + (size_t)y * a.W + x, mk<T>(orr, oi));
        }
    }
}

template <typename T, int REM>
cudaError_t launch_rem(const ColArgs<T>& a, bool has_b, int G, size_t smem, cudaStream_t s) {
    constexpr int R = ColCfg<T>::R;
    auto kern = has_b ? col_kernel<T, REM, true> : col_kernel<T, REM, false>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const int TY = G * R;
    dim3 grid((a.W + 31) / 32, (a.H + TY - 1) / TY, a.njobs * a.batch);
    kern<<<grid, dim3(32, G), smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace

template <typename T> size_t col_smem(int nt, int G) {
    constexpr int R = ColCfg<T>::R;
    return sizeof(cx_t<T>) * ((size_t)((nt + 1) & ~1) + (size_t)(G * R + nt - 1) * 32);
}

template <typename T> cudaError_t launch_col(const ColArgs<T>& a, bool has_b, cudaStream_t s) {
    constexpr int R = ColCfg<T>::R;
    int G = 8;
    // small images: fewer rows per CTA keeps enough CTAs in flight
    while (G > 1 && (size_t)((a.W + 31) / 32) * ((a.H + G * R - 1) / (G * R)) * a.njobs * a.batch < 2 * 148) G /= 2;
    while (G > 1 && col_smem<T>(a.nt, G) > 200 * 1024) G /= 2;
    const size_t smem = col_smem<T>(a.nt, G);
    if (smem > 220 * 1024) return cudaErrorInvalidConfiguration;
    switch (a.nt % R) {
        case 0: return launch_rem<T, 0>(a, has_b, G, smem, s);
        case 1: return launch_rem<T, 1>(a, has_b, G, smem, s);
        case 2: return launch_rem<T, 2>(a, has_b, G, smem, s);
        case 3: return launch_rem<T, 3>(a, has_b, G, smem, s);
        default: break;
    }
    if constexpr (R > 4) {
        switch (a.nt % R) {
            case 4: return launch_rem<T, 4 % R>(a, has_b, G, smem, s);
            case 5: return launch_rem<T, 5 % R>(a, has_b, G, smem, s);
            case 6: return launch_rem<T, 6 % R>(a, has_b, G, smem, s);
            case 7: return launch_rem<T, 7 % R>(a, has_b, G, smem, s);
            default: break;
        }
    }
    return cudaErrorInvalidValue;
}

template size_t col_smem<float>(int, int);
template size_t col_smem<double>(int, int);
template cudaError_t launch_col<float>(const ColArgs<float>&, bool, cudaStream_t);
template cudaError_t launch_col<double>(const ColArgs<double>&, bool, cudaStream_t);

}  // namespace fgb
