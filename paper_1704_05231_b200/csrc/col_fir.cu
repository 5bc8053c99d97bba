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
// Layout: CTA = 32 columns x G row-groups x one segment of S rows of one
// job; each thread owns one column and R consecutive rows per TY = G*R row
// chunk.  The segment's (S + nt - 1)-row tile (rows clamped = replicate pad,
// or zeroed for the box window) is requested up front with cp.async, one
// commit group per chunk, so chunk i computes while chunks > i stream in and
// the 2h halo is fetched once per segment.  Taps run in chunks of R with a
// (2R-1)-deep register window: every J load feeds 4R FFMAs and each
// (ka, kb) tap pair is one broadcast LDS.  REM = nt % R is a template
// parameter so no taps are padded.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace fgb {

namespace {

template <typename T> struct ColCfg;
template <> struct ColCfg<float> { static constexpr int R = 8; };
template <> struct ColCfg<double> { static constexpr int R = 4; };

template <typename T, int R, int REM, bool HASB>
__device__ __forceinline__ void col_accumulate(const cx_t<T>* tb, const cx_t<T>* wts, int nt, T* Ar, T* Ai, T* Br,
                                               T* Bi) {
    using C = cx_t<T>;
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
}

__device__ __forceinline__ void cp_async_wait_pending(int n) {
    switch (n) {
        case 0: asm volatile("cp.async.wait_group 0;\n" ::: "memory"); break;
        case 1: asm volatile("cp.async.wait_group 1;\n" ::: "memory"); break;
        case 2: asm volatile("cp.async.wait_group 2;\n" ::: "memory"); break;
        case 3: asm volatile("cp.async.wait_group 3;\n" ::: "memory"); break;
        case 4: asm volatile("cp.async.wait_group 4;\n" ::: "memory"); break;
        case 5: asm volatile("cp.async.wait_group 5;\n" ::: "memory"); break;
        case 6: asm volatile("cp.async.wait_group 6;\n" ::: "memory"); break;
        default: asm volatile("cp.async.wait_group 7;\n" ::: "memory"); break;
    }
}

template <typename T, int REM>
__global__ void __launch_bounds__(256) col_kernel(ColArgs<T> a) {
    constexpr int R = ColCfg<T>::R;
    using C = cx_t<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int G = blockDim.y;
    const int TY = G * R;
    const int nt = a.nt;
    const int S = a.seg;
    C* wts = reinterpret_cast<C*>(smem_raw);
    C* tile = wts + ((nt + 1) & ~1);

    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * 32 + tx;
    const int job = blockIdx.z % a.njobs;
    const int b = blockIdx.z / a.njobs;
    const ColJob<T>* jb = a.jobs + job;
    const int x = blockIdx.x * 32 + tx;
    const int xc = x < a.W ? x : a.W - 1;
    const int ys = blockIdx.y * S;
    const int rows_out = min(S, a.H - ys);
    const int nch = (rows_out + TY - 1) / TY;

    // job descriptor -> registers before any global store (no aliasing reloads)
    const int64_t src_off = jb->src_off;
    const int wofs = jb->wofs;
    const int has_b = jb->has_b;
    const int nout = jb->nout;
    int64_t doff[4];
    T phr[4], phi[4];
    int bse[4], cnj[4];
#pragma unroll
    for (int o = 0; o < 4; ++o) {
        doff[o] = jb->dst_off[o];
        phr[o] = jb->phase_re[o];
        phi[o] = jb->phase_im[o];
        bse[o] = jb->base[o];
        cnj[o] = jb->conj[o];
    }

    {
        const C* wg = a.weights + wofs;
        for (int i = tid; i < nt; i += 32 * G) cp_async<sizeof(C)>(wts + i, wg + i);
        const C* src = a.src_base + src_off + (size_t)b * a.src_bstride + xc;
        for (int ch = 0; ch < nch; ++ch) {
            const int j0 = ch == 0 ? 0 : ch * TY + nt - 1;
            const int j1 = min((ch + 1) * TY, rows_out) + nt - 1;
            for (int j = j0 + ty; j < j1; j += G) {
                int yy = ys + a.t0 + j;
                if (a.zero_boundary && (yy < 0 || yy >= a.H)) {
                    tile[j * 32 + tx] = mk<T>(T(0), T(0));
                } else {
                    yy = clampi(yy, 0, a.H - 1);
                    cp_async<sizeof(C)>(tile + j * 32 + tx, src + (size_t)yy * a.W);
                }
            }
            asm volatile("cp.async.commit_group;\n" ::: "memory");
        }
    }

    C* dst = a.dst_base + (size_t)b * a.dst_bstride;
    for (int ch = 0; ch < nch; ++ch) {
        cp_async_wait_pending(min(nch - 1 - ch, 7));
        __syncthreads();
        T Ar[R], Ai[R], Br[R], Bi[R];
#pragma unroll
        for (int r = 0; r < R; ++r) { Ar[r] = Ai[r] = Br[r] = Bi[r] = T(0); }
        const C* tb = tile + (ch * TY + ty * R) * 32 + tx;
        if (has_b) col_accumulate<T, R, REM, true>(tb, wts, nt, Ar, Ai, Br, Bi);
        else col_accumulate<T, R, REM, false>(tb, wts, nt, Ar, Ai, Br, Bi);
        if (x < a.W) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int yl = ch * TY + ty * R + r;
                if (yl >= rows_out) break;
                const T xr = Ar[r] + Bi[r], xi = Ai[r] - Br[r];  // X = A - iB
                const T yr = Ar[r] - Bi[r], yi = Ai[r] + Br[r];  // Y = A + iB
                const size_t pix = (size_t)(ys + yl) * a.W + x;
#pragma unroll
                for (int o = 0; o < 4; ++o) {
                    if (o >= nout) break;
                    T re = bse[o] ? yr : xr;
                    T im = bse[o] ? yi : xi;
                    if (cnj[o]) im = -im;
                    if (phi[o] != T(0) || phr[o] != T(1)) {
                        const T orr = phr[o] * re - phi[o] * im;
                        im = phr[o] * im + phi[o] * re;
                        re = orr;
                    }
                    st_cs(dst + doff[o] + pix, mk<T>(re, im));
                }
            }
        }
    }
}

template <typename T, int REM>
cudaError_t launch_rem(const ColArgs<T>& a, int G, size_t smem, cudaStream_t s) {
    auto kern = col_kernel<T, REM>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    dim3 grid((a.W + 31) / 32, (a.H + a.seg - 1) / a.seg, a.njobs * a.batch);
    kern<<<grid, dim3(32, G), smem, s>>>(a);
    return cudaGetLastError();
}

int g_sm_count = 0;

}  // namespace

template <typename T> size_t col_smem(int nt, int rows) {
    return sizeof(cx_t<T>) * ((size_t)((nt + 1) & ~1) + (size_t)(rows + nt - 1) * 32);
}

template <typename T> cudaError_t launch_col(const ColArgs<T>& a_in, bool has_b, cudaStream_t s) {
    constexpr int R = ColCfg<T>::R;
    (void)has_b;
    ColArgs<T> a = a_in;
    if (g_sm_count == 0) {
        int dev = 0;
        g_sm_count = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
    }
    int G = 8;
    const size_t cols = (size_t)((a.W + 31) / 32) * a.njobs * a.batch;
    while (G > 1 && cols * ((a.H + G * R - 1) / (G * R)) < 2 * (size_t)g_sm_count) G /= 2;
    const int TY = G * R;
    // segment length S in {TY, 2TY, .., 8TY}: minimise waves x per-CTA work
    double best = 1e300;
    int bestS = 0;
    const int hr = (a.H + TY - 1) / TY * TY;
    for (int k = 1; k <= 8; k *= 2) {
        const int S = k * TY;
        if (S > hr && k > 1) break;
        const size_t smem = col_smem<T>(a.nt, S);
        if (smem > 200 * 1024) break;
        const int per_sm_smem = (int)((227 * 1024) / (smem + 1024));
        const int per_sm_thr = 2048 / (32 * G);
        const int per_sm = std::max(1, std::min(per_sm_smem, per_sm_thr));
        if (per_sm < 2 && k > 1) break;  // keep >= 2 CTAs per SM for latency hiding
        // throughput-bound SMs: time ~ (CTAs on the busiest SM) x per-CTA work
        const double ctas = (double)cols * ((a.H + S - 1) / S);
        const double per_sm_ctas = std::ceil(ctas / g_sm_count);
        const double work = (double)S * a.nt + 6.0 * (S + a.nt - 1) + 16.0 * S;  // fma + loads + epilogue
        const double cost = per_sm_ctas * work;
        if (cost < best * 0.999) {
            best = cost;
            bestS = S;
        }
    }
    if (bestS == 0) {
        if (col_smem<T>(a.nt, TY) > 220 * 1024) return cudaErrorInvalidConfiguration;
        bestS = TY;
    }
    a.seg = bestS;
    const size_t smem = col_smem<T>(a.nt, bestS);
    switch (a.nt % R) {
        case 0: return launch_rem<T, 0>(a, G, smem, s);
        case 1: return launch_rem<T, 1>(a, G, smem, s);
        case 2: return launch_rem<T, 2>(a, G, smem, s);
        case 3: return launch_rem<T, 3>(a, G, smem, s);
        default: break;
    }
    if constexpr (R > 4) {
        switch (a.nt % R) {
            case 4: return launch_rem<T, 4 % R>(a, G, smem, s);
            case 5: return launch_rem<T, 5 % R>(a, G, smem, s);
            case 6: return launch_rem<T, 6 % R>(a, G, smem, s);
            case 7: return launch_rem<T, 7 % R>(a, G, smem, s);
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
