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
// Layout (both variants): a CTA owns a column tile x one segment of S rows of
// one job.  The segment's (S + nt - 1)-row tile (rows clamped = replicate pad,
// or zeroed for the box window) is requested up front with cp.async, one
// commit group per chunk of rows, so chunk i computes while chunks > i stream
// in and the 2h halo is fetched once per segment.  Taps run in chunks of R
// with a (2R-1)-deep register window; REM = nt % R is a template parameter so
// no taps are padded.  Tap tables travel in the kernel parameters (constant
// bank -> uniform-register operands) when they fit, else in shared memory.
//  * col_kernel2 (fp32, even widths): two adjacent columns per thread (16-byte
//    cp.async / LDS.128 / STG.128), 8 rows per thread, packed FFMA2
//    accumulation (A and B of both columns: 4 FFMA2 per tap and row); CTA =
//    16 or 32 columns (CP = 8 / 16 column pairs) x 4 warps.
//  * col_kernel (fp64 validation build, odd widths): one column per thread,
//    scalar FMAs, CTA = 32 columns x G row groups.
//  * col_kernel_gmem: supports beyond shared memory (sigma 50 at radius 6).
// launch_col picks the variant, tile width and S with a small cost model.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace fgb {

namespace {

template <typename T> struct ColCfg;
template <> struct ColCfg<float> { static constexpr int R = 8; };
template <> struct ColCfg<double> { static constexpr int R = 4; };

template <typename T, int R, int REM, bool HASB, typename WF>
__device__ __forceinline__ void col_accumulate(const cx_t<T>* tb, WF wts, int nt, T* Ar, T* Ai, T* Br, T* Bi) {
    using C = cx_t<T>;
    const int nfull = (nt - REM) / R;
#pragma unroll 1
    for (int c = 0; c < nfull; ++c) {
        C v[2 * R - 1];
#pragma unroll
        for (int m = 0; m < 2 * R - 1; ++m) v[m] = tb[(c * R + m) * 32];
#pragma unroll
        for (int tt = 0; tt < R; ++tt) {
            const C w = wts(c * R + tt);
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
            const C w = wts(c * R + tt);
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

// CAP > 0: the launch's tap pairs travel in the kernel parameters (constant
// bank); the warp-uniform (ka, kb) loads become uniform-register operands
// of the FFMAs, which then read only two vector registers (measured on
// B200: 72.6 TFLOP/s vs 60.6 with a register multiplier).  CAP == 0: taps
// staged in shared memory (many jobs / long kernels).
template <typename T, int REM, int CAP>
__global__ void __launch_bounds__(256) col_kernel(const __grid_constant__ ColArgs<T> a,
                                                  const __grid_constant__ ColWParam<T, CAP> pw) {
    constexpr int R = ColCfg<T>::R;
    using C = cx_t<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int G = blockDim.y;
    const int TY = G * R;
    const int nt = a.nt;
    const int S = a.seg;
    C* wts = reinterpret_cast<C*>(smem_raw);
    C* tile = CAP > 0 ? wts : wts + ((nt + 1) & ~1);

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
        if (CAP == 0) {
            const C* wg = a.weights + wofs;
            for (int i = tid; i < nt; i += 32 * G) cp_async<sizeof(C)>(wts + i, wg + i);
        }
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
        if constexpr (CAP > 0) {
            const int pbase = job * nt;
            auto wf = [&](int i) { return pw.w[pbase + i]; };
            if (has_b) col_accumulate<T, R, REM, true>(tb, wf, nt, Ar, Ai, Br, Bi);
            else col_accumulate<T, R, REM, false>(tb, wf, nt, Ar, Ai, Br, Bi);
        } else {
            auto wf = [&](int i) { return wts[i]; };
            if (has_b) col_accumulate<T, R, REM, true>(tb, wf, nt, Ar, Ai, Br, Bi);
            else col_accumulate<T, R, REM, false>(tb, wf, nt, Ar, Ai, Br, Bi);
        }
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

// fp32 variant with two adjacent columns per thread: J pairs move as 16-byte
// cp.async / LDS.128 / STG.128, halving load, weight and store instructions
// per FFMA (needs an even W).  CTA = 64 columns x G row groups.
// Packed-FP32 accumulation (sm_100 FFMA2): (Ar, Ai) += ka * (Jr, Ji) and
// (Br, Bi) += kb * (Jr, Ji) are one FFMA2 each with the tap broadcast from a
// uniform register -- half the FMA-pipe instructions of scalar FFMA, so the
// loads and address arithmetic issue in the FMA pipe's spare slots.
template <int R, int REM, bool HASB, int RS, typename WF>
__device__ __forceinline__ void col_accumulate2(const float4* tb, WF wts, int nt, float2 (&A)[2][R], float2 (&Bv)[2][R]) {
    const int nfull = (nt - REM) / R;
#pragma unroll 1
    for (int c = 0; c < nfull; ++c) {
        float4 v[2 * R - 1];
#pragma unroll
        for (int m = 0; m < 2 * R - 1; ++m) v[m] = tb[(c * R + m) * RS];
#pragma unroll
        for (int tt = 0; tt < R; ++tt) {
            const float2 w = wts(c * R + tt);
            const float2 wa = make_float2(w.x, w.x), wb = make_float2(w.y, w.y);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const float4 q = v[r + tt];
                const float2 lo = make_float2(q.x, q.y), hi = make_float2(q.z, q.w);
                A[0][r] = __ffma2_rn(wa, lo, A[0][r]);
                A[1][r] = __ffma2_rn(wa, hi, A[1][r]);
                if (HASB) {
                    Bv[0][r] = __ffma2_rn(wb, lo, Bv[0][r]);
                    Bv[1][r] = __ffma2_rn(wb, hi, Bv[1][r]);
                }
            }
        }
    }
    if constexpr (REM > 0) {
        const int c = nfull;
        float4 v[R + REM - 1];
#pragma unroll
        for (int m = 0; m < R + REM - 1; ++m) v[m] = tb[(c * R + m) * RS];
#pragma unroll
        for (int tt = 0; tt < REM; ++tt) {
            const float2 w = wts(c * R + tt);
            const float2 wa = make_float2(w.x, w.x), wb = make_float2(w.y, w.y);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const float4 q = v[r + tt];
                const float2 lo = make_float2(q.x, q.y), hi = make_float2(q.z, q.w);
                A[0][r] = __ffma2_rn(wa, lo, A[0][r]);
                A[1][r] = __ffma2_rn(wa, hi, A[1][r]);
                if (HASB) {
                    Bv[0][r] = __ffma2_rn(wb, lo, Bv[0][r]);
                    Bv[1][r] = __ffma2_rn(wb, hi, Bv[1][r]);
                }
            }
        }
    }
}

// Real-J variant (ColJob::realj): A and B of the two columns from Re J only,
// (A0, A1) += ka (J0r, J1r), (B0, B1) += kb (J0r, J1r) -- two FFMA2 per tap
// and row instead of four.
template <int R, int REM, int RS, typename WF>
__device__ __forceinline__ void col_accumulate2_real(const float4* tb, WF wts, int nt, float2 (&A)[R], float2 (&Bv)[R]) {
    const int nfull = (nt - REM) / R;
#pragma unroll 1
    for (int c = 0; c < nfull; ++c) {
        float2 v[2 * R - 1];
#pragma unroll
        for (int m = 0; m < 2 * R - 1; ++m) {
            const float4 q = tb[(c * R + m) * RS];
            v[m] = make_float2(q.x, q.z);
        }
#pragma unroll
        for (int tt = 0; tt < R; ++tt) {
            const float2 w = wts(c * R + tt);
            const float2 wa = make_float2(w.x, w.x), wb = make_float2(w.y, w.y);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                A[r] = __ffma2_rn(wa, v[r + tt], A[r]);
                Bv[r] = __ffma2_rn(wb, v[r + tt], Bv[r]);
            }
        }
    }
    if constexpr (REM > 0) {
        const int c = nfull;
        float2 v[R + REM - 1];
#pragma unroll
        for (int m = 0; m < R + REM - 1; ++m) {
            const float4 q = tb[(c * R + m) * RS];
            v[m] = make_float2(q.x, q.z);
        }
#pragma unroll
        for (int tt = 0; tt < REM; ++tt) {
            const float2 w = wts(c * R + tt);
            const float2 wa = make_float2(w.x, w.x), wb = make_float2(w.y, w.y);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                A[r] = __ffma2_rn(wa, v[r + tt], A[r]);
                Bv[r] = __ffma2_rn(wb, v[r + tt], Bv[r]);
            }
        }
    }
}

// CP = column pairs per CTA (16 -> 32 columns, 8 -> 16 columns for long
// kernels whose (S + nt - 1)-row tile would otherwise limit occupancy).
template <int REM, int CAP, int CP>
__global__ void __launch_bounds__(128) col_kernel2(const __grid_constant__ ColArgs<float> a,
                                                   const __grid_constant__ ColWParam<float, CAP> pw) {
    constexpr int R = 8;
    constexpr int RGW = 32 / CP;  // row groups per warp
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // warp = CP column pairs x RGW row groups; CTA = 2 CP columns x (RGW G) row groups
    const int G2 = RGW * blockDim.y;
    const int TY = G2 * R;
    const int nt = a.nt;
    const int S = a.seg;
    float2* wts = reinterpret_cast<float2*>(smem_raw);
    float4* tile = reinterpret_cast<float4*>(CAP > 0 ? smem_raw : smem_raw + sizeof(float2) * ((nt + 1) & ~1));

    const int tid = threadIdx.y * 32 + threadIdx.x;
    const int cx = threadIdx.x % CP;                        // column pair
    const int rg = threadIdx.x / CP + RGW * threadIdx.y;    // row group
    const int job = blockIdx.z % a.njobs;
    const int b = blockIdx.z / a.njobs;
    const ColJob<float>* jb = a.jobs + job;
    const int x = blockIdx.x * 2 * CP + 2 * cx;  // first of the two columns
    const int ys = blockIdx.y * S;
    const int rows_out = min(S, a.H - ys);
    const int nch = (rows_out + TY - 1) / TY;
    const int H = a.H, W = a.W;

    const int64_t src_off = jb->src_off;
    const int wofs = jb->wofs;
    const int has_b = jb->has_b;
    const int nout = jb->nout;
    const int emode = jb->mode;
    // output o: re = Ar + sa*Bi, im = sc*Ai + sd*Br, then * phase
    float sa[4], sc[4], sd[4], phr[4], phi[4];
    int64_t doff[4];
#pragma unroll
    for (int o = 0; o < 4; ++o) {
        const int yb = jb->base[o], cj = jb->conj[o];
        sa[o] = yb ? -1.f : 1.f;
        sc[o] = cj ? -1.f : 1.f;
        sd[o] = (yb ? 1.f : -1.f) * (cj ? -1.f : 1.f);
        phr[o] = jb->phase_re[o];
        phi[o] = jb->phase_im[o];
        doff[o] = jb->dst_off[o];
    }

    {
        if (CAP == 0) {
            const float2* wg = a.weights + wofs;
            for (int i = tid; i < nt; i += 32 * blockDim.y) cp_async<8>(wts + i, wg + i);
        }
        // loader mapping: CP threads per tile row
        const int lc = tid % CP, lr = tid / CP, lstep = (32 * blockDim.y) / CP;
        const int xl = blockIdx.x * 2 * CP + 2 * lc;
        const float2* src = a.src_base + src_off + (size_t)b * a.src_bstride + (xl < W ? xl : W - 2);
        const int r0 = ys + a.t0;  // image row of tile row 0
        const bool interior = r0 >= 0 && r0 + rows_out + nt - 1 <= H && !a.zero_boundary;
        for (int ch = 0; ch < nch; ++ch) {
            const int j0 = ch == 0 ? 0 : ch * TY + nt - 1;
            const int j1 = min((ch + 1) * TY, rows_out) + nt - 1;
            if (interior) {
                const float2* p = src + (size_t)(r0 + j0 + lr) * W;
                for (int j = j0 + lr; j < j1; j += lstep, p += (size_t)lstep * W) cp_async16(tile + j * CP + lc, p);
            } else {
                for (int j = j0 + lr; j < j1; j += lstep) {
                    int yy = r0 + j;
                    if (a.zero_boundary && (yy < 0 || yy >= H)) {
                        tile[j * CP + lc] = make_float4(0.f, 0.f, 0.f, 0.f);
                    } else {
                        yy = clampi(yy, 0, H - 1);
                        cp_async16(tile + j * CP + lc, src + (size_t)yy * W);
                    }
                }
            }
            asm volatile("cp.async.commit_group;\n" ::);
        }
    }

    float2* dst = a.dst_base + (size_t)b * a.dst_bstride + x;
    if (jb->realj) {  // theta = pi/2 (mode 1, has_b): X = A - iB from Re J
        for (int ch = 0; ch < nch; ++ch) {
            cp_async_wait_pending(min(nch - 1 - ch, 7));
            __syncthreads();
            float2 A2[R], B2[R];
#pragma unroll
            for (int r = 0; r < R; ++r) { A2[r] = make_float2(0.f, 0.f); B2[r] = make_float2(0.f, 0.f); }
            const float4* tb = tile + (ch * TY + rg * R) * CP + cx;
            if constexpr (CAP > 0) {
                const int pbase = job * nt;
                col_accumulate2_real<R, REM, CP>(tb, [&](int i) { return pw.w[pbase + i]; }, nt, A2, B2);
            } else {
                col_accumulate2_real<R, REM, CP>(tb, [&](int i) { return wts[i]; }, nt, A2, B2);
            }
            if (x < W) {
                float2* d0 = dst + doff[0];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int yl = ch * TY + rg * R + r;
                    if (yl >= rows_out) break;
                    __stcs(reinterpret_cast<float4*>(d0 + (size_t)(ys + yl) * W),
                           make_float4(A2[r].x, -B2[r].x, A2[r].y, -B2[r].y));
                }
            }
        }
        return;
    }
    for (int ch = 0; ch < nch; ++ch) {
        cp_async_wait_pending(min(nch - 1 - ch, 7));
        __syncthreads();
        float2 A2[2][R], B2[2][R];
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int r = 0; r < R; ++r) { A2[q][r] = make_float2(0.f, 0.f); B2[q][r] = make_float2(0.f, 0.f); }
        const float4* tb = tile + (ch * TY + rg * R) * CP + cx;
        if constexpr (CAP > 0) {
            const int pbase = job * nt;
            auto wf = [&](int i) { return pw.w[pbase + i]; };
            if (has_b) col_accumulate2<R, REM, true, CP>(tb, wf, nt, A2, B2);
            else col_accumulate2<R, REM, false, CP>(tb, wf, nt, A2, B2);
        } else {
            auto wf = [&](int i) { return wts[i]; };
            if (has_b) col_accumulate2<R, REM, true, CP>(tb, wf, nt, A2, B2);
            else col_accumulate2<R, REM, false, CP>(tb, wf, nt, A2, B2);
        }
        float Ar[2][R], Ai[2][R], Br[2][R], Bi[2][R];
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int r = 0; r < R; ++r) {
                Ar[q][r] = A2[q][r].x; Ai[q][r] = A2[q][r].y;
                Br[q][r] = B2[q][r].x; Bi[q][r] = B2[q][r].y;
            }
        if (x < W) {
            if (emode == 2) {  // Gabor theta / pi-theta: X = A - iB, conj(Y) = (Ar - Bi, -(Ai + Br))
                float2* d0 = dst + doff[0];
                float2* d1 = dst + doff[1];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int yl = ch * TY + rg * R + r;
                    if (yl >= rows_out) break;
                    const size_t pix = (size_t)(ys + yl) * W;
                    __stcs(reinterpret_cast<float4*>(d0 + pix),
                           make_float4(Ar[0][r] + Bi[0][r], Ai[0][r] - Br[0][r], Ar[1][r] + Bi[1][r], Ai[1][r] - Br[1][r]));
                    __stcs(reinterpret_cast<float4*>(d1 + pix), make_float4(Ar[0][r] - Bi[0][r], -(Ai[0][r] + Br[0][r]),
                                                                            Ar[1][r] - Bi[1][r], -(Ai[1][r] + Br[1][r])));
                }
            } else if (emode == 1) {  // Gabor single orientation: X
                float2* d0 = dst + doff[0];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int yl = ch * TY + rg * R + r;
                    if (yl >= rows_out) break;
                    const size_t pix = (size_t)(ys + yl) * W;
                    __stcs(reinterpret_cast<float4*>(d0 + pix),
                           make_float4(Ar[0][r] + Bi[0][r], Ai[0][r] - Br[0][r], Ar[1][r] + Bi[1][r], Ai[1][r] - Br[1][r]));
                }
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int yl = ch * TY + rg * R + r;
                    if (yl >= rows_out) break;
                    float2* drow = dst + (size_t)(ys + yl) * W;
#pragma unroll
                    for (int o = 0; o < 4; ++o) {
                        if (o >= nout) break;
                        float v[4];
#pragma unroll
                        for (int q = 0; q < 2; ++q) {
                            float re = fmaf(sa[o], Bi[q][r], Ar[q][r]);
                            float im = fmaf(sd[o], Br[q][r], sc[o] * Ai[q][r]);
                            const float orr = phr[o] * re - phi[o] * im;
                            im = phr[o] * im + phi[o] * re;
                            v[2 * q] = orr;
                            v[2 * q + 1] = im;
                        }
                        __stcs(reinterpret_cast<float4*>(drow + doff[o]), make_float4(v[0], v[1], v[2], v[3]));
                    }
                }
            }
        }
    }
}

template <typename T, int REM, int CAP>
cudaError_t launch_cap(const ColArgs<T>& a, const cx_t<T>* pw_host, int G, size_t smem, cudaStream_t s) {
    auto kern = col_kernel<T, REM, CAP>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    static ColWParam<T, CAP> pw;  // host staging of the parameter block (launches are serialised by the engine lock)
    if constexpr (CAP > 0) std::memcpy(pw.w, pw_host, sizeof(cx_t<T>) * (size_t)a.njobs * a.nt);
    dim3 grid((a.W + 31) / 32, (a.H + a.seg - 1) / a.seg, a.njobs * a.batch);
    kern<<<grid, dim3(32, G), smem, s>>>(a, pw);
    return cudaGetLastError();
}

template <int REM, int CAP>
cudaError_t launch_cap2(const ColArgs<float>& a, const float2* pw_host, int G, size_t smem, cudaStream_t s) {
    auto kern = a.col2 == 2 ? col_kernel2<REM, CAP, 8> : col_kernel2<REM, CAP, 16>;
    const int cw = a.col2 == 2 ? 16 : 32;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    static ColWParam<float, CAP> pw;
    if constexpr (CAP > 0) std::memcpy(pw.w, pw_host, sizeof(float2) * (size_t)a.njobs * a.nt);
    dim3 grid((a.W + cw - 1) / cw, (a.H + a.seg - 1) / a.seg, a.njobs * a.batch);
    kern<<<grid, dim3(32, G), smem, s>>>(a, pw);
    return cudaGetLastError();
}

template <typename T, int REM>
cudaError_t launch_rem(const ColArgs<T>& a, const cx_t<T>* pw_host, int G, size_t smem, cudaStream_t s) {
    const size_t need = (size_t)a.njobs * a.nt;
    if constexpr (sizeof(T) == 4) {
        if (a.col2) {
            // two columns per thread, 32-column tiles (same footprint as the 1-column tile)
            const size_t tile2 = smem;
            if (pw_host && need <= (size_t)ColWCap<T>::kSmall) return launch_cap2<REM, ColWCap<T>::kSmall>(a, pw_host, G, tile2, s);
            if (pw_host && need <= (size_t)ColWCap<T>::kLarge) return launch_cap2<REM, ColWCap<T>::kLarge>(a, pw_host, G, tile2, s);
            return launch_cap2<REM, 0>(a, nullptr, G, tile2 + sizeof(float2) * ((a.nt + 1) & ~1), s);
        }
    }
    if (pw_host && need <= (size_t)ColWCap<T>::kSmall) return launch_cap<T, REM, ColWCap<T>::kSmall>(a, pw_host, G, smem, s);
    if (pw_host && need <= (size_t)ColWCap<T>::kLarge) return launch_cap<T, REM, ColWCap<T>::kLarge>(a, pw_host, G, smem, s);
    return launch_cap<T, REM, 0>(a, nullptr, G, smem + sizeof(cx_t<T>) * ((a.nt + 1) & ~1), s);
}

int g_sm_count = 0;

// Fallback for very long kernels (the (S + nt - 1)-row tile would not fit in
// shared memory, e.g. sigma = 50 at radius 6 -> 605 taps): each thread reads
// its column straight from global memory (L1/L2 cached), R rows per thread.
template <typename T>
__global__ void __launch_bounds__(256) col_kernel_gmem(ColArgs<T> a) {
    constexpr int R = 4;
    using C = cx_t<T>;
    const int job = blockIdx.z % a.njobs, b = blockIdx.z / a.njobs;
    const ColJob<T>* jb = a.jobs + job;
    const int x = blockIdx.x * 32 + threadIdx.x;
    const int y0 = (blockIdx.y * blockDim.y + threadIdx.y) * R;
    if (x >= a.W || y0 >= a.H) return;
    const C* src = a.src_base + jb->src_off + (size_t)b * a.src_bstride + x;
    const C* w = a.weights + jb->wofs;
    T Ar[R] = {}, Ai[R] = {}, Br[R] = {}, Bi[R] = {};
    for (int q = 0; q < a.nt; ++q) {
        const C k = __ldg(w + q);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            int yy = y0 + r + a.t0 + q;
            C v;
            if (a.zero_boundary && (yy < 0 || yy >= a.H)) {
                v = mk<T>(T(0), T(0));
            } else {
                yy = clampi(yy, 0, a.H - 1);
                v = __ldg(src + (size_t)yy * a.W);
            }
            Ar[r] = fma(k.x, v.x, Ar[r]);
            Ai[r] = fma(k.x, v.y, Ai[r]);
            Br[r] = fma(k.y, v.x, Br[r]);
            Bi[r] = fma(k.y, v.y, Bi[r]);
        }
    }
    const size_t ob = (size_t)b * a.dst_bstride;
    for (int r = 0; r < R; ++r) {
        const int y = y0 + r;
        if (y >= a.H) break;
        const T xr = Ar[r] + Bi[r], xi = Ai[r] - Br[r], yr = Ar[r] - Bi[r], yi = Ai[r] + Br[r];
        for (int o = 0; o < jb->nout; ++o) {
            T re = jb->base[o] ? yr : xr, im = jb->base[o] ? yi : xi;
            if (jb->conj[o]) im = -im;
            const T pr = jb->phase_re[o], pi = jb->phase_im[o];
            a.dst_base[jb->dst_off[o] + ob + (size_t)y * a.W + x] = mk<T>(pr * re - pi * im, pr * im + pi * re);
        }
    }
}

}  // namespace

template <typename T> size_t col_smem(int nt, int rows) {  // tile only (+ taps when not in params)
    return sizeof(cx_t<T>) * ((size_t)(rows + nt - 1) * 32);
}

template <typename T> cudaError_t launch_col(const ColArgs<T>& a_in, const cx_t<T>* pw_host, cudaStream_t s) {
    constexpr int R = ColCfg<T>::R;
    ColArgs<T> a = a_in;
    if (g_sm_count == 0) {
        int dev = 0;
        g_sm_count = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
    }
    const bool c2ok = (sizeof(T) == 4 && a.W % 2 == 0 && a.W >= 2 && !knobs().col1);
    // candidates: (mode, S) with mode 0 = 1 column/thread (32-col tiles, G=8),
    // 1 = 2 columns/thread 32-col tiles, 2 = 2 columns/thread 16-col tiles (G=4)
    double best = 1e300;
    int bestS = 0, bestMode = c2ok ? 1 : 0, bestG = c2ok ? 4 : 8;
    for (int mode = c2ok ? 1 : 0; mode <= (c2ok ? 2 : 0); ++mode) {
        const int cw = mode == 2 ? 16 : 32;
        int G = mode == 0 ? 8 : 4;
        const size_t cols = (size_t)((a.W + cw - 1) / cw) * a.njobs * a.batch;
        if (mode == 0)
            while (G > 1 && cols * ((a.H + G * R - 1) / (G * R)) < 2 * (size_t)g_sm_count) G /= 2;
        const int TY = mode == 0 ? G * R : (32 / (cw / 2)) * G * R;
        const size_t rowb = (size_t)cw * sizeof(cx_t<T>);
        const int hr = (a.H + TY - 1) / TY * TY;
        for (int k = 1; k <= 8; k *= 2) {
            const int S = k * TY;
            if (S > hr && k > 1) break;
            const size_t smem = rowb * (size_t)(S + a.nt - 1);
            if (smem > 200 * 1024) break;
            const int per_sm_smem = (int)((227 * 1024) / (smem + 1024));
            const int per_sm_thr = mode == 0 ? 2048 / (32 * G) : 5;  // ~96 registers x 128 threads
            const int per_sm = std::max(1, std::min(per_sm_smem, per_sm_thr));
            if (per_sm < 2 && k > 1) break;
            const double ctas = (double)cols * ((a.H + S - 1) / S);
            const double per_sm_ctas = std::ceil(ctas / g_sm_count);
            // per-CTA work in "FFMA-slot" units: taps x rows x columns, halo loads, epilogue;
            // few resident warps issue slower (~2 warps/scheduler is ~85%)
            const double warps = (double)per_sm * G;
            const double issue = warps >= 16 ? 1.0 : (warps >= 12 ? 0.95 : (warps >= 8 ? 0.88 : 0.75));
            const double work = ((double)S * a.nt * cw + 6.0 * (S + a.nt - 1) * cw + 16.0 * S * cw) / issue;
            const double cost = per_sm_ctas * work;
            if (cost < best * 0.999) {
                best = cost;
                bestS = S;
                bestMode = mode;
                bestG = G;
            }
        }
    }
    if (knobs().col_mode >= 0) {  // experiment knobs: force mode / segment rows
        const int m = knobs().col_mode;
        if (m >= 0 && m <= 2 && (m == 0 || c2ok)) { bestMode = m; bestG = m == 0 ? 8 : 4; }
    }
    if (knobs().col_seg > 0) {
        const int TY = bestMode == 0 ? bestG * R : (bestMode == 2 ? 4 : 2) * bestG * R;
        const int S = knobs().col_seg / TY * TY;
        if (S > 0) bestS = S;
    }
    a.col2 = bestMode;
    const int G = bestG;
    const int TY = bestMode == 0 ? G * R : (bestMode == 2 ? 4 : 2) * G * R;
    if (bestS == 0) {
        if (col_smem<T>(a.nt, TY) > 200 * 1024) {
            dim3 grid((a.W + 31) / 32, (a.H + 4 * 8 - 1) / (4 * 8), a.njobs * a.batch);
            col_kernel_gmem<T><<<grid, dim3(32, 8), 0, s>>>(a);
            return cudaGetLastError();
        }
        bestS = TY;
    }
    a.seg = bestS;
    const size_t smem = col_smem<T>(a.nt, bestS) / (bestMode == 2 ? 2 : 1);
    switch (a.nt % R) {
        case 0: return launch_rem<T, 0>(a, pw_host, G, smem, s);
        case 1: return launch_rem<T, 1>(a, pw_host, G, smem, s);
        case 2: return launch_rem<T, 2>(a, pw_host, G, smem, s);
        case 3: return launch_rem<T, 3>(a, pw_host, G, smem, s);
        default: break;
    }
    if constexpr (R > 4) {
        switch (a.nt % R) {
            case 4: return launch_rem<T, 4 % R>(a, pw_host, G, smem, s);
            case 5: return launch_rem<T, 5 % R>(a, pw_host, G, smem, s);
            case 6: return launch_rem<T, 6 % R>(a, pw_host, G, smem, s);
            case 7: return launch_rem<T, 7 % R>(a, pw_host, G, smem, s);
            default: break;
        }
    }
    return cudaErrorInvalidValue;
}

template size_t col_smem<float>(int, int);
template size_t col_smem<double>(int, int);
template cudaError_t launch_col<float>(const ColArgs<float>&, const float2*, cudaStream_t);
template cudaError_t launch_col<double>(const ColArgs<double>&, const double2*, cudaStream_t);

}  // namespace fgb
