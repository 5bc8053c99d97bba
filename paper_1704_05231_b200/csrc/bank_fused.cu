// K5: fused row + column Gabor stages for one frequency, small half-widths.
//
// For sigma <= 4 (h <= 12 at radius 3) the separate row / column launches are
// bound by the J round trip through memory (nd x 8 B written + read per
// pixel) and by launch latency, not by arithmetic.  This kernel keeps J in
// shared memory: one CTA = 32 columns x TY output rows x ALL direct
// orientations of the frequency.
//   1. stage the clamped input tile (TY+2h) x (32+2h)             (cp.async)
//   2. row stage (gabor.py:107-132, taps w e^{-i wc t}, symmetric pairs shared
//      across orientations) for the TY+2h rows -> J_k tiles in shared memory
//   3. column stage (gabor.py:135-164 + bank.py:68-74) per orientation:
//      A = sum ka J, B = sum kb J -> F_theta = A - iB, F_{pi-theta} = conj(A + iB)
// Tap tables travel in the kernel parameters (uniform-register FFMA operands).
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace fgb {

namespace {

constexpr int kBfTX = 32;
constexpr int kBfWarps = 8;

template <int ND, int R>
__global__ void __launch_bounds__(kBfTX * kBfWarps) bank_fused_kernel(const __grid_constant__ BankFusedArgs a,
                                                                      const __grid_constant__ BankFusedW pw) {
    constexpr int NDP = (ND + 1) & ~1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int h = a.h, nt = 2 * a.h + 1;
    const int ntp = (nt + R - 1) / R * R;  // taps padded with zero weights to whole register chunks
    const int TY = R * kBfWarps;
    const int NR = TY + 2 * h;          // J rows holding data
    const int NRA = TY + ntp - 1;       // J rows allocated (zero padded)
    const int NC = kBfTX + 2 * h;       // input columns
    float2* js = reinterpret_cast<float2*>(smem_raw);                  // [ND][NRA][32]
    float* fin = reinterpret_cast<float*>(js + (size_t)ND * NRA * kBfTX);  // [NR][NC]

    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * kBfTX + tx;
    const int b = blockIdx.z;
    const int x0 = blockIdx.x * kBfTX, y0 = blockIdx.y * TY;
    const int H = a.H, W = a.W;

    {
        const float* src = a.img + (size_t)b * a.img_bstride;
        for (int i = tid; i < NR * NC; i += kBfTX * kBfWarps) {
            const int r = i / NC, q = i - r * NC;
            const int yy = clampi(y0 - h + r, 0, H - 1);
            const int xx = clampi(x0 - h + q, 0, W - 1);
            cp_async4(fin + i, src + (size_t)yy * a.pitch + xx);
        }
    }
    for (int i = tid; i < ND * (NRA - NR) * kBfTX; i += kBfTX * kBfWarps) {
        const int k = i / ((NRA - NR) * kBfTX), rem = i - k * (NRA - NR) * kBfTX;
        js[((size_t)k * NRA + NR) * kBfTX + rem] = make_float2(0.f, 0.f);
    }
    cp_async_wait_all();
    __syncthreads();

    // ---- row stage: J_k(r, c) for every direct orientation ----
    for (int pos = tid; pos < NR * kBfTX; pos += kBfTX * kBfWarps) {
        const int r = pos / kBfTX, c = pos - r * kBfTX;
        const float* f = fin + (size_t)r * NC + c + h;  // f[t] = input at column c + t
        float jr[ND], ji[ND];
        const float f0 = f[0];
#pragma unroll
        for (int k = 0; k < ND; ++k) {
            jr[k] = pw.w[2 * k] * f0;
            ji[k] = 0.f;
        }
        for (int t = 1; t <= h; ++t) {
            const float p = f[t], m = f[-t];
            const float s = p + m, d = p - m;
            const int wr = t * NDP * 2;
#pragma unroll
            for (int k = 0; k < ND; ++k) {
                jr[k] = fmaf(pw.w[wr + 2 * k], s, jr[k]);
                ji[k] = fmaf(pw.w[wr + 2 * k + 1], d, ji[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < ND; ++k) js[((size_t)k * NRA + r) * kBfTX + c] = make_float2(jr[k], ji[k]);
    }
    __syncthreads();

    // ---- column stage per orientation ----
    const int x = x0 + tx;
    if (x >= W) return;
    const float* wcol = pw.w + a.col_w_off;  // [ND][ntp] (ka, kb) pairs, zero beyond nt
#pragma unroll 1
    for (int k = 0; k < ND; ++k) {
        float Ar[R], Ai[R], Br[R], Bi[R];
#pragma unroll
        for (int r = 0; r < R; ++r) Ar[r] = Ai[r] = Br[r] = Bi[r] = 0.f;
        const float2* jc = js + ((size_t)k * NRA + ty * R) * kBfTX + tx;  // J_k rows ty*R + q (tile coords)
        const float* wk = wcol + 2 * k * ntp;
#pragma unroll 1
        for (int c0 = 0; c0 < ntp; c0 += R) {
            float2 v[2 * R - 1];
#pragma unroll
            for (int m = 0; m < 2 * R - 1; ++m) v[m] = jc[(c0 + m) * kBfTX];
#pragma unroll
            for (int tt = 0; tt < R; ++tt) {
                const float ka = wk[2 * (c0 + tt)], kb = wk[2 * (c0 + tt) + 1];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    Ar[r] = fmaf(ka, v[r + tt].x, Ar[r]);
                    Ai[r] = fmaf(ka, v[r + tt].y, Ai[r]);
                    Br[r] = fmaf(kb, v[r + tt].x, Br[r]);
                    Bi[r] = fmaf(kb, v[r + tt].y, Bi[r]);
                }
            }
        }
        const BankFusedOut& o = a.out[k];
        float2* base = a.dst + (size_t)b * a.dst_bstride + x;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int y = y0 + ty * R + r;
            if (y >= H) break;
            const size_t pix = (size_t)y * W;
            // F_theta = A - iB ; F_{pi-theta} = conj(A + iB)
            __stcs(base + o.direct + pix, make_float2(Ar[r] + Bi[r], Ai[r] - Br[r]));
            if (o.mirror >= 0) __stcs(base + o.mirror + pix, make_float2(Ar[r] - Bi[r], -(Ai[r] + Br[r])));
        }
    }
}

template <int ND>
cudaError_t launch_nd(const BankFusedArgs& a, const BankFusedW& w, cudaStream_t s) {
    const int R = bank_fused_r(a.h);
    const int TY = R * kBfWarps;
    const size_t smem = bank_fused_smem(a.h, ND, TY);
    auto kern = R == 8 ? bank_fused_kernel<ND, 8> : bank_fused_kernel<ND, 4>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    dim3 grid((a.W + kBfTX - 1) / kBfTX, (a.H + TY - 1) / TY, a.batch);
    kern<<<grid, dim3(kBfTX, kBfWarps), smem, s>>>(a, w);
    return cudaGetLastError();
}

}  // namespace

size_t bank_fused_smem(int h, int nd, int TY) {
    const int R = TY / kBfWarps, nt = 2 * h + 1, ntp = (nt + R - 1) / R * R;
    const int NR = TY + 2 * h, NRA = TY + ntp - 1, NC = kBfTX + 2 * h;
    return (size_t)nd * NRA * kBfTX * sizeof(float2) + (size_t)NR * NC * sizeof(float);
}

bool bank_fused_ok(int h, int nd) {
    if (nd < 1 || nd > kMaxND || h > 12) return false;
    const int R = bank_fused_r(h);
    const int ntp = (2 * h + 1 + R - 1) / R * R;
    const size_t need_w = (size_t)(h + 1) * ((nd + 1) & ~1) * 2 + (size_t)nd * ntp * 2;
    return bank_fused_smem(h, nd, R * kBfWarps) <= 200 * 1024 && need_w <= (size_t)BankFusedW::kCap;
}

cudaError_t launch_bank_fused(const BankFusedArgs& a, const BankFusedW& w, cudaStream_t s) {
    switch (a.nd) {
        case 1: return launch_nd<1>(a, w, s);
        case 2: return launch_nd<2>(a, w, s);
        case 3: return launch_nd<3>(a, w, s);
        case 4: return launch_nd<4>(a, w, s);
        case 5: return launch_nd<5>(a, w, s);
        case 6: return launch_nd<6>(a, w, s);
        case 7: return launch_nd<7>(a, w, s);
        case 8: return launch_nd<8>(a, w, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace fgb
