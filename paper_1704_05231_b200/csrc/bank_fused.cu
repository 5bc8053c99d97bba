// K5: fused row + column Gabor stages for one frequency, small half-widths.
//
// For small sigma the separate row / column launches are bound by the J round
// trip through memory (nd x 8 B written + read per pixel) and by per-launch
// overheads, not by arithmetic.  This kernel keeps J in shared memory: one
// CTA = a 32 x 32 output tile x ALL direct orientations of the frequency.
//   0. stage the clamped input tile (32 + 2hp) x (32 + 2hp)          (cp.async)
//   1. row stage (gabor.py:107-132, taps w e^{-i wc t}): each thread makes 4
//      consecutive J values of one row for every orientation; the symmetric
//      pair (f[x+t] + f[x-t], f[x+t] - f[x-t]) is formed once and shared by
//      all orientations, and one FFMA2 accumulates (jr, ji) per orientation
//   2. column stage (gabor.py:135-164 + bank.py:68-74): each thread makes 2
//      columns x 4 rows of one orientation, A = sum ka J, B = sum kb J with
//      FFMA2 over a register window -> F_theta = A - iB, F_{pi-theta} = conj(A + iB)
// Row and column tap tables travel in the kernel parameters (uniform-register
// FFMA2 operands); taps are zero-padded to whole 4-tap chunks.
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace fgb {

namespace {

constexpr int kFT = 32;        // output tile (32 x 32)
constexpr int kFThreads = 256;

__host__ __device__ inline int fused_pitch(int hp) { return (kFT + 2 * hp) | 1; }  // odd: conflict-free rows

// HH > 0: the half-width is a compile-time constant (exact tap loops, fully
// unrolled, static tap offsets); HH = 0: runtime h with zero-padded chunks.
template <int ND, int HH>
__global__ void __launch_bounds__(kFThreads) bank_fused_kernel(const __grid_constant__ BankFusedArgs a,
                                                               const __grid_constant__ BankFusedW pw) {
    constexpr int NDP = (ND + 1) & ~1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int h = HH > 0 ? HH : a.h;
    const int hp = (h + 3) & ~3;            // row taps padded to 4-tap chunks
    const int ntp = (2 * h + 1 + 3) & ~3;   // column taps padded to 4-tap chunks
    const int NR = kFT + 2 * h;             // J rows holding data
    const int NRA = kFT + ntp + 3;          // J rows allocated (zero rows past NR)
    const int NC = kFT + 2 * hp;            // staged input columns
    float2* js = reinterpret_cast<float2*>(smem_raw);                        // [ND][NRA][32]
    const int pitch = fused_pitch(hp);
    float* fin = reinterpret_cast<float*>(js + (size_t)ND * NRA * kFT);     // [NR][pitch]

    const int tid = threadIdx.x;
    const int b = blockIdx.z;
    const int x0 = blockIdx.x * kFT, y0 = blockIdx.y * kFT;
    const int H = a.H, W = a.W;

    // ---- 0: input tile, replicate-clamped; fin[r][c] = f[y0 - h + r][x0 - hp + c] ----
    {
        const float* src = a.img + (size_t)b * a.img_bstride;
        for (int i = tid; i < NR * NC; i += kFThreads) {
            const int r = i / NC, c = i - r * NC;
            const int yy = clampi(y0 - h + r, 0, H - 1);
            const int xx = clampi(x0 - hp + c, 0, W - 1);
            cp_async4(fin + r * pitch + c, src + (size_t)yy * a.pitch + xx);
        }
        for (int i = tid; i < ND * (NRA - NR) * kFT; i += kFThreads) {
            const int k = i / ((NRA - NR) * kFT), rem = i - k * (NRA - NR) * kFT;
            js[((size_t)k * NRA + NR) * kFT + rem] = make_float2(0.f, 0.f);
        }
        cp_async_wait_all();
        __syncthreads();
    }

    // ---- 1: row stage, 4 consecutive J columns of one row per task ----
    for (int task = tid; task < NR * 8; task += kFThreads) {
        const int r = task >> 3, q = task & 7;
        const float* f = fin + r * pitch + hp + 4 * q;  // f[j] = input at x = x0 + 4q + j
        float2 acc[ND][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float v = f[j];
#pragma unroll
            for (int k = 0; k < ND; ++k) acc[k][j] = make_float2(pw.w[2 * k] * v, 0.f);
        }
        constexpr int kRowTrip = HH > 0 ? (HH + 3) / 4 : 1;
#pragma unroll
        for (int ci = 0; ci < (HH > 0 ? kRowTrip : (hp >> 2)); ++ci) {
            const int t0 = 1 + 4 * ci;
            // right window f[t0 .. t0 + 6], left window f[-t0 - 3 .. 3 - t0]
            float rv[7], lv[7];
#pragma unroll
            for (int m = 0; m < 7; ++m) {
                rv[m] = f[t0 + m];
                lv[m] = f[-t0 - 3 + m];
            }
#pragma unroll
            for (int tt = 0; tt < 4; ++tt) {
                if (HH > 0 && t0 + tt > HH) break;  // exact tap count (compile-time)
                const int wrow = (t0 + tt) * NDP * 2;
                float2 wk[ND];
#pragma unroll
                for (int k = 0; k < ND; ++k) wk[k] = make_float2(pw.w[wrow + 2 * k], pw.w[wrow + 2 * k + 1]);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float p = rv[j + tt], m = lv[j - tt + 3];
                    const float2 sd = make_float2(p + m, p - m);
#pragma unroll
                    for (int k = 0; k < ND; ++k) acc[k][j] = __ffma2_rn(wk[k], sd, acc[k][j]);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < ND; ++k) {
            float4* d = reinterpret_cast<float4*>(js + ((size_t)k * NRA + r) * kFT + 4 * q);
            d[0] = make_float4(acc[k][0].x, acc[k][0].y, acc[k][1].x, acc[k][1].y);
            d[1] = make_float4(acc[k][2].x, acc[k][2].y, acc[k][3].x, acc[k][3].y);
        }
    }
    __syncthreads();

    // ---- 2: column stage, 2 columns x 4 rows of one orientation per task ----
    for (int task = tid; task < ND * 128; task += kFThreads) {
        const int k = task >> 7, rem = task & 127;
        const int g = rem >> 4, cp = rem & 15;  // warp: 16 column pairs x 2 row groups
        const float4* jc = reinterpret_cast<const float4*>(js + ((size_t)k * NRA + 4 * g) * kFT) + cp;
        const float* wc = pw.w + a.col_w_off + 2 * k * ntp;
        float2 A[2][4], B[2][4];
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
            for (int i = 0; i < 4; ++i) A[s][i] = B[s][i] = make_float2(0.f, 0.f);
        constexpr int kColTrip = HH > 0 ? (2 * HH + 1 + 3) / 4 : 1;
#pragma unroll
        for (int ci = 0; ci < (HH > 0 ? kColTrip : (ntp >> 2)); ++ci) {
            const int c0 = 4 * ci;
            float4 v[7];
#pragma unroll
            for (int m = 0; m < 7; ++m)
                if (HH == 0 || c0 + m < 2 * HH + 4) v[m] = jc[(c0 + m) * (kFT / 2)];
#pragma unroll
            for (int tt = 0; tt < 4; ++tt) {
                if (HH > 0 && c0 + tt > 2 * HH) break;  // exact tap count (compile-time)
                const float ka = wc[2 * (c0 + tt)], kb = wc[2 * (c0 + tt) + 1];
                const float2 wa = make_float2(ka, ka), wb = make_float2(kb, kb);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float4 qv = v[i + tt];
                    const float2 lo = make_float2(qv.x, qv.y), hi = make_float2(qv.z, qv.w);
                    A[0][i] = __ffma2_rn(wa, lo, A[0][i]);
                    A[1][i] = __ffma2_rn(wa, hi, A[1][i]);
                    B[0][i] = __ffma2_rn(wb, lo, B[0][i]);
                    B[1][i] = __ffma2_rn(wb, hi, B[1][i]);
                }
            }
        }
        const BankFusedOut o = a.out[k];
        const int x = x0 + 2 * cp;
        if (x >= W) continue;
        const bool two = x + 1 < W;
        float2* base = a.dst + (size_t)b * a.dst_bstride + x;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int y = y0 + 4 * g + i;
            if (y >= H) break;
            const size_t pix = (size_t)y * W;
            // F_theta = A - iB ; F_{pi-theta} = conj(A + iB)
            const float2 d0 = make_float2(A[0][i].x + B[0][i].y, A[0][i].y - B[0][i].x);
            const float2 d1 = make_float2(A[1][i].x + B[1][i].y, A[1][i].y - B[1][i].x);
            if (two && (W & 1) == 0) {
                __stcs(reinterpret_cast<float4*>(base + o.direct + pix), make_float4(d0.x, d0.y, d1.x, d1.y));
            } else {
                __stcs(base + o.direct + pix, d0);
                if (two) __stcs(base + o.direct + pix + 1, d1);
            }
            if (o.mirror >= 0) {
                const float2 m0 = make_float2(A[0][i].x - B[0][i].y, -(A[0][i].y + B[0][i].x));
                const float2 m1 = make_float2(A[1][i].x - B[1][i].y, -(A[1][i].y + B[1][i].x));
                if (two && (W & 1) == 0) {
                    __stcs(reinterpret_cast<float4*>(base + o.mirror + pix), make_float4(m0.x, m0.y, m1.x, m1.y));
                } else {
                    __stcs(base + o.mirror + pix, m0);
                    if (two) __stcs(base + o.mirror + pix + 1, m1);
                }
            }
        }
    }
}

template <int ND>
cudaError_t launch_nd(const BankFusedArgs& a, const BankFusedW& w, cudaStream_t s) {
    const size_t smem = bank_fused_smem(a.h, ND, kFT);
    auto kern = a.h == 6 ? bank_fused_kernel<ND, 6> : bank_fused_kernel<ND, 0>;  // h = 6: sigma 2 at radius 3
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    dim3 grid((a.W + kFT - 1) / kFT, (a.H + kFT - 1) / kFT, a.batch);
    kern<<<grid, kFThreads, smem, s>>>(a, w);
    return cudaGetLastError();
}

}  // namespace

size_t bank_fused_smem(int h, int nd, int /*TY*/) {
    const int hp = (h + 3) & ~3, ntp = (2 * h + 1 + 3) & ~3;
    const int NR = kFT + 2 * h, NRA = kFT + ntp + 3;
    return (size_t)nd * NRA * kFT * sizeof(float2) + (size_t)NR * fused_pitch(hp) * sizeof(float);
}

bool bank_fused_ok(int h, int nd) {
    if (nd < 1 || nd > kMaxND || h < 1 || h > 24) return false;
    const int hp = (h + 3) & ~3, ntp = (2 * h + 1 + 3) & ~3;
    const size_t need_w = (size_t)(hp + 1) * ((nd + 1) & ~1) * 2 + (size_t)nd * ntp * 2;
    return bank_fused_smem(h, nd, kFT) <= 112 * 1024 && need_w <= (size_t)BankFusedW::kCap;
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
