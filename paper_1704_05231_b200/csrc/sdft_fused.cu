// K3: fused localized SDFT for power-of-two square windows (FIR Gaussian).
//
// Reference: sdft.py:75-213 (Algorithm 2).  With the modulation folded into
// the taps, one stage computes  J_u(x) = sum_t w[t] e^{i phi_u (c+t)} z[x+t],
// phi_u = 2 pi u / M.  The phase is periodic in s = (c+t) mod M, so
//     g_s(x) = sum_{t : (c+t) = s mod M} w[t] z[x+t]      (2h+1 FMAs)
//     J_u(x) = sum_s g_s e^{+2 pi i u s / M}             (one M-point FFT)
// gives EVERY bin of the stage at once.  The row stage (real input) writes
// J_u for the pair heads u <= M/2 to shared memory; the column stage folds
// J_u over rows and FFTs again, producing F_{u,v} for all v.  Bins of the
// mirrored row M-u come from the same registers:
//     F_{M-u,v} = conj(F_{u,(M-v) mod M})   (sdft.py:202-203 + 209-212),
// so one CTA writes all 2M bins of a pair head straight from registers and
// the kernel is bound by the complex64 output stream (8 B per px*bin).
//
// CTA: 32 columns x TY rows x one pair head, blockDim (32, 8).  Shared
// memory: clamped input tile (TY+2h) x (32+2h), the Gaussian taps and J_u of
// the head; the row stage of one head is a fold plus an M-term DFT.
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace fgb {

namespace {

constexpr int kSdTX = 32;
constexpr int kSdWarps = 8;

// cos(2 pi k / 32), k = 0..31 -- twiddles of every power-of-two M <= 32.
// __constant__ tables: compile-time indices become constant-bank operands
// (a function-local constexpr table would be materialised in local memory).
#define FGB_TW32                                                                                            \
    {1.0, 0.98078528040323043, 0.92387953251128674, 0.83146961230254524, 0.70710678118654757,              \
     0.55557023301960218, 0.38268343236508984, 0.19509032201612833, 0.0, -0.19509032201612833,             \
     -0.38268343236508984, -0.55557023301960218, -0.70710678118654757, -0.83146961230254524,               \
     -0.92387953251128674, -0.98078528040323043, -1.0, -0.98078528040323043, -0.92387953251128674,         \
     -0.83146961230254524, -0.70710678118654757, -0.55557023301960218, -0.38268343236508984,               \
     -0.19509032201612833, 0.0, 0.19509032201612833, 0.38268343236508984, 0.55557023301960218,             \
     0.70710678118654757, 0.83146961230254524, 0.92387953251128674, 0.98078528040323043}
__constant__ double c_tw64[32] = FGB_TW32;
__constant__ float c_tw32[32] = FGB_TW32;
template <typename T> __device__ __forceinline__ T tw_cos(int k);
template <> __device__ __forceinline__ float tw_cos<float>(int k) { return c_tw32[k & 31]; }
template <> __device__ __forceinline__ double tw_cos<double>(int k) { return c_tw64[k & 31]; }
template <typename T> __device__ __forceinline__ T tw_sin(int k) { return tw_cos<T>(k - 8); }

__host__ __device__ constexpr int bitrev(int x, int bits) {
    int r = 0;
    for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1) << (bits - 1 - i);
    return r;
}
__host__ __device__ constexpr int ilog2(int m) { return m <= 1 ? 0 : 1 + ilog2(m / 2); }

// In-register radix-2 DIT FFT with the + sign: X[v] = sum_s x[s] e^{+2 pi i v s / M}.
// Trivial twiddles (1, i) are special-cased at compile time.
// compile-time bit-reversal permutation (a runtime-evaluated index would
// demote the register arrays to local memory)
template <typename T, int M, int I>
__device__ __forceinline__ void bitrev_perm(T (&re)[M], T (&im)[M]) {
    if constexpr (I < M) {
        constexpr int J = bitrev(I, ilog2(M));
        if constexpr (J > I) {
            T t = re[I]; re[I] = re[J]; re[J] = t;
            t = im[I]; im[I] = im[J]; im[J] = t;
        }
        bitrev_perm<T, M, I + 1>(re, im);
    }
}

template <typename T, int M, int LEN>
__device__ __forceinline__ void fft_stage(T (&re)[M], T (&im)[M]) {
    if constexpr (LEN <= M) {
#pragma unroll
        for (int i = 0; i < M; i += LEN) {
#pragma unroll
            for (int j = 0; j < LEN / 2; ++j) {
                const int k = j * (32 / LEN);  // twiddle e^{+2 pi i j / LEN} = W32^k
                const int a = i + j, b = i + j + LEN / 2;
                T tr, ti;
                if (k == 0) {
                    tr = re[b]; ti = im[b];
                } else if (k == 8) {  // multiply by +i
                    tr = -im[b]; ti = re[b];
                } else {
                    const T wr = tw_cos<T>(k), wi = tw_sin<T>(k);
                    tr = wr * re[b] - wi * im[b];
                    ti = wr * im[b] + wi * re[b];
                }
                re[b] = re[a] - tr; im[b] = im[a] - ti;
                re[a] = re[a] + tr; im[a] = im[a] + ti;
            }
        }
        fft_stage<T, M, 2 * LEN>(re, im);
    }
}

// In-register radix-2 DIT FFT with the + sign: X[v] = sum_s x[s] e^{+2 pi i v s / M};
// every index is a compile-time constant (stages unrolled by template recursion).
template <typename T, int M>
__device__ __forceinline__ void fft_pos(T (&re)[M], T (&im)[M]) {
    bitrev_perm<T, M, 0>(re, im);
    fft_stage<T, M, 2>(re, im);
}

// Fold of 2h+1 taps into M phase residues: g[s] = sum_{(c+t) = s mod M} w[t] v[t].
// HC > 0: compile-time half-width (exact taps, fully unrolled).  HC == 0:
// runtime h over zero-padded blocks of M taps (t = -c + M j + s).
template <typename T, int M, int HC, typename V, typename Acc>
__device__ __forceinline__ void fold(const T* w, V v, int j0, int j1, Acc acc) {
    constexpr int c = M / 2;
    if constexpr (HC > 0) {
#pragma unroll
        for (int t = -HC; t <= HC; ++t) acc(((c + t) % M + M) % M, w[t], v(t));
    } else {
        for (int j = j0; j <= j1; ++j) {
#pragma unroll
            for (int s = 0; s < M; ++s) {
                const int t = -c + M * j + s;
                acc(s, w[t], v(t));
            }
        }
    }
}

// One CTA = one 32 x TY tile x ONE pair head u.  Heads are the slowest grid
// dimension, so the CTAs in flight all write the same 2M output planes
// (writing all M^2 planes per CTA thrashes the TLB: 8.6 GB of outputs).
template <typename T, int M, int HC>
__global__ void __launch_bounds__(kSdTX * kSdWarps) sdft_fused_kernel(SdftFusedArgs<T> a, int TY) {
    using C = cx_t<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int c = M / 2;  // phase centre, sdft.py:118 (x_hat = x - M//2)
    const int h = HC > 0 ? HC : a.h;
    // tap span [tl, tr]: exact for HC > 0, padded to whole residue blocks otherwise
    const int j0 = HC > 0 ? 0 : (int)floorf((float)(c - h) / M);
    const int j1 = HC > 0 ? 0 : (int)floorf((float)(c + h) / M);
    const int tl = HC > 0 ? -h : -c + M * j0;
    const int tr = HC > 0 ? h : -c + M * (j1 + 1) - 1;
    const int NR = TY + tr - tl;        // rows of J / input rows
    const int NC = kSdTX + tr - tl;     // input columns
    const int nw = tr - tl + 1;
    C* js = reinterpret_cast<C*>(smem_raw);                // [NR][32]
    T* fs = reinterpret_cast<T*>(js + (size_t)NR * kSdTX);  // [NR][NC]
    T* wsm = fs + (size_t)NR * NC;                          // [nw], wsm[t - tl]
    T* ecs = wsm + ((nw + 1) & ~1);                         // [M][2]: e^{+2 pi i u s / M}

    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * kSdTX + tx;
    const int k = blockIdx.z / a.batch;
    const int b = blockIdx.z - k * a.batch;
    const int u = a.heads[k];
    const int x0 = blockIdx.x * kSdTX, y0 = blockIdx.y * TY;

    // ---- stage the clamped input tile, the (zero-padded) taps, the head twiddles ----
    {
        const T* src = a.img + (size_t)b * a.img_bstride;
        for (int i = tid; i < NR * NC; i += kSdTX * kSdWarps) {
            const int r = i / NC, q = i - r * NC;
            const int yy = clampi(y0 + tl + r, 0, a.H - 1);
            const int xx = clampi(x0 + tl + q, 0, a.W - 1);
            cp_async<sizeof(T)>(fs + i, src + (size_t)yy * a.pitch + xx);
        }
        for (int i = tid; i < nw; i += kSdTX * kSdWarps) {
            const int t = tl + i;
            wsm[i] = (t >= -h && t <= h) ? a.w[t + h] : T(0);
        }
        if (tid < M) {
            const int kk = ((u * tid) % M) * (32 / M);
            ecs[2 * tid] = tw_cos<T>(kk);
            ecs[2 * tid + 1] = tw_sin<T>(kk);
        }
    }
    cp_async_wait_all();
    __syncthreads();
    const T* wc = wsm - tl;  // wc[t], t in [tl, tr]

    // ---- row stage for head u: J_u = sum_s g_s e^{+2 pi i u s/M} ----
    T er[M], ei[M];
#pragma unroll
    for (int s2 = 0; s2 < M; ++s2) { er[s2] = ecs[2 * s2]; ei[s2] = ecs[2 * s2 + 1]; }
    for (int r = ty; r < NR; r += kSdWarps) {
        T g[M];
#pragma unroll
        for (int s2 = 0; s2 < M; ++s2) g[s2] = T(0);
        const T* frow = fs + (size_t)r * NC + tx - tl;  // frow[t] = f[x + t]
        fold<T, M, HC>(wc, [&](int t) { return frow[t]; }, j0, j1,
                       [&](int s2, T w, T v) { g[s2] = fma(w, v, g[s2]); });
        T jr = T(0), ji = T(0);
#pragma unroll
        for (int s2 = 0; s2 < M; ++s2) {
            jr = fma(g[s2], er[s2], jr);
            ji = fma(g[s2], ei[s2], ji);
        }
        js[(size_t)r * kSdTX + tx] = mk<T>(jr, ji);
    }
    __syncthreads();

    // ---- column stage: fold J_u over rows, FFT, write the head's 2M bins ----
    const int x = x0 + tx;
    if (x >= a.W) return;
    const size_t HW = (size_t)a.H * a.W;
    const int s0 = a.head_slot[2 * k], s1 = a.head_slot[2 * k + 1];
    for (int yl = ty; yl < TY; yl += kSdWarps) {
        const int y = y0 + yl;
        if (y >= a.H) break;
        const size_t pix = (size_t)b * a.out_bstride + (size_t)y * a.W + x;
        const C* jcol = js + (size_t)(yl - tl) * kSdTX + tx;  // jcol[t * 32] = J_u[y + t]
        T gr[M], gi[M];
#pragma unroll
        for (int s2 = 0; s2 < M; ++s2) { gr[s2] = T(0); gi[s2] = T(0); }
        fold<T, M, HC>(wc, [&](int t) { return jcol[t * kSdTX]; }, j0, j1, [&](int s2, T w, C v) {
            gr[s2] = fma(w, v.x, gr[s2]);
            gi[s2] = fma(w, v.y, gi[s2]);
        });
        fft_pos<T, M>(gr, gi);
        C* o0 = a.out + (size_t)s0 * HW + pix;
#pragma unroll
        for (int v = 0; v < M; ++v) st_cs(o0 + (size_t)v * HW, mk<T>(gr[v], gi[v]));
        if (s1 >= 0) {
            C* o1 = a.out + (size_t)s1 * HW + pix;
#pragma unroll
            for (int v = 0; v < M; ++v) {
                const int vm = (M - v) & (M - 1);
                st_cs(o1 + (size_t)v * HW, mk<T>(gr[vm], -gi[vm]));
            }
        }
    }
}

// geometry of the padded tap span
inline void sd_span(int M, int h, int hc, int* tl, int* tr) {
    const int c = M / 2;
    if (hc > 0) {
        *tl = -h;
        *tr = h;
        return;
    }
    const int j0 = (int)std::floor((double)(c - h) / M), j1 = (int)std::floor((double)(c + h) / M);
    *tl = -c + M * j0;
    *tr = -c + M * (j1 + 1) - 1;
}

inline int sd_hc(int h) { return (h == 3 || h == 6 || h == 12 || h == 24) ? h : 0; }

template <typename T> size_t sdft_fused_smem(int M, int h, int nh, int TY) {
    int tl, tr;
    sd_span(M, h, sd_hc(h), &tl, &tr);
    const int NR = TY + tr - tl, NC = kSdTX + tr - tl;
    (void)nh;
    return (size_t)NR * kSdTX * sizeof(cx_t<T>) + (size_t)NR * NC * sizeof(T) + (tr - tl + 2 + 2 * M) * sizeof(T) + 16;
}

template <typename T> int sdft_fused_ty(int M, int h, int nh) {
    for (int ty : {32, 16, 8}) {
        if (sdft_fused_smem<T>(M, h, nh, ty) <= 56 * 1024) return ty;  // >= 4 CTAs per SM
    }
    if (sdft_fused_smem<T>(M, h, nh, 8) <= 220 * 1024) return 8;
    return 0;
}

template <typename T, int M, int HC>
cudaError_t launch_mh(const SdftFusedArgs<T>& a, int TY, size_t smem, cudaStream_t s) {
    auto kern = sdft_fused_kernel<T, M, HC>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    dim3 grid((a.W + kSdTX - 1) / kSdTX, (a.H + TY - 1) / TY, a.batch * a.nheads);
    kern<<<grid, dim3(kSdTX, kSdWarps), smem, s>>>(a, TY);
    return cudaGetLastError();
}

template <typename T, int M>
cudaError_t launch_m(const SdftFusedArgs<T>& a, cudaStream_t s) {
    const int TY = sdft_fused_ty<T>(M, a.h, a.nheads);
    if (TY == 0) return cudaErrorInvalidConfiguration;
    const size_t smem = sdft_fused_smem<T>(M, a.h, a.nheads, TY);
    switch (sd_hc(a.h)) {
        case 3: return launch_mh<T, M, 3>(a, TY, smem, s);
        case 6: return launch_mh<T, M, 6>(a, TY, smem, s);
        case 12: return launch_mh<T, M, 12>(a, TY, smem, s);
        case 24: return launch_mh<T, M, 24>(a, TY, smem, s);
        default: return launch_mh<T, M, 0>(a, TY, smem, s);
    }
}

}  // namespace

bool sdft_fused_supported(int M, int h, size_t elem) {
    if (M != 4 && M != 8 && M != 16 && M != 32) return false;
    const int nh = M / 2 + 1;
    return elem == 4 ? sdft_fused_ty<float>(M, h, nh) > 0 : sdft_fused_ty<double>(M, h, nh) > 0;
}

template <typename T> cudaError_t launch_sdft_fused(const SdftFusedArgs<T>& a, int M, cudaStream_t s) {
    switch (M) {
        case 4: return launch_m<T, 4>(a, s);
        case 8: return launch_m<T, 8>(a, s);
        case 16: return launch_m<T, 16>(a, s);
        case 32: return launch_m<T, 32>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

template cudaError_t launch_sdft_fused<float>(const SdftFusedArgs<float>&, int, cudaStream_t);
template cudaError_t launch_sdft_fused<double>(const SdftFusedArgs<double>&, int, cudaStream_t);

}  // namespace fgb
