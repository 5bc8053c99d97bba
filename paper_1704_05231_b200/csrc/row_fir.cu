// K1: fused horizontal stage for symmetric FIR taps (ExactFIR / SDFT rows).
//
// Reference semantics (gabor.py:107-132, sdft.py:75-131): replicate-pad the
// row, modulate by cos/sin(freq * x_true), smooth both planes with the
// sampled Gaussian, crop, recombine.  Folding the modulation/demodulation
// into the taps gives the exact identity
//     J(x) = phase * sum_{t=-h..h} w[t] e^{-i s freq t} f[clamp(x+t)]
// (s = +1 Gabor, s = -1 SDFT; phase = 1 Gabor, e^{i freq c} SDFT), so the
// kernel needs no per-pixel trig and no large-phase fp32 products.  The
// Gaussian is even, so taps t and -t share one add/sub of the input pair,
// and every direct orientation of one frequency (up to kMaxND per launch)
// shares those adds:  per tap pair 2 FADD + 2*ND FFMA instead of 4*ND FFMA
// (fp32: one packed FFMA2 (Jr, Ji) += (kr, ki) * (f+ + f-, f+ - f-) per
// orientation; the (kr, ki) pairs come from the kernel-parameter bank as
// uniform-register operands).
//
// Layout: CTA = 64 threads x kRowTY rows, each thread R=4 consecutive outputs of one
// row (256 px per CTA row).  The clamped row segment lives in shared memory
// split into R residue sub-arrays (element i at (i%R)*S + i/R) so the
// stride-R register windows load conflict-free with immediate offsets.
#include <cstdint>
#include <cstring>

#include "common.cuh"
#include "kernels.h"
#include "umma.cuh"

namespace fgb {

namespace {

constexpr int kRowR = 4;
constexpr int kRowTX = 64;
constexpr int kRowTY = 1;  // one image row per CTA: finer blocks shorten the last wave (config 2 rows -6%, config 3 -3%)
constexpr int kRowSpan = kRowR * kRowTX;  // outputs per CTA row

template <typename T> __host__ __device__ constexpr int row_stride_mod() { return (128 / (int)sizeof(T)); }

// Sub-array length S >= need with S == banks/R (mod banks): conflict-free stores.
template <typename T> __host__ __device__ inline int row_sub_len(int need) {
    const int banks = row_stride_mod<T>();
    const int want = banks / kRowR;
    int s = need;
    int r = ((s - want) % banks + banks) % banks;
    if (r) s += banks - r;
    return s;
}

// fp32 row pitch: room for the 16-byte window reads past the segment end,
// a multiple of 4 floats (16-byte aligned rows).
__host__ __device__ inline int row_vec_pitch(int nseg) { return (nseg + 4 + 3) / 4 * 4; }
// Vector windows for fp32 up to 6 orientations per launch (measured: config 2 / 3
// +1-2%; at 8 orientations the extra live registers made config 5's rows 27% slower).
template <typename T> __host__ __device__ constexpr bool row_vec(int nd) { return sizeof(T) == 4 && nd <= 6; }

// CAP > 0: the group's tap table travels in the kernel parameters (constant
// bank) so the FFMA multipliers are uniform-register operands; CAP == 0:
// table staged in shared memory.
template <typename T, int ND, int CAP, bool LR>
__global__ void __launch_bounds__(kRowTX * kRowTY) row_sym_kernel(const __grid_constant__ RowArgs<T> a,
                                                                  const __grid_constant__ RowGroup<T> g,
                                                                  const __grid_constant__ RowWParam<T, CAP> pw) {
    constexpr int R = kRowR;
    constexpr int NDP = (ND + 1) & ~1;  // weight rows padded to an even count
    using C = cx_t<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* wsm = reinterpret_cast<T*>(smem_raw);  // [(hp+1)][NDP][2]
    const int hp = a.hp;
    // fp32: each CTA row is contiguous (pitch S4, 16-byte aligned) and the
    // windows are read as 16-byte vectors; fp64: R residue sub-arrays of
    // length S (element i at (i%R)*S + i/R) so scalar windows are conflict-free
    constexpr bool VEC = row_vec<T>(ND);
    const int nseg = kRowSpan + 2 * hp;
    const int S = row_sub_len<T>((nseg + R - 1) / R);
    const int S4 = row_vec_pitch(nseg);
    T* rows = CAP > 0 ? wsm : wsm + (size_t)(hp + 1) * NDP * 2;  // [kRowTY][R][S] or [kRowTY][S4]
    auto W = [&](int i) -> T { if constexpr (CAP > 0) return pw.w[i]; else return wsm[i]; };

    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = ty * kRowTX + tx;
    const int b = blockIdx.z;
    const int x0 = blockIdx.x * kRowSpan;
    const int y = blockIdx.y * kRowTY + ty;

    // weights: global table already laid out [(hp+1)][NDP][2]
    if (CAP == 0) {
        // [(hp+1)][NDP][2] table: a multiple of 16 bytes, 16-byte aligned
        const T* wg = a.weights + g.wofs;
        constexpr int per16 = 16 / sizeof(T);
        const int n = (hp + 1) * NDP * 2 / per16;
        for (int i = tid; i < n; i += kRowTX * kRowTY) cp_async16(wsm + i * per16, wg + i * per16);
    }
    T* my = rows + (size_t)ty * (VEC ? S4 : R * S);
    if (y < a.H) {
        const T* src = a.img + (size_t)b * a.img_bstride + (size_t)y * a.pitch;
        if constexpr (VEC) {
            // interior rows with a 16-byte aligned source: 16-byte copies
            const int xs = x0 - hp;
            const bool inner = xs >= 0 && xs + nseg <= a.W && ((reinterpret_cast<uintptr_t>(src + xs) & 15) == 0);
            if (inner) {
                for (int i = 4 * tx; i < nseg; i += 4 * kRowTX) cp_async16(my + i, src + xs + i);
            } else {
                for (int i = tx; i < nseg; i += kRowTX) cp_async<sizeof(T)>(my + i, src + clampi(xs + i, 0, a.W - 1));
            }
        } else {
            for (int i = tx; i < nseg; i += kRowTX) {
                int x = clampi(x0 - hp + i, 0, a.W - 1);
                cp_async<sizeof(T)>(my + (i % R) * S + i / R, src + x);
            }
        }
    }
    cp_async_wait_all();
    __syncthreads();
    if (y >= a.H) return;

    // accumulators (Jr, Ji) per orientation and output: one FFMA2 (fp32) per
    // orientation per tap pair: (Jr, Ji) += (kr, ki) * (f[x+t] + f[x-t], f[x+t] - f[x-t])
    C acc[ND][R];
    // centre tap t = 0: element R*tx + hp + r
    {
        T cv[R];
        if constexpr (VEC) {
            const float4 c4 = *reinterpret_cast<const float4*>(my + R * tx + hp);
            cv[0] = c4.x; cv[1] = c4.y; cv[2] = c4.z; cv[3] = c4.w;
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) cv[r] = my[r * S + tx + hp / R];
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
#pragma unroll
            for (int k = 0; k < ND; ++k) acc[k][r] = mk<T>(W(k * 2) * cv[r], T(0));
        }
    }
    const int nch = hp / R;
#pragma unroll 1
    for (int c = 0; c < nch; ++c) {
        // right window: f[x + r + t], t = 1 + cR + tt  ->  q = r + tt in [0, 2R-2]
        // left  window: f[x + r - t]                    ->  q' = r - tt + R - 1
        // right window element R*tx + hp + R*c + 1 + q, left R*tx + hp - R*c - R + q
        T rv[2 * R - 1], lv[2 * R - 1];
        if constexpr (VEC) {
            const float4* r4 = reinterpret_cast<const float4*>(my + R * tx + hp + R * c);
            const float4* l4 = reinterpret_cast<const float4*>(my + R * tx + hp - R * c - R);
            const float4 ra = r4[0], rb4 = r4[1], la = l4[0], lb4 = l4[1];
            rv[0] = ra.y; rv[1] = ra.z; rv[2] = ra.w; rv[3] = rb4.x; rv[4] = rb4.y; rv[5] = rb4.z; rv[6] = rb4.w;
            lv[0] = la.x; lv[1] = la.y; lv[2] = la.z; lv[3] = la.w; lv[4] = lb4.x; lv[5] = lb4.y; lv[6] = lb4.z;
        } else {
            const int rb = tx + hp / R + c;
            const int lb = tx + hp / R - c - 1;
#pragma unroll
            for (int q = 0; q < 2 * R - 1; ++q) {
                rv[q] = my[((1 + q) % R) * S + rb + (1 + q) / R];
                lv[q] = my[(q % R) * S + lb + q / R];
            }
        }
#pragma unroll
        for (int tt = 0; tt < R; ++tt) {
            const int wrow = (1 + c * R + tt) * NDP * 2;
            T wr[NDP], wi[NDP];
            if constexpr (CAP > 0) {
                if constexpr (sizeof(T) == 4) {
                    // (kr, ki) as one 8-byte uniform load (LDCU.64) instead of two LDCU.32:
                    // the tap loads were 24% of the ND = 8 kernel's instructions
                    const float2* p2 = reinterpret_cast<const float2*>(pw.w) + wrow / 2;
#pragma unroll
                    for (int k = 0; k < NDP; ++k) {
                        const float2 kk = p2[k];
                        wr[k] = kk.x;
                        wi[k] = kk.y;
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < NDP; ++k) { wr[k] = W(wrow + 2 * k); wi[k] = W(wrow + 2 * k + 1); }
                }
            } else {
#pragma unroll
                for (int k = 0; k < NDP; k += 2) {
                    if constexpr (sizeof(T) == 4) {
                        float4 w4 = *reinterpret_cast<const float4*>(wsm + wrow + 2 * k);
                        wr[k] = w4.x; wi[k] = w4.y; wr[k + 1] = w4.z; wi[k + 1] = w4.w;
                    } else {
                        double2 w0 = *reinterpret_cast<const double2*>(wsm + wrow + 2 * k);
                        double2 w1 = *reinterpret_cast<const double2*>(wsm + wrow + 2 * k + 2);
                        wr[k] = w0.x; wi[k] = w0.y; wr[k + 1] = w1.x; wi[k + 1] = w1.y;
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const T p = rv[r + tt], m = lv[r - tt + R - 1];
                const C sd = mk<T>(p + m, p - m);
#pragma unroll
                for (int k = 0; k < ND; ++k) {
                    if (LR && k == ND - 1) {  // real J (RowGroup::last_real): Im stays 0
                        acc[k][r].x = fma(wr[k], sd.x, acc[k][r].x);
                    } else if constexpr (sizeof(T) == 4) {
                        acc[k][r] = __ffma2_rn(make_float2(wr[k], wi[k]), sd, acc[k][r]);
                    } else {
                        acc[k][r].x = fma(wr[k], sd.x, acc[k][r].x);
                        acc[k][r].y = fma(wi[k], sd.y, acc[k][r].y);
                    }
                }
            }
        }
    }

    const int xb = x0 + R * tx;
    if constexpr (sizeof(T) == 4) {
        if (a.j16) {
            // split-fp16 J for the tensor-core column pass (col_umma.cu): J 2^e = hi + lo per
            // component, half2 (re, im) per element, strip-major planes; the edge rows also fill the
            // jpad pad rows
            if (xb >= a.W) return;
            const float sc = ldexpf(1.f, jscale_exp(a.maxbits[b]));
            const int r0 = y == 0 ? 0 : y + a.jpad;
            const int r1 = y == a.H - 1 ? a.H + 2 * a.jpad - 1 : y + a.jpad;
#pragma unroll
            for (int k = 0; k < ND; ++k) {
                uint32_t hw[R], lw[R];
#pragma unroll
                for (int r = 0; r < R; ++r) umma::split_f16x2(acc[k][r].x * sc, acc[k][r].y * sc, hw[r], lw[r]);
                // strip-major plane: [W / 64 strips][H + 2 jpad rows][64]
                uint32_t* hp0 = reinterpret_cast<uint32_t*>(a.dst_base + g.dst_off[k] + (size_t)b * a.out_bstride) +
                                (size_t)(xb >> 6) * (a.H + 2 * a.jpad) * 64 + (xb & 63);
                for (int rr = r0; rr <= r1; ++rr) {
                    uint32_t* ph = hp0 + (size_t)rr * 64;
                    *reinterpret_cast<uint4*>(ph) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                    *reinterpret_cast<uint4*>(ph + a.j16_plane) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
                }
            }
            return;
        }
    }
    const size_t ob = (size_t)b * a.out_bstride + (size_t)y * a.W;
#pragma unroll
    for (int k = 0; k < ND; ++k) {
        C* dst = a.dst_base + g.dst_off[k] + ob;
        C v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            T re = acc[k][r].x, im = acc[k][r].y;
            if (g.has_phase) {
                const T pr = g.phase_re[k], pi = g.phase_im[k];
                T nr = pr * re - pi * im;
                T ni = pr * im + pi * re;
                re = nr; im = ni;
            }
            v[r] = mk<T>(re, im);
        }
        if (xb + R <= a.W && (a.W % 2) == 0 && sizeof(T) == 4) {
            // 2 x 16-byte stores
            float4* d4 = reinterpret_cast<float4*>(dst + xb);
            const float* f = reinterpret_cast<const float*>(v);
            d4[0] = make_float4(f[0], f[1], f[2], f[3]);
            d4[1] = make_float4(f[4], f[5], f[6], f[7]);
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (xb + r < a.W) dst[xb + r] = v[r];
        }
    }
}

}  // namespace

template <typename T> size_t row_sym_smem(int hp, int nd, bool taps_in_smem) {
    const int ndp = (nd + 1) & ~1;
    const int nseg = kRowSpan + 2 * hp;
    const int S = row_sub_len<T>((nseg + kRowR - 1) / kRowR);
    const size_t rows = row_vec<T>(nd) ? (size_t)kRowTY * row_vec_pitch(nseg) : (size_t)kRowTY * kRowR * S;
    return sizeof(T) * ((taps_in_smem ? (size_t)(hp + 1) * ndp * 2 : 0) + rows);
}

template <typename T> int row_sym_pad(int h) { return (h + kRowR - 1) / kRowR * kRowR; }

template <typename T, int ND, int CAP, bool LR = false>
static cudaError_t launch_cap(const RowArgs<T>& a, const RowGroup<T>& g, const T* pw_host, cudaStream_t s) {
    const size_t smem = row_sym_smem<T>(a.hp, ND, CAP == 0);
    auto kern = row_sym_kernel<T, ND, CAP, LR>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    static RowWParam<T, CAP> pw;  // host staging (launches are serialised by the engine lock)
    constexpr int NDP = (ND + 1) & ~1;
    if constexpr (CAP > 0) std::memcpy(pw.w, pw_host, sizeof(T) * (size_t)(a.hp + 1) * NDP * 2);
    dim3 grid((a.W + kRowSpan - 1) / kRowSpan, (a.H + kRowTY - 1) / kRowTY, a.batch);
    dim3 block(kRowTX, kRowTY);
    kern<<<grid, block, smem, s>>>(a, g, pw);
    return cudaGetLastError();
}

template <typename T, int ND>
static cudaError_t launch_nd(const RowArgs<T>& a, const RowGroup<T>& g, const T* pw_host, cudaStream_t s) {
    constexpr int NDP = (ND + 1) & ~1;
    const size_t need = (size_t)(a.hp + 1) * NDP * 2;
    if constexpr (sizeof(T) == 4) {
        if (g.last_real && pw_host && need <= (size_t)RowWCap<T>::kSmall)
            return launch_cap<T, ND, RowWCap<T>::kSmall, true>(a, g, pw_host, s);
        if (g.last_real && pw_host && need <= (size_t)RowWCap<T>::kLarge)
            return launch_cap<T, ND, RowWCap<T>::kLarge, true>(a, g, pw_host, s);
    }
    if (pw_host && need <= (size_t)RowWCap<T>::kSmall) return launch_cap<T, ND, RowWCap<T>::kSmall>(a, g, pw_host, s);
    if (pw_host && need <= (size_t)RowWCap<T>::kLarge) return launch_cap<T, ND, RowWCap<T>::kLarge>(a, g, pw_host, s);
    return launch_cap<T, ND, 0>(a, g, nullptr, s);
}

template <typename T>
cudaError_t launch_row_sym(const RowArgs<T>& a, const RowGroup<T>& g, const T* pw_host, cudaStream_t s) {
    switch (g.nd) {
        case 1: return launch_nd<T, 1>(a, g, pw_host, s);
        case 2: return launch_nd<T, 2>(a, g, pw_host, s);
        case 3: return launch_nd<T, 3>(a, g, pw_host, s);
        case 4: return launch_nd<T, 4>(a, g, pw_host, s);
        case 5: return launch_nd<T, 5>(a, g, pw_host, s);
        case 6: return launch_nd<T, 6>(a, g, pw_host, s);
        case 7: return launch_nd<T, 7>(a, g, pw_host, s);
        case 8: return launch_nd<T, 8>(a, g, pw_host, s);
        default: return cudaErrorInvalidValue;
    }
}

template size_t row_sym_smem<float>(int, int, bool);
template size_t row_sym_smem<double>(int, int, bool);
template int row_sym_pad<float>(int);
template int row_sym_pad<double>(int);
template cudaError_t launch_row_sym<float>(const RowArgs<float>&, const RowGroup<float>&, const float*, cudaStream_t);
template cudaError_t launch_row_sym<double>(const RowArgs<double>&, const RowGroup<double>&, const double*,
                                            cudaStream_t);

}  // namespace fgb
