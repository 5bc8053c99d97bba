// K4: recursive-Gaussian (RecursiveIIR) stage, fp64 recursion state,
// segment-parallel, for both directions of the separable pipeline.
//
// Restates gaussian.py:215-228 (_iir_lines with assume_padded: the stage
// already replicate-padded by P = ceil(5 sigma)+2, gaussian.py:211) inside
// the modulate / smooth / recombine stages of gabor.py:107-164 and
// sdft.py:75-131:
//   forward : y[n] = B z[n] - a1 y[n-1] - a2 y[n-2] - a3 y[n-3],
//             y[-1] = y[-2] = y[-3] = z[0]  (lfilter_zi * x[0] steady state)
//   backward: u[n] = B y[n] - a1 u[n+1] - a2 u[n+2] - a3 u[n+3],
//             u[L] = u[L+1] = u[L+2] = y[L-1]
// The recursion runs in fp64 (an fp32 recursion misses 1e-5 by up to 125x
// at sigma = 32).
//
// A "line" is one independent recursion (an image column for the vertical
// stage, an image row for the horizontal stage); lines are adjacent threads
// and the source / destination are addressed through (line, sample) strides,
// so the horizontal stage reads the image rows and writes J in place -- no
// transposes.  Scratch is [z][plane][sample][line] (lines contiguous) in
// both modes.
//
// Parallelisation is EXACT (no warm-up approximation): each line is cut into
// NS segments.  A segment runs its recursion from a zero state; with the
// companion matrix A = [[-a1,-a2,-a3],[1,0,0],[0,1,0]] the true output is
//     y[a+m] = y_loc[a+m] + g_m . s_in,   g_m = first row of A^(m+1),
// where s_in is the true 3-sample state entering the segment, and the states
// chain as s_out = s_loc_end + A^len s_in (a 3x3 scan over segments).  The
// backward pass is the same recursion on reversed indices.  Five kernels:
//   fwd    : modulate, local forward recursion -> y_loc (storage type), end states
//   scan<0>: end states -> carry-ins (sequential per line, batched loads)
//   bwd    : correct y, local backward recursion -> u_loc, start states
//   scan<1>: start states -> carry-ins from above
//   out    : correct u, recombine -> outputs
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace fgb {

namespace {

constexpr int kIirTX = 32;  // lines per block (one warp)
constexpr int kIirSY = 4;   // segments per block
constexpr int kIirMinBlocks = 8;  // 64 registers: more resident warps for the latency-bound passes
constexpr int kIirUB = 3;   // scratch samples per load batch (backward / output passes)

struct IirScanMats {
    double Aseg[9], Alast[9];
};



// Recursion step writing y[n] into the slot that held y[n-3]: with three
// named registers whose roles rotate every sample, a 3x unrolled loop needs
// no state moves (y[n] = B z - a1 y[n-1] - a2 y[n-2] - a3 y[n-3]).
__device__ __forceinline__ void rec_into(double& oldest, double z, double ym1, double ym2, const IirCoef& c) {
    const double t = fma(c.B, z, -(c.a2 * ym2 + c.a3 * oldest));
    oldest = fma(-c.a1, ym1, t);
}

// one recursion step on a (y[n-1], y[n-2], y[n-3]) state; returns y[n]
__device__ __forceinline__ double rec_step(double* p, double zin, const IirCoef& c) {
    const double t = fma(c.B, zin, -(c.a2 * p[1] + c.a3 * p[2]));
    const double y = fma(-c.a1, p[0], t);
    p[2] = p[1];
    p[1] = p[0];
    p[0] = y;
    return y;
}


template <typename T, bool REAL> struct SrcT;
template <typename T> struct SrcT<T, true> { using type = T; };
template <typename T> struct SrcT<T, false> { using type = cx_t<T>; };

__device__ __forceinline__ double2 ld_d2(const float* p) { return make_double2((double)*p, 0.0); }
__device__ __forceinline__ double2 ld_d2(const double* p) { return make_double2(*p, 0.0); }
__device__ __forceinline__ double2 ld_d2(const float2* p) { const float2 v = *p; return make_double2(v.x, v.y); }
__device__ __forceinline__ double2 ld_d2(const double2* p) { return *p; }

// Every job is ONE modulation pair (two real planes a, b); the host splits a
// Gabor theta / pi - theta job into its two pairs, so a thread carries 2 x 3
// fp64 states and the kernels stay at a high occupancy.
__device__ __forceinline__ void modulate_pair(int pair, double jr, double ji, double2 cs, double& za, double& zb) {
    if (pair == 0) {
        za = fma(jr, cs.x, ji * cs.y);
        zb = fma(jr, cs.y, -ji * cs.x);
    } else {
        za = fma(jr, cs.x, -ji * cs.y);
        zb = fma(jr, cs.y, ji * cs.x);
    }
}

// ---- pass 1: modulate + zero-state forward recursion per segment ----
// STAGE (horizontal stage: lines are image rows, real input): the CTA's
// 32 rows x (kIirSY * seglen) samples are fetched row-contiguously into shared
// memory first instead of one strided element per thread and sample.
template <typename T, bool REAL, bool STAGE>
__global__ void __launch_bounds__(128, kIirMinBlocks) iir_fwd(const IirArgs<T> a) {
    using S = typename SrcT<T, REAL>::type;
    static_assert(!STAGE || REAL, "staging is for the real-input horizontal stage");
    const int x = blockIdx.x * kIirTX + threadIdx.x;
    const int seg = blockIdx.y * kIirSY + threadIdx.y;
    const int jb = blockIdx.z % a.njobs;
    const int b = blockIdx.z / a.njobs;
    const IirJob<T>& job = a.jobs[jb];
    const int len = a.len, P = a.P, L = len + 2 * P, NL = a.lines;
    const int n0 = seg * a.seglen, n1 = min(L, n0 + a.seglen);
    const S* src = reinterpret_cast<const S*>(a.src_base) + job.src_off + (int64_t)b * a.src_bstride +
                   (int64_t)x * a.src_ls;
    int64_t ss = a.src_ss;
    if constexpr (STAGE) {
        extern __shared__ __align__(16) unsigned char smem_raw[];
        T* tile = reinterpret_cast<T*>(smem_raw);
        const int sw = kIirSY * a.seglen, swp = sw | 1;  // odd row pitch: conflict-free column reads
        const int nb0 = blockIdx.y * kIirSY * a.seglen;
        const S* base = reinterpret_cast<const S*>(a.src_base) + job.src_off + (int64_t)b * a.src_bstride;
        const int tid = threadIdx.y * kIirTX + threadIdx.x;
        for (int r = threadIdx.y; r < kIirTX; r += kIirSY) {  // row r of the CTA, samples across the warp
            const int line = blockIdx.x * kIirTX + r;
            if (line >= NL) continue;
            const S* row = base + (int64_t)line * a.src_ls;
            for (int cc = threadIdx.x; cc < sw; cc += kIirTX) {
                const int n = nb0 + cc;
                if (n < L) tile[r * swp + cc] = row[clampi(n - P, 0, len - 1)];
            }
        }
        (void)tid;
        __syncthreads();
        // thread view: sample n of this line at tile[threadIdx.x * swp + (n - nb0)]
        src = reinterpret_cast<const S*>(tile) + threadIdx.x * swp - nb0 + P;
        ss = 1;
    }
    if (x >= a.lines || seg >= a.nseg) return;
    const double2* tabm = a.tab_base + job.tabm_off;
    const int64_t plane = (int64_t)L * NL;
    T* sc = a.scratch + (int64_t)blockIdx.z * 2 * plane + x;
    const IirCoef c = a.c;
    const int pair = job.need >> 1;
    double pa[3], pb[3];
    if (seg == 0) {  // the reference's steady-state init on the first padded sample
        const double2 v = ld_d2(src + (STAGE ? -P : 0));
        double za, zb;
        modulate_pair(pair, v.x, v.y, tabm[0], za, zb);
        pa[0] = pa[1] = pa[2] = za;
        pb[0] = pb[1] = pb[2] = zb;
    } else {
        pa[0] = pa[1] = pa[2] = pb[0] = pb[1] = pb[2] = 0.0;
    }
    // Three samples per iteration: their inputs are loaded before the
    // dependent recursion consumes them (the scratch stores would otherwise
    // keep the compiler from hoisting loads), and the state registers rotate
    // roles (r0, r1, r2) -> (r2, r0, r1) per sample, so no moves.
    double a0 = pa[0], a1 = pa[1], a2 = pa[2], b0 = pb[0], b1 = pb[1], b2 = pb[2];
    auto in_at = [&](int n) { return ld_d2(src + (STAGE ? n - P : clampi(n - P, 0, len - 1) * ss)); };
    T* o = sc + (int64_t)n0 * NL;
    const int64_t NL64 = NL;
    int n = n0;
    for (; n + 3 <= n1; n += 3) {
        const double2 v0 = in_at(n), v1 = in_at(n + 1), v2 = in_at(n + 2);
        double za, zb;
        modulate_pair(pair, v0.x, v0.y, tabm[n], za, zb);
        rec_into(a2, za, a0, a1, c);  // y[n] -> a2
        rec_into(b2, zb, b0, b1, c);
        o[0] = (T)a2;
        o[plane] = (T)b2;
        o += NL64;
        modulate_pair(pair, v1.x, v1.y, tabm[n + 1], za, zb);
        rec_into(a1, za, a2, a0, c);  // y[n+1] -> a1
        rec_into(b1, zb, b2, b0, c);
        o[0] = (T)a1;
        o[plane] = (T)b1;
        o += NL64;
        modulate_pair(pair, v2.x, v2.y, tabm[n + 2], za, zb);
        rec_into(a0, za, a1, a2, c);  // y[n+2] -> a0; roles back to (a0, a1, a2)
        rec_into(b0, zb, b1, b2, c);
        o[0] = (T)a0;
        o[plane] = (T)b0;
        o += NL64;
    }
    pa[0] = a0; pa[1] = a1; pa[2] = a2;
    pb[0] = b0; pb[1] = b1; pb[2] = b2;
    for (; n < n1; ++n) {  // 0-2 remaining samples
        const double2 v = in_at(n);
        double za, zb;
        modulate_pair(pair, v.x, v.y, tabm[n], za, zb);
        o[0] = (T)rec_step(pa, za, c);
        o[plane] = (T)rec_step(pb, zb, c);
        o += NL64;
    }
    // local end state (y[end], y[end-1], y[end-2]) per plane
    double* st = a.state + (((int64_t)blockIdx.z * a.nseg + seg) * 6) * NL + x;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        st[(int64_t)k * NL] = pa[k];
        st[(int64_t)(3 + k) * NL] = pb[k];
    }
}

// ---- pass 2: forward carry + correction, zero-state backward recursion ----
template <typename T>
__global__ void __launch_bounds__(128, kIirMinBlocks) iir_bwd(const IirArgs<T> a) {
    const int x = blockIdx.x * kIirTX + threadIdx.x;
    const int seg = blockIdx.y * kIirSY + threadIdx.y;
    if (x >= a.lines || seg >= a.nseg) return;
    const int len = a.len, P = a.P, L = len + 2 * P, NL = a.lines;
    const int n0 = seg * a.seglen, n1 = min(L, n0 + a.seglen);
    const int64_t plane = (int64_t)L * NL;
    T* sc = a.scratch + (int64_t)blockIdx.z * 2 * plane + x;
    const IirCoef c = a.c;
    const double* st_all = a.state + ((int64_t)blockIdx.z * a.nseg * 6) * NL + x;
    // true state entering this segment (iir_scan_seq<0> turned the local end states into carry-ins)
    double sa[3], sb[3];
    {
        const double* sj = st_all + (int64_t)seg * 6 * NL;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            sa[k] = sj[(int64_t)k * NL];
            sb[k] = sj[(int64_t)(3 + k) * NL];
        }
    }
    const double* gt = a.g;
    const bool first = seg == 0;
    // backward local recursion from the segment end, on the corrected forward output
    double ua[3], ub[3];
    if (seg == a.nseg - 1) {  // u[L..L+2] = y[L-1] (true value)
        const T* o = sc + (int64_t)(n1 - 1) * NL;
        const double* g = gt + 3 * (n1 - 1 - n0);
        const double ya = first ? (double)o[0] : (double)o[0] + g[0] * sa[0] + g[1] * sa[1] + g[2] * sa[2];
        const double yb = first ? (double)o[plane] : (double)o[plane] + g[0] * sb[0] + g[1] * sb[1] + g[2] * sb[2];
        ua[0] = ua[1] = ua[2] = ya;
        ub[0] = ub[1] = ub[2] = yb;
    } else {
        ua[0] = ua[1] = ua[2] = ub[0] = ub[1] = ub[2] = 0.0;
    }
    // three samples per iteration, rotating state roles (see iir_fwd)
    double a0 = ua[0], a1 = ua[1], a2 = ua[2], b0 = ub[0], b1 = ub[1], b2 = ub[2];
    const double sa0 = sa[0], sa1 = sa[1], sa2 = sa[2], sb0 = sb[0], sb1 = sb[1], sb2 = sb[2];
    const int64_t NL64 = NL;
    T* o = sc + (int64_t)(n1 - 1) * NL;
    const double* g = gt + 3 * (n1 - 1 - n0);  // correction row of the current sample
    // forward value of this segment corrected by the carried-in state (segment 0: exact already)
    auto corr2 = [&](T ya, T yb, const double* gg, double& va, double& vb) {
        va = ya;
        vb = yb;
        if (!first) {
            const double g0 = gg[0], g1 = gg[1], g2 = gg[2];
            va += g0 * sa0 + g1 * sa1 + g2 * sa2;
            vb += g0 * sb0 + g1 * sb1 + g2 * sb2;
        }
    };
    int n = n1 - 1;
    for (; n - 2 >= n0; n -= 3) {
        const T y0a = o[0], y0b = o[plane];
        const T y1a = o[-NL64], y1b = o[plane - NL64];
        const T y2a = o[-2 * NL64], y2b = o[plane - 2 * NL64];
        double va, vb;
        corr2(y0a, y0b, g, va, vb);
        rec_into(a2, va, a0, a1, c);
        rec_into(b2, vb, b0, b1, c);
        o[0] = (T)a2;
        o[plane] = (T)b2;
        corr2(y1a, y1b, g - 3, va, vb);
        rec_into(a1, va, a2, a0, c);
        rec_into(b1, vb, b2, b0, c);
        o[-NL64] = (T)a1;
        o[plane - NL64] = (T)b1;
        corr2(y2a, y2b, g - 6, va, vb);
        rec_into(a0, va, a1, a2, c);
        rec_into(b0, vb, b1, b2, c);
        o[-2 * NL64] = (T)a0;
        o[plane - 2 * NL64] = (T)b0;
        o -= 3 * NL64;
        g -= 9;
    }
    ua[0] = a0; ua[1] = a1; ua[2] = a2;
    ub[0] = b0; ub[1] = b1; ub[2] = b2;
    for (; n >= n0; --n) {  // 0-2 remaining samples
        double va, vb;
        corr2(o[0], o[plane], g, va, vb);
        o[0] = (T)rec_step(ua, va, c);
        o[plane] = (T)rec_step(ub, vb, c);
        o -= NL64;
        g -= 3;
    }
    // local start state (u[start], u[start+1], u[start+2]) -> the backward half of the state buffer
    double* st = a.state + ((int64_t)a.njobs * a.batch * a.nseg * 6) * NL +
                 (((int64_t)blockIdx.z * a.nseg + seg) * 6) * NL + x;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        st[(int64_t)k * NL] = ua[k];
        st[(int64_t)(3 + k) * NL] = ub[k];
    }
}

// ---- pass 3 for the horizontal stage: staged, row-contiguous output ----
template <typename T>
__device__ __forceinline__ void iir_out_rows(const IirArgs<T>& a, const IirJob<T>& job, int x, int seg, int b, int n0,
                                             int n1) {
    using C = cx_t<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tile = reinterpret_cast<C*>(smem_raw);
    const int len = a.len, P = a.P, L = len + 2 * P, NL = a.lines;
    const int sw = kIirSY * a.seglen, swp = sw | 1;
    const int nb0 = blockIdx.y * kIirSY * a.seglen;
    const bool live = x < NL && seg < a.nseg && n1 > P && n0 < P + len;
    if (live) {
        const int64_t plane = (int64_t)L * NL;
        const T* sc = a.scratch + (int64_t)blockIdx.z * 2 * plane + x;
        const double* sj = a.state + ((int64_t)a.njobs * a.batch * a.nseg * 6) * NL +
                           (((int64_t)blockIdx.z * a.nseg + seg) * 6) * NL + x;
        double ta[3], tb[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            ta[k] = sj[(int64_t)k * NL];
            tb[k] = sj[(int64_t)(3 + k) * NL];
        }
        const bool last = seg == a.nseg - 1;
        const double osg = (job.sdft ? -1.0 : 1.0) * (job.conj[0] ? -1.0 : 1.0);
        const double2* tabr = a.tab_base + job.tabr_off;
        const int lo = max(n0, P), hi = min(n1, P + len);
        C* trow = tile + threadIdx.x * swp - nb0;
        for (int nb = lo; nb < hi; nb += kIirUB) {
            T ua[kIirUB], ub[kIirUB];
#pragma unroll
            for (int k = 0; k < kIirUB; ++k) {
                const T* o = sc + (int64_t)(nb + k) * NL;
                if (nb + k < hi) { ua[k] = o[0]; ub[k] = o[plane]; }
            }
#pragma unroll
            for (int k = 0; k < kIirUB; ++k) {
                const int n = nb + k;
                if (n >= hi) break;
                double va = ua[k], vb = ub[k];
                if (!last) {
                    const double* g = a.g + 3 * (n1 - 1 - n);
                    const double g0 = g[0], g1 = g[1], g2 = g[2];
                    va += g0 * ta[0] + g1 * ta[1] + g2 * ta[2];
                    vb += g0 * tb[0] + g1 * tb[1] + g2 * tb[2];
                }
                const double2 cs = tabr[n - P];
                trow[n] = mk<T>((T)fma(cs.x, va, cs.y * vb), (T)(osg * fma(cs.y, va, -cs.x * vb)));
            }
        }
    }
    __syncthreads();
    // row-contiguous write-out of the CTA's 32 rows x sw samples (crop window only)
    C* dst = a.dst_base + job.dst_off[0] + (int64_t)b * a.dst_bstride;
    const int tid = threadIdx.y * kIirTX + threadIdx.x;
    (void)tid;
    for (int r = threadIdx.y; r < kIirTX; r += kIirSY) {
        const int line = blockIdx.x * kIirTX + r;
        if (line >= NL) continue;
        C* row = dst + (int64_t)line * a.dst_ls - P;
        const int c0 = max(0, P - nb0), c1 = min(sw, min(P + len, L) - nb0);
        for (int cc = c0 + threadIdx.x; cc < c1; cc += kIirTX) row[nb0 + cc] = tile[r * swp + cc];
    }
}

// ---- pass 3: backward carry + correction, recombination, outputs ----
// STAGE (horizontal stage, one output per job): results go to a shared tile
// and leave row-contiguously instead of one strided element per thread.
template <typename T, bool STAGE>
__global__ void __launch_bounds__(128, kIirMinBlocks) iir_out(const IirArgs<T> a) {
    const int x = blockIdx.x * kIirTX + threadIdx.x;
    const int seg = blockIdx.y * kIirSY + threadIdx.y;
    const int jb = blockIdx.z % a.njobs;
    const int b = blockIdx.z / a.njobs;
    const IirJob<T>& job = a.jobs[jb];
    const int len = a.len, P = a.P, L = len + 2 * P, NL = a.lines;
    const int n0 = seg * a.seglen, n1 = min(L, n0 + a.seglen);
    if constexpr (STAGE) {
        iir_out_rows<T>(a, job, x, seg, b, n0, n1);
        return;
    }
    if (x >= a.lines || seg >= a.nseg) return;
    if (n1 <= P || n0 >= P + len) return;  // nothing of this segment survives the crop
    const int64_t plane = (int64_t)L * NL;
    const T* sc = a.scratch + (int64_t)blockIdx.z * 2 * plane + x;
    const double* st_all = a.state + ((int64_t)a.njobs * a.batch * a.nseg * 6) * NL +
                           ((int64_t)blockIdx.z * a.nseg * 6) * NL + x;
    // true state entering this segment from above (iir_scan_seq<1> turned the local start states into carry-ins)
    double ta[3], tb[3];
    {
        const double* sj = st_all + (int64_t)seg * 6 * NL;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            ta[k] = sj[(int64_t)k * NL];
            tb[k] = sj[(int64_t)(3 + k) * NL];
        }
    }
    const bool last = seg == a.nseg - 1;
    // outputs (all of this job's pair): pointers + conjugation flags in registers
    const int nout = job.nout;
    const double isg = job.sdft ? -1.0 : 1.0;  // Gabor im = s Sa - c Sb; SDFT im = c Sb - s Sa
    cx_t<T>* dptr[4];
    double osg[4];
    const int64_t dss = a.dst_ss;
#pragma unroll
    for (int o = 0; o < 4; ++o) {
        dptr[o] = a.dst_base + (o < nout ? job.dst_off[o] : 0) + (int64_t)b * a.dst_bstride + (int64_t)x * a.dst_ls;
        osg[o] = (o < nout && job.conj[o]) ? -isg : isg;
    }
    const double2* tabr = a.tab_base + job.tabr_off;
    const int lo = max(n0, P), hi = min(n1, P + len);
    const double* gt = a.g;
    for (int nb = lo; nb < hi; nb += kIirUB) {
        T ua[kIirUB], ub[kIirUB];
#pragma unroll
        for (int k = 0; k < kIirUB; ++k) {
            const T* o = sc + (int64_t)(nb + k) * NL;
            if (nb + k < hi) { ua[k] = o[0]; ub[k] = o[plane]; }
        }
#pragma unroll
        for (int k = 0; k < kIirUB; ++k) {
            const int n = nb + k;
            if (n >= hi) break;
            const int yo = n - P;
            const double2 cs = tabr[yo];
            double va = ua[k], vb = ub[k];
            if (!last) {
                const double* g = gt + 3 * (n1 - 1 - n);
                const double g0 = g[0], g1 = g[1], g2 = g[2];
                va += g0 * ta[0] + g1 * ta[1] + g2 * ta[2];
                vb += g0 * tb[0] + g1 * tb[1] + g2 * tb[2];
            }
            const T re = (T)fma(cs.x, va, cs.y * vb);
            const double im = fma(cs.y, va, -cs.x * vb);
            const int64_t dof = (int64_t)yo * dss;
            dptr[0][dof] = mk<T>(re, (T)(osg[0] * im));
            if (nout > 1) {  // SDFT jobs: the conjugate-symmetric fills
#pragma unroll
                for (int o = 1; o < 4; ++o)
                    if (o < nout) dptr[o][dof] = mk<T>(re, (T)(osg[o] * im));
            }
        }
    }
}

// ---- carry scans: local segment states -> true incoming states, in place ----
// DIR 0 (after iir_fwd): s_in[0] = 0, s_in[j+1] = Aseg s_in[j] + end_loc[j]
// DIR 1 (after iir_bwd): t_in[n-1] = 0, t_in[j-1] = A_j t_in[j] + start_loc[j]
//                        (A_j = Alast for the shorter last segment)
// One thread per (line, plane) walks its segments in scan order, loading
// kSeqB segments' states per round trip (the loads do not depend on the
// running state; the writes go to slots already read).
constexpr int kSeqB = 16;
template <int DIR>
__global__ void __launch_bounds__(128) iir_scan_seq(double* state, int64_t sec_off, int lines, int nseg,
                                                   const __grid_constant__ IirScanMats m) {
    const int x = blockIdx.x * 64 + (threadIdx.x & 63);
    const int q = threadIdx.x >> 6;  // plane
    if (x >= lines) return;
    const int NL = lines, ns = nseg;
    double* st = state + sec_off + ((int64_t)blockIdx.z * ns * 6) * NL + (int64_t)(q * 3) * NL + x;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int r0 = 0; r0 < ns; r0 += kSeqB) {
        double l[kSeqB][3];
#pragma unroll
        for (int i = 0; i < kSeqB; ++i) {
            const int r = r0 + i;
            if (r < ns) {
                const double* p = st + (int64_t)(DIR == 0 ? r : ns - 1 - r) * 6 * NL;
                l[i][0] = p[0];
                l[i][1] = p[NL];
                l[i][2] = p[2 * (int64_t)NL];
            }
        }
#pragma unroll
        for (int i = 0; i < kSeqB; ++i) {
            const int r = r0 + i;
            if (r >= ns) break;
            const int j = DIR == 0 ? r : ns - 1 - r;
            double* p = st + (int64_t)j * 6 * NL;
            p[0] = s0;
            p[NL] = s1;
            p[2 * (int64_t)NL] = s2;
            const double* A = (DIR == 1 && j == ns - 1) ? m.Alast : m.Aseg;
            const double n0 = A[0] * s0 + A[1] * s1 + A[2] * s2 + l[i][0];
            const double n1 = A[3] * s0 + A[4] * s1 + A[5] * s2 + l[i][1];
            const double n2 = A[6] * s0 + A[7] * s1 + A[8] * s2 + l[i][2];
            s0 = n0;
            s1 = n1;
            s2 = n2;
        }
    }
}

}  // namespace

template <typename T> size_t iir_scratch_elems(int len, int lines, int P, int njobs, int batch) {
    if (sizeof(T) == 4 && iir32_enabled()) return 0;  // iir32.cu keeps no sequences
    return (size_t)njobs * batch * 2 * (size_t)(len + 2 * P) * lines;
}

// (iir32.cu keeps [z][nseg + ceil(nseg / 4)][12][lines] floats plus one arrival counter per 32-line block and z
// in the same region: the extra z * lines doubles cover the counters when nseg is tiny)
size_t iir_state_doubles(int lines, int nseg, int njobs, int batch) {
    return 2 * (size_t)njobs * batch * nseg * 6 * lines + (size_t)njobs * batch * lines;
}

template <typename T> cudaError_t launch_iir(const IirArgs<T>& a, cudaStream_t s) {
    dim3 block(kIirTX, kIirSY);
    dim3 grid((a.lines + kIirTX - 1) / kIirTX, (a.nseg + kIirSY - 1) / kIirSY, a.njobs * a.batch);
    IirScanMats m;
    std::memcpy(m.Aseg, a.Aseg, sizeof(m.Aseg));
    std::memcpy(m.Alast, a.Alast, sizeof(m.Alast));
    const int64_t bwd_sec = (int64_t)a.njobs * a.batch * a.nseg * 6 * a.lines;
    // horizontal stage (real rows in, one output per job): stage through shared memory
    const size_t sw = (size_t)(kIirSY * a.seglen) | 1;
    const size_t in_smem = kIirTX * sw * sizeof(T), out_smem = kIirTX * sw * sizeof(cx_t<T>);
    const bool stage = a.real_in && a.src_ss == 1 && a.dst_ss == 1 && a.one_out && out_smem <= 48 * 1024;
    if (stage) iir_fwd<T, true, true><<<grid, block, in_smem, s>>>(a);
    else if (a.real_in) iir_fwd<T, true, false><<<grid, block, 0, s>>>(a);
    else iir_fwd<T, false, false><<<grid, block, 0, s>>>(a);
    const dim3 qgrid((a.lines + 63) / 64, 1, a.njobs * a.batch);
    iir_scan_seq<0><<<qgrid, 128, 0, s>>>(a.state, 0, a.lines, a.nseg, m);
    iir_bwd<T><<<grid, block, 0, s>>>(a);
    iir_scan_seq<1><<<qgrid, 128, 0, s>>>(a.state, bwd_sec, a.lines, a.nseg, m);
    if (stage) iir_out<T, true><<<grid, block, out_smem, s>>>(a);
    else iir_out<T, false><<<grid, block, 0, s>>>(a);
    return cudaGetLastError();
}

template size_t iir_scratch_elems<float>(int, int, int, int, int);
template size_t iir_scratch_elems<double>(int, int, int, int, int);
template cudaError_t launch_iir<float>(const IirArgs<float>&, cudaStream_t);
template cudaError_t launch_iir<double>(const IirArgs<double>&, cudaStream_t);

}  // namespace fgb
