// K4 (fp32 build): RecursiveIIR stage in PARALLEL FORM, segment-parallel,
// two passes over the input and no scratch planes.
//
// The reference filter (gaussian.py:215-228; restated in iir.cu) is the
// direct-form 3rd-order recursion y[n] = B z[n] - a1 y[n-1] - a2 y[n-2] -
// a3 y[n-3], forward then backward, with steady-state inits.  Its transfer
// function B / (1 + a1 z^-1 + a2 z^-2 + a3 z^-3) has one real pole q_r and a
// complex pair q_c, conj(q_c), so it is exactly the sum of first-order
// sections
//     s_r[n] = q_r s_r[n-1] + c_r z[n],   s_c[n] = q_c s_c[n-1] + c_c z[n],
//     y[n]   = s_r[n] + 2 Re s_c[n]
// with residues c_k = B / prod_{j != k} (1 - q_j / q_k), and the reference's
// steady-state init (y[-1..-3] = z[0]) is the sections' steady state
// s_k = c_k z[0] / (1 - q_k).  The direct form needs fp64 state to meet
// 1e-5 (its coefficients are ill-conditioned near the unit circle: SURVEY
// Appendix B); the parallel form does not -- each pole is stored as
// 1 - d (d exact to fp32 relative precision) and s - d s is one FMA -- so
// the recursion runs in fp32 FFMA2 (planes a and b of a modulation pair
// packed), with no fp32 <-> fp64 conversions (each costs ~4 DFMA issue
// slots on B200: tools/probes/f64_probe.cu).  Measured emulation error vs
// the fp64 reference: <= 2e-6 (sigma = 32), see DESIGN.md §4.
//
// Segment parallelism is exact.  A line is cut into segments of kM samples.
//   pass 1 (iir32_sum): per segment, modulate and run the forward sections
//     from a zero state (segment 0: the true init); keep the end state e and
//     the backward-start sums b = sum_i c q^i y_loc[n0 + i] (the start state
//     the backward sections would reach over this segment's local output).
//   carry (iir32_carry): per line, forward s_in[j+1] = q^m s_in[j] + e[j];
//     the backward init from the true y[L-1]; then backward
//     t_in[j-1] = q^m t_in[j] + b[j] + Mb s_in[j]   (Mb: the backward-start
//     response to a forward carry-in, host-computed).
//   pass 2 (iir32_fin): per segment, forward sections from the true s_in
//     (exact y, kept in registers), backward sections from the true t_in,
//     recombination, outputs.
// Lines are adjacent threads; the horizontal stage (lines = image rows)
// stages its rows through shared memory both ways.
#include <complex>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace fgb {

namespace {

constexpr int kM = kIir32M;  // samples per segment (register window of pass 2)
constexpr int kTX = 32;      // lines per CTA
constexpr int kSY = 4;       // segments per CTA

struct Iir32Par {
    float ndr, cr;           // real section:    s = s + ndr s + cr z     (ndr = -(1 - q_r))
    float ndc, nqi, qi;      // complex section: pole (1 + ndc) + i qi, nqi = -qi
    float ccr, cci;          // complex residue
    float gr, gcr, gci;      // steady state per unit constant input: c / (1 - q)
    float wr[kM], wcr[kM], wci[kM];  // backward-start weights c q^i
    float Q[2][3];           // q^kM, q^mlast: (real, complex re, complex im)
    float Mb[2][9];          // b contribution of a forward carry-in (s_r, s_cr, s_ci) -> (b_r, b_cr, b_ci)
};

__device__ __forceinline__ float2 dup(float v) { return make_float2(v, v); }

struct Sec {
    float2 r, cr, ci;  // (plane a, plane b)
};

// one sample of the three sections on both planes; returns y = s_r + 2 Re s_c
__device__ __forceinline__ float2 sec_step(Sec& s, float2 z, const Iir32Par& q) {
    s.r = __ffma2_rn(dup(q.ndr), s.r, s.r);
    s.r = __ffma2_rn(dup(q.cr), z, s.r);
    float2 tr = __ffma2_rn(dup(q.ndc), s.cr, s.cr);
    tr = __ffma2_rn(dup(q.nqi), s.ci, tr);
    tr = __ffma2_rn(dup(q.ccr), z, tr);
    float2 ti = __ffma2_rn(dup(q.ndc), s.ci, s.ci);
    ti = __ffma2_rn(dup(q.qi), s.cr, ti);
    ti = __ffma2_rn(dup(q.cci), z, ti);
    s.cr = tr;
    s.ci = ti;
    return __ffma2_rn(dup(2.f), s.cr, s.r);
}

__device__ __forceinline__ void sec_steady(Sec& s, float2 z0, const Iir32Par& q) {
    s.r = make_float2(q.gr * z0.x, q.gr * z0.y);
    s.cr = make_float2(q.gcr * z0.x, q.gcr * z0.y);
    s.ci = make_float2(q.gci * z0.x, q.gci * z0.y);
}

// modulation pair (see kernels.h): pair 0: (jr c + ji s, jr s - ji c); pair 1: (jr c - ji s, jr s + ji c)
__device__ __forceinline__ float2 modz(float sgn, float jr, float ji, float2 cs) {
    const float sj = sgn * ji;
    return make_float2(fmaf(jr, cs.x, sj * cs.y), fmaf(jr, cs.y, -sj * cs.x));
}

// Source access of one line.  STAGE: the CTA's rows sit in shared memory
// (samples nb0 .. nb0 + kSY kM - 1 of each row, already clamped).
template <bool REAL, bool STAGE> struct Src {
    const void* p;
    int64_t ss;
    int P, len, nb0;
    const float2* tab;
    float sgn;
    __device__ __forceinline__ float2 z(int n) const {
        const float2 cs = tab[n];
        if constexpr (STAGE) {
            const float f = reinterpret_cast<const float*>(p)[n - nb0];
            return make_float2(f * cs.x, f * cs.y);
        } else if constexpr (REAL) {
            const float f = reinterpret_cast<const float*>(p)[(int64_t)clampi(n - P, 0, len - 1) * ss];
            return make_float2(f * cs.x, f * cs.y);
        } else {
            const float2 v = reinterpret_cast<const float2*>(p)[(int64_t)clampi(n - P, 0, len - 1) * ss];
            return modz(sgn, v.x, v.y, cs);
        }
    }
};

// Row staging of the horizontal stage: the CTA's 32 rows x (kSY kM) samples,
// row-contiguous loads, odd pitch for conflict-free per-thread reads.
__device__ __forceinline__ void stage_rows(float* tile, const IirArgs<float>& a, const IirJob<float>& job, int b) {
    constexpr int sw = kSY * kM, swp = sw | 1;
    const int len = a.len, P = a.P, L = len + 2 * P;
    const int nb0 = blockIdx.y * sw;
    const float* base = reinterpret_cast<const float*>(a.src_base) + job.src_off + (int64_t)b * a.src_bstride;
    for (int r = threadIdx.y; r < kTX; r += kSY) {
        const int line = blockIdx.x * kTX + r;
        if (line >= a.lines) continue;
        const float* row = base + (int64_t)line * a.src_ls;
        for (int cc = threadIdx.x; cc < sw; cc += kTX) {
            const int n = nb0 + cc;
            if (n < L) tile[r * swp + cc] = row[clampi(n - P, 0, len - 1)];
        }
    }
}

template <bool REAL, bool STAGE>
__device__ __forceinline__ Src<REAL, STAGE> make_src(const IirArgs<float>& a, const IirJob<float>& job, int x, int b,
                                                     const float* tile) {
    Src<REAL, STAGE> s;
    s.P = a.P;
    s.len = a.len;
    s.nb0 = blockIdx.y * kSY * kM;
    s.tab = a.tab32 + job.tabm_off;
    s.sgn = (job.need >> 1) ? -1.f : 1.f;
    if constexpr (STAGE) {
        s.p = tile + threadIdx.x * ((kSY * kM) | 1);
        s.ss = 1;
    } else if constexpr (REAL) {
        s.p = reinterpret_cast<const float*>(a.src_base) + job.src_off + (int64_t)b * a.src_bstride + (int64_t)x * a.src_ls;
        s.ss = a.src_ss;
    } else {
        s.p = reinterpret_cast<const float2*>(a.src_base) + job.src_off + (int64_t)b * a.src_bstride + (int64_t)x * a.src_ls;
        s.ss = a.src_ss;
    }
    return s;
}

// ---- pass 1: local forward sections -> end state e, backward-start sums b ----
template <bool REAL, bool STAGE, bool FULL>
__device__ __forceinline__ void sum_body(const Src<REAL, STAGE>& src, int n0, int m, Sec& s, float2& br, float2& bcr,
                                         float2& bci, const Iir32Par& q) {
#pragma unroll
    for (int i = 0; i < kM; ++i) {
        if (FULL || i < m) {
            const float2 y = sec_step(s, src.z(n0 + i), q);
            br = __ffma2_rn(dup(q.wr[i]), y, br);
            bcr = __ffma2_rn(dup(q.wcr[i]), y, bcr);
            bci = __ffma2_rn(dup(q.wci[i]), y, bci);
        }
    }
}

template <bool REAL, bool STAGE>
__global__ void __launch_bounds__(128) iir32_sum(const IirArgs<float> a, const __grid_constant__ Iir32Par q) {
    const int x = blockIdx.x * kTX + threadIdx.x;
    const int seg = blockIdx.y * kSY + threadIdx.y;
    const int jb = blockIdx.z % a.njobs, b = blockIdx.z / a.njobs;
    const IirJob<float>& job = a.jobs[jb];
    const int L = a.len + 2 * a.P, NL = a.lines;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* tile = reinterpret_cast<float*>(smem_raw);
    if constexpr (STAGE) {
        stage_rows(tile, a, job, b);
        __syncthreads();
    }
    const int n0 = seg * kM;
    if (x >= NL || n0 >= L) return;
    const int m = min(kM, L - n0);
    const Src<REAL, STAGE> src = make_src<REAL, STAGE>(a, job, x, b, tile);
    Sec s;
    if (seg == 0) sec_steady(s, src.z(0), q);
    else s.r = s.cr = s.ci = dup(0.f);
    float2 br = dup(0.f), bcr = dup(0.f), bci = dup(0.f);
    if (m == kM) sum_body<REAL, STAGE, true>(src, n0, m, s, br, bcr, bci, q);
    else sum_body<REAL, STAGE, false>(src, n0, m, s, br, bcr, bci, q);
    float* st = a.state32 + ((int64_t)blockIdx.z * a.nseg + seg) * 12 * NL + x;
    const float v[12] = {s.r.x, s.cr.x, s.ci.x, s.r.y, s.cr.y, s.ci.y, br.x, bcr.x, bci.x, br.y, bcr.y, bci.y};
#pragma unroll
    for (int k = 0; k < 12; ++k) st[(int64_t)k * NL] = v[k];
}

// ---- carries: one thread per (line, plane), segments in order, loads batched ----
constexpr int kCB = 8;
__global__ void __launch_bounds__(128) iir32_carry(float* state, int lines, int nseg, const __grid_constant__ Iir32Par q) {
    const int x = blockIdx.x * 64 + (threadIdx.x & 63);
    const int pl = threadIdx.x >> 6;
    if (x >= lines) return;
    const int64_t NL = lines, SS = 12 * NL;  // slot / segment strides
    float* base = state + (int64_t)blockIdx.z * nseg * SS + x;
    float* e0 = base + 3 * pl * NL;        // e (then s_in) of this plane
    float* b0 = base + (6 + 3 * pl) * NL;  // b (then t_in) of this plane
    float sr = 0.f, scr = 0.f, sci = 0.f;
    for (int j0 = 0; j0 < nseg; j0 += kCB) {
        float e[kCB][3];
#pragma unroll
        for (int i = 0; i < kCB; ++i)
            if (j0 + i < nseg) {
                const float* p = e0 + (j0 + i) * SS;
                e[i][0] = p[0];
                e[i][1] = p[NL];
                e[i][2] = p[2 * NL];
            }
#pragma unroll
        for (int i = 0; i < kCB; ++i) {
            const int j = j0 + i;
            if (j >= nseg) break;
            float* p = e0 + j * SS;
            p[0] = sr;
            p[NL] = scr;
            p[2 * NL] = sci;
            const float* Q = q.Q[j == nseg - 1];
            const float nr = fmaf(Q[0], sr, e[i][0]);
            const float ncr = fmaf(Q[1], scr, fmaf(-Q[2], sci, e[i][1]));
            const float nci = fmaf(Q[1], sci, fmaf(Q[2], scr, e[i][2]));
            sr = nr;
            scr = ncr;
            sci = nci;
        }
    }
    // true y[L-1] -> the backward sections' steady-state init
    const float yL = fmaf(2.f, scr, sr);
    float tr = q.gr * yL, tcr = q.gcr * yL, tci = q.gci * yL;
    for (int j0 = nseg - 1; j0 >= 0; j0 -= kCB) {
        float bb[kCB][3], si[kCB][3];
#pragma unroll
        for (int i = 0; i < kCB; ++i)
            if (j0 - i >= 0) {
                const float* p = b0 + (j0 - i) * SS;
                const float* r = e0 + (j0 - i) * SS;
                bb[i][0] = p[0];
                bb[i][1] = p[NL];
                bb[i][2] = p[2 * NL];
                si[i][0] = r[0];
                si[i][1] = r[NL];
                si[i][2] = r[2 * NL];
            }
#pragma unroll
        for (int i = 0; i < kCB; ++i) {
            const int j = j0 - i;
            if (j < 0) break;
            float* p = b0 + j * SS;
            p[0] = tr;
            p[NL] = tcr;
            p[2 * NL] = tci;
            const int lt = j == nseg - 1;
            const float* Q = q.Q[lt];
            const float* M = q.Mb[lt];
            const float c0 = fmaf(M[0], si[i][0], fmaf(M[1], si[i][1], fmaf(M[2], si[i][2], bb[i][0])));
            const float c1 = fmaf(M[3], si[i][0], fmaf(M[4], si[i][1], fmaf(M[5], si[i][2], bb[i][1])));
            const float c2 = fmaf(M[6], si[i][0], fmaf(M[7], si[i][1], fmaf(M[8], si[i][2], bb[i][2])));
            const float nr = fmaf(Q[0], tr, c0);
            const float ncr = fmaf(Q[1], tcr, fmaf(-Q[2], tci, c1));
            const float nci = fmaf(Q[1], tci, fmaf(Q[2], tcr, c2));
            tr = nr;
            tcr = ncr;
            tci = nci;
        }
    }
}

// ---- pass 2: exact forward (registers), exact backward, recombination ----
template <bool REAL, bool STAGE, bool FULL>
__device__ __forceinline__ void fin_fwd(const Src<REAL, STAGE>& src, int n0, int m, Sec& s, float2 (&y)[kM],
                                        const Iir32Par& q) {
#pragma unroll
    for (int i = 0; i < kM; ++i)
        if (FULL || i < m) y[i] = sec_step(s, src.z(n0 + i), q);
}

template <bool FULL, typename EMIT>
__device__ __forceinline__ void fin_bwd(int m, Sec& t, const float2 (&y)[kM], const Iir32Par& q, EMIT emit) {
#pragma unroll
    for (int i = kM - 1; i >= 0; --i)
        if (FULL || i < m) emit(i, sec_step(t, y[i], q));
}

template <bool REAL, bool STAGE>
__global__ void __launch_bounds__(128) iir32_fin(const IirArgs<float> a, const __grid_constant__ Iir32Par q) {
    const int x = blockIdx.x * kTX + threadIdx.x;
    const int seg = blockIdx.y * kSY + threadIdx.y;
    const int jb = blockIdx.z % a.njobs, b = blockIdx.z / a.njobs;
    const IirJob<float>& job = a.jobs[jb];
    const int len = a.len, P = a.P, L = len + 2 * P, NL = a.lines;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* tile = reinterpret_cast<float*>(smem_raw);
    if constexpr (STAGE) {
        stage_rows(tile, a, job, b);
        __syncthreads();
    }
    const int n0 = seg * kM;
    const int m = min(kM, L - n0);
    // segments that leave nothing inside the crop [P, P + len) only fed the carries
    const bool live = x < NL && n0 < L && n0 + m > P && n0 < P + len;
    const float* st = a.state32 + ((int64_t)blockIdx.z * a.nseg + seg) * 12 * NL + x;
    float2 y[kM];
    if (live) {
        const Src<REAL, STAGE> src = make_src<REAL, STAGE>(a, job, x, b, tile);
        Sec s;
        if (seg == 0) {
            sec_steady(s, src.z(0), q);
        } else {
            s.r = make_float2(st[0], st[3 * (int64_t)NL]);
            s.cr = make_float2(st[(int64_t)NL], st[4 * (int64_t)NL]);
            s.ci = make_float2(st[2 * (int64_t)NL], st[5 * (int64_t)NL]);
        }
        if (m == kM) fin_fwd<REAL, STAGE, true>(src, n0, m, s, y, q);
        else fin_fwd<REAL, STAGE, false>(src, n0, m, s, y, q);
    }
    const float2* tabr = a.tab32 + job.tabr_off;
    const float isg = job.sdft ? -1.f : 1.f;  // Gabor im = s Sa - c Sb; SDFT im = c Sb - s Sa
    if constexpr (STAGE) {
        __syncthreads();  // every input sample consumed: the tile becomes the output tile
        float2* otile = reinterpret_cast<float2*>(smem_raw);
        constexpr int sw = kSY * kM, swp = sw | 1;
        const int nb0 = blockIdx.y * sw;
        if (live) {
            Sec t;
            t.r = make_float2(st[6 * (int64_t)NL], st[9 * (int64_t)NL]);
            t.cr = make_float2(st[7 * (int64_t)NL], st[10 * (int64_t)NL]);
            t.ci = make_float2(st[8 * (int64_t)NL], st[11 * (int64_t)NL]);
            const float osg = isg * (job.conj[0] ? -1.f : 1.f);
            float2* trow = otile + threadIdx.x * swp - nb0;
            auto emit = [&](int i, float2 u) {
                const int n = n0 + i;
                if (n >= P && n < P + len) {
                    const float2 cs = tabr[n - P];
                    trow[n] = make_float2(fmaf(cs.x, u.x, cs.y * u.y), osg * fmaf(cs.y, u.x, -cs.x * u.y));
                }
            };
            if (m == kM) fin_bwd<true>(m, t, y, q, emit);
            else fin_bwd<false>(m, t, y, q, emit);
        }
        __syncthreads();
        float2* dst = a.dst_base + job.dst_off[0] + (int64_t)b * a.dst_bstride;
        for (int r = threadIdx.y; r < kTX; r += kSY) {
            const int line = blockIdx.x * kTX + r;
            if (line >= NL) continue;
            float2* row = dst + (int64_t)line * a.dst_ls - P;
            const int c0 = max(0, P - nb0), c1 = min(sw, min(P + len, L) - nb0);
            for (int cc = c0 + threadIdx.x; cc < c1; cc += kTX) row[nb0 + cc] = otile[r * swp + cc];
        }
        return;
    } else {
        if (!live) return;
        Sec t;
        t.r = make_float2(st[6 * (int64_t)NL], st[9 * (int64_t)NL]);
        t.cr = make_float2(st[7 * (int64_t)NL], st[10 * (int64_t)NL]);
        t.ci = make_float2(st[8 * (int64_t)NL], st[11 * (int64_t)NL]);
        const int nout = job.nout;
        float2* dptr[4];
        float osg[4];
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            dptr[o] = a.dst_base + (o < nout ? job.dst_off[o] : 0) + (int64_t)b * a.dst_bstride + (int64_t)x * a.dst_ls;
            osg[o] = (o < nout && job.conj[o]) ? -isg : isg;
        }
        const int64_t dss = a.dst_ss;
        auto emit = [&](int i, float2 u) {
            const int n = n0 + i;
            if (n >= P && n < P + len) {
                const int yo = n - P;
                const float2 cs = tabr[yo];
                const float re = fmaf(cs.x, u.x, cs.y * u.y);
                const float im = fmaf(cs.y, u.x, -cs.x * u.y);
                const int64_t dof = (int64_t)yo * dss;
                __stcs(dptr[0] + dof, make_float2(re, osg[0] * im));
                if (nout > 1) {
#pragma unroll
                    for (int o = 1; o < 4; ++o)
                        if (o < nout) __stcs(dptr[o] + dof, make_float2(re, osg[o] * im));
                }
            }
        };
        if (m == kM) fin_bwd<true>(m, t, y, q, emit);
        else fin_bwd<false>(m, t, y, q, emit);
    }
}

// ---- host: parallel-form parameters from the direct-form coefficients ----
using cd = std::complex<double>;

void iir32_params(const IirCoef& c, int mlast, Iir32Par* out) {
    // roots of z^3 + a1 z^2 + a2 z + a3 (Durand-Kerner, then Newton polish)
    auto poly = [&](cd z) { return ((z + c.a1) * z + c.a2) * z + c.a3; };
    cd r[3] = {cd(0.4, 0.9), cd(0.4, 0.9) * cd(0.4, 0.9), cd(0.4, 0.9) * cd(0.4, 0.9) * cd(0.4, 0.9)};
    for (int it = 0; it < 500; ++it)
        for (int k = 0; k < 3; ++k) {
            cd d(1.0, 0.0);
            for (int j = 0; j < 3; ++j)
                if (j != k) d *= r[k] - r[j];
            r[k] -= poly(r[k]) / d;
        }
    for (int k = 0; k < 3; ++k)
        for (int it = 0; it < 3; ++it) {
            const cd dp = (3.0 * r[k] + 2.0 * c.a1) * r[k] + c.a2;
            if (std::abs(dp) > 0) r[k] -= poly(r[k]) / dp;
        }
    int ir = 0;
    for (int k = 1; k < 3; ++k)
        if (std::abs(r[k].imag()) < std::abs(r[ir].imag())) ir = k;
    int ic = -1;
    for (int k = 0; k < 3; ++k)
        if (k != ir && (ic < 0 || r[k].imag() > r[ic].imag())) ic = k;
    const cd qr(r[ir].real(), 0.0), qc = r[ic];
    const cd qs[3] = {qr, qc, std::conj(qc)};
    auto resid = [&](int k) {
        cd d(1.0, 0.0);
        for (int j = 0; j < 3; ++j)
            if (j != k) d *= 1.0 - qs[j] / qs[k];
        return c.B / d;
    };
    const cd cr = resid(0), cc = resid(1);
    Iir32Par& p = *out;
    std::memset(&p, 0, sizeof(p));
    p.ndr = (float)-(1.0 - qr.real());
    p.cr = (float)cr.real();
    p.ndc = (float)-(1.0 - qc.real());
    p.qi = (float)qc.imag();
    p.nqi = -p.qi;
    p.ccr = (float)cc.real();
    p.cci = (float)cc.imag();
    const cd gr = cr / (1.0 - qr), gc = cc / (1.0 - qc);
    p.gr = (float)gr.real();
    p.gcr = (float)gc.real();
    p.gci = (float)gc.imag();
    for (int i = 0; i < kM; ++i) {
        const cd wr = cr * std::pow(qr, i), wc = cc * std::pow(qc, i);
        p.wr[i] = (float)wr.real();
        p.wcr[i] = (float)wc.real();
        p.wci[i] = (float)wc.imag();
    }
    const int ms[2] = {kM, mlast};
    for (int t = 0; t < 2; ++t) {
        const int m = ms[t];
        const cd Qr = std::pow(qr, m), Qc = std::pow(qc, m);
        p.Q[t][0] = (float)Qr.real();
        p.Q[t][1] = (float)Qc.real();
        p.Q[t][2] = (float)Qc.imag();
        // corr_i(s) = s_r qr^(i+1) + 2 (s_cr Re qc^(i+1) - s_ci Im qc^(i+1))
        double Mr[3] = {0, 0, 0};
        cd Mc[3] = {0.0, 0.0, 0.0};
        for (int i = 0; i < m; ++i) {
            const cd qr1 = std::pow(qr, i + 1), qc1 = std::pow(qc, i + 1);
            const double basis[3] = {qr1.real(), 2.0 * qc1.real(), -2.0 * qc1.imag()};
            const cd wr = cr * std::pow(qr, i), wc = cc * std::pow(qc, i);
            for (int k = 0; k < 3; ++k) {
                Mr[k] += wr.real() * basis[k];
                Mc[k] += wc * basis[k];
            }
        }
        for (int k = 0; k < 3; ++k) {
            p.Mb[t][k] = (float)Mr[k];
            p.Mb[t][3 + k] = (float)Mc[k].real();
            p.Mb[t][6 + k] = (float)Mc[k].imag();
        }
    }
}

template <bool REAL, bool STAGE>
cudaError_t launch_passes(const IirArgs<float>& a, const Iir32Par& q, dim3 grid, dim3 block, size_t smem, cudaStream_t s) {
    if (smem > 48 * 1024) {
        cudaFuncSetAttribute(iir32_sum<REAL, STAGE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(iir32_fin<REAL, STAGE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    iir32_sum<REAL, STAGE><<<grid, block, STAGE ? smem / 2 : 0, s>>>(a, q);
    const dim3 cgrid((a.lines + 63) / 64, 1, a.njobs * a.batch);
    iir32_carry<<<cgrid, 128, 0, s>>>(a.state32, a.lines, a.nseg, q);
    iir32_fin<REAL, STAGE><<<grid, block, STAGE ? smem : 0, s>>>(a, q);
    return cudaGetLastError();
}

}  // namespace

bool iir32_enabled() {
    static const bool on = !std::getenv("FGB_IIR64");
    return on;
}

cudaError_t launch_iir32(const IirArgs<float>& a_in, cudaStream_t s) {
    IirArgs<float> a = a_in;
    const int L = a.len + 2 * a.P;
    if (a.seglen != kM || a.nseg != (L + kM - 1) / kM) return cudaErrorInvalidValue;
    a.state32 = reinterpret_cast<float*>(a.state);
    Iir32Par q;
    iir32_params(a.c, L - (a.nseg - 1) * kM, &q);
    const dim3 block(kTX, kSY);
    const dim3 grid((a.lines + kTX - 1) / kTX, (a.nseg + kSY - 1) / kSY, a.njobs * a.batch);
    const size_t out_smem = (size_t)kTX * ((kSY * kM) | 1) * sizeof(float2);
    const bool stage = a.real_in && a.src_ss == 1 && a.dst_ss == 1 && a.one_out;
    if (stage) return launch_passes<true, true>(a, q, grid, block, out_smem, s);
    if (a.real_in) return launch_passes<true, false>(a, q, grid, block, 0, s);
    return launch_passes<false, false>(a, q, grid, block, 0, s);
}

}  // namespace fgb
