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
// the fp64 reference: <= 2e-6 (sigma = 32, tests/test_iir_parallel_form.py).
//
// Segment parallelism is exact.  A line is cut into segments of kM = 32
// samples; a CTA owns 32 lines x kSY = 4 consecutive segments (a
// "super-segment") of one job, with the input tile and the trig tables
// staged in shared memory (column stages: one bulk async copy per 256-byte
// sample row, completing on an mbarrier; row stages: cp.async).
//   pass 1 (iir32_sum): per segment, modulate and run the forward sections
//     from a zero state (segment 0: the true init); the end state e and the
//     backward-start sums b = sum_i c q^i y_loc[n0 + i] (the start state the
//     backward sections would reach over this segment's local output).  The
//     CTA folds its 4 segments into super-segment summaries (e_S, b_S) and
//     keeps each segment's local chains (s_loc, T_loc).
//   carries: the last CTA of a 32-line block to finish (arrival counter)
//     scans the block's super-segments: s_in[j+1] = q^m s_in[j] + e[j]; the
//     backward init from the true y[L-1]; t_in[j-1] = q^m t_in[j] + b[j] +
//     Mb s_in[j]  (Mb: the backward-start response to a forward carry-in,
//     host-computed).  The scans overlap the rest of pass 1.
//   pass 2 (iir32_fin): per segment, its true carries from the super ones
//     (s_in = QF s_S + s_loc, t_in = QB t_S + T_loc + G s_S, host-computed
//     operators), forward sections from s_in (exact y, written over the
//     thread's own tile slots), backward sections from t_in, recombination,
//     outputs.
// Lines are adjacent threads; the horizontal stage (lines = image rows)
// stages its rows through shared memory both ways.
#include <algorithm>
#include <array>
#include <map>
#include <complex>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace fgb {

namespace {

constexpr int kM = kIir32M;  // samples per segment (the unrolled inner loops)
constexpr int kTX = 32;      // lines per CTA
constexpr int kSY = 4;       // segments per CTA

struct Iir32Par {
    float ndr, cr;           // real section:    s = s + ndr s + cr z     (ndr = -(1 - q_r))
    float ndc, nqi, qi;      // complex section: pole (1 + ndc) + i qi, nqi = -qi
    float ccr, cci;          // complex residue
    float gr, gcr, gci;      // steady state per unit constant input: c / (1 - q)
    float wr[kM], wcr[kM], wci[kM];  // backward-start weights c q^i
    // pass 1 of a full segment as dot products with the segment's modulated input (no recursion
    // chain): end states e = sum_k E[k] z_k, backward-start sums b = sum_k B[k] z_k
    float ER[kM], ECR[kM], ECI[kM], BR[kM], BCR[kM], BCI[kM];
    float Q[2][3];           // q^kM, q^mlast: (real, complex re, complex im)
    float Mb[2][9];          // b contribution of a forward carry-in (s_r, s_cr, s_ci) -> (b_r, b_cr, b_ci)
    float QS[2][3];          // the same for super-segments (the kSY segments of a CTA): q^(kSY kM), q^mlastS
    float MbS[2][9];
    // expansion of the super-segment carries (s_S, t_S) to sub-segment k of a
    // [regular, last] super-segment:  s_in_k = QF[k] s_S + s_loc_k,
    // t_in_k = QB[.][k] t_S + T_loc_k + G[.][k] s_S   (3-vectors (r, c re, c im))
    float QF[kSY][3];
    float QB[2][kSY][3];
    float G[2][kSY][9];
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

// CTA tile: 32 lines x kSY segments (kSW samples from nb0) of one job.
// Shared memory: the modulation table of the tile's samples, the
// recombination table, then the input tile of float2 slots:
//   ROWS (horizontal stage, real rows): [32 rows][kSW | 1] (odd pitch)
//   COLS (lines contiguous in memory):  [kSW samples][32 lines]
constexpr int kSW = kSY * kM;

// Grid: x = segment blocks (fastest, so the CTAs of one line block run
// back to back and its carry scan starts early), y = 32-line blocks, z = jobs.
__device__ __forceinline__ int sblk() { return blockIdx.x; }
__device__ __forceinline__ int lblk() { return blockIdx.y; }
// tables (float4 per sample, so modulation and recombination are one
// FMUL2 + one FFMA2 each):  tabm[i] = (c, s, sgn s, -sgn c) of sample nb0 + i,
// (za, zb) = jr (c, s) + ji (sgn s, -sgn c);  tabr[i] = (c, o s, s, -o c) of
// output sample nb0 + i - P, (re, im) = Sa (c, o s) + Sb (s, -o c), o = the
// sign of output 0's imaginary part.
constexpr int kTabBytes = 2 * kSW * (int)sizeof(float4);

// Every tile slot is a float2 (real inputs fill .x): pass 2 overwrites a
// thread's own slots in place with y, and (ROWS) with the outputs.
template <bool ROWS, bool CPLX> struct Tile {
    static constexpr size_t smem = kTabBytes + (ROWS ? (size_t)kTX * (kSW | 1) : (size_t)kSW * kTX) * sizeof(float2);
};
// slot of sample i (relative to the tile start) of this thread's line
template <bool ROWS> __device__ __forceinline__ int slot(int i) {
    return ROWS ? threadIdx.x * (kSW | 1) + i : i * kTX + threadIdx.x;
}

// cp.async the tile (clamped = replicate pad) and both tables; one wait.
template <bool ROWS, bool CPLX>
__device__ __forceinline__ void stage_tile(unsigned char* smem, const IirArgs<float>& a, const IirJob<float>& job, int b,
                                           bool want_tabr) {
    const int len = a.len, P = a.P, L = len + 2 * P;
    const int nb0 = sblk() * kSW;
    const int tid = threadIdx.y * kTX + threadIdx.x;
    // the tables are built AFTER the input copies are issued (their global loads then overlap
    // the tile's flight instead of delaying its issue)
    auto tables = [&]() {
        float4* tabm = reinterpret_cast<float4*>(smem);
        float4* tabr = tabm + kSW;
        const float sgn = (job.need >> 1) ? -1.f : 1.f;
        const float osg = (job.sdft ? -1.f : 1.f) * (job.conj[0] ? -1.f : 1.f);
        for (int i = tid; i < kSW; i += kTX * kSY) {
            const int n = nb0 + i;
            if (n < L) {
                const float2 cs = a.tab32[job.tabm_off + n];
                tabm[i] = make_float4(cs.x, cs.y, sgn * cs.y, -sgn * cs.x);
            }
            if (want_tabr && n >= P && n < P + len) {
                const float2 cs = a.tab32[job.tabr_off + (n - P)];
                tabr[i] = make_float4(cs.x, osg * cs.y, cs.y, -osg * cs.x);
            }
        }
    };
    unsigned char* tile = smem + kTabBytes;
    // tile samples [nb0, nb0 + kSW) need no clamping when they map into [0, len)
    const bool inner = nb0 >= P && nb0 + kSW <= P + len;
    if constexpr (ROWS) {
        constexpr int swp = kSW | 1;
        const float* base = reinterpret_cast<const float*>(a.src_base) + job.src_off + (int64_t)b * a.src_bstride;
        float2* t = reinterpret_cast<float2*>(tile);
        // lanes along the row (coalesced), warps over rows; pointers step by 4 rows
        const int line0 = lblk() * kTX + threadIdx.y;
        const float* row = base + (int64_t)line0 * a.src_ls;
        float2* d = t + threadIdx.y * swp + threadIdx.x;
        const int64_t rstep = (int64_t)kSY * a.src_ls;
        for (int r = threadIdx.y; r < kTX && lblk() * kTX + r < a.lines; r += kSY, row += rstep, d += kSY * swp) {
            if (inner) {
                const float* rp = row + (nb0 - P) + threadIdx.x;
#pragma unroll
                for (int k = 0; k < kSW / kTX; ++k) cp_async4(d + k * kTX, rp + k * kTX);
            } else {
#pragma unroll
                for (int k = 0; k < kSW / kTX; ++k) {
                    const int n = nb0 + threadIdx.x + k * kTX;
                    if (n < L) cp_async4(d + k * kTX, row + clampi(n - P, 0, len - 1));
                }
            }
        }
    } else {
        const int x = min(lblk() * kTX + threadIdx.x, a.lines - 1);
        if constexpr (CPLX) {
            const float2* blk = reinterpret_cast<const float2*>(a.src_base) + job.src_off + (int64_t)b * a.src_bstride +
                                lblk() * kTX;
            float2* t = reinterpret_cast<float2*>(tile);
            // a whole 32-line block: each sample row is one contiguous 256-byte run -> one bulk copy per row
            const bool bulk = lblk() * kTX + kTX <= a.lines && (a.src_ss & 1) == 0 &&
                              ((reinterpret_cast<uintptr_t>(blk) & 15) == 0);
            if (bulk) {
                __shared__ alignas(8) uint64_t bar;
                const int nrows = min(kSW, L - nb0);
                if (tid == 0) {
                    mbar_init(&bar, 1);
                    mbar_arrive_expect_tx(&bar, (unsigned)(nrows * kTX * sizeof(float2)));
                }
                __syncthreads();
                for (int r = tid; r < nrows; r += kTX * kSY)
                    bulk_g2s(t + r * kTX, blk + (int64_t)clampi(nb0 + r - P, 0, len - 1) * a.src_ss,
                             kTX * sizeof(float2), &bar);
                tables();
                mbar_wait(&bar, 0);
                // each warp built exactly the table entries of its own segment (entry i = tid,
                // segment ty = samples [32 ty, 32 ty + 32)) and every thread waited on the tile's
                // mbarrier itself: a warp barrier is enough
                __syncwarp();
                return;
            }
            const float2* src = blk + threadIdx.x;
            (void)x;
            for (int cc = threadIdx.y; cc < kSW; cc += kSY) {
                const int n = nb0 + cc;
                if (n < L && lblk() * kTX + threadIdx.x < a.lines)
                    cp_async8(t + cc * kTX + threadIdx.x, src + (int64_t)clampi(n - P, 0, len - 1) * a.src_ss);
            }
        } else {
            const float* src = reinterpret_cast<const float*>(a.src_base) + job.src_off + (int64_t)b * a.src_bstride + x;
            float2* t = reinterpret_cast<float2*>(tile);
            for (int cc = threadIdx.y; cc < kSW; cc += kSY) {
                const int n = nb0 + cc;
                if (n < L) cp_async4(t + cc * kTX + threadIdx.x, src + (int64_t)clampi(n - P, 0, len - 1) * a.src_ss);
            }
        }
    }
    tables();
    cp_async_wait_all();
    __syncthreads();
}

// modulated input (za, zb) of tile sample i (relative to nb0) for this thread's line
template <bool ROWS, bool CPLX> struct In {
    float2* tile;
    const float4* tabm;
    __device__ __forceinline__ float2 z(int i) const {
        const float4 t = tabm[i];
        const float2 v = tile[slot<ROWS>(i)];
        if constexpr (CPLX) return __ffma2_rn(make_float2(t.x, t.y), dup(v.x), __fmul2_rn(make_float2(t.z, t.w), dup(v.y)));
        else return __fmul2_rn(make_float2(t.x, t.y), dup(v.x));
    }
};

// (re, im) of output 0 from the smoothed pair u = (Sa, Sb)
__device__ __forceinline__ float2 recombine(const float4 t, float2 u) {
    return __ffma2_rn(make_float2(t.x, t.y), dup(u.x), __fmul2_rn(make_float2(t.z, t.w), dup(u.y)));
}

template <bool ROWS, bool CPLX>
__device__ __forceinline__ In<ROWS, CPLX> make_in(unsigned char* smem, const IirJob<float>& job) {
    In<ROWS, CPLX> in;
    in.tabm = reinterpret_cast<const float4*>(smem);
    in.tile = reinterpret_cast<float2*>(smem + kTabBytes);
    return in;
}

// Column stages, pass 1: no input tile.  Lines are adjacent threads and contiguous in
// memory, so each sample row of a warp is one coalesced 256-byte (complex) / 128-byte
// (real) load straight into registers; the thread never shares its samples, and pass 1
// keeps nothing for later, so the 32 KB tile only cost occupancy (6 CTAs / SM).  Shared
// memory holds the warp's own modulation-table entries, then the CTA summaries.
template <bool CPLX> struct InS {
    const float4* tabm;  // [i]: padded sample nb0 + i (this CTA's entries, built per warp)
    const void* src;     // this thread's line (clamped to the last line)
    int64_t ss;          // source elements between samples
    int nb0, P, len;
    __device__ __forceinline__ float2 z(int i) const {
        const float4 t = tabm[i];
        const int64_t n = clampi(nb0 + i - P, 0, len - 1);
        if constexpr (CPLX) {
            const float2 v = __ldg(reinterpret_cast<const float2*>(src) + n * ss);
            return __ffma2_rn(make_float2(t.x, t.y), dup(v.x), __fmul2_rn(make_float2(t.z, t.w), dup(v.y)));
        } else {
            const float v = __ldg(reinterpret_cast<const float*>(src) + n * ss);
            return __fmul2_rn(make_float2(t.x, t.y), dup(v));
        }
    }
};

// ---- pass 1: local forward sections -> end state e, backward-start sums b ----
template <bool FULL, typename IN>
__device__ __forceinline__ void sum_body(const IN& in, int i0, int m, Sec& s, float2& br, float2& bcr, float2& bci,
                                         const Iir32Par& q) {
    // the short last segment of a line runs rolled (keeps the kernel's code small)
#pragma unroll(FULL ? kM : 1)
    for (int i = 0; i < (FULL ? kM : m); ++i) {
        {
            const float2 y = sec_step(s, in.z(i0 + i), q);
            br = __ffma2_rn(dup(q.wr[i]), y, br);
            bcr = __ffma2_rn(dup(q.wcr[i]), y, bcr);
            bci = __ffma2_rn(dup(q.wci[i]), y, bci);
        }
    }
}

// ---- carries ----
// The last CTA of a 32-line block to finish pass 1 (an arrival counter per
// block) scans that block's states, so the scans overlap the rest of pass 1
// instead of running as a separate latency-bound launch.  States are staged
// through the CTA's shared memory in chunks of kCS segments
// ([kCS][12 slots][32 lines], 128-byte line runs); warp 0 scans plane a,
// warp 1 plane b (lane = line); all four warps move the data.
constexpr int kCL = kTX;
__device__ __forceinline__ void carry_io(float* sm, float* g, int64_t NL, int j0, int nj, int nl, int k0, int k1, bool load) {
    const int tid = threadIdx.y * kTX + threadIdx.x;
    if (nl == kCL && (NL & 3) == 0 && ((uintptr_t)g & 15) == 0) {  // 16-byte runs: thread = 4 lines of one (segment, slot)
        constexpr int kGroups = kTX * kSY / 8;  // row groups of 8 threads
        const int l4 = (tid & 7) * 4, r0 = tid >> 3;
        const int nk = k1 - k0;
        for (int r = r0; r < nj * nk; r += kGroups) {
            const int jj = r / nk, k = k0 + r - jj * nk;
            float* gp = g + ((int64_t)(j0 + jj) * 12 + k) * NL + l4;
            float* sp = sm + (jj * 12 + k) * kCL + l4;
            if (load) cp_async16(sp, gp);
            else *reinterpret_cast<float4*>(gp) = *reinterpret_cast<const float4*>(sp);
        }
    } else {
        const int l = tid & 31, grp = tid >> 5;
        if (l < nl)
            for (int jj = 0; jj < nj; ++jj) {
                float* gp = g + (int64_t)(j0 + jj) * 12 * NL + l;
                float* sp = sm + jj * 12 * kCL + l;
                for (int k = k0 + grp; k < k1; k += kSY) {
                    if (load) sp[k * kCL] = __ldcg(gp + (int64_t)k * NL);  // L2 (other CTAs' states)
                    else gp[(int64_t)k * NL] = sp[k * kCL];
                }
            }
    }
    if (load) cp_async_wait_all();
    __syncthreads();
}

// g: the block's states ([nseg][12][NL] from line x0); sm: kCS segments of staging
__device__ void carry_block(float* sm, int kCS, float* g, int64_t NL, int nl, int nseg, const Iir32Par& q,
                            const float (*QT)[3], const float (*MT)[9]) {
    const int l = threadIdx.x, pl = threadIdx.y;  // scanning threads: pl < 2
    const bool scan = pl < 2 && l < nl;
    const int es = 3 * pl, bs = 6 + 3 * pl;  // slots of e (then s_in) and b (then t_in) of this plane
    const bool one = nseg <= kCS;
    // forward: s_in[j] = carry-in, s_{j+1} = q^m s_j + e_j
    float sr = 0.f, scr = 0.f, sci = 0.f;
    const float Q0r = QT[0][0], Q0c = QT[0][1], Q0s = QT[0][2];
    for (int j0 = 0; j0 < nseg; j0 += kCS) {
        const int nj = min(kCS, nseg - j0);
        carry_io(sm, g, NL, j0, nj, nl, 0, one ? 12 : 6, true);
        if (scan) {
            float* p = sm + l;
#pragma unroll 4
            for (int jj = 0; jj < nj; ++jj, p += 12 * kCL) {
                const float e0 = p[es * kCL], e1 = p[(es + 1) * kCL], e2 = p[(es + 2) * kCL];
                p[es * kCL] = sr;
                p[(es + 1) * kCL] = scr;
                p[(es + 2) * kCL] = sci;
                const bool lt = j0 + jj == nseg - 1;
                const float Qr = lt ? QT[1][0] : Q0r, Qc = lt ? QT[1][1] : Q0c, Qs = lt ? QT[1][2] : Q0s;
                const float nr = fmaf(Qr, sr, e0);
                const float ncr = fmaf(Qc, scr, fmaf(-Qs, sci, e1));
                const float nci = fmaf(Qc, sci, fmaf(Qs, scr, e2));
                sr = nr;
                scr = ncr;
                sci = nci;
            }
        }
        __syncthreads();
        if (!one) carry_io(sm, g, NL, j0, nj, nl, 0, 6, false);
    }
    // true y[L-1] -> the backward sections' steady-state init
    const float yL = fmaf(2.f, scr, sr);
    float tr = q.gr * yL, tcr = q.gcr * yL, tci = q.gci * yL;
    float M0[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) M0[k] = MT[0][k];
    for (int j0 = (nseg - 1) / kCS * kCS; j0 >= 0; j0 -= kCS) {
        const int nj = min(kCS, nseg - j0);
        if (!one) carry_io(sm, g, NL, j0, nj, nl, 0, 12, true);
        if (scan) {
            float* p = sm + (nj - 1) * 12 * kCL + l;
#pragma unroll 4
            for (int jj = nj - 1; jj >= 0; --jj, p -= 12 * kCL) {
                const float b0 = p[bs * kCL], b1 = p[(bs + 1) * kCL], b2 = p[(bs + 2) * kCL];
                const float i0 = p[es * kCL], i1 = p[(es + 1) * kCL], i2 = p[(es + 2) * kCL];  // s_in of this plane
                p[bs * kCL] = tr;
                p[(bs + 1) * kCL] = tcr;
                p[(bs + 2) * kCL] = tci;
                const bool lt = j0 + jj == nseg - 1;
                float M[9];
#pragma unroll
                for (int k = 0; k < 9; ++k) M[k] = lt ? MT[1][k] : M0[k];
                const float Qr = lt ? QT[1][0] : Q0r, Qc = lt ? QT[1][1] : Q0c, Qs = lt ? QT[1][2] : Q0s;
                const float c0 = fmaf(M[0], i0, fmaf(M[1], i1, fmaf(M[2], i2, b0)));
                const float c1 = fmaf(M[3], i0, fmaf(M[4], i1, fmaf(M[5], i2, b1)));
                const float c2 = fmaf(M[6], i0, fmaf(M[7], i1, fmaf(M[8], i2, b2)));
                const float nr = fmaf(Qr, tr, c0);
                const float ncr = fmaf(Qc, tcr, fmaf(-Qs, tci, c1));
                const float nci = fmaf(Qc, tci, fmaf(Qs, tcr, c2));
                tr = nr;
                tcr = ncr;
                tci = nci;
            }
        }
        __syncthreads();
        carry_io(sm, g, NL, j0, nj, nl, one ? 0 : 6, 12, false);
    }
}

template <bool ROWS, bool CPLX, bool STREAM>
__global__ void __launch_bounds__(kTX * kSY, STREAM ? 8 : 1) iir32_sum(const IirArgs<float> a, const __grid_constant__ Iir32Par q,
                                                                     int* counters) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int jb = blockIdx.z % a.njobs, b = blockIdx.z / a.njobs;
    const IirJob<float>& job = a.jobs[jb];
    const int x = lblk() * kTX + threadIdx.x;
    const int seg = sblk() * kSY + threadIdx.y;
    const int L = a.len + 2 * a.P, NL = a.lines;
    const int n0 = seg * kM;
    if constexpr (STREAM) {
        // each warp builds the table entries of its own segment (entry i = tid)
        const int i = threadIdx.y * kTX + threadIdx.x, n = sblk() * kSW + i;
        if (n < L) {
            const float sgn = (job.need >> 1) ? -1.f : 1.f;
            const float2 cs = a.tab32[job.tabm_off + n];
            reinterpret_cast<float4*>(smem)[i] = make_float4(cs.x, cs.y, sgn * cs.y, -sgn * cs.x);
        }
        __syncwarp();
    } else {
        stage_tile<ROWS, CPLX>(smem, a, job, b, false);
    }
    float sub[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) sub[k] = 0.f;
    if (x < NL && n0 < L) {
        const int m = min(kM, L - n0);
        const int i0 = threadIdx.y * kM;
        float2 br = dup(0.f), bcr = dup(0.f), bci = dup(0.f);
        Sec s;
        auto run = [&](const auto& in) {
            if (m == kM) {
                // full segment: six independent dot products (FFMA2 with uniform weights)
                float2 er = dup(0.f), ecr = dup(0.f), eci = dup(0.f);
#pragma unroll
                for (int i = 0; i < kM; ++i) {
                    const float2 z = in.z(i0 + i);
                    er = __ffma2_rn(dup(q.ER[i]), z, er);
                    ecr = __ffma2_rn(dup(q.ECR[i]), z, ecr);
                    eci = __ffma2_rn(dup(q.ECI[i]), z, eci);
                    br = __ffma2_rn(dup(q.BR[i]), z, br);
                    bcr = __ffma2_rn(dup(q.BCR[i]), z, bcr);
                    bci = __ffma2_rn(dup(q.BCI[i]), z, bci);
                }
                if (seg == 0) {
                    // the reference's steady-state init: its free response over the segment
                    Sec s0;
                    sec_steady(s0, in.z(0), q);
                    const float* Q = q.Q[0];
                    const float* M = q.Mb[0];
                    er = __ffma2_rn(dup(Q[0]), s0.r, er);
                    ecr = __ffma2_rn(dup(Q[1]), s0.cr, __ffma2_rn(dup(-Q[2]), s0.ci, ecr));
                    eci = __ffma2_rn(dup(Q[1]), s0.ci, __ffma2_rn(dup(Q[2]), s0.cr, eci));
                    br = __ffma2_rn(dup(M[0]), s0.r, __ffma2_rn(dup(M[1]), s0.cr, __ffma2_rn(dup(M[2]), s0.ci, br)));
                    bcr = __ffma2_rn(dup(M[3]), s0.r, __ffma2_rn(dup(M[4]), s0.cr, __ffma2_rn(dup(M[5]), s0.ci, bcr)));
                    bci = __ffma2_rn(dup(M[6]), s0.r, __ffma2_rn(dup(M[7]), s0.cr, __ffma2_rn(dup(M[8]), s0.ci, bci)));
                }
                s.r = er;
                s.cr = ecr;
                s.ci = eci;
            } else {  // the short last segment: the recursion (rolled)
                if (seg == 0) sec_steady(s, in.z(0), q);
                else s.r = s.cr = s.ci = dup(0.f);
                sum_body<false>(in, i0, m, s, br, bcr, bci, q);
            }
        };
        if constexpr (STREAM) {
            InS<CPLX> in;
            in.tabm = reinterpret_cast<const float4*>(smem);
            const int64_t bo = job.src_off + (int64_t)b * a.src_bstride;
            if constexpr (CPLX) in.src = reinterpret_cast<const float2*>(a.src_base) + bo + x;
            else in.src = reinterpret_cast<const float*>(a.src_base) + bo + x;
            in.ss = a.src_ss;
            in.nb0 = sblk() * kSW;
            in.P = a.P;
            in.len = a.len;
            run(in);
        } else {
            run(make_in<ROWS, CPLX>(smem, job));
        }
        const float v[12] = {s.r.x, s.cr.x, s.ci.x, s.r.y, s.cr.y, s.ci.y, br.x, bcr.x, bci.x, br.y, bcr.y, bci.y};
#pragma unroll
        for (int k = 0; k < 12; ++k) sub[k] = v[k];
    }
    // super-segment summary (this CTA's kSY segments as one segment): the
    // carries then scan kSY times fewer steps; pass 2 expands them again
    __syncthreads();  // the tile is dead: it holds the sub-segment summaries now
    float* sm = reinterpret_cast<float*>(smem);  // [kSY][12][kTX]
#pragma unroll
    for (int k = 0; k < 12; ++k) sm[(threadIdx.y * 12 + k) * kTX + threadIdx.x] = sub[k];
    __syncthreads();
    const int nS = gridDim.x, K = min(kSY, a.nseg - sblk() * kSY);
    if (x < NL) {
        // local chains with zero super carries: s_loc_k (forward, entering sub k) and
        // T_loc_k (backward, entering sub k from above); e_S / b_S close them.  All four
        // warps work: warps 0 / 1 (planes a / b) write the forward chain, warps 2 / 3 redo
        // that short chain for their plane and run + write the backward one.
        const int pl = threadIdx.y & 1;
        const bool bwd = threadIdx.y >= 2;
        float sl[kSY][3];
        float r0 = 0.f, r1 = 0.f, r2 = 0.f;
#pragma unroll
        for (int k = 0; k < kSY; ++k) {
            if (k >= K) break;
            const float* p = sm + (k * 12 + 3 * pl) * kTX + threadIdx.x;
            sl[k][0] = r0; sl[k][1] = r1; sl[k][2] = r2;
            const float* Q = q.Q[sblk() * kSY + k == a.nseg - 1];
            const float n0_ = fmaf(Q[0], r0, p[0]);
            const float n1_ = fmaf(Q[1], r1, fmaf(-Q[2], r2, p[kTX]));
            const float n2_ = fmaf(Q[1], r2, fmaf(Q[2], r1, p[2 * kTX]));
            r0 = n0_; r1 = n1_; r2 = n2_;
        }
        float* sb = a.state32 + ((int64_t)blockIdx.z * a.nseg + sblk() * kSY) * 12 * NL + x;  // sub 0 of this CTA
        float* su = a.state32 + ((int64_t)gridDim.z * a.nseg + (int64_t)blockIdx.z * nS + sblk()) * 12 * NL + x;
        if (!bwd) {
#pragma unroll
            for (int k = 0; k < kSY; ++k) {
                if (k >= K) break;
                float* d = sb + (int64_t)k * 12 * NL;
                d[(int64_t)(3 * pl) * NL] = sl[k][0];
                d[(int64_t)(3 * pl + 1) * NL] = sl[k][1];
                d[(int64_t)(3 * pl + 2) * NL] = sl[k][2];
            }
            su[(int64_t)(3 * pl) * NL] = r0;
            su[(int64_t)(3 * pl + 1) * NL] = r1;
            su[(int64_t)(3 * pl + 2) * NL] = r2;
        } else {
            float t0 = 0.f, t1 = 0.f, t2 = 0.f;
#pragma unroll
            for (int k = kSY - 1; k >= 0; --k) {
                if (k >= K) continue;
                float* d = sb + (int64_t)k * 12 * NL;
                d[(int64_t)(6 + 3 * pl) * NL] = t0;
                d[(int64_t)(7 + 3 * pl) * NL] = t1;
                d[(int64_t)(8 + 3 * pl) * NL] = t2;
                const float* p = sm + (k * 12 + 6 + 3 * pl) * kTX + threadIdx.x;
                const int lt = sblk() * kSY + k == a.nseg - 1;
                const float* Q = q.Q[lt];
                const float* M = q.Mb[lt];
                const float c0 = fmaf(M[0], sl[k][0], fmaf(M[1], sl[k][1], fmaf(M[2], sl[k][2], p[0])));
                const float c1 = fmaf(M[3], sl[k][0], fmaf(M[4], sl[k][1], fmaf(M[5], sl[k][2], p[kTX])));
                const float c2 = fmaf(M[6], sl[k][0], fmaf(M[7], sl[k][1], fmaf(M[8], sl[k][2], p[2 * kTX])));
                const float n0_ = fmaf(Q[0], t0, c0);
                const float n1_ = fmaf(Q[1], t1, fmaf(-Q[2], t2, c1));
                const float n2_ = fmaf(Q[1], t2, fmaf(Q[2], t1, c2));
                t0 = n0_; t1 = n1_; t2 = n2_;
            }
            su[(int64_t)(6 + 3 * pl) * NL] = t0;
            su[(int64_t)(7 + 3 * pl) * NL] = t1;
            su[(int64_t)(8 + 3 * pl) * NL] = t2;
        }
    }
    // arrival: the last CTA of this line block runs its carries
    // (the barrier orders the CTA's state writes before thread 0's cumulative
    // gpu-scope fence; only one thread pays the membar)
    __shared__ int last;
    __syncthreads();
    int* cnt = counters + (int64_t)blockIdx.z * gridDim.y + lblk();
    if (threadIdx.x == 0 && threadIdx.y == 0) {
        __threadfence();
        last = atomicAdd(cnt, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int x0 = lblk() * kTX;
    unsigned dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    const int kCS = (int)(dyn / (12 * kCL * sizeof(float)));
    carry_block(reinterpret_cast<float*>(smem), kCS,
                a.state32 + ((int64_t)gridDim.z * a.nseg + (int64_t)blockIdx.z * nS) * 12 * NL + x0, NL, min(kTX, NL - x0),
                nS, q, q.QS, q.MbS);
    if (threadIdx.x == 0 && threadIdx.y == 0) *cnt = 0;  // ready for the next launch
}

// ---- pass 2: exact forward (y into the thread's own tile slots), exact backward, recombination ----
// FULL (interior segments): unrolled; otherwise (segments at the pad
// boundaries, the short last one) rolled, so the kernel's code stays small
template <bool ROWS, bool CPLX, bool FULL>
__device__ __forceinline__ void fin_fwd(const In<ROWS, CPLX>& in, int i0, int m, Sec& s, const Iir32Par& q) {
#pragma unroll(FULL ? kM : 1)
    for (int i = 0; i < (FULL ? kM : m); ++i) {
        const float2 z = in.z(i0 + i);
        in.tile[slot<ROWS>(i0 + i)] = sec_step(s, z, q);
    }
}

template <bool ROWS, bool FULL, typename EMIT>
__device__ __forceinline__ void fin_bwd(const float2* tile, int i0, int m, Sec& t, const Iir32Par& q, EMIT emit) {
#pragma unroll(FULL ? kM : 1)
    for (int i = (FULL ? kM : m) - 1; i >= 0; --i) emit(i, sec_step(t, tile[slot<ROWS>(i0 + i)], q));
}

template <bool ROWS, bool CPLX>
__global__ void __launch_bounds__(kTX * kSY) iir32_fin(const IirArgs<float> a, const __grid_constant__ Iir32Par q) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int jb = blockIdx.z % a.njobs, b = blockIdx.z / a.njobs;
    const IirJob<float>& job = a.jobs[jb];
    const int x = lblk() * kTX + threadIdx.x;
    const int seg = sblk() * kSY + threadIdx.y;
    const int len = a.len, P = a.P, L = len + 2 * P, NL = a.lines;
    // carries of this segment: its local chains (s_loc, T_loc) and the super-segment carries (s_S, t_S)
    float lc[12], sc[12];
    {
        const bool ok = x < NL && seg < a.nseg;
        const float* st = a.state32 + ((int64_t)blockIdx.z * a.nseg + seg) * 12 * NL + x;
        const float* su = a.state32 + ((int64_t)gridDim.z * a.nseg + (int64_t)blockIdx.z * gridDim.x + sblk()) * 12 * NL + x;
#pragma unroll
        for (int k = 0; k < 12; ++k) {
            lc[k] = ok ? st[(int64_t)k * NL] : 0.f;
            sc[k] = ok ? su[(int64_t)k * NL] : 0.f;
        }
    }
    stage_tile<ROWS, CPLX>(smem, a, job, b, true);
    const int n0 = seg * kM;
    const int m = min(kM, L - n0);
    const int i0 = threadIdx.y * kM;
    // segments that leave nothing inside the crop [P, P + len) only fed the carries
    const bool live = x < NL && n0 < L && n0 + m > P && n0 < P + len;
    // interior: a whole segment inside the crop (no per-sample checks)
    const bool interior = m == kM && n0 >= P && n0 + kM <= P + len;
    const float4* tabr = reinterpret_cast<const float4*>(smem) + kSW;  // [i]: output sample nb0 + i - P
    float2* tile = reinterpret_cast<float2*>(smem + kTabBytes);
    Sec t;
    if (live) {
        const In<ROWS, CPLX> in = make_in<ROWS, CPLX>(smem, job);
        // true carries: s_in = QF s_S + s_loc,  t_in = QB t_S + T_loc + G s_S
        const int kk = threadIdx.y, lt = sblk() == (int)gridDim.x - 1;
        const float* QF = q.QF[kk];
        const float* QB = q.QB[lt][kk];
        const float* G = q.G[lt][kk];
        float si[2][3], ti[2][3];
#pragma unroll
        for (int pl = 0; pl < 2; ++pl) {
            const float* S = sc + 3 * pl;  // s_S of this plane
            const float* T = sc + 6 + 3 * pl;
            si[pl][0] = fmaf(QF[0], S[0], lc[3 * pl]);
            si[pl][1] = fmaf(QF[1], S[1], fmaf(-QF[2], S[2], lc[3 * pl + 1]));
            si[pl][2] = fmaf(QF[1], S[2], fmaf(QF[2], S[1], lc[3 * pl + 2]));
            const float g0 = fmaf(G[0], S[0], fmaf(G[1], S[1], fmaf(G[2], S[2], lc[6 + 3 * pl])));
            const float g1 = fmaf(G[3], S[0], fmaf(G[4], S[1], fmaf(G[5], S[2], lc[7 + 3 * pl])));
            const float g2 = fmaf(G[6], S[0], fmaf(G[7], S[1], fmaf(G[8], S[2], lc[8 + 3 * pl])));
            ti[pl][0] = fmaf(QB[0], T[0], g0);
            ti[pl][1] = fmaf(QB[1], T[1], fmaf(-QB[2], T[2], g1));
            ti[pl][2] = fmaf(QB[1], T[2], fmaf(QB[2], T[1], g2));
        }
        Sec s;
        if (seg == 0) {
            sec_steady(s, in.z(0), q);
        } else {
            s.r = make_float2(si[0][0], si[1][0]);
            s.cr = make_float2(si[0][1], si[1][1]);
            s.ci = make_float2(si[0][2], si[1][2]);
        }
        t.r = make_float2(ti[0][0], ti[1][0]);
        t.cr = make_float2(ti[0][1], ti[1][1]);
        t.ci = make_float2(ti[0][2], ti[1][2]);
        if (interior) fin_fwd<ROWS, CPLX, true>(in, i0, m, s, q);
        else fin_fwd<ROWS, CPLX, false>(in, i0, m, s, q);
    }
    if constexpr (ROWS) {
        constexpr int swp = kSW | 1;
        const int nb0 = sblk() * kSW;
        float2* otile = tile;  // outputs replace y in the same slots
        if (live) {
            float2* trow = otile + threadIdx.x * swp + i0;
            if (interior) {
                fin_bwd<ROWS, true>(tile, i0, m, t, q, [&](int i, float2 u) { trow[i] = recombine(tabr[i0 + i], u); });
            } else {
                auto emit = [&](int i, float2 u) {
                    const int n = n0 + i;
                    if (n >= P && n < P + len) trow[i] = recombine(tabr[i0 + i], u);
                };
                fin_bwd<ROWS, false>(tile, i0, m, t, q, emit);
            }
        }
        __syncthreads();
        // row-contiguous write-out (lanes along the row), pointers stepped per row
        const int c0 = max(0, P - nb0), c1 = min(kSW, min(P + len, L) - nb0);
        float2* row = a.dst_base + job.dst_off[0] + (int64_t)b * a.dst_bstride +
                      (int64_t)(lblk() * kTX + threadIdx.y) * a.dst_ls - P + nb0;
        const float2* orow = otile + threadIdx.y * swp;
        const int64_t rstep = (int64_t)kSY * a.dst_ls;
        if (c0 == 0 && c1 == kSW) {
            for (int r = threadIdx.y; r < kTX && lblk() * kTX + r < NL; r += kSY, row += rstep, orow += kSY * swp) {
#pragma unroll
                for (int k = 0; k < kSW / kTX; ++k) __stcs(row + threadIdx.x + k * kTX, orow[threadIdx.x + k * kTX]);
            }
        } else {
            for (int r = threadIdx.y; r < kTX && lblk() * kTX + r < NL; r += kSY, row += rstep, orow += kSY * swp)
                for (int cc = c0 + threadIdx.x; cc < c1; cc += kTX) __stcs(row + cc, orow[cc]);
        }
    } else {
        if (!live) return;
        // outputs 1..3 (SDFT conjugate fills) = output 0 with im scaled by rel[o] = +-1
        const int nout = job.nout;
        float2* d0 = a.dst_base + job.dst_off[0] + (int64_t)b * a.dst_bstride + (int64_t)x * a.dst_ls;
        int64_t dlt[4];
        float rel[4];
#pragma unroll
        for (int o = 0; o < 4; ++o) {
            dlt[o] = o < nout ? job.dst_off[o] - job.dst_off[0] : 0;
            rel[o] = (o < nout && job.conj[o] != job.conj[0]) ? -1.f : 1.f;
        }
        const int64_t dss = a.dst_ss;
        auto put = [&](float2* p, float2 v) {
            __stcs(p, v);
            if (nout > 1) {
#pragma unroll
                for (int o = 1; o < 4; ++o)
                    if (o < nout) __stcs(p + dlt[o], make_float2(v.x, rel[o] * v.y));
            }
        };
        if (interior) {
            float2* p = d0 + (int64_t)(n0 + kM - 1 - P) * dss;  // walks up with the backward pass
            fin_bwd<ROWS, true>(tile, i0, m, t, q, [&](int i, float2 u) {
                put(p, recombine(tabr[i0 + i], u));
                p -= dss;
            });
        } else {
            auto emit = [&](int i, float2 u) {
                const int n = n0 + i;
                if (n >= P && n < P + len) put(d0 + (int64_t)(n - P) * dss, recombine(tabr[i0 + i], u));
            };
            fin_bwd<ROWS, false>(tile, i0, m, t, q, emit);
        }
    }
}

// ---- host: parallel-form parameters from the direct-form coefficients ----
using cd = std::complex<double>;

// L = padded samples per line
// parallel form of the direct-form coefficients: real pole qr, complex pole qc (Im > 0), residues cr, cc
void sections(const IirCoef& c, cd& qr, cd& qc, cd& cr, cd& cc) {
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
    qr = cd(r[ir].real(), 0.0);
    qc = r[ic];
    const cd qs[3] = {qr, qc, std::conj(qc)};
    auto resid = [&](int k) {
        cd d(1.0, 0.0);
        for (int j = 0; j < 3; ++j)
            if (j != k) d *= 1.0 - qs[j] / qs[k];
        return c.B / d;
    };
    cr = resid(0);
    cc = resid(1);
}

void iir32_params(const IirCoef& c, int L, Iir32Par* out) {
    const int nseg = (L + kM - 1) / kM, mlast = L - (nseg - 1) * kM;
    const int nS = (nseg + kSY - 1) / kSY, mlastS = L - (nS - 1) * kSW, Klast = nseg - (nS - 1) * kSY;
    cd qr, qc, cr, cc;
    sections(c, qr, qc, cr, cc);

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
    // full-segment pass-1 weights: forward impulse response g_n = c_r q_r^n + 2 Re(c_c q_c^n);
    // E[k] = c q^(kM-1-k); B[k] = sum_{i >= k} (c q^i) g_(i-k)  (fp64, rounded once)
    {
        double g[kM];
        for (int n = 0; n < kM; ++n) g[n] = (cr * std::pow(qr, n)).real() + 2.0 * (cc * std::pow(qc, n)).real();
        for (int k = 0; k < kM; ++k) {
            const cd er = cr * std::pow(qr, kM - 1 - k), ec = cc * std::pow(qc, kM - 1 - k);
            p.ER[k] = (float)er.real();
            p.ECR[k] = (float)ec.real();
            p.ECI[k] = (float)ec.imag();
            double br = 0.0;
            cd bc = 0.0;
            for (int i = k; i < kM; ++i) {
                br += (cr * std::pow(qr, i)).real() * g[i - k];
                bc += cc * std::pow(qc, i) * g[i - k];
            }
            p.BR[k] = (float)br;
            p.BCR[k] = (float)bc.real();
            p.BCI[k] = (float)bc.imag();
        }
    }
    // transfer q^m and Mb of a run of m samples: segments (kM, mlast) and super-segments (kSW, mlastS)
    auto run = [&](int m, float* Q, float* Mb) {
        const cd Qr = std::pow(qr, m), Qc = std::pow(qc, m);
        Q[0] = (float)Qr.real();
        Q[1] = (float)Qc.real();
        Q[2] = (float)Qc.imag();
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
            Mb[k] = (float)Mr[k];
            Mb[3 + k] = (float)Mc[k].real();
            Mb[6 + k] = (float)Mc[k].imag();
        }
    };
    run(kM, p.Q[0], p.Mb[0]);
    run(mlast, p.Q[1], p.Mb[1]);
    run(kSW, p.QS[0], p.MbS[0]);
    run(mlastS, p.QS[1], p.MbS[1]);
    // super-segment -> sub-segment expansion (3x3 operators on (r, c re, c im), in double)
    using M3 = std::array<double, 9>;
    auto mat = [](cd a, cd b) { return M3{a.real(), 0, 0, 0, b.real(), -b.imag(), 0, b.imag(), b.real()}; };
    auto mul = [](const M3& A, const M3& B) {
        M3 C{};
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) C[3 * i + j] = A[3 * i] * B[j] + A[3 * i + 1] * B[3 + j] + A[3 * i + 2] * B[6 + j];
        return C;
    };
    M3 Mbd[2];
    for (int t = 0; t < 2; ++t)
        for (int k = 0; k < 9; ++k) Mbd[t][k] = p.Mb[t][k];
    // (Mb recomputed in double would be marginally more exact; the fp32 copies are what pass 1 used)
    for (int k = 0; k < kSY; ++k) {
        const cd a = std::pow(qr, kM * k), b = std::pow(qc, kM * k);
        p.QF[k][0] = (float)a.real();
        p.QF[k][1] = (float)b.real();
        p.QF[k][2] = (float)b.imag();
    }
    for (int t = 0; t < 2; ++t) {
        const int K = t ? Klast : kSY;
        for (int k = 0; k < kSY; ++k) {
            cd ar(1.0, 0.0), bc(1.0, 0.0);  // prod_{j=k+1}^{K-1} q^{m_j}
            M3 P = mat(1.0, 1.0), G{};       // running prod_{j=k+1}^{i-1} Q_j, accumulated G
            for (int i = k + 1; i < K; ++i) {
                const bool last = t && i == K - 1;
                const int m = last ? mlast : kM;
                const M3 term = mul(mul(P, Mbd[last ? 1 : 0]), mat(std::pow(qr, kM * i), std::pow(qc, kM * i)));
                for (int e = 0; e < 9; ++e) G[e] += term[e];
                P = mul(P, mat(std::pow(qr, m), std::pow(qc, m)));
                ar *= std::pow(qr, m);
                bc *= std::pow(qc, m);
            }
            p.QB[t][k][0] = (float)ar.real();
            p.QB[t][k][1] = (float)bc.real();
            p.QB[t][k][2] = (float)bc.imag();
            for (int e = 0; e < 9; ++e) p.G[t][k][e] = (float)G[e];
        }
    }
}

template <bool ROWS, bool CPLX>
cudaError_t launch_passes(const IirArgs<float>& a, const Iir32Par& q, cudaStream_t s) {
    // (pass 1's carry scans stage their states in chunks of what the tile
    // leaves: reserving room for a single chunk cost more in occupancy)
    constexpr size_t smem = Tile<ROWS, CPLX>::smem;
    // column stages stream pass 1 (no tile): tables, then summaries / carry staging
    constexpr bool kStream = !ROWS;
    constexpr size_t smem1 = kStream ? 12 * 1024 : smem;
    static bool attr = false;  // launches are serialised by the engine lock
    if (!attr) {
        cudaFuncSetAttribute(iir32_sum<ROWS, CPLX, kStream>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
        cudaFuncSetAttribute(iir32_fin<ROWS, CPLX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    const dim3 block(kTX, kSY);
    const dim3 grid((a.nseg + kSY - 1) / kSY, (a.lines + kTX - 1) / kTX, a.njobs * a.batch);
    // arrival counters (one int per 32-line block and job): a library-owned buffer zeroed
    // once at allocation; every launch leaves them zero again (the last CTA of a block
    // resets its counter), so no memset launch per stage
    int* counters = a.counters;
    iir32_sum<ROWS, CPLX, kStream><<<grid, block, smem1, s>>>(a, q, counters);
    iir32_fin<ROWS, CPLX><<<grid, block, smem, s>>>(a, q);
    return cudaGetLastError();
}

}  // namespace

void iir32_sections(const IirCoef& c, double out[6]) {
    cd qr, qc, cr, cc;
    sections(c, qr, qc, cr, cc);
    const double v[6] = {qr.real(), qc.real(), qc.imag(), cr.real(), cc.real(), cc.imag()};
    std::memcpy(out, v, sizeof(v));
}

bool iir32_enabled() {
    const bool on = !knobs().iir64;
    return on;
}

cudaError_t launch_iir32(const IirArgs<float>& a_in, cudaStream_t s) {
    IirArgs<float> a = a_in;
    const int L = a.len + 2 * a.P;
    if (a.seglen != kM || a.nseg != (L + kM - 1) / kM) return cudaErrorInvalidValue;
    a.state32 = reinterpret_cast<float*>(a.state);
    // parameters per (coefficients, last segment length), computed once (launches are serialised by the engine lock)
    static std::map<std::array<double, 5>, Iir32Par> cache;
    const std::array<double, 5> key = {a.c.B, a.c.a1, a.c.a2, a.c.a3, (double)L};
    auto it = cache.find(key);
    if (it == cache.end()) {
        Iir32Par p;
        iir32_params(a.c, L, &p);
        it = cache.emplace(key, p).first;
    }
    const Iir32Par& q = it->second;
    if (a.src_ls == 1) return a.real_in ? launch_passes<false, false>(a, q, s) : launch_passes<false, true>(a, q, s);
    // horizontal stage: real rows in, one output per job, rows written in place
    if (a.real_in && a.src_ss == 1 && a.dst_ss == 1 && a.one_out) return launch_passes<true, false>(a, q, s);
    return cudaErrorInvalidValue;
}

}  // namespace fgb
