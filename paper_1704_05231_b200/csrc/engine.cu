// libfgb200 host engine: coefficient math, plan building, execution, C ABI.
//
// A call is compiled into an immutable, cached Plan: a list of kernel steps
// plus one device blob holding every tap table, job table and trig table
// the steps read.  Per call only the base pointers (image, output,
// workspace) change, so steady-state calls issue kernel launches only.
//
// Schedules restated here (paths relative to /root/reference/pkg/src/fastgabor):
//   bank (Algorithm 1)   bank.py:90-129 / :132-157 -- per frequency: one fused
//                        row launch for every directly computed orientation
//                        k <= N/2, then one column launch emitting theta_k
//                        and pi - theta_k from the same J (bank.py:109-116);
//                        small half-widths (h <= 6): one fused row+column
//                        launch with J in shared memory.  Frequencies run on
//                        up to 4 stream lanes, heaviest first.
//   filter / stages      gabor.py:107-176, bank.py:68-74
//   SDFT (Algorithm 2)   sdft.py:178-213 -- J_u for u <= Mx/2 once, every
//                        (u, v<=My/2) column job writes bin(u,v), the mirror
//                        bin(Mx-u,v) from conj(J_u) (sdft.py:202-203) and the
//                        conjugate-symmetric fills (sdft.py:209-212).
//
// Sections: errors | host coefficient math (sampled Gaussian, IIR poles,
// pad radius) | device memory | plans (Step, Plan) and builders | descriptor
// validation | Gabor plans | SDFT plans | execution (lanes, chunks, live
// profile) | plan cache keys | GPU brute-force oracles | C ABI (device,
// host-buffer with pipelined D2H, planar host, GBNK, probes).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <type_traits>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/fgb200.h"
#include "kernels.h"

namespace fgb {

template <typename T> double probe_fma_tflops();
int gbnk_write_device(const char* path, const double* params, int n_entries, int H, int W, int dtype,
                      const void* dev_entries, int sdft, cudaStream_t s, std::string* err);
template <typename T> double probe_fma_reg_tflops(int mode);
double probe_ffma2_tflops(int mode);

// ===========================================================================
// errors
// ===========================================================================
static thread_local std::string g_err;
struct NvtxRange {  // scoped NVTX range (balanced on every return path)
    explicit NvtxRange(const char* n) { nvtxRangePushA(n); }
    ~NvtxRange() { nvtxRangePop(); }
};
static int32_t fail(int32_t code, const std::string& msg) {
    g_err = msg;
    return code;
}
#define FGB_CUDA(x)                                                                          \
    do {                                                                                     \
        cudaError_t e_ = (x);                                                                \
        if (e_ != cudaSuccess) return fail(FGB_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)
#define FGB_TRY(x)                     \
    do {                               \
        int32_t r_ = (x);              \
        if (r_ != FGB_OK) return r_;   \
    } while (0)

// ===========================================================================
// host coefficient math
// ===========================================================================

// gaussian.py:198-212
static int pad_radius(const fgb_smoother& k, double sigma) {
    if (k.kind == FGB_SMOOTH_FIR) return std::max(1, (int)std::ceil(k.radius * sigma));
    if (k.kind == FGB_SMOOTH_IIR) return (int)std::ceil(5.0 * sigma) + 2;
    return 0;
}

// numpy's pairwise summation (np.add.reduce on a contiguous float64 array):
// 8-way unrolled blocks of <= 128, recursive halving above.  Reproducing it
// makes the tap weights bit-identical to the reference's kernel.sum().
static double np_pairwise_sum(const double* a, size_t n) {
    if (n < 8) {
        double res = 0.;
        for (size_t i = 0; i < n; ++i) res += a[i];
        return res;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        size_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    size_t n2 = n / 2;
    n2 -= n2 % 8;
    return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
}

// gaussian.py:188-195: unit-sum sampled Gaussian on [-h, h].
static std::vector<double> sampled_gaussian(double sigma, double radius, int* half) {
    const int h = std::max(1, (int)std::ceil(radius * sigma));
    std::vector<double> w(2 * h + 1);
    for (int i = 0; i <= 2 * h; ++i) {
        const double x = (double)(i - h);
        w[i] = std::exp(-(x * x) / (2.0 * sigma * sigma));
    }
    const double s = np_pairwise_sum(w.data(), w.size());
    for (double& v : w) v /= s;
    *half = h;
    return w;
}

// Pole-parameter knots of the third-order recursion; data table of
// gaussian.py:78-105 (log2 sigma = -1 .. 5 step 0.25; (log(r-1), phi, log(d-1))).
static const double kKnots[25][3] = {
    {1.4935547894, 1.7389422874, 1.4116802788},    {1.0124325346, 1.6028888671, 0.9948121036},
    {0.7060188604, 1.4246405642, 0.7655646807},    {0.3711981889, 1.3035671168, 0.4599139117},
    {0.0723219048, 1.1741421430, 0.1988303275},    {-0.0657826821, 1.0609426640, 0.0641342325},
    {-0.1084526360, 0.8746229033, 0.0520603916},   {-0.3079872798, 0.7888980715, -0.2103392209},
    {-0.4435572915, 0.6681318749, -0.3543999555},  {-0.5826541508, 0.5511044975, -0.4681767292},
    {-0.6341889379, 0.4375707759, -0.4950920113},  {-0.9438814088, 0.3960503190, -0.8422106914},
    {-1.1264093957, 0.3331316708, -1.0232036316},  {-1.3323529220, 0.2853777435, -1.2419374903},
    {-1.5043108087, 0.2384505949, -1.4119365035},  {-1.6909017377, 0.2010996380, -1.6007291308},
    {-1.8639872273, 0.1677245302, -1.7693707791},  {-2.0526626380, 0.1419695700, -1.9627706878},
    {-2.2480922032, 0.1206592327, -2.1643322734},  {-2.4183618584, 0.1007997229, -2.3318115898},
    {-2.6108636240, 0.0856583363, -2.5302995718},  {-2.7812366868, 0.0716083982, -2.6981612487},
    {-2.9595594412, 0.0602521009, -2.8771310090},  {-3.1353804585, 0.0506201753, -3.0527659020},
    {-3.3165061207, 0.0427250483, -3.2360423517},
};

using cd = std::complex<double>;

static void poles_from(const double prm[3], cd p[3]) {
    // gaussian.py:136-142
    const double r = 1.0 + std::exp(prm[0]);
    const double d = 1.0 + std::exp(prm[2]);
    p[0] = r * cd(std::cos(prm[1]), std::sin(prm[1]));
    p[1] = r * cd(std::cos(-prm[1]), std::sin(-prm[1]));
    p[2] = cd(d, 0.0);
}

static double cascade_var(const cd p[3]) {
    // gaussian.py:145-147
    cd s(0.0, 0.0);
    for (int i = 0; i < 3; ++i) s += 2.0 * p[i] / ((p[i] - 1.0) * (p[i] - 1.0));
    return s.real();
}

// Brent's root finder (Brent 1973), the algorithm of scipy.optimize.brentq
// used by gaussian.py:160 with its default tolerances.
template <typename F> static double brent(F f, double xa, double xb) {
    const double xtol = 2e-12, rtol = 8.881784197001252e-16;
    double xpre = xa, xcur = xb, xblk = 0.0, fpre = f(xpre), fcur = f(xcur), fblk = 0.0, spre = 0.0, scur = 0.0;
    if (fpre == 0) return xpre;
    if (fcur == 0) return xcur;
    for (int it = 0; it < 200; ++it) {
        if (fpre != 0 && fcur != 0 && (std::signbit(fpre) != std::signbit(fcur))) {
            xblk = xpre;
            fblk = fpre;
            spre = scur = xcur - xpre;
        }
        if (std::fabs(fblk) < std::fabs(fcur)) {
            xpre = xcur; xcur = xblk; xblk = xpre;
            fpre = fcur; fcur = fblk; fblk = fpre;
        }
        const double delta = (xtol + rtol * std::fabs(xcur)) / 2;
        const double sbis = (xblk - xcur) / 2;
        if (fcur == 0 || std::fabs(sbis) < delta) return xcur;
        if (std::fabs(spre) > delta && std::fabs(fcur) < std::fabs(fpre)) {
            double stry;
            if (xpre == xblk) {
                stry = -fcur * (xcur - xpre) / (fcur - fpre);
            } else {
                const double dpre = (fpre - fcur) / (xpre - xcur);
                const double dblk = (fblk - fcur) / (xblk - xcur);
                stry = -fcur * (fblk * dblk - fpre * dpre) / (dblk * dpre * (fblk - fpre));
            }
            if (2 * std::fabs(stry) < std::min(std::fabs(spre), 3 * std::fabs(sbis) - delta)) {
                spre = scur;
                scur = stry;
            } else {
                spre = sbis;
                scur = sbis;
            }
        } else {
            spre = sbis;
            scur = sbis;
        }
        xpre = xcur;
        fpre = fcur;
        if (std::fabs(scur) > delta) xcur += scur;
        else xcur += (sbis > 0 ? delta : -delta);
        fcur = f(xcur);
    }
    return xcur;
}

// gaussian.py:164-185: (B, a1, a2, a3) with B = sum(a), a = poly(1/poles).
static int32_t iir_coeffs(double sigma, double out[4]) {
    if (!(sigma > 0)) return fail(FGB_EINVAL, "sigma must be positive");
    if (sigma < 0.5)
        return fail(FGB_EINVAL,
                    "sigma below 0.5 is outside the recursive filter's validity range; use the ExactFIR smoother instead");
    cd p[3];
    if (sigma <= 32.0) {
        double l2 = std::log2(sigma);
        l2 = std::min(std::max(l2, -1.0), 5.0);
        double prm[3];
        // np.interp on the uniform knot grid -1 + 0.25 j
        int j = (int)std::floor((l2 + 1.0) / 0.25);
        if (j >= 24) {
            for (int c = 0; c < 3; ++c) prm[c] = kKnots[24][c];
        } else {
            if (j < 0) j = 0;
            const double x0 = -1.0 + 0.25 * j, x1 = -1.0 + 0.25 * (j + 1);
            for (int c = 0; c < 3; ++c) {
                const double slope = (kKnots[j + 1][c] - kKnots[j][c]) / (x1 - x0);
                prm[c] = slope * (l2 - x0) + kKnots[j][c];
            }
        }
        poles_from(prm, p);
    } else {
        cd top[3];
        poles_from(kKnots[24], top);
        auto mismatch = [&](double q) {
            cd t[3];
            for (int i = 0; i < 3; ++i) t[i] = std::pow(top[i], 1.0 / q);
            return cascade_var(t) - sigma * sigma;
        };
        double hi = 2.0;
        while (mismatch(hi) < 0.0) hi *= 2.0;
        const double q = brent(mismatch, 0.5, hi);
        for (int i = 0; i < 3; ++i) p[i] = std::pow(top[i], 1.0 / q);
    }
    // np.poly(1/p): a = [1]; a = conv(a, [1, -q_k]) for k = 0, 1, 2
    cd a[4] = {cd(1, 0), cd(0, 0), cd(0, 0), cd(0, 0)};
    for (int k = 0; k < 3; ++k) {
        const cd q = 1.0 / p[k];
        for (int m = k + 1; m >= 1; --m) a[m] = a[m] - q * a[m - 1];
    }
    const double a1 = a[1].real(), a2 = a[2].real(), a3 = a[3].real();
    out[0] = 1.0 + a1 + a2 + a3;
    out[1] = a1;
    out[2] = a2;
    out[3] = a3;
    return FGB_OK;
}

// ===========================================================================
// device memory
// ===========================================================================
struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
    ~DevBuf() { reset(); }
    void reset() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    int32_t ensure(size_t bytes) {
        if (bytes <= n) return FGB_OK;
        reset();
        if (bytes == 0) return FGB_OK;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess) {
            p = nullptr;
            cudaGetLastError();
            return fail(FGB_ENOMEM, std::string("cudaMalloc workspace: ") + cudaGetErrorString(e));
        }
        n = bytes;
        return FGB_OK;
    }
};

// ===========================================================================
// plans
// ===========================================================================
enum Sel { SEL_IMG = 0, SEL_IMGC = 1, SEL_OUT = 2, SEL_WS = 3, SEL_WSR = 4 };
struct Ref {
    int sel = SEL_WS;
    int64_t off = 0;  // elements of the referenced type (T for real, C for complex)
};

enum StepKind { ST_ROW = 0, ST_COL, ST_IIR, ST_TR_RC, ST_TR_CC, ST_TR_RR, ST_SDFTF, ST_BANKF, ST_COLU, ST_ROWU, ST_BANKU };

template <typename T> struct Step {
    int kind = 0;
    int lane = 0;            // stream lane (independent frequencies run concurrently)
    const char* name = "";
    double flops = 0.0;      // reference-counter flops (M + A) per image
    double bytes = 0.0;      // compulsory bytes per image (input read + output written)
    int H = 0, W = 0;     // dims seen by the kernel
    Ref src, dst;
    int64_t src_pitch = -1;  // real inputs: -1 = descriptor pitch
    // ST_ROW
    RowGroup<T> rg{};
    int hp = 0;
    int j16 = 0;             // fp32: split-fp16 J planes for the tensor-core column pass (ST_COLU)
    // ST_COL
    int job0 = 0, njobs = 0, t0 = 0, nt = 0, zero_bnd = 0, has_b = 1;
    std::vector<cx_t<T>> pw;  // ST_COL: tap pairs packed in job order (kernel-parameter path)
    // ST_IIR
    int P = 0;
    IirCoef coef{};
    int64_t scratch_off = 0;  // T elements into the workspace scratch region
    int nseg = 1, seglen = 1;
    int iir_row = 0;          // lines are image rows (horizontal stage): strided in place, no transposes
    int iir_real = 0;         // real source (the image) instead of complex J
    int64_t g_off = 0;        // into Plan::dbls: [seglen][3]
    double Aseg[9] = {0}, Alast[9] = {0};
    // ST_BANKF (fp32): tap tables + per-orientation outputs
    std::vector<float> bf_w;
    std::vector<BankFusedOut> bf_out;
    int bf_colw_off = 0;
    // ST_SDFTF
    int M = 0, h = 0, nheads = 0;
    int64_t heads_off = 0, slots_off = 0, w_off = 0;
};

struct PlanBase {
    virtual ~PlanBase() {}
};

template <typename T> struct Plan : PlanBase {
    using C = cx_t<T>;
    std::vector<Step<T>> steps;
    // host blobs (uploaded once into `blob`)
    std::vector<T> wrow;          // row tap tables
    std::vector<C> wcol;          // column tap pairs
    std::vector<ColJob<T>> cjobs;
    std::vector<BankUJob> bjobs;  // ST_BANKU (fp32)
    std::vector<IirJob<T>> ijobs;
    std::vector<double2> tabs;
    std::vector<int32_t> ints;
    std::vector<double> dbls;
    DevBuf blob;
    size_t off_wrow = 0, off_wcol = 0, off_cjobs = 0, off_bjobs = 0, off_ijobs = 0, off_tabs = 0, off_tabs32 = 0, off_ints = 0, off_dbls = 0;
    // workspace per image (bytes), scratch (T elements per image-chunk) and chunking
    int64_t ws_img_c = 0;         // complex elements per image
    int64_t scratch_img_t = 0;    // T elements per image (IIR scratch)
    int64_t state_img_d = 0;      // doubles per image (IIR segment states)
    int64_t out_img_c = 0;        // complex elements per output image
    int H = 0, W = 0;
    int jbuf = 0;                 // > 0: J slots are split-fp16 planes with jbuf replicate rows (ST_COLU)
    int xbuf = 0;                 // > 0: some row stages run on the tensor cores (ST_ROWU / ST_BANKU) from the prep planes
    bool banku = false;           // fp32 FIR bank plan: some frequencies run as ST_BANKU (J in shared memory)
    std::set<int> banku_h;        // their half-widths
    int64_t hpw = 0;              // (H + 2 jbuf) * W64: complex elements per J slot (= u32 per fp16 plane)
    int chunk = 1;
    int nlanes = 1;               // concurrent stream lanes used by the steps

    int32_t upload() {
        auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
        size_t o = 0;
        off_wrow = o; o = al(o + wrow.size() * sizeof(T));
        off_wcol = o; o = al(o + wcol.size() * sizeof(C));
        off_cjobs = o; o = al(o + cjobs.size() * sizeof(ColJob<T>));
        off_bjobs = o; o = al(o + bjobs.size() * sizeof(BankUJob));
        off_ijobs = o; o = al(o + ijobs.size() * sizeof(IirJob<T>));
        off_tabs = o; o = al(o + tabs.size() * sizeof(double2));
        off_tabs32 = o; o = al(o + tabs.size() * sizeof(float2));
        off_ints = o; o = al(o + ints.size() * sizeof(int32_t));
        off_dbls = o; o = al(o + dbls.size() * sizeof(double));
        FGB_TRY(blob.ensure(std::max<size_t>(o, 256)));
        std::vector<char> h(o, 0);
        if (!wrow.empty()) std::memcpy(h.data() + off_wrow, wrow.data(), wrow.size() * sizeof(T));
        if (!wcol.empty()) std::memcpy(h.data() + off_wcol, wcol.data(), wcol.size() * sizeof(C));
        if (!cjobs.empty()) std::memcpy(h.data() + off_cjobs, cjobs.data(), cjobs.size() * sizeof(ColJob<T>));
        if (!bjobs.empty()) std::memcpy(h.data() + off_bjobs, bjobs.data(), bjobs.size() * sizeof(BankUJob));
        if (!ijobs.empty()) std::memcpy(h.data() + off_ijobs, ijobs.data(), ijobs.size() * sizeof(IirJob<T>));
        if (!tabs.empty()) std::memcpy(h.data() + off_tabs, tabs.data(), tabs.size() * sizeof(double2));
        for (size_t i = 0; i < tabs.size(); ++i) {  // fp32 copy (each value rounded once from the fp64 table)
            const float2 v = make_float2((float)tabs[i].x, (float)tabs[i].y);
            std::memcpy(h.data() + off_tabs32 + i * sizeof(float2), &v, sizeof(v));
        }
        if (!ints.empty()) std::memcpy(h.data() + off_ints, ints.data(), ints.size() * sizeof(int32_t));
        if (!dbls.empty()) std::memcpy(h.data() + off_dbls, dbls.data(), dbls.size() * sizeof(double));
        FGB_CUDA(cudaMemcpy(blob.p, h.data(), o, cudaMemcpyHostToDevice));
        return FGB_OK;
    }
    const T* d_wrow() const { return (const T*)((char*)blob.p + off_wrow); }
    const C* d_wcol() const { return (const C*)((char*)blob.p + off_wcol); }
    const ColJob<T>* d_cjobs() const { return (const ColJob<T>*)((char*)blob.p + off_cjobs); }
    const BankUJob* d_bjobs() const { return (const BankUJob*)((char*)blob.p + off_bjobs); }
    const IirJob<T>* d_ijobs() const { return (const IirJob<T>*)((char*)blob.p + off_ijobs); }
    const double2* d_tabs() const { return (const double2*)((char*)blob.p + off_tabs); }
    const float2* d_tabs32() const { return (const float2*)((char*)blob.p + off_tabs32); }
    const int32_t* d_ints() const { return (const int32_t*)((char*)blob.p + off_ints); }
    const double* d_dbls() const { return (const double*)((char*)blob.p + off_dbls); }
};

// ---------------------------------------------------------------------------
// builders
// ---------------------------------------------------------------------------
template <typename T> struct Builder {
    using C = cx_t<T>;
    Plan<T>& p;
    int lane = 0;  // lane stamped on every step this builder emits
    explicit Builder(Plan<T>& pl) : p(pl) {}
    void push(Step<T>& st) {
        st.lane = lane;
        p.steps.push_back(st);
    }

    // Row group over symmetric taps w[0..2h] for nd jobs with frequencies
    // f_k and sign s: J_k = phase_k sum_t w[t] e^{-i s f_k t} f[x+t].
    void row_group(const std::vector<double>& w, int h, const std::vector<double>& freq, double sgn,
                   const std::vector<cd>& phase, const std::vector<int64_t>& dst_off, Ref src, Ref dst, int H, int W,
                   double sflops) {
        const int nd = (int)freq.size();
        const int hp = row_sym_pad<T>(h);
        const int ndp = (nd + 1) & ~1;
        Step<T> st;
        st.kind = ST_ROW;
        st.name = "row_fir";
        st.flops = nd * (2.0 * sflops + 8.0) * H * W;
        st.bytes = (double)H * W * sizeof(T) + (double)nd * H * W * sizeof(C);
        st.H = H;
        st.W = W;
        st.src = src;
        st.dst = dst;
        st.hp = hp;
        st.rg.wofs = (int32_t)p.wrow.size();
        st.rg.nd = nd;
        st.rg.has_phase = 0;
        // theta = pi/2 (last direct of a Gabor group): the phase step omega cos(theta) ~ 1e-17 leaves
        // Im J <= 1e-12 |J|, so the fp32 kernel accumulates Re J only (the column pass reads Re J, realj)
        st.rg.last_real = sizeof(T) == 4 && std::fabs(freq[nd - 1]) * (W + 2.0 * (h + 1)) < 1e-12 &&
                          phase[nd - 1] == cd(1.0, 0.0) && !knobs().no_realj;
        for (int k = 0; k < nd; ++k) {
            st.rg.dst_off[k] = dst_off[k];
            st.rg.phase_re[k] = (T)phase[k].real();
            st.rg.phase_im[k] = (T)phase[k].imag();
            if (phase[k] != cd(1.0, 0.0)) st.rg.has_phase = 1;
        }
        for (int t = 0; t <= hp; ++t) {
            for (int k = 0; k < ndp; ++k) {
                double kr = 0.0, ki = 0.0;
                if (k < nd && t <= h) {
                    const double wt = w[h + t];
                    kr = wt * std::cos(freq[k] * t);
                    ki = -sgn * wt * std::sin(freq[k] * t);
                }
                p.wrow.push_back((T)kr);
                p.wrow.push_back((T)ki);
            }
        }
        push(st);
    }

    // Column job with taps t0..t0+nt-1: ka = w cos(f t), kb = w sin(f t).
    int col_weights(const std::vector<double>& w, int t0, double f) {
        const int off = (int)p.wcol.size();
        for (size_t q = 0; q < w.size(); ++q) {
            const double t = (double)(t0 + (int)q);
            p.wcol.push_back(mk<T>((T)(w[q] * std::cos(f * t)), (T)(w[q] * std::sin(f * t))));
        }
        return off;
    }

    struct Out {
        int64_t dst_off;
        int base;  // 0 X, 1 Y
        int conj;
        cd phase;
    };
    ColJob<T> col_job(int64_t src_off, int wofs, const std::vector<Out>& outs, int has_b = 1) {
        ColJob<T> j{};
        j.src_off = src_off;
        j.wofs = wofs;
        j.has_b = has_b;
        j.nout = (int)outs.size();
        j.mode = 0;
        bool unit_phase = true;
        for (const auto& o : outs) unit_phase = unit_phase && o.phase == cd(1.0, 0.0);
        if (unit_phase && outs.size() == 1 && outs[0].base == 0 && !outs[0].conj) j.mode = 1;
        if (unit_phase && outs.size() == 2 && outs[0].base == 0 && !outs[0].conj && outs[1].base == 1 && outs[1].conj)
            j.mode = 2;
        for (size_t o = 0; o < outs.size(); ++o) {
            j.dst_off[o] = outs[o].dst_off;
            j.base[o] = (int8_t)outs[o].base;
            j.conj[o] = (int8_t)outs[o].conj;
            j.phase_re[o] = (T)outs[o].phase.real();
            j.phase_im[o] = (T)outs[o].phase.imag();
        }
        return j;
    }
    void col_step(const std::vector<ColJob<T>>& jobs, Ref src, Ref dst, int H, int W, int t0, int nt, int zero_bnd,
                  int has_b, double sflops = 0.0, int counted = -1, bool real_in = false) {
        if (jobs.empty()) return;
        Step<T> st;
        st.kind = ST_COL;
        st.name = "col_fir";
        int nout = 0;
        for (const auto& j : jobs) nout += j.nout;
        if (counted < 0) counted = nout;
        st.flops = counted * (2.0 * sflops + (real_in ? 8.0 : 12.0)) * H * W;
        st.bytes = ((double)nout + jobs.size()) * H * W * sizeof(C);
        st.H = H;
        st.W = W;
        st.src = src;
        st.dst = dst;
        st.job0 = (int)p.cjobs.size();
        st.njobs = (int)jobs.size();
        st.t0 = t0;
        st.nt = nt;
        st.zero_bnd = zero_bnd;
        st.has_b = has_b;
        for (const auto& j : jobs)
            for (int q = 0; q < nt; ++q) st.pw.push_back(p.wcol[j.wofs + q]);
        p.cjobs.insert(p.cjobs.end(), jobs.begin(), jobs.end());
        push(st);
    }
    int64_t table(double f, int lo, int n) {
        const int64_t off = (int64_t)p.tabs.size();
        for (int i = 0; i < n; ++i) {
            const double x = (double)(lo + i);
            p.tabs.push_back(make_double2(std::cos(f * x), std::sin(f * x)));
        }
        return off;
    }
    // H = samples per line (unpadded), W = number of lines.  row_mode: lines
    // are image rows read / written in place (source real when real_in).
    void iir_step(const std::vector<IirJob<T>>& jobs_in, Ref src, Ref dst, int H, int W, int P, const IirCoef& c,
                  int64_t scratch_off, int counted = -1, bool real_in = false, bool row_mode = false) {
        if (jobs_in.empty()) return;
        // one modulation pair per kernel job: a two-pair job (Gabor theta and
        // pi - theta, SDFT bin and mirror) becomes two jobs sharing the source
        std::vector<IirJob<T>> jobs;
        for (const auto& j : jobs_in)
            for (int pr = 0; pr < 2; ++pr) {
                if (!((j.need >> pr) & 1)) continue;
                IirJob<T> q = j;
                q.nout = 0;
                q.need = 1 << pr;
                for (int o = 0; o < j.nout; ++o)
                    if (j.pair[o] == pr) {
                        q.dst_off[q.nout] = j.dst_off[o];
                        q.pair[q.nout] = (int8_t)pr;
                        q.conj[q.nout] = j.conj[o];
                        q.nout++;
                    }
                if (q.nout > 0) jobs.push_back(q);
            }
        Step<T> st;
        st.kind = ST_IIR;
        st.name = "iir";
        int nout = 0;
        for (const auto& j : jobs) nout += j.nout;
        if (counted < 0) counted = nout;
        st.flops = counted * (2.0 * 12.0 + (real_in ? 8.0 : 12.0)) * H * W;
        st.bytes = ((double)nout + jobs.size()) * H * W * sizeof(C);
        st.H = H;
        st.W = W;
        st.src = src;
        st.dst = dst;
        st.job0 = (int)p.ijobs.size();
        st.njobs = (int)jobs.size();
        st.P = P;
        st.coef = c;
        st.scratch_off = scratch_off;
        st.iir_row = row_mode ? 1 : 0;
        st.iir_real = real_in ? 1 : 0;
        // segment-parallel recursion: enough (column, job, segment) threads to fill the GPU
        const int L = H + 2 * P;
        const double threads = (double)W * jobs.size();
        static const double iir_threads = std::getenv("FGB_IIR_THREADS") ? std::atof(std::getenv("FGB_IIR_THREADS")) : 12288.0;
        int nseg = (int)std::ceil(148.0 * iir_threads / std::max(1.0, threads));
        nseg = std::max(1, std::min(nseg, std::max(1, L / 32)));  // segments >= 32 samples (measured: 24 / 16 / 12 slower)
        nseg = std::min(nseg, 128);
        // whole CTAs: the IIR kernels put 4 segments of 32 lines in a CTA, so a
        // segment count that is not a multiple of 4 leaves threads idle
        // (config 4: 5 segments 8.95 ms, 4 segments 8.30 ms per step)
        nseg = (nseg + 3) / 4 * 4;
        if (nseg > L / 8 && L / 8 >= 4) nseg = (L / 8) / 4 * 4;  // keep segments >= 8 samples
        int seglen = (L + nseg - 1) / nseg;
        nseg = (L + seglen - 1) / seglen;
        if (sizeof(T) == 4 && iir32_enabled()) {  // iir32.cu: fixed register-window segments
            seglen = kIir32M;
            nseg = (L + seglen - 1) / seglen;
        }
        st.nseg = nseg;
        st.seglen = seglen;
        // companion matrix A, g_m = first row of A^(m+1), A^seglen, A^last
        const double A[9] = {-c.a1, -c.a2, -c.a3, 1, 0, 0, 0, 1, 0};
        double Pm[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};  // A^0
        auto mul = [](const double* X, const double* Y, double* Z) {
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) Z[3 * i + j] = X[3 * i] * Y[j] + X[3 * i + 1] * Y[3 + j] + X[3 * i + 2] * Y[6 + j];
        };
        st.g_off = (int64_t)p.dbls.size();
        const int last_len = L - (nseg - 1) * seglen;
        for (int m = 1; m <= seglen; ++m) {
            double Q[9];
            mul(A, Pm, Q);
            std::memcpy(Pm, Q, sizeof(Q));  // Pm = A^m
            p.dbls.push_back(Pm[0]);
            p.dbls.push_back(Pm[1]);
            p.dbls.push_back(Pm[2]);
            if (m == last_len) std::memcpy(st.Alast, Pm, sizeof(Pm));
            if (m == seglen) std::memcpy(st.Aseg, Pm, sizeof(Pm));
        }
        p.ijobs.insert(p.ijobs.end(), jobs.begin(), jobs.end());
        push(st);
    }
    void tr(int kind, Ref src, Ref dst, int H, int W) {
        Step<T> st;
        st.kind = kind;
        st.name = "transpose";
        st.bytes = 2.0 * H * W * (kind == ST_TR_RR ? sizeof(T) : sizeof(C));
        st.H = H;
        st.W = W;
        st.src = src;
        st.dst = dst;
        push(st);
    }
};

static Ref R(int sel, int64_t off) {
    Ref r;
    r.sel = sel;
    r.off = off;
    return r;
}

// ---------------------------------------------------------------------------
// descriptor validation
// ---------------------------------------------------------------------------
static int32_t check_image(const fgb_image& im, bool complex_in = false) {
    if (im.height < 1 || im.width < 1) return fail(FGB_EINVAL, "image dimensions must be at least 1x1");
    if (im.dtype != FGB_F32 && im.dtype != FGB_F64) return fail(FGB_EINVAL, "dtype must be FGB_F32 or FGB_F64");
    if (im.batch < 1) return fail(FGB_EINVAL, "batch must be >= 1");
    if (im.pitch < im.width) return fail(FGB_EINVAL, "pitch must be >= width");
    if (complex_in && im.pitch != im.width) return fail(FGB_EINVAL, "complex inputs must be dense (pitch == width)");
    if (im.batch > 1 && im.batch_stride < (int64_t)im.height * im.pitch)
        return fail(FGB_EINVAL, "batch_stride must be >= height*pitch");
    return FGB_OK;
}

static int32_t check_smoother(const fgb_smoother& k, double sigma) {
    if (k.kind == FGB_SMOOTH_FIR) {
        if (k.radius < 3) return fail(FGB_EINVAL, "truncation radius must be at least 3 sigma");
        return FGB_OK;
    }
    if (k.kind == FGB_SMOOTH_IIR) {
        double c[4];
        return iir_coeffs(sigma, c);
    }
    if (k.kind == FGB_SMOOTH_BOX) {
        if (k.box_half < 0) return fail(FGB_EINVAL, "box half-width must be non-negative");
        return FGB_OK;
    }
    return fail(FGB_EUNSUPPORTED, "unknown smoother kind");
}

static double norm_theta(double th) {
    // Python's float % (sign of the divisor)
    double r = std::fmod(th, M_PI);
    if (r != 0.0 && (r < 0) != (M_PI < 0)) r += M_PI;
    return r;
}

// ===========================================================================
// Gabor plans
// ===========================================================================
struct DirectJob {
    double wc, ws;        // omega cos(theta), omega sin(theta)
    int64_t out_direct;   // entry slot (complex elems offset) or -1
    int64_t out_mirror;   // mirrored slot or -1
};

// Fused row+column kernel (J kept in shared memory) for half-widths up to
// 6 and <= 5 direct orientations per launch (balanced groups): config 2's
// sigma = 2 frequency 30 us instead of 42 us for the two launches (step
// +4.5%); at h = 12 the halo and shared-memory footprint make it a wash
// (measured).  FGB_FUSED_BANK=<max h> overrides (0 disables).
static bool fused_bank_used(int h, int nj, int H, int W) {
    static const int fused_max_h = std::getenv("FGB_FUSED_BANK") ? std::atoi(std::getenv("FGB_FUSED_BANK")) : 6;
    const int ng = (nj + 4) / 5;
    return h <= fused_max_h && (int64_t)H * W >= 4096 && bank_fused_ok(h, (nj + ng - 1) / ng);
}

// Tensor-core column pass (col_umma.cu) for an fp32 FIR bank frequency of half-width h
// (FGB_COL_FFMA=1 keeps the FFMA column kernel; FGB_UMMA_MIN_H sets the smallest h).
static bool rowu_used(int h, int W) {
    static const bool off = std::getenv("FGB_ROW_FFMA") != nullptr;
    return !off && row_umma_supported(h, W);
}
static bool umma_freq_used(int h, int nj, int H, int W) {
    static const bool off = std::getenv("FGB_COL_FFMA") != nullptr;
    static const int min_h = std::getenv("FGB_UMMA_MIN_H") ? std::atoi(std::getenv("FGB_UMMA_MIN_H")) : 7;
    return !off && h >= min_h && H >= 16 && col_umma_supported(h, W) && !fused_bank_used(h, nj, H, W);
}

// Row + column passes of one frequency in one tensor-core kernel, J in shared memory
// (bank_umma.cu; h <= 48).  Where the plan gives it enough tiles per SM it also takes the small
// half-widths of the FFMA fused kernel (config 5 sigma = 2: one 2.3 ms launch instead of two 1.5 ms
// ones, step +2.3 %).  FGB_BANK_UMMA=0 keeps the separate passes.
static bool banku_used(int h, int nj, int H, int W) {
    static const bool off = std::getenv("FGB_BANK_UMMA") && std::atoi(std::getenv("FGB_BANK_UMMA")) == 0;
    static const bool coloff = std::getenv("FGB_COL_FFMA") != nullptr;
    (void)nj;
    return !off && !coloff && H >= 16 && bank_umma_supported(h, W);
}

// One frequency worth of Gabor work: row stage for `jobs`, column stage with
// direct / mirrored outputs.  J planes live in ws at [ws_j0 + j*H*W].
template <typename T>
static int32_t build_gabor_freq(Builder<T>& b, const fgb_smoother& sm, double sigma, const std::vector<DirectJob>& jobs,
                                int H, int W, int64_t ws_j0, int64_t ws_aux, Ref img, Ref out, bool row_only,
                                bool col_only, int64_t* ws_need, int64_t jslot = -1) {
    const int64_t HW = (int64_t)H * W;
    if (jslot < 0) jslot = HW;  // complex elements per J slot (larger for split-fp16 padded slots)
    const int nj = (int)jobs.size();
    if (nj == 0) return FGB_OK;
    int64_t need = ws_j0 + (row_only || col_only ? 0 : (int64_t)nj * jslot);
    if (sm.kind == FGB_SMOOTH_FIR || sm.kind == FGB_SMOOTH_BOX) {
        std::vector<double> w;
        int h = 0, t0 = 0;
        const bool box = sm.kind == FGB_SMOOTH_BOX;
        if (box) {
            h = sm.box_half;
            w.assign(2 * h + 1, 1.0);
        } else {
            w = sampled_gaussian(sigma, sm.radius, &h);
        }
        t0 = -h;
        const int nt = 2 * h + 1;
        // ---- fused small-sigma path: J stays in shared memory ----
        if constexpr (std::is_same<T, float>::value) {
            // More than 5 directs (config 5: 9 per frequency) run as balanced groups of <= 5, one
            // fused launch each: config 5's sigma = 2 frequency 2.5 ms instead of 3.4 ms for the
            // row + column launches (profiles/r02/unit_costs_c5.json).
            const int ng = (nj + 4) / 5;
            if (!box && !row_only && !col_only && fused_bank_used(h, nj, H, W) && !b.p.banku_h.count(h)) {
                for (int gi = 0; gi < ng; ++gi) {
                    const int g0 = gi * nj / ng, g1 = (gi + 1) * nj / ng, gn = g1 - g0;
                    Step<T> st;
                    st.kind = ST_BANKF;
                    st.name = "bank_fused";
                    st.H = H;
                    st.W = W;
                    st.src = img;
                    st.dst = out;
                    st.h = h;
                    st.nheads = gn;  // nd
                    const int ndp = (gn + 1) & ~1;
                    const int hp = bank_fused_pad(h);
                    const int ntp = bank_fused_pad(nt);
                    for (int t = 0; t <= hp; ++t)
                        for (int k = 0; k < ndp; ++k) {
                            double kr = 0.0, ki = 0.0;
                            if (k < gn && t <= h) {
                                kr = w[h + t] * std::cos(jobs[g0 + k].wc * t);
                                ki = -w[h + t] * std::sin(jobs[g0 + k].wc * t);
                            }
                            st.bf_w.push_back((float)kr);
                            st.bf_w.push_back((float)ki);
                        }
                    st.bf_colw_off = (int)st.bf_w.size();
                    int counted = 0;
                    for (int k = 0; k < gn; ++k) {
                        const DirectJob& jb = jobs[g0 + k];
                        for (int q = 0; q < ntp; ++q) {
                            double ka = 0.0, kb = 0.0;
                            if (q < nt) {
                                const double t = (double)(q - h);
                                ka = w[q] * std::cos(jb.ws * t);
                                kb = w[q] * std::sin(jb.ws * t);
                            }
                            st.bf_w.push_back((float)ka);
                            st.bf_w.push_back((float)kb);
                        }
                        BankFusedOut o;
                        o.direct = jb.out_direct;
                        o.mirror = jb.out_mirror;
                        st.bf_out.push_back(o);
                        counted += 1 + (jb.out_mirror >= 0 ? 1 : 0);
                    }
                    const double sfl = 4.0 * h + 1;
                    st.flops = ((double)gn * (2.0 * sfl + 8.0) + (double)counted * (2.0 * sfl + 12.0)) * H * W;
                    st.bytes = (double)H * W * sizeof(T) + (double)counted * H * W * sizeof(cx_t<T>);
                    b.push(st);
                }
                *ws_need = std::max(*ws_need, need - (int64_t)nj * jslot);
                return FGB_OK;
            }
        }
        // row + column passes in one tensor-core kernel (no J planes)
        if constexpr (std::is_same<T, float>::value) {
            if (!box && !row_only && !col_only && b.p.banku_h.count(h) && b.p.xbuf >= 32) {
                Step<T> st;
                st.kind = ST_BANKU;
                st.name = "bank_umma";
                st.H = H;
                st.W = W;
                st.h = h;
                st.src = img;
                st.dst = out;
                st.job0 = (int)b.p.bjobs.size();
                st.njobs = nj;
                int counted = 0;
                for (int j = 0; j < nj; ++j) {
                    BankUJob q{};
                    q.rofs = (int32_t)b.p.wcol.size();
                    double mr = 0.0, mc = 0.0;
                    for (int t = 0; t <= h; ++t) {
                        const double kr = w[h + t] * std::cos(jobs[j].wc * t), ki = -w[h + t] * std::sin(jobs[j].wc * t);
                        b.p.wcol.push_back(mk<T>((T)kr, (T)ki));
                        mr = std::max(mr, std::max(std::fabs(kr), std::fabs(ki)));
                    }
                    q.cofs = b.col_weights(w, t0, jobs[j].ws);
                    for (int qq = 0; qq < nt; ++qq)
                        mc = std::max(mc, std::max(std::fabs((double)b.p.wcol[q.cofs + qq].x), std::fabs((double)b.p.wcol[q.cofs + qq].y)));
                    int ex = 0;
                    if (mr > 0.0) std::frexp(mr, &ex);
                    q.rexp = 10 - ex;
                    ex = 0;
                    if (mc > 0.0) std::frexp(mc, &ex);
                    q.cexp = 10 - ex;
                    q.dst_off[0] = jobs[j].out_direct;
                    q.dst_off[1] = jobs[j].out_mirror >= 0 ? jobs[j].out_mirror : jobs[j].out_direct;
                    q.nout = jobs[j].out_mirror >= 0 ? 2 : 1;
                    counted += q.nout;
                    b.p.bjobs.push_back(q);
                }
                const double sfl = 4.0 * h + 1;
                st.flops = ((double)nj * (2.0 * sfl + 8.0) + (double)counted * (2.0 * sfl + 12.0)) * H * W;
                st.bytes = (double)H * W * sizeof(T) + (double)counted * H * W * sizeof(cx_t<T>);
                b.push(st);
                *ws_need = std::max(*ws_need, need - (int64_t)nj * jslot);
                return FGB_OK;
            }
        }
        // tensor-core column pass: the plan's J slots are split-fp16 planes (Plan::jbuf > 0)
        const bool umma = std::is_same<T, float>::value && !box && !row_only && !col_only && b.p.jbuf > 0 &&
                          umma_freq_used(h, nj, H, W) && col_umma_jpad(h) <= b.p.jbuf;
        // ---- row stage ----
        if (!col_only && umma && b.p.xbuf > 0 && rowu_used(h, W) && row_umma_jpad(h) <= b.p.xbuf) {
            // tensor-core row pass: every direct of the frequency in one persistent launch
            Step<T> st;
            st.kind = ST_ROWU;
            st.name = "row_umma";
            const double sflops = 4.0 * h + 1;
            st.flops = nj * (2.0 * sflops + 8.0) * H * W;
            st.bytes = (double)H * W * sizeof(T) + (double)nj * H * W * sizeof(cx_t<T>);
            st.H = H;
            st.W = W;
            st.h = h;
            st.src = img;
            st.dst = R(SEL_WS, 0);
            st.job0 = (int)b.p.cjobs.size();
            st.njobs = nj;
            for (int j = 0; j < nj; ++j) {
                ColJob<T> q{};
                q.wofs = (int32_t)b.p.wcol.size();
                double mx = 0.0;
                for (int t = 0; t <= h; ++t) {
                    const double kr = w[h + t] * std::cos(jobs[j].wc * t), ki = -w[h + t] * std::sin(jobs[j].wc * t);
                    b.p.wcol.push_back(mk<T>((T)kr, (T)ki));
                    mx = std::max(mx, std::max(std::fabs(kr), std::fabs(ki)));
                }
                int ex = 0;
                if (mx > 0.0) std::frexp(mx, &ex);
                q.wexp = 10 - ex;
                q.nout = 1;
                q.dst_off[0] = ws_j0 + (int64_t)j * jslot;
                b.p.cjobs.push_back(q);
            }
            b.push(st);
        } else if (!col_only) {
            if (!box) {
                // row launches of <= gmax directs, balanced (9 -> 5 + 4 with gmax 5)
                static const int gmax = std::max(1, std::min(kMaxND, std::getenv("FGB_ROW_GROUP") ? std::atoi(std::getenv("FGB_ROW_GROUP")) : kMaxND));
                const int ngr = (nj + gmax - 1) / gmax;
                for (int gi = 0; gi < ngr; ++gi) {
                    const int g0 = gi * nj / ngr, g1 = (gi + 1) * nj / ngr;
                    std::vector<double> fr;
                    std::vector<cd> ph;
                    std::vector<int64_t> dst;
                    for (int j = g0; j < g1; ++j) {
                        fr.push_back(jobs[j].wc);
                        ph.push_back(cd(1.0, 0.0));
                        dst.push_back(row_only ? jobs[j].out_direct : ws_j0 + (int64_t)j * jslot);
                    }
                    b.row_group(w, h, fr, +1.0, ph, dst, img, row_only ? out : R(SEL_WS, 0), H, W, 4.0 * h + 1);
                    if (umma) b.p.steps.back().j16 = 1;
                }
            } else {
                // zero-padded box: transpose -> column kernel -> transpose back
                const int64_t t_img = ws_aux, t_j = ws_aux + HW;
                need = std::max(need, t_j + (int64_t)nj * HW);
                b.tr(ST_TR_RC, img, R(SEL_WS, t_img), H, W);
                std::vector<ColJob<T>> cj;
                for (int j = 0; j < nj; ++j) {
                    const int wo = b.col_weights(w, t0, jobs[j].wc);
                    cj.push_back(b.col_job(0, wo, {{t_j + (int64_t)j * HW, 0, 0, cd(1, 0)}}));
                }
                b.col_step(cj, R(SEL_WS, t_img), R(SEL_WS, 0), W, H, t0, nt, 1, 1, 2.0 * h, nj, true);
                for (int j = 0; j < nj; ++j)
                    b.tr(ST_TR_CC, R(SEL_WS, t_j + (int64_t)j * HW),
                         row_only ? R(out.sel, jobs[j].out_direct) : R(SEL_WS, ws_j0 + (int64_t)j * jslot), W, H);
            }
        }
        // ---- column stage ----
        if (!row_only) {
            std::vector<ColJob<T>> cj_b, cj_nob;
            for (int j = 0; j < nj; ++j) {
                const int wo = b.col_weights(w, t0, jobs[j].ws);
                std::vector<typename Builder<T>::Out> outs;
                if (jobs[j].out_direct >= 0) outs.push_back({jobs[j].out_direct, 0, 0, cd(1, 0)});
                if (jobs[j].out_mirror >= 0) outs.push_back({jobs[j].out_mirror, 1, 1, cd(1, 0)});
                ColJob<T> job = b.col_job(col_only ? 0 : ws_j0 + (int64_t)j * jslot, wo, outs, jobs[j].ws != 0.0);
                if (umma) {
                    // taps scaled by 2^wexp so |scaled| < 2^10 (fp16 hi / lo split without underflow)
                    double mx = 0.0;
                    for (int q = 0; q < nt; ++q)
                        mx = std::max(mx, std::max(std::fabs((double)b.p.wcol[wo + q].x), std::fabs((double)b.p.wcol[wo + q].y)));
                    int ex = 0;
                    if (mx > 0.0) std::frexp(mx, &ex);
                    job.wexp = 10 - ex;
                }
                // theta = pi/2: the row stage's phase step omega cos(theta) ~ 1e-17 leaves Im J at
                // ~1e-12 of |J| or less, so the fp32 column kernel reads Re J only (half the FMAs)
                if (sizeof(T) == 4 && !col_only && !box && job.mode == 1 && job.has_b &&
                    std::fabs(jobs[j].wc) * (W + 2.0 * (h + 1)) < 1e-12 && !knobs().no_realj)
                    job.realj = 1;
                // theta = 0 (ws = 0) jobs need A only (half the work): they share the
                // launch (per-CTA branch) and go last so heavy CTAs start first
                if (jobs[j].ws == 0.0) cj_nob.push_back(job);
                else cj_b.push_back(job);
            }
            const Ref src = col_only ? img : R(SEL_WS, 0);
            const double sfl = box ? 2.0 * h : 4.0 * h + 1;
            cj_b.insert(cj_b.end(), cj_nob.begin(), cj_nob.end());
            b.col_step(cj_b, src, out, H, W, t0, nt, box ? 1 : 0, 1, sfl);
            if (umma) {
                Step<T>& cs = b.p.steps.back();
                cs.kind = ST_COLU;
                cs.name = "col_umma";
                cs.h = h;
            }
        }
    } else {
        // ---- RecursiveIIR ----
        double cf[4];
        FGB_TRY(iir_coeffs(sigma, cf));
        IirCoef c{cf[0], cf[1], cf[2], cf[3]};
        const int P = pad_radius(sm, sigma);
        int64_t scratch = 0;  // T elements, region after all complex regions (set by caller via ws_need)
        if (!col_only) {
            std::vector<IirJob<T>> ij;
            for (int j = 0; j < nj; ++j) {
                IirJob<T> q{};
                q.src_off = 0;
                q.tabm_off = b.table(jobs[j].wc, -P, W + 2 * P);
                q.tabr_off = q.tabm_off + P;
                q.dst_off[0] = row_only ? jobs[j].out_direct : ws_j0 + (int64_t)j * jslot;
                q.pair[0] = 0;
                q.conj[0] = 0;
                q.nout = 1;
                q.need = 1;
                q.sdft = 0;
                ij.push_back(q);
            }
            // lines = image rows (H of them), W samples each, straight from the image
            b.iir_step(ij, img, row_only ? out : R(SEL_WS, 0), W, H, P, c, scratch, -1, true, true);
        }
        if (!row_only) {
            std::vector<IirJob<T>> ij;
            for (int j = 0; j < nj; ++j) {
                IirJob<T> q{};
                q.src_off = col_only ? 0 : ws_j0 + (int64_t)j * jslot;
                q.tabm_off = b.table(jobs[j].ws, -P, H + 2 * P);
                q.tabr_off = q.tabm_off + P;
                q.nout = 0;
                q.need = 0;
                if (jobs[j].out_direct >= 0) {
                    q.dst_off[q.nout] = jobs[j].out_direct;
                    q.pair[q.nout] = 0;
                    q.conj[q.nout] = 0;
                    q.nout++;
                    q.need |= 1;
                }
                if (jobs[j].out_mirror >= 0) {
                    q.dst_off[q.nout] = jobs[j].out_mirror;
                    q.pair[q.nout] = 1;
                    q.conj[q.nout] = 0;
                    q.nout++;
                    q.need |= 2;
                }
                q.sdft = 0;
                ij.push_back(q);
            }
            b.iir_step(ij, col_only ? img : R(SEL_WS, 0), out, H, W, P, c, scratch);
        }
    }
    *ws_need = std::max(*ws_need, need);
    return FGB_OK;
}

// IIR scratch need (T elements per image) for a plan: max over IIR steps.
template <typename T> static int64_t iir_scratch_need(const Plan<T>& p) {
    int64_t m = 0;
    for (const auto& s : p.steps)
        if (s.kind == ST_IIR) m = std::max<int64_t>(m, (int64_t)iir_scratch_elems<T>(s.H, s.W, s.P, s.njobs, 1));
    return (m + 63) / 64 * 64;  // lane / image bases stay 256-byte aligned (16-byte vector paths)
}
template <typename T> static int64_t iir_state_need(const Plan<T>& p) {
    int64_t m = 0;
    for (const auto& s : p.steps)
        if (s.kind == ST_IIR) m = std::max<int64_t>(m, (int64_t)iir_state_doubles(s.W, s.nseg, s.njobs, 1));
    return (m + 31) / 32 * 32;  // per-lane state bases 256-byte aligned (iir32 carry_io's 16-byte copies)
}

static int64_t ws_budget_bytes() {
    const char* e = std::getenv("FGB_WS_BUDGET_MB");
    const int64_t mb = e ? std::atoll(e) : 2048;  // 2 GB of 180: batches of up to 16 1024² images per chunk (config 3: +5%)
    return std::max<int64_t>(mb, 1) << 20;
}

template <typename T> static void finish_chunking(Plan<T>& p, int batch) {
    p.scratch_img_t = iir_scratch_need(p) * p.nlanes;
    p.state_img_d = iir_state_need(p) * p.nlanes;
    const int64_t per = p.ws_img_c * (int64_t)sizeof(cx_t<T>) + p.scratch_img_t * (int64_t)sizeof(T) +
                        p.state_img_d * (int64_t)sizeof(double);
    int64_t c = per > 0 ? ws_budget_bytes() / per : batch;
    p.chunk = (int)std::max<int64_t>(1, std::min<int64_t>(c, batch));
}

template <typename T>
static int32_t build_bank(Plan<T>& p, const fgb_bank_desc& d) {
    Builder<T> b(p);
    const int H = d.img.height, W = d.img.width, N = d.orientations;
    const int64_t HW = (int64_t)H * W;
    const int nh = N / 2;
    p.H = H;
    p.W = W;
    // work units / output slots
    std::vector<std::vector<DirectJob>> per_f(d.n_freq);
    int64_t slot = 0;
    if (d.units) {
        for (int u = 0; u < d.n_units; ++u) {
            const int unit = d.units[u];
            const int i = unit / (nh + 1), k = unit % (nh + 1);
            if (unit < 0 || i >= d.n_freq) return fail(FGB_EINVAL, "work unit out of range");
            const double th = norm_theta(k * M_PI / N);
            DirectJob j{d.omegas[i] * std::cos(th), d.omegas[i] * std::sin(th), slot * HW, -1};
            slot++;
            if (nh < N - k && N - k < N) j.out_mirror = (slot++) * HW;
            per_f[i].push_back(j);
        }
    } else {
        for (int i = 0; i < d.n_freq; ++i) {
            const int nk = d.reuse ? nh + 1 : N;
            for (int k = 0; k < nk; ++k) {
                const double th = norm_theta(k * M_PI / N);
                DirectJob j{d.omegas[i] * std::cos(th), d.omegas[i] * std::sin(th), ((int64_t)i * N + k) * HW, -1};
                if (d.reuse && nh < N - k && N - k < N) j.out_mirror = ((int64_t)i * N + (N - k)) * HW;
                per_f[i].push_back(j);
            }
        }
        slot = (int64_t)d.n_freq * N;
    }
    p.out_img_c = slot * HW;
    int64_t max_nj = 0;
    int nfreq_used = 0;
    for (auto& v : per_f) {
        max_nj = std::max<int64_t>(max_nj, (int64_t)v.size());
        nfreq_used += v.empty() ? 0 : 1;
    }
    // Frequencies are independent until their outputs: each runs its row -> column
    // chain on its own stream lane, so memory/latency-bound small-sigma launches
    // overlap the FP32-bound large-sigma ones.  Each lane owns its J (and aux) planes.
    const char* le = std::getenv("FGB_LANES");
    const int max_lanes = le ? std::max(1, std::atoi(le)) : 4;
    const int NL = std::max(1, std::min(max_lanes, nfreq_used));
    const bool plain_fir = d.smoother.kind == FGB_SMOOTH_FIR;
    // fp32 FIR banks: frequencies whose column pass runs on the tensor cores get split-fp16 J
    // slots with jbuf replicate rows above and below (one slot size for every lane)
    if (std::is_same<T, float>::value && plain_fir) {
        for (int i = 0; i < d.n_freq; ++i) {
            if (per_f[i].empty()) continue;
            const int h = std::max(1, (int)std::ceil(d.smoother.radius * d.sigmas[i]));
            // the persistent fused kernel needs >= 16 tiles (64 x 64 outputs of one direct) per SM
            // (config 2, 1024^2 x 5 directs: 9 per SM, 168 vs 195 G px*filters/s with the separate passes)
            const int64_t tiles = (int64_t)((H + 63) / 64) * ((W + 63) / 64) * (int64_t)per_f[i].size() *
                                  std::min(d.img.batch, 16);
            static const bool force = std::getenv("FGB_BANK_UMMA") && std::atoi(std::getenv("FGB_BANK_UMMA")) == 2;
            if (banku_used(h, (int)per_f[i].size(), H, W) && (force || tiles >= 16 * 148)) {
                p.banku = true;
                p.banku_h.insert(h);
                p.xbuf = std::max(p.xbuf, h > 32 ? 64 : 32);
            } else if (umma_freq_used(h, (int)per_f[i].size(), H, W)) {
                p.jbuf = std::max(p.jbuf, col_umma_jpad(h));
            }
        }
    }
    if (p.jbuf > 0) {
        for (int i = 0; i < d.n_freq; ++i) {
            if (per_f[i].empty()) continue;
            const int h = std::max(1, (int)std::ceil(d.smoother.radius * d.sigmas[i]));
            // the persistent row kernel needs enough 128 x 64 tiles per SM to amortise its pipeline fill
            // (config 2, 1024^2 x 5 directs: 4 tiles per SM, FFMA rows 21 us vs 32 us per launch)
            const int64_t tiles = (int64_t)((H + 127) / 128) * ((W + 63) / 64) * (int64_t)per_f[i].size() *
                                  std::min(d.img.batch, 16);
            static const bool force = std::getenv("FGB_ROW_UMMA") != nullptr;  // tests: small images too
            if (!p.banku_h.count(h) && umma_freq_used(h, (int)per_f[i].size(), H, W) &&
                rowu_used(h, W) && (force || tiles >= 16 * 148))
                p.xbuf = std::max(p.xbuf, row_umma_jpad(h));
        }
    }
    // split-fp16 J slot: per plane [strip of 64 columns][H + 2 jbuf rows][64 half2] (a column strip is contiguous)
    const int64_t jslot = p.jbuf > 0 ? (int64_t)(H + 2 * p.jbuf) * ((W + 63) / 64 * 64) : HW;
    p.hpw = jslot;
    const int64_t lane_stride = plain_fir ? max_nj * jslot : (2 * max_nj + 1) * HW;
    int64_t need = 0;
    int li = 0;
    // emit the heaviest frequency first: the longest lane chain starts first and the
    // small-sigma kernels fill its gaps (FGB_FREQ_ORDER=asc restores reference order)
    std::vector<int> order;
    for (int i = 0; i < d.n_freq; ++i) order.push_back(i);
    const char* fo = std::getenv("FGB_FREQ_ORDER");
    if (!(fo && std::string(fo) == "asc"))
        std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
            return d.sigmas[x] * (double)per_f[x].size() > d.sigmas[y] * (double)per_f[y].size();
        });
    for (int i : order) {
        if (per_f[i].empty()) continue;
        b.lane = li % NL;
        const int64_t j0 = b.lane * lane_stride;
        FGB_TRY(build_gabor_freq<T>(b, d.smoother, d.sigmas[i], per_f[i], H, W, j0, j0 + max_nj * HW, R(SEL_IMG, 0),
                                    R(SEL_OUT, 0), false, false, &need, plain_fir ? jslot : HW));
        ++li;
    }
    p.nlanes = NL;
    p.ws_img_c = need;  // lanes whose frequency runs fused (no J planes) reserve nothing
    finish_chunking(p, d.img.batch);
    return p.upload();
}

// mode: 0 full filter, 1 horizontal stage only, 2 vertical stage, 3 vertical conjugate
template <typename T>
static int32_t build_filter(Plan<T>& p, const fgb_filter_desc& d, int mode) {
    Builder<T> b(p);
    const int H = d.img.height, W = d.img.width;
    const int64_t HW = (int64_t)H * W;
    p.H = H;
    p.W = W;
    const double th = norm_theta(d.theta);
    DirectJob j{d.omega * std::cos(th), d.omega * std::sin(th), 0, -1};
    if (mode == 3) {
        j.out_direct = -1;
        j.out_mirror = 0;
    }
    p.out_img_c = HW;
    int64_t need = 0;
    const Ref in = (mode >= 2) ? R(SEL_IMGC, 0) : R(SEL_IMG, 0);
    FGB_TRY(build_gabor_freq<T>(b, d.smoother, d.sigma, {j}, H, W, 0, (mode == 0 ? HW : 0), in, R(SEL_OUT, 0),
                                mode == 1, mode >= 2, &need));
    p.ws_img_c = need;
    finish_chunking(p, d.img.batch);
    return p.upload();
}

// ===========================================================================
// SDFT plans
// ===========================================================================
static double sdft_sigma(const fgb_sdft_desc& d) {
    if (d.sigma > 0) return d.sigma;
    return (double)(std::min(d.mx, d.my) / 2) / 3.0;
}

// Window taps of one SDFT axis (sdft.py:68-72 + gaussian.py): Gaussian
// [-h, h] (replicate) or the asymmetric box [-(m/2), m-1-m/2] (zero padded).
static void sdft_axis_taps(const fgb_smoother& sm, double sigma, int m, std::vector<double>* w, int* t0) {
    if (sm.kind == FGB_SMOOTH_BOX) {
        const int lo = -(m / 2), hi = m - 1 - m / 2;
        w->assign(hi - lo + 1, 1.0);
        *t0 = lo;
    } else {
        int h;
        *w = sampled_gaussian(sigma, sm.radius, &h);
        *t0 = -h;
    }
}

// head list -> bin slots.  full layout: bin = u*my + v.  compact: per head u,
// rows (u, 0..my-1) then (mx-u, 0..my-1) if distinct.
struct BinMap {
    std::vector<int> heads;
    std::map<int, int64_t> row_slot;  // u -> first bin slot of row u
    int64_t nbins = 0;
};
static int32_t make_binmap(const fgb_sdft_desc& d, BinMap* bm) {
    const int mx = d.mx, my = d.my;
    if (!d.u_heads) {
        for (int u = 0; u <= mx / 2; ++u) bm->heads.push_back(u);
        for (int u = 0; u < mx; ++u) bm->row_slot[u] = (int64_t)u * my;
        bm->nbins = (int64_t)mx * my;
        return FGB_OK;
    }
    int64_t s = 0;
    for (int i = 0; i < d.n_heads; ++i) {
        const int u = d.u_heads[i];
        if (u < 0 || u > mx / 2) return fail(FGB_EINVAL, "SDFT pair head outside [0, mx/2]");
        if (bm->row_slot.count(u)) return fail(FGB_EINVAL, "duplicate SDFT pair head");
        bm->heads.push_back(u);
        bm->row_slot[u] = s;
        s += my;
        const int um = (mx - u) % mx;
        if (um != u) {
            bm->row_slot[um] = s;
            s += my;
        }
    }
    bm->nbins = s;
    return FGB_OK;
}

// Full SDFT on an image of H x W read from `img` (real).  The horizontal
// stage writes J_u into ws planes [0, nh); bins go to `out` at slot*HW.
template <typename T>
static int32_t build_sdft_core(Builder<T>& b, const fgb_sdft_desc& d, const BinMap& bm, int H, int W, Ref img,
                               Ref out, int64_t out_base, int64_t ws0, int64_t* ws_need) {
    const int mx = d.mx, my = d.my;
    const int64_t HW = (int64_t)H * W;
    const double sigma = sdft_sigma(d);
    const fgb_smoother& sm = d.smoother;
    const int cx = mx / 2, cy = my / 2;
    const double w0x = 2.0 * M_PI / mx, w0y = 2.0 * M_PI / my;
    const int nh = (int)bm.heads.size();
    int64_t need = (int64_t)nh * HW;  // J_u planes
    const int64_t aux = need;
    auto slot = [&](int u, int v) { return out_base + (bm.row_slot.at(u) + v) * HW; };

    if (sm.kind == FGB_SMOOTH_FIR && mx == my && ws0 == 0 && !knobs().sdft_unfused) {
        int h = 0;
        std::vector<double> w = sampled_gaussian(sigma, sm.radius, &h);
        if (sdft_fused_supported(mx, h, sizeof(T)) && out.sel == SEL_OUT) {
            Step<T> st;
            st.kind = ST_SDFTF;
            st.name = "sdft_fused";
            st.H = H;
            st.W = W;
            st.src = img;
            st.dst = out;
            st.M = mx;
            st.h = h;
            st.nheads = nh;
            st.w_off = (int64_t)b.p.wrow.size();
            for (double v : w) b.p.wrow.push_back((T)v);
            while (b.p.wrow.size() % 4) b.p.wrow.push_back((T)0);
            st.heads_off = (int64_t)b.p.ints.size();
            for (int u : bm.heads) b.p.ints.push_back(u);
            st.slots_off = (int64_t)b.p.ints.size();
            int counted = 0;
            for (int u : bm.heads) {
                const int um = (mx - u) % mx;
                b.p.ints.push_back((int32_t)(out_base / HW + bm.row_slot.at(u)));
                b.p.ints.push_back(um != u ? (int32_t)(out_base / HW + bm.row_slot.at(um)) : -1);
                counted += (um != u) ? 2 : 1;
            }
            const double T_ = 2.0 * h + 1;
            st.flops = ((double)nh * (4 * T_ + 6) + (double)counted * (my / 2 + 1) * (4 * T_ + 10)) * HW;
            st.bytes = (double)HW * sizeof(T) + (double)bm.nbins * HW * sizeof(cx_t<T>);
            b.p.steps.push_back(st);
            *ws_need = std::max(*ws_need, (int64_t)0);
            return FGB_OK;
        }
    }
    if (sm.kind == FGB_SMOOTH_FIR || sm.kind == FGB_SMOOTH_BOX) {
        std::vector<double> wx, wy;
        int t0x, t0y;
        sdft_axis_taps(sm, sigma, mx, &wx, &t0x);
        sdft_axis_taps(sm, sigma, my, &wy, &t0y);
        const bool box = sm.kind == FGB_SMOOTH_BOX;
        // ---- horizontal stage: J_u = sum_t w e^{i phi (c + t)} f[x+t] ----
        if (!box) {
            const int h = -t0x;
            for (int g0 = 0; g0 < nh; g0 += kMaxND) {
                const int g1 = std::min(nh, g0 + kMaxND);
                std::vector<double> fr;
                std::vector<cd> ph;
                std::vector<int64_t> dst;
                for (int i = g0; i < g1; ++i) {
                    const double phi = w0x * bm.heads[i];
                    fr.push_back(phi);
                    ph.push_back(cd(std::cos(phi * cx), std::sin(phi * cx)));
                    dst.push_back((int64_t)i * HW);
                }
                b.row_group(wx, h, fr, -1.0, ph, dst, img, R(SEL_WS, ws0 + 0), H, W, 4.0 * h + 1);
            }
        } else {
            need = std::max(need, aux + HW + (int64_t)nh * HW);
            b.tr(ST_TR_RC, img, R(SEL_WS, ws0 + aux), H, W);
            std::vector<ColJob<T>> cj;
            for (int i = 0; i < nh; ++i) {
                const double phi = w0x * bm.heads[i];
                const int wo = b.col_weights(wx, t0x, phi);
                cj.push_back(b.col_job(0, wo, {{aux + HW + (int64_t)i * HW, 1, 0, cd(std::cos(phi * cx), std::sin(phi * cx))}}));
            }
            b.col_step(cj, R(SEL_WS, ws0 + aux), R(SEL_WS, ws0 + 0), W, H, t0x, (int)wx.size(), 1, 1, (double)(wx.size() - 1), -1, true);
            for (int i = 0; i < nh; ++i) b.tr(ST_TR_CC, R(SEL_WS, ws0 + aux + HW + (int64_t)i * HW), R(SEL_WS, ws0 + (int64_t)i * HW), W, H);
        }
        // ---- vertical stage + conjugate fills ----
        std::vector<ColJob<T>> cj_b, cj_nob;
        int cnt_b = 0, cnt_nob = 0;
        for (int i = 0; i < nh; ++i) {
            const int u = bm.heads[i];
            const int um = (mx - u) % mx;
            for (int v = 0; v <= my / 2; ++v) {
                const double phi = w0y * v;
                const cd P(std::cos(phi * cy), std::sin(phi * cy));
                const int wo = b.col_weights(wy, t0y, phi);
                std::vector<typename Builder<T>::Out> outs;
                outs.push_back({slot(u, v), 1, 0, P});                    // bin(u,v) = P Y
                const bool mir = (um != u);
                const bool fill = (v != 0) && (2 * v != my);
                if (mir) outs.push_back({slot(um, v), 0, 1, P});          // bin(mx-u,v) = P conj X
                if (fill) outs.push_back({slot(um, my - v), 1, 1, std::conj(P)});  // conj(bin(u,v))
                if (mir && fill) outs.push_back({slot(u, my - v), 0, 0, std::conj(P)});  // conj(bin(mx-u,v))
                ColJob<T> job = b.col_job((int64_t)i * HW, wo, outs, phi != 0.0);
                cj_b.push_back(job);
                cnt_b += 1 + (mir ? 1 : 0);
            }
        }
        const double sfl = box ? (double)(wy.size() - 1) : 2.0 * wy.size() - 1;
        b.col_step(cj_b, R(SEL_WS, ws0 + 0), out, H, W, t0y, (int)wy.size(), box ? 1 : 0, 1, sfl, cnt_b);
        b.col_step(cj_nob, R(SEL_WS, ws0 + 0), out, H, W, t0y, (int)wy.size(), box ? 1 : 0, 0, sfl, cnt_nob);
    } else {
        double cf[4];
        FGB_TRY(iir_coeffs(sigma, cf));
        IirCoef c{cf[0], cf[1], cf[2], cf[3]};
        const int P = pad_radius(sm, sigma);
        std::vector<IirJob<T>> ij;
        for (int i = 0; i < nh; ++i) {
            const double phi = w0x * bm.heads[i];
            IirJob<T> q{};
            q.src_off = 0;
            q.tabm_off = b.table(phi, -P, W + 2 * P);
            q.tabr_off = b.table(phi, -cx, W);
            q.dst_off[0] = (int64_t)i * HW;
            q.pair[0] = 1;
            q.nout = 1;
            q.need = 2;
            q.sdft = 1;
            ij.push_back(q);
        }
        b.iir_step(ij, img, R(SEL_WS, ws0 + 0), W, H, P, c, 0, -1, true, true);
        std::vector<IirJob<T>> cj;
        int cnt = 0;
        for (int i = 0; i < nh; ++i) {
            const int u = bm.heads[i];
            const int um = (mx - u) % mx;
            for (int v = 0; v <= my / 2; ++v) {
                const double phi = w0y * v;
                IirJob<T> q{};
                q.src_off = (int64_t)i * HW;
                q.tabm_off = b.table(phi, -P, H + 2 * P);
                q.tabr_off = b.table(phi, -cy, H);
                q.sdft = 1;
                const bool mir = (um != u);
                const bool fill = (v != 0) && (2 * v != my);
                auto add = [&](int64_t dst, int pair, int conj) {
                    q.dst_off[q.nout] = dst;
                    q.pair[q.nout] = (int8_t)pair;
                    q.conj[q.nout] = (int8_t)conj;
                    q.nout++;
                    q.need |= (1 << pair);
                };
                add(slot(u, v), 1, 0);
                cnt += 1 + (mir ? 1 : 0);
                if (mir) add(slot(um, v), 0, 0);
                if (fill) add(slot(um, my - v), 1, 1);
                if (mir && fill) add(slot(u, my - v), 0, 1);
                cj.push_back(q);
            }
        }
        b.iir_step(cj, R(SEL_WS, ws0 + 0), out, H, W, P, c, 0, cnt);
    }
    *ws_need = std::max(*ws_need, ws0 + need);
    return FGB_OK;
}

template <typename T>
static int32_t build_sdft(Plan<T>& p, const fgb_sdft_desc& d) {
    Builder<T> b(p);
    const int H = d.img.height, W = d.img.width;
    const int64_t HW = (int64_t)H * W;
    p.H = H;
    p.W = W;
    BinMap bm;
    FGB_TRY(make_binmap(d, &bm));
    p.out_img_c = bm.nbins * HW;
    int64_t need = 0;
    if (d.my >= d.mx) {
        FGB_TRY(build_sdft_core<T>(b, d, bm, H, W, R(SEL_IMG, 0), R(SEL_OUT, 0), 0, 0, &need));
    } else {
        // sdft.py:185-195: transpose, swap extents, transpose bins back.
        if (d.u_heads) return fail(FGB_EINVAL, "pair-head sharding needs my >= mx");
        fgb_sdft_desc dt = d;
        std::swap(dt.mx, dt.my);
        BinMap bt;
        FGB_TRY(make_binmap(dt, &bt));
        // ws layout: [transposed image (real, as HW/2 complex)][bins' planes][core ws]
        const int64_t img_c = (HW + 1) / 2;
        const int64_t bins_off = img_c;
        const int64_t core_off = bins_off + bt.nbins * HW;
        b.tr(ST_TR_RR, R(SEL_IMG, 0), R(SEL_WSR, 0), H, W);
        // core on the transposed image (W rows x H cols), its ws after the bins
        int64_t core_need = 0;
        FGB_TRY(build_sdft_core<T>(b, dt, bt, W, H, R(SEL_WSR, 0), R(SEL_WS, bins_off), 0, core_off, &core_need));
        need = core_need;
        // bins'[v][u] (W x H planes) -> bins[u][v] (H x W)
        for (int u = 0; u < d.mx; ++u)
            for (int v = 0; v < d.my; ++v)
                b.tr(ST_TR_CC, R(SEL_WS, bins_off + ((int64_t)v * d.mx + u) * HW), R(SEL_OUT, ((int64_t)u * d.my + v) * HW), W, H);
    }
    p.ws_img_c = need;
    finish_chunking(p, d.img.batch);
    return p.upload();
}

// single bin / horizontal stage, direct (sdft.py:134-175): no reuse.
template <typename T>
static int32_t build_sdft_single(Plan<T>& p, const fgb_sdft_desc& d, int u, int v) {
    Builder<T> b(p);
    const int H = d.img.height, W = d.img.width;
    const int64_t HW = (int64_t)H * W;
    p.H = H;
    p.W = W;
    p.out_img_c = HW;
    const double sigma = sdft_sigma(d);
    const fgb_smoother& sm = d.smoother;
    const double phx = 2.0 * M_PI / d.mx * u;
    const int cx = d.mx / 2, cy = d.my / 2;
    const bool only_h = v < 0;
    int64_t need = only_h ? 0 : HW;
    const Ref jdst = only_h ? R(SEL_OUT, 0) : R(SEL_WS, 0);
    if (sm.kind == FGB_SMOOTH_FIR) {
        std::vector<double> w;
        int t0;
        sdft_axis_taps(sm, sigma, d.mx, &w, &t0);
        b.row_group(w, -t0, {phx}, -1.0, {cd(std::cos(phx * cx), std::sin(phx * cx))}, {0}, R(SEL_IMG, 0), jdst, H, W,
                    2.0 * w.size() - 1);
    } else if (sm.kind == FGB_SMOOTH_BOX) {
        std::vector<double> w;
        int t0;
        sdft_axis_taps(sm, sigma, d.mx, &w, &t0);
        const int64_t aux = need;
        need = aux + 2 * HW;
        b.tr(ST_TR_RC, R(SEL_IMG, 0), R(SEL_WS, aux), H, W);
        const int wo = b.col_weights(w, t0, phx);
        b.col_step({b.col_job(0, wo, {{aux + HW, 1, 0, cd(std::cos(phx * cx), std::sin(phx * cx))}})}, R(SEL_WS, aux),
                   R(SEL_WS, 0), W, H, t0, (int)w.size(), 1, 1);
        b.tr(ST_TR_CC, R(SEL_WS, aux + HW), jdst, W, H);
    } else {
        double cf[4];
        FGB_TRY(iir_coeffs(sigma, cf));
        IirCoef c{cf[0], cf[1], cf[2], cf[3]};
        const int P = pad_radius(sm, sigma);
        IirJob<T> q{};
        q.tabm_off = b.table(phx, -P, W + 2 * P);
        q.tabr_off = b.table(phx, -cx, W);
        q.dst_off[0] = jdst.off;
        q.pair[0] = 1;
        q.nout = 1;
        q.need = 2;
        q.sdft = 1;
        b.iir_step({q}, R(SEL_IMG, 0), R(jdst.sel, 0), W, H, P, c, 0, -1, true, true);
    }
    if (!only_h) {
        const double phy = 2.0 * M_PI / d.my * v;
        const cd Pp(std::cos(phy * cy), std::sin(phy * cy));
        if (sm.kind == FGB_SMOOTH_IIR) {
            double cf[4];
            FGB_TRY(iir_coeffs(sigma, cf));
            IirCoef c{cf[0], cf[1], cf[2], cf[3]};
            const int P = pad_radius(sm, sigma);
            IirJob<T> q{};
            q.tabm_off = b.table(phy, -P, H + 2 * P);
            q.tabr_off = b.table(phy, -cy, H);
            q.pair[0] = 1;
            q.nout = 1;
            q.need = 2;
            q.sdft = 1;
            b.iir_step({q}, R(SEL_WS, 0), R(SEL_OUT, 0), H, W, P, c, 0);
        } else {
            std::vector<double> w;
            int t0;
            sdft_axis_taps(sm, sigma, d.my, &w, &t0);
            const int wo = b.col_weights(w, t0, phy);
            b.col_step({b.col_job(0, wo, {{0, 1, 0, Pp}}, phy != 0.0)}, R(SEL_WS, 0), R(SEL_OUT, 0), H, W, t0, (int)w.size(),
                       sm.kind == FGB_SMOOTH_BOX ? 1 : 0, phy != 0.0);
        }
    }
    p.ws_img_c = need;
    finish_chunking(p, d.img.batch);
    return p.upload();
}

// ===========================================================================
// execution
// ===========================================================================
struct Ctx {
    std::vector<cudaStream_t> lanes;
    std::vector<cudaEvent_t> lane_ev;
    cudaEvent_t fork_ev = nullptr;
    ~Ctx() {
        if (copy_stream) cudaStreamDestroy(copy_stream);
        for (auto e : piece_ev) cudaEventDestroy(e);
        for (auto st : lanes) cudaStreamDestroy(st);
        for (auto e : lane_ev) cudaEventDestroy(e);
        if (fork_ev) cudaEventDestroy(fork_ev);
        if (ws_ev) cudaEventDestroy(ws_ev);
    }
    DevBuf ws;
    std::map<std::string, std::shared_ptr<PlanBase>> plans;
    DevBuf hin, hout;  // device staging of the *_host entry points
    cudaStream_t copy_stream = nullptr;    // D2H of finished pieces while later pieces compute
    std::vector<cudaEvent_t> piece_ev;
    DevBuf hpl, hflag; // planar f64 staging + non-finite flag of the *_host_planar entry points
    // The workspace is shared by every call on this device: each execute records ws_ev on its
    // stream when it has enqueued its last use, and a call on a different stream first waits
    // on it, so calls on distinct streams never overlap on the same J / state buffers.
    cudaEvent_t ws_ev = nullptr;
    cudaStream_t ws_stream = nullptr;
    bool ws_pending = false;
    std::map<std::string, std::unique_ptr<DevBuf>> line_taps;  // fgb_smooth_lines tap tables (immutable)
    DevBuf ser_scratch;                                         // fgb_ser_sums partials
    DevBuf maxbits;                                             // max|f| bits per image (split-fp16 J scale)
    DevBuf fprep;                                               // x-padded split-fp16 image planes (ST_ROWU)
    int sms = 0;                                                // SM count (persistent grids)
    DevBuf iir_cnt;                                             // iir32 arrival counters, zero between launches
    size_t iir_cnt_zeroed = 0;                                  // bytes of iir_cnt known to be zero
};
static int32_t ws_acquire(Ctx& cx, cudaStream_t s) {
    if (!cx.ws_ev) FGB_CUDA(cudaEventCreateWithFlags(&cx.ws_ev, cudaEventDisableTiming));
    if (cx.ws_pending && cx.ws_stream != s) FGB_CUDA(cudaStreamWaitEvent(s, cx.ws_ev, 0));
    return FGB_OK;
}
static int32_t ws_release(Ctx& cx, cudaStream_t s) {
    FGB_CUDA(cudaEventRecord(cx.ws_ev, s));
    cx.ws_stream = s;
    cx.ws_pending = true;
    return FGB_OK;
}
static std::mutex g_mu;
static std::map<int, std::unique_ptr<Ctx>> g_ctx;

// ---- live per-kernel profiling (CUDA events on the launching stream) ----
struct ProfRec {
    std::string name;
    cudaEvent_t e0, e1;
    double flops, bytes;
};
static bool g_prof = false;
static int64_t g_launches = 0;
static std::vector<ProfRec> g_prof_pending;
static std::vector<cudaEvent_t> g_event_pool;
static cudaEvent_t pool_event() {
    if (!g_event_pool.empty()) {
        cudaEvent_t e = g_event_pool.back();
        g_event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

static Ctx& ctx() {
    int dev = 0;
    cudaGetDevice(&dev);
    auto& c = g_ctx[dev];
    if (!c) c.reset(new Ctx());
    return *c;
}

// Device workspace a call of this plan needs (J planes, IIR scratch and
// segment states for one chunk of images); the library keeps it grow-only.
template <typename T> static int64_t plan_ws_bytes(const Plan<T>& p, int batch) {
    const int chunk = std::min(p.chunk, batch);
    const int64_t ws_img_bytes = p.ws_img_c * (int64_t)sizeof(cx_t<T>);
    const int64_t scr_bytes = p.scratch_img_t * (int64_t)sizeof(T);
    const int64_t stt_bytes = p.state_img_d * (int64_t)sizeof(double);
    return (ws_img_bytes * chunk + 255) / 256 * 256 + scr_bytes * chunk + stt_bytes * chunk + 512;
}

template <typename T>
static int32_t execute(Plan<T>& p, Ctx& cx, const fgb_image& im, const void* img, void* out, cudaStream_t s) {
    using C = cx_t<T>;
    const int batch = im.batch;
    const int chunk = std::min(p.chunk, batch);
    const int64_t ws_img_bytes = p.ws_img_c * (int64_t)sizeof(C);
    const int64_t scr_bytes = p.scratch_img_t * (int64_t)sizeof(T);
    FGB_TRY(cx.ws.ensure((size_t)plan_ws_bytes(p, batch)));
    C* ws = (C*)cx.ws.p;
    // region bases and per-lane strides are multiples of 256 bytes (iir_*_need round the per-lane needs)
    const int64_t scr0 = (ws_img_bytes * chunk + 255) / 256 * 256;
    T* scratch = (T*)((char*)cx.ws.p + scr0);
    const int64_t scratch_lane = p.scratch_img_t / std::max(1, p.nlanes) * chunk;
    double* states = (double*)((char*)cx.ws.p + scr0 + scr_bytes * chunk);
    const int64_t state_lane = p.state_img_d / std::max(1, p.nlanes) * chunk;
    // lane streams: lane 0 is the caller's stream; lanes >= 1 are library streams forked
    // from / joined into it with events, per image chunk
    // live per-kernel profiling serialises the lanes so each kernel's events time it alone
    const int nl = g_prof ? 1 : p.nlanes;
    std::vector<cudaStream_t> lane_s(p.nlanes, s);
    for (int l = 1; l < nl; ++l) {
        while ((int)cx.lanes.size() < l) {
            cudaStream_t ns;
            FGB_CUDA(cudaStreamCreateWithFlags(&ns, cudaStreamNonBlocking));
            cx.lanes.push_back(ns);
            cudaEvent_t e;
            FGB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            cx.lane_ev.push_back(e);
        }
        lane_s[l] = cx.lanes[l - 1];
    }
    if (!cx.fork_ev) FGB_CUDA(cudaEventCreateWithFlags(&cx.fork_ev, cudaEventDisableTiming));
    FGB_TRY(ws_acquire(cx, s));
    if (p.jbuf > 0 || p.xbuf > 0) {
        FGB_TRY(cx.maxbits.ensure(sizeof(unsigned) * (size_t)chunk));
        if (p.xbuf > 0) FGB_TRY(cx.fprep.ensure(row_umma_fprep_bytes(p.H, p.W, p.xbuf, chunk)));
        if (cx.sms == 0) {
            int dev = 0;
            FGB_CUDA(cudaGetDevice(&dev));
            FGB_CUDA(cudaDeviceGetAttribute(&cx.sms, cudaDevAttrMultiProcessorCount, dev));
        }
    }
    // iir32 arrival counters (shared like the workspace, so after ws_acquire): one int per
    // 32-line block, job and image of a chunk, per lane; zeroed once when (re)allocated
    size_t cnt_lane = 0;
    for (const auto& st : p.steps)
        if (st.kind == ST_IIR) cnt_lane = std::max(cnt_lane, (size_t)((st.W + 31) / 32) * st.njobs * chunk);
    int* cnt = nullptr;
    if (cnt_lane) {
        const size_t need = cnt_lane * std::max(1, p.nlanes) * sizeof(int);
        if (need > cx.iir_cnt_zeroed) {
            FGB_TRY(cx.iir_cnt.ensure(need));
            FGB_CUDA(cudaMemsetAsync(cx.iir_cnt.p, 0, cx.iir_cnt.n, s));
            cx.iir_cnt_zeroed = cx.iir_cnt.n;
        }
        cnt = (int*)cx.iir_cnt.p;
    }
    const int64_t img_bs = (batch > 1) ? im.batch_stride : (int64_t)im.height * im.pitch;
    for (int b0 = 0; b0 < batch; b0 += chunk) {
        const int nb = std::min(chunk, batch - b0);
        const T* imgb = (const T*)img + (size_t)b0 * img_bs;
        if constexpr (std::is_same<T, float>::value) {
            if (p.jbuf > 0 || p.xbuf > 0) {  // split-fp16 J scale per image, before the lanes fork
                ++g_launches;
                FGB_CUDA(launch_absmax(imgb, im.pitch, img_bs, p.H, p.W, nb, (unsigned*)cx.maxbits.p, cx.sms, s));
                if (p.xbuf > 0) {
                    ++g_launches;
                    FGB_CUDA(launch_row_umma_prep(imgb, im.pitch, img_bs, p.H, p.W, p.xbuf, nb,
                                                  (const unsigned*)cx.maxbits.p, cx.fprep.p, s));
                }
            }
        }
        if (nl > 1) {
            FGB_CUDA(cudaEventRecord(cx.fork_ev, s));
            for (int l = 1; l < nl; ++l) FGB_CUDA(cudaStreamWaitEvent(lane_s[l], cx.fork_ev, 0));
        }
        C* imgcb = (C*)img + (size_t)b0 * img_bs;  // complex inputs: strides in complex elements
        C* outb = (C*)out + (size_t)b0 * p.out_img_c;
        auto baseC = [&](const Ref& r) -> C* {
            switch (r.sel) {
                case SEL_IMGC: return imgcb + r.off;  // complex input (dense)
                case SEL_OUT: return outb + r.off;
                case SEL_WS: return ws + r.off;
                default: return nullptr;
            }
        };
        auto bsC = [&](const Ref& r) -> int64_t {
            switch (r.sel) {
                case SEL_IMGC: return img_bs;
                case SEL_OUT: return p.out_img_c;
                default: return p.ws_img_c;
            }
        };
        auto baseT = [&](const Ref& r, int64_t* pitch, int64_t* bs) -> const T* {
            if (r.sel == SEL_IMG) {
                *pitch = im.pitch;
                *bs = img_bs;
                return imgb + r.off;
            }
            // SEL_WSR: real plane inside ws (dense; the caller sets the row length)
            *pitch = 0;
            *bs = 2 * p.ws_img_c;
            return (const T*)ws + r.off;
        };
        const bool detail = knobs().prof_detail;
        int sidx = 0;
        for (const Step<T>& st : p.steps) {
            cudaStream_t s = lane_s[st.lane];  // shadows the caller's stream for this step
            ProfRec pr{detail ? std::string(st.name) + "." + std::to_string(sidx) : std::string(st.name), nullptr, nullptr,
                       st.flops * nb, st.bytes * nb};
            ++sidx;
            const NvtxRange nvtx_step(st.name);  // per-step NVTX range (no-op without an attached tool)
            if (g_prof) {
                pr.e0 = pool_event();
                pr.e1 = pool_event();
                cudaEventRecord(pr.e0, s);
            }
            // kernels per step: IIR = sum (with the carry scans), fin (fp32 parallel form; plus a
            // driver memset of the arrival counters, not counted) or fwd, scan, bwd, scan, out
            g_launches += st.kind == ST_IIR ? ((sizeof(T) == 4 && iir32_enabled()) ? 2 : 5) : 1;
            switch (st.kind) {
                case ST_ROW: {
                    RowArgs<T> a{};
                    int64_t pitch, bs;
                    a.img = baseT(st.src, &pitch, &bs);
                    a.pitch = (st.src.sel == SEL_WSR) ? st.W : pitch;
                    a.img_bstride = bs;
                    a.dst_base = baseC(st.dst);
                    a.out_bstride = bsC(st.dst);
                    a.weights = p.d_wrow();
                    a.H = st.H;
                    a.W = st.W;
                    a.hp = st.hp;
                    a.batch = nb;
                    a.j16 = st.j16;
                    a.jpad = p.jbuf;
                    a.j16_plane = p.hpw;
                    a.maxbits = (const unsigned*)cx.maxbits.p;
                    FGB_CUDA(launch_row_sym<T>(a, st.rg, knobs().row_smem_taps ? nullptr : p.wrow.data() + st.rg.wofs, s));
                    break;
                }
                case ST_BANKU: {
                    if constexpr (std::is_same<T, float>::value) {
                        BankUArgs a{};
                        a.jobs = p.d_bjobs() + st.job0;
                        a.weights = p.d_wcol();
                        a.dst_base = baseC(st.dst);
                        a.dst_bstride = bsC(st.dst);
                        a.maxbits = (const unsigned*)cx.maxbits.p;
                        a.H = st.H;
                        a.W = st.W;
                        a.h = st.h;
                        a.njobs = st.njobs;
                        a.batch = nb;
                        a.xbuf = p.xbuf;
                        a.dst_planes = (int64_t)nb * bsC(st.dst) / ((int64_t)st.H * st.W);
                        FGB_CUDA(launch_bank_umma(a, cx.fprep.p, cx.sms, s));
                    }
                    break;
                }
                case ST_ROWU: {
                    if constexpr (std::is_same<T, float>::value) {
                        RowUArgs a{};
                        a.jobs = p.d_cjobs() + st.job0;
                        a.weights = p.d_wcol();
                        a.dst_base = ws;
                        a.dst_bstride = p.ws_img_c;
                        a.hpw = p.hpw;
                        a.H = st.H;
                        a.W = st.W;
                        a.h = st.h;
                        a.njobs = st.njobs;
                        a.batch = nb;
                        a.jbuf = p.jbuf;
                        a.xbuf = p.xbuf;
                        FGB_CUDA(launch_row_umma(a, cx.fprep.p, cx.sms, s));
                    }
                    break;
                }
                case ST_COLU: {
                    if constexpr (std::is_same<T, float>::value) {
                        ColUArgs a{};
                        a.jobs = p.d_cjobs() + st.job0;
                        a.weights = p.d_wcol();
                        a.dst_base = baseC(st.dst);
                        a.dst_bstride = bsC(st.dst);
                        a.maxbits = (const unsigned*)cx.maxbits.p;
                        a.ws_img_c = p.ws_img_c;
                        a.hpw = p.hpw;
                        a.H = st.H;
                        a.W = st.W;
                        a.h = st.h;
                        a.jbuf = p.jbuf;
                        a.njobs = st.njobs;
                        a.batch = nb;
                        a.dst_planes = (int64_t)nb * bsC(st.dst) / ((int64_t)st.H * st.W);
                        FGB_CUDA(launch_col_umma(a, cx.ws.p, ws_img_bytes * chunk, cx.sms, s));
                    }
                    break;
                }
                case ST_COL: {
                    ColArgs<T> a{};
                    a.jobs = p.d_cjobs() + st.job0;
                    a.weights = p.d_wcol();
                    a.src_base = baseC(st.src);
                    a.dst_base = baseC(st.dst);
                    a.src_bstride = bsC(st.src);
                    a.dst_bstride = bsC(st.dst);
                    a.H = st.H;
                    a.W = st.W;
                    a.t0 = st.t0;
                    a.nt = st.nt;
                    a.zero_boundary = st.zero_bnd;
                    a.njobs = st.njobs;
                    a.batch = nb;
                    FGB_CUDA(launch_col<T>(a, knobs().col_smem_taps ? nullptr : st.pw.data(), s));
                    break;
                }
                case ST_IIR: {
                    IirArgs<T> a{};
                    a.jobs = p.d_ijobs() + st.job0;
                    a.tab_base = p.d_tabs();
                    if (st.iir_real) {
                        int64_t pitch = 0, bs = 0;
                        a.src_base = baseT(st.src, &pitch, &bs);
                        if (st.src.sel == SEL_WSR) pitch = st.H;
                        a.src_bstride = bs;
                        a.src_ls = st.iir_row ? pitch : 1;
                        a.src_ss = st.iir_row ? 1 : pitch;
                    } else {
                        a.src_base = baseC(st.src);
                        a.src_bstride = bsC(st.src);
                        a.src_ls = st.iir_row ? st.H : 1;
                        a.src_ss = st.iir_row ? 1 : st.W;
                    }
                    a.dst_base = baseC(st.dst);
                    a.dst_bstride = bsC(st.dst);
                    a.dst_ls = st.iir_row ? st.H : 1;
                    a.dst_ss = st.iir_row ? 1 : st.W;
                    a.real_in = st.iir_real;
                    a.one_out = 1;
                    for (int j = 0; j < st.njobs; ++j) a.one_out &= p.ijobs[st.job0 + j].nout == 1;
                    a.scratch = scratch + st.lane * scratch_lane;
                    a.state = states + st.lane * state_lane;
                    std::memcpy(a.Aseg, st.Aseg, sizeof(a.Aseg));
                    std::memcpy(a.Alast, st.Alast, sizeof(a.Alast));
                    a.nseg = st.nseg;
                    a.seglen = st.seglen;
                    a.c = st.coef;
                    a.len = st.H;
                    a.lines = st.W;
                    a.P = st.P;
                    a.njobs = st.njobs;
                    a.batch = nb;
                    if ((int64_t)iir_scratch_elems<T>(st.H, st.W, st.P, st.njobs, nb) > scratch_lane)
                        return fail(FGB_EINVAL, "internal: IIR scratch too small");
                    a.g = p.d_dbls() + st.g_off;
                    a.tab32 = p.d_tabs32();
                    a.counters = cnt + (size_t)st.lane * cnt_lane;
                    if constexpr (sizeof(T) == 4) {
                        if (iir32_enabled()) {
                            FGB_CUDA(launch_iir32(a, s));
                            break;
                        }
                    }
                    FGB_CUDA(launch_iir<T>(a, s));
                    break;
                }
                case ST_TR_RC: {
                    int64_t pitch, bs;
                    const T* in = baseT(st.src, &pitch, &bs);
                    if (st.src.sel == SEL_WSR) pitch = st.W;
                    FGB_CUDA(launch_transpose_real_to_cx<T>(in, pitch, bs, baseC(st.dst), bsC(st.dst), st.H, st.W, nb, s));
                    break;
                }
                case ST_TR_CC:
                    FGB_CUDA(launch_transpose_cx<T>(baseC(st.src), bsC(st.src), baseC(st.dst), bsC(st.dst), st.H, st.W,
                                                    nb, s));
                    break;
                case ST_SDFTF: {
                    SdftFusedArgs<T> a{};
                    int64_t pitch, bs;
                    a.img = baseT(st.src, &pitch, &bs);
                    a.pitch = pitch;
                    a.img_bstride = bs;
                    a.out = baseC(st.dst);
                    a.out_bstride = bsC(st.dst);
                    a.w = p.d_wrow() + st.w_off;
                    a.heads = p.d_ints() + st.heads_off;
                    a.head_slot = p.d_ints() + st.slots_off;
                    a.nheads = st.nheads;
                    a.H = st.H;
                    a.W = st.W;
                    a.h = st.h;
                    a.batch = nb;
                    FGB_CUDA(launch_sdft_fused<T>(a, st.M, s));
                    break;
                }
                case ST_BANKF: {
                    if constexpr (std::is_same<T, float>::value) {
                        BankFusedArgs a{};
                        int64_t pitch, bs;
                        a.img = baseT(st.src, &pitch, &bs);
                        a.pitch = pitch;
                        a.img_bstride = bs;
                        a.dst = baseC(st.dst);
                        a.dst_bstride = bsC(st.dst);
                        a.H = st.H;
                        a.W = st.W;
                        a.h = st.h;
                        a.nd = st.nheads;
                        a.batch = nb;
                        a.col_w_off = st.bf_colw_off;
                        for (int k = 0; k < st.nheads; ++k) a.out[k] = st.bf_out[k];
                        // per-call parameter block (28 KB, copied into the launch's constant bank)
                        auto w = std::make_unique<BankFusedW>();
                        std::memcpy(w->w, st.bf_w.data(), st.bf_w.size() * sizeof(float));
                        FGB_CUDA(launch_bank_fused(a, *w, s));
                    }
                    break;
                }
                case ST_TR_RR: {
                    int64_t pitch, bs;
                    const T* in = baseT(st.src, &pitch, &bs);
                    T* o = (T*)ws + st.dst.off;
                    FGB_CUDA(launch_transpose_real<T>(in, pitch, bs, o, 2 * p.ws_img_c, st.H, st.W, nb, s));
                    break;
                }
            }
            if (g_prof) {
                cudaEventRecord(pr.e1, s);
                g_prof_pending.push_back(pr);
            }
        }
        if (nl > 1) {
            for (int l = 1; l < nl; ++l) {
                FGB_CUDA(cudaEventRecord(cx.lane_ev[l - 1], lane_s[l]));
                FGB_CUDA(cudaStreamWaitEvent(s, cx.lane_ev[l - 1], 0));
            }
        }
    }
    return ws_release(cx, s);
}

// ---------------------------------------------------------------------------
// plan cache keys
// ---------------------------------------------------------------------------
static void key_img(std::ostringstream& k, const fgb_image& im) {
    k << im.height << 'x' << im.width << 'p' << im.pitch << 'd' << im.dtype << '|';
}
static void key_sm(std::ostringstream& k, const fgb_smoother& s) {
    k.precision(17);
    k << 's' << s.kind << ',' << s.box_half << ',' << s.radius << '|';
}

template <typename T, typename BuildF>
static int32_t get_plan(Ctx& cx, const std::string& key, BuildF bf, Plan<T>** out) {
    auto it = cx.plans.find(key);
    if (it != cx.plans.end()) {
        *out = static_cast<Plan<T>*>(it->second.get());
        return FGB_OK;
    }
    auto p = std::make_shared<Plan<T>>();
    FGB_TRY(bf(*p));
    cx.plans[key] = p;
    *out = p.get();
    return FGB_OK;
}

static int32_t validate_bank(const fgb_bank_desc* d) {
    if (!d) return fail(FGB_EINVAL, "null descriptor");
    FGB_TRY(check_image(d->img));
    if (d->orientations < 1) return fail(FGB_EINVAL, "orientation count must be at least 1");
    if (d->n_freq < 1 || !d->omegas || !d->sigmas)
        return fail(FGB_EINVAL, "frequencies must be a non-empty list of positive values");
    for (int i = 0; i < d->n_freq; ++i) {
        if (!(d->omegas[i] > 0)) return fail(FGB_EINVAL, "frequencies must be a non-empty list of positive values");
        if (!(d->sigmas[i] > 0)) return fail(FGB_EINVAL, "sigma must be positive");
        FGB_TRY(check_smoother(d->smoother, d->sigmas[i]));
    }
    if (d->units && !d->reuse) return fail(FGB_EINVAL, "work units need reuse mode");
    return FGB_OK;
}

template <typename T> static int32_t bank_plan(const fgb_bank_desc* d, Plan<T>** p) {
    std::ostringstream k;
    k.precision(17);
    k << "bank|";
    key_img(k, d->img);
    key_sm(k, d->smoother);
    k << d->orientations << '|' << d->reuse << '|' << d->img.batch << '|';
    for (int i = 0; i < d->n_freq; ++i) k << d->omegas[i] << ',' << d->sigmas[i] << ';';
    if (d->units)
        for (int i = 0; i < d->n_units; ++i) k << 'u' << d->units[i];
    return get_plan<T>(ctx(), k.str(), [&](Plan<T>& pl) { return build_bank<T>(pl, *d); }, p);
}

template <typename T> static int32_t bank_t(const fgb_bank_desc* d, const void* img, void* out, cudaStream_t s) {
    Plan<T>* p = nullptr;
    FGB_TRY(bank_plan<T>(d, &p));
    return execute<T>(*p, ctx(), d->img, img, out, s);
}

static int32_t validate_filter(const fgb_filter_desc* d, bool complex_in) {
    if (!d) return fail(FGB_EINVAL, "null descriptor");
    FGB_TRY(check_image(d->img, complex_in));
    if (!(d->omega > 0)) return fail(FGB_EINVAL, "omega must be positive");
    if (!(d->sigma > 0)) return fail(FGB_EINVAL, "sigma must be positive");
    return check_smoother(d->smoother, d->sigma);
}

template <typename T>
static int32_t filter_t(const fgb_filter_desc* d, int mode, const void* img, void* out, cudaStream_t s) {
    std::ostringstream k;
    k.precision(17);
    k << "filter|" << mode << '|';
    key_img(k, d->img);
    key_sm(k, d->smoother);
    k << d->omega << ',' << d->theta << ',' << d->sigma << '|' << d->img.batch;
    Ctx& cx = ctx();
    Plan<T>* p = nullptr;
    FGB_TRY(get_plan<T>(cx, k.str(), [&](Plan<T>& pl) { return build_filter<T>(pl, *d, mode); }, &p));
    return execute<T>(*p, cx, d->img, img, out, s);
}

static int32_t validate_sdft(const fgb_sdft_desc* d) {
    if (!d) return fail(FGB_EINVAL, "null descriptor");
    FGB_TRY(check_image(d->img));
    if (d->mx < 1 || d->my < 1) return fail(FGB_EINVAL, "window extents must be at least 1");
    if (d->sigma < 0) return fail(FGB_EINVAL, "sigma must be positive");
    return check_smoother(d->smoother, sdft_sigma(*d));
}

template <typename T> static int32_t sdft_plan(const fgb_sdft_desc* d, int u, int v, Plan<T>** pp) {
    std::ostringstream k;
    k.precision(17);
    k << "sdft|" << u << ',' << v << '|';
    key_img(k, d->img);
    key_sm(k, d->smoother);
    k << d->mx << ',' << d->my << ',' << sdft_sigma(*d) << '|' << d->img.batch;
    if (d->u_heads)
        for (int i = 0; i < d->n_heads; ++i) k << 'h' << d->u_heads[i];
    Ctx& cx = ctx();
    if (u < 0) return get_plan<T>(cx, k.str(), [&](Plan<T>& pl) { return build_sdft<T>(pl, *d); }, pp);
    return get_plan<T>(cx, k.str(), [&](Plan<T>& pl) { return build_sdft_single<T>(pl, *d, u, v); }, pp);
}

template <typename T>
static int32_t sdft_t(const fgb_sdft_desc* d, int u, int v, const void* img, void* out, cudaStream_t s) {
    Plan<T>* p = nullptr;
    FGB_TRY(sdft_plan<T>(d, u, v, &p));
    return execute<T>(*p, ctx(), d->img, img, out, s);
}

// ===========================================================================
// 1-D line smoothing (smooth_lines gaussian.py:245-285)
// ===========================================================================
static int32_t validate_lines(const fgb_lines_desc* d) {
    if (!d) return fail(FGB_EINVAL, "null descriptor");
    if (d->n_lines < 0 || d->len < 1) return fail(FGB_EINVAL, "signal must be a non-empty 1-D array");
    if (d->dtype != FGB_F32 && d->dtype != FGB_F64) return fail(FGB_EINVAL, "dtype must be FGB_F32 or FGB_F64");
    if (d->pitch < d->len) return fail(FGB_EINVAL, "pitch must be >= len");
    const fgb_smoother& k = d->smoother;
    if (k.kind == FGB_SMOOTH_BOX) {
        if (d->box_lo > d->box_hi) return fail(FGB_EINVAL, "box offsets need lo <= hi");
        return FGB_OK;
    }
    if (k.kind == FGB_SMOOTH_FIR && !(d->sigma > 0)) return fail(FGB_EINVAL, "sigma must be positive");
    return check_smoother(k, d->sigma);
}

template <typename T> static int32_t smooth_lines_t(const fgb_lines_desc* d, const void* in, void* out, cudaStream_t s) {
    Ctx& cx = ctx();
    const fgb_smoother& k = d->smoother;
    if (d->n_lines == 0) return FGB_OK;
    if (k.kind == FGB_SMOOTH_IIR) {
        double c[4];
        FGB_TRY(iir_coeffs(d->sigma, c));
        LinesIirArgs<T> a{};
        a.in = (const T*)in;
        a.out = (T*)out;
        a.pitch = d->pitch;
        a.out_pitch = d->len;
        a.n_lines = d->n_lines;
        a.len = d->len;
        a.P = d->assume_padded ? 0 : (int)std::ceil(5.0 * d->sigma) + 2;
        a.c = IirCoef{c[0], c[1], c[2], c[3]};
        FGB_TRY(ws_acquire(cx, s));
        FGB_TRY(cx.ws.ensure((size_t)(d->len + 2 * a.P) * d->n_lines * sizeof(double)));
        a.scratch = (double*)cx.ws.p;
        ++g_launches;
        FGB_CUDA(launch_lines_iir<T>(a, s));
        return ws_release(cx, s);
    }
    // FIR / box: correlation with a cached, immutable device tap table
    std::ostringstream key;
    key.precision(17);
    int t0 = 0;
    std::vector<double> w;
    if (k.kind == FGB_SMOOTH_FIR) {
        int half = 0;
        w = sampled_gaussian(d->sigma, k.radius, &half);
        t0 = -half;
        key << "fir|" << sizeof(T) << '|' << d->sigma << '|' << k.radius;
    } else {
        w.assign((size_t)(d->box_hi - d->box_lo + 1), 1.0);
        t0 = d->box_lo;
        key << "box|" << sizeof(T) << '|' << w.size();
    }
    auto& buf = cx.line_taps[key.str()];
    if (!buf) {
        std::vector<T> wt(w.begin(), w.end());
        std::unique_ptr<DevBuf> nb(new DevBuf());
        FGB_TRY(nb->ensure(wt.size() * sizeof(T)));
        FGB_CUDA(cudaMemcpy(nb->p, wt.data(), wt.size() * sizeof(T), cudaMemcpyHostToDevice));
        buf = std::move(nb);
    }
    LinesCorrArgs<T> a{};
    a.in = (const T*)in;
    a.out = (T*)out;
    a.w = (const T*)buf->p;
    a.pitch = d->pitch;
    a.out_pitch = d->len;
    a.n_lines = d->n_lines;
    a.len = d->len;
    a.t0 = t0;
    a.nt = (int)w.size();
    a.zero_boundary = k.kind == FGB_SMOOTH_BOX;
    ++g_launches;
    FGB_CUDA(launch_lines_corr<T>(a, s));
    return FGB_OK;
}

// ===========================================================================
// brute-force 2-D oracles on the GPU (oracle.py:53-109)
// ===========================================================================
template <typename T>
static int32_t direct2d_run(const fgb_image& im, const std::vector<cd>& k, int ky, int kx, int oy, int ox, int zero,
                            const void* img, void* out, cudaStream_t s) {
    using C = cx_t<T>;
    std::vector<C> hk(k.size());
    for (size_t i = 0; i < k.size(); ++i) hk[i] = mk<T>((T)k[i].real(), (T)k[i].imag());
    C* dk = nullptr;
    FGB_CUDA(cudaMallocAsync((void**)&dk, hk.size() * sizeof(C), s));
    FGB_CUDA(cudaMemcpyAsync(dk, hk.data(), hk.size() * sizeof(C), cudaMemcpyHostToDevice, s));
    Direct2DArgs<T> a{};
    a.img = (const T*)img;
    a.pitch = im.pitch;
    a.img_bstride = im.batch > 1 ? im.batch_stride : (int64_t)im.height * im.pitch;
    a.out = (C*)out;
    a.out_bstride = (int64_t)im.height * im.width;
    a.kern = dk;
    a.ky = ky;
    a.kx = kx;
    a.oy = oy;
    a.ox = ox;
    a.zero_boundary = zero;
    a.H = im.height;
    a.W = im.width;
    a.batch = im.batch;
    cudaError_t e = launch_direct2d<T>(a, s);
    cudaFreeAsync(dk, s);
    if (e == cudaErrorInvalidConfiguration) return fail(FGB_EINVAL, "oracle kernel support too large for the direct GPU path");
    FGB_CUDA(e);
    FGB_CUDA(cudaStreamSynchronize(s));  // the host kernel table must outlive the H2D copy
    return FGB_OK;
}

// fir_gabor (oracle.py:53-66): env * e^{i w (dx cos + dy sin)}, reversed, replicate pad by half
static void fir_gabor_kernel(const fgb_filter_desc& d, double radius, std::vector<cd>* k, int* half) {
    int h;
    std::vector<double> g = sampled_gaussian(d.sigma, radius, &h);
    const double th = norm_theta(d.theta);
    const int n = 2 * h + 1;
    k->assign((size_t)n * n, cd(0, 0));
    for (int iy = 0; iy < n; ++iy)
        for (int ix = 0; ix < n; ++ix) {
            // reversed: kernel row iy holds dy = h - iy, column ix holds dx = h - ix
            const double dy = (double)(h - iy), dx = (double)(h - ix);
            const double ph = d.omega * (std::cos(th) * dx + std::sin(th) * dy);
            const double env = g[h - iy + h] * g[h - ix + h];
            (*k)[(size_t)iy * n + ix] = cd(env * std::cos(ph), env * std::sin(ph));
        }
    *half = h;
}

// localized_dft (oracle.py:69-109)
static void ldft_kernel(const fgb_sdft_desc& d, int u, int v, double radius, std::vector<cd>* k, int* ky, int* kx,
                        int* oy, int* ox, int* zero) {
    const int mx = d.mx, my = d.my;
    std::vector<double> gx, gy;
    int lox, hix, loy, hiy;
    if (d.smoother.kind == FGB_SMOOTH_BOX) {
        lox = -(mx / 2); hix = mx - 1 - mx / 2;
        loy = -(my / 2); hiy = my - 1 - my / 2;
        gx.assign(hix - lox + 1, 1.0);
        gy.assign(hiy - loy + 1, 1.0);
        *zero = 1;
    } else {
        int hx, hy;
        const double s = sdft_sigma(d);
        gx = sampled_gaussian(s, radius, &hx);
        gy = sampled_gaussian(s, radius, &hy);
        lox = -hx; hix = hx; loy = -hy; hiy = hy;
        *zero = 0;
    }
    *ky = hiy - loy + 1;
    *kx = hix - lox + 1;
    *oy = -loy;
    *ox = -lox;
    const double w0x = 2.0 * M_PI / mx, w0y = 2.0 * M_PI / my;
    k->assign((size_t)(*ky) * (*kx), cd(0, 0));
    for (int iy = 0; iy < *ky; ++iy)
        for (int ix = 0; ix < *kx; ++ix) {
            const double dm = (double)(lox + ix), dn = (double)(loy + iy);
            const double ph = w0x * u * (mx / 2 + dm) + w0y * v * (my / 2 + dn);
            const double env = gy[iy] * gx[ix];
            (*k)[(size_t)iy * (*kx) + ix] = cd(env * std::cos(ph), env * std::sin(ph));
        }
}

}  // namespace fgb

// ===========================================================================
// C ABI
// ===========================================================================
using namespace fgb;

namespace fgb {
static size_t elem_size(int32_t dtype) { return dtype == FGB_F64 ? 8 : 4; }
static size_t img_bytes(const fgb_image& im) {
    const int64_t bs = im.batch > 1 ? im.batch_stride : (int64_t)im.height * im.pitch;
    return (size_t)((int64_t)(im.batch - 1) * bs + (int64_t)(im.height - 1) * im.pitch + im.width) * elem_size(im.dtype);
}

// host-buffer variants: H2D, compute, D2H on one stream (synchronous)
template <typename F>
static int32_t host_call(const fgb_image& im, int64_t out_elems_c, const void* in_h, void* out_h, F compute) {
    Ctx& cx = ctx();
    const size_t in_b = img_bytes(im);
    const size_t out_b = (size_t)out_elems_c * 2 * elem_size(im.dtype);
    FGB_TRY(cx.hin.ensure(in_b));
    FGB_TRY(cx.hout.ensure(out_b));
    cudaStream_t s = 0;
    FGB_CUDA(cudaMemcpyAsync(cx.hin.p, in_h, in_b, cudaMemcpyHostToDevice, s));
    FGB_TRY(compute(cx.hin.p, cx.hout.p, s));
    FGB_CUDA(cudaMemcpyAsync(out_h, cx.hout.p, out_b, cudaMemcpyDeviceToHost, s));
    FGB_CUDA(cudaStreamSynchronize(s));
    return FGB_OK;
}

// Same as host_call, but the result reaches the host as the reference's
// ComplexImage layout: [entries][2][plane] float64 (re plane, im plane),
// converted on the GPU, with a finiteness flag so the host can skip its own
// per-element checks.
template <typename F>
static int32_t host_call_planar(const fgb_image& im, int64_t out_elems_c, int64_t plane, const void* in_h,
                                double* out_h, int32_t* nonfinite, F compute) {
    Ctx& cx = ctx();
    const size_t in_b = img_bytes(im);
    const size_t out_b = (size_t)out_elems_c * 2 * elem_size(im.dtype);
    const size_t pl_b = (size_t)out_elems_c * 2 * sizeof(double);
    FGB_TRY(cx.hin.ensure(in_b));
    FGB_TRY(cx.hout.ensure(out_b));
    FGB_TRY(cx.hpl.ensure(pl_b));
    FGB_TRY(cx.hflag.ensure(sizeof(int)));
    cudaStream_t s = 0;
    FGB_CUDA(cudaMemsetAsync(cx.hflag.p, 0, sizeof(int), s));
    FGB_CUDA(cudaMemcpyAsync(cx.hin.p, in_h, in_b, cudaMemcpyHostToDevice, s));
    FGB_TRY(compute(cx.hin.p, cx.hout.p, s));
    if (im.dtype == FGB_F32)
        FGB_CUDA(launch_entries_planar<float>((const float2*)cx.hout.p, out_elems_c, plane, (double*)cx.hpl.p,
                                              (int*)cx.hflag.p, s));
    else
        FGB_CUDA(launch_entries_planar<double>((const double2*)cx.hout.p, out_elems_c, plane, (double*)cx.hpl.p,
                                               (int*)cx.hflag.p, s));
    int flag = 0;
    FGB_CUDA(cudaMemcpyAsync(out_h, cx.hpl.p, pl_b, cudaMemcpyDeviceToHost, s));
    FGB_CUDA(cudaMemcpyAsync(&flag, cx.hflag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    FGB_CUDA(cudaStreamSynchronize(s));
    if (nonfinite) *nonfinite = flag;
    return FGB_OK;
}

}  // namespace fgb

extern "C" {

const char* fgb_last_error(void) { return g_err.c_str(); }
int32_t fgb_version(void) { return 1 * 10000 + 0 * 100 + 0; }
int32_t fgb_device_sm_count(void) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return fail(FGB_ECUDA, "no CUDA device");
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return fail(FGB_ECUDA, "cudaDeviceGetAttribute failed");
    return n;
}

int32_t fgb_pad_radius(const fgb_smoother* kind, double sigma) {
    if (!kind) return fail(FGB_EINVAL, "null smoother");
    return pad_radius(*kind, sigma);
}

int32_t fgb_sampled_gaussian(double sigma, double radius, double* out, int32_t cap, int32_t* half) {
    if (!(sigma > 0)) return fail(FGB_EINVAL, "sigma must be positive");
    int h;
    std::vector<double> w = sampled_gaussian(sigma, radius, &h);
    if (half) *half = h;
    if (out) {
        if (cap < (int32_t)w.size()) return fail(FGB_EINVAL, "output capacity too small");
        std::memcpy(out, w.data(), w.size() * sizeof(double));
    }
    return FGB_OK;
}

int32_t fgb_iir_coeffs(double sigma, double out[4]) { return iir_coeffs(sigma, out); }
int32_t fgb_iir_sections(double sigma, double out[6]) {
    double cf[4];
    FGB_TRY(iir_coeffs(sigma, cf));
    iir32_sections(IirCoef{cf[0], cf[1], cf[2], cf[3]}, out);
    return FGB_OK;
}

int64_t fgb_bank_entries(const fgb_bank_desc* d) {
    if (!d) return fail(FGB_EINVAL, "null descriptor");
    if (!d->units) return (int64_t)d->n_freq * d->orientations;
    const int N = d->orientations, nh = N / 2;
    int64_t n = 0;
    for (int i = 0; i < d->n_units; ++i) {
        const int k = d->units[i] % (nh + 1);
        n += 1 + ((nh < N - k && N - k < N) ? 1 : 0);
    }
    return n;
}

int64_t fgb_sdft_bins(const fgb_sdft_desc* d) {
    if (!d) return fail(FGB_EINVAL, "null descriptor");
    BinMap bm;
    int32_t r = make_binmap(*d, &bm);
    if (r != FGB_OK) return r;
    return bm.nbins;
}

int64_t fgb_bank_workspace_bytes(const fgb_bank_desc* d) {
    FGB_TRY(validate_bank(d));
    std::lock_guard<std::mutex> lk(g_mu);
    if (d->img.dtype == FGB_F32) {
        Plan<float>* p = nullptr;
        FGB_TRY(bank_plan<float>(d, &p));
        return plan_ws_bytes(*p, d->img.batch);
    }
    Plan<double>* p = nullptr;
    FGB_TRY(bank_plan<double>(d, &p));
    return plan_ws_bytes(*p, d->img.batch);
}

int64_t fgb_sdft_workspace_bytes(const fgb_sdft_desc* d) {
    FGB_TRY(validate_sdft(d));
    std::lock_guard<std::mutex> lk(g_mu);
    if (d->img.dtype == FGB_F32) {
        Plan<float>* p = nullptr;
        FGB_TRY(sdft_plan<float>(d, -1, -1, &p));
        return plan_ws_bytes(*p, d->img.batch);
    }
    Plan<double>* p = nullptr;
    FGB_TRY(sdft_plan<double>(d, -1, -1, &p));
    return plan_ws_bytes(*p, d->img.batch);
}

int32_t fgb_bank(const fgb_bank_desc* d, const void* img, void* out, void* stream) {
    FGB_TRY(validate_bank(d));
    std::lock_guard<std::mutex> lk(g_mu);
    cudaStream_t s = (cudaStream_t)stream;
    return d->img.dtype == FGB_F32 ? bank_t<float>(d, img, out, s) : bank_t<double>(d, img, out, s);
}

int32_t fgb_filter(const fgb_filter_desc* d, const void* img, void* out, void* stream) {
    FGB_TRY(validate_filter(d, false));
    std::lock_guard<std::mutex> lk(g_mu);
    cudaStream_t s = (cudaStream_t)stream;
    return d->img.dtype == FGB_F32 ? filter_t<float>(d, 0, img, out, s) : filter_t<double>(d, 0, img, out, s);
}

int32_t fgb_horizontal_stage(const fgb_filter_desc* d, const void* img, void* j_out, void* stream) {
    FGB_TRY(validate_filter(d, false));
    std::lock_guard<std::mutex> lk(g_mu);
    cudaStream_t s = (cudaStream_t)stream;
    return d->img.dtype == FGB_F32 ? filter_t<float>(d, 1, img, j_out, s) : filter_t<double>(d, 1, img, j_out, s);
}

int32_t fgb_vertical_stage(const fgb_filter_desc* d, const void* j_in, void* out, int32_t conjugate, void* stream) {
    FGB_TRY(validate_filter(d, true));
    std::lock_guard<std::mutex> lk(g_mu);
    cudaStream_t s = (cudaStream_t)stream;
    const int mode = conjugate ? 3 : 2;
    return d->img.dtype == FGB_F32 ? filter_t<float>(d, mode, j_in, out, s) : filter_t<double>(d, mode, j_in, out, s);
}

int32_t fgb_sdft(const fgb_sdft_desc* d, const void* img, void* out, void* stream) {
    FGB_TRY(validate_sdft(d));
    std::lock_guard<std::mutex> lk(g_mu);
    cudaStream_t s = (cudaStream_t)stream;
    return d->img.dtype == FGB_F32 ? sdft_t<float>(d, -1, -1, img, out, s) : sdft_t<double>(d, -1, -1, img, out, s);
}

int32_t fgb_sdft_bin(const fgb_sdft_desc* d, int32_t u, int32_t v, const void* img, void* out, void* stream) {
    FGB_TRY(validate_sdft(d));
    if (u < 0 || u >= d->mx) return fail(FGB_EINVAL, "bin index u=" + std::to_string(u) + " outside [0, " + std::to_string(d->mx) + ")");
    if (v < 0 || v >= d->my) return fail(FGB_EINVAL, "bin index v=" + std::to_string(v) + " outside [0, " + std::to_string(d->my) + ")");
    std::lock_guard<std::mutex> lk(g_mu);
    cudaStream_t s = (cudaStream_t)stream;
    return d->img.dtype == FGB_F32 ? sdft_t<float>(d, u, v, img, out, s) : sdft_t<double>(d, u, v, img, out, s);
}

int32_t fgb_ser_sums(const void* approx, const void* truth, int64_t n, int32_t dtype, double out[4], void* stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (n < 0 || !out) return fail(FGB_EINVAL, "bad SER arguments");
    if (dtype != FGB_F32 && dtype != FGB_F64) return fail(FGB_EINVAL, "dtype must be FGB_F32 or FGB_F64");
    if (n == 0) {
        for (int k = 0; k < 4; ++k) out[k] = 0.0;
        return FGB_OK;
    }
    Ctx& cx = ctx();
    cudaStream_t s = (cudaStream_t)stream;
    FGB_TRY(cx.ser_scratch.ensure(ser_scratch_doubles() * sizeof(double)));
    double* scr = (double*)cx.ser_scratch.p;
    g_launches += 2;
    if (dtype == FGB_F32) FGB_CUDA(launch_ser<float>((const float2*)approx, (const float2*)truth, n, scr, s));
    else FGB_CUDA(launch_ser<double>((const double2*)approx, (const double2*)truth, n, scr, s));
    FGB_CUDA(cudaMemcpyAsync(out, scr, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
    FGB_CUDA(cudaStreamSynchronize(s));
    return FGB_OK;
}
int32_t fgb_smooth_lines(const fgb_lines_desc* d, const void* lines, void* out, void* stream) {
    std::lock_guard<std::mutex> lk(g_mu);
    FGB_TRY(validate_lines(d));
    return d->dtype == FGB_F64 ? smooth_lines_t<double>(d, lines, out, (cudaStream_t)stream)
                               : smooth_lines_t<float>(d, lines, out, (cudaStream_t)stream);
}
int32_t fgb_smooth_lines_host(const fgb_lines_desc* d, const void* lines_host, void* out_host) {
    std::lock_guard<std::mutex> lk(g_mu);
    FGB_TRY(validate_lines(d));
    if (d->n_lines == 0) return FGB_OK;
    Ctx& cx = ctx();
    const size_t es = elem_size(d->dtype);
    const size_t in_b = ((size_t)(d->n_lines - 1) * d->pitch + d->len) * es;
    const size_t out_b = (size_t)d->n_lines * d->len * es;
    FGB_TRY(cx.hin.ensure(in_b));
    FGB_TRY(cx.hout.ensure(out_b));
    cudaStream_t s = 0;
    FGB_CUDA(cudaMemcpyAsync(cx.hin.p, lines_host, in_b, cudaMemcpyHostToDevice, s));
    FGB_TRY(d->dtype == FGB_F64 ? smooth_lines_t<double>(d, cx.hin.p, cx.hout.p, s)
                                : smooth_lines_t<float>(d, cx.hin.p, cx.hout.p, s));
    FGB_CUDA(cudaMemcpyAsync(out_host, cx.hout.p, out_b, cudaMemcpyDeviceToHost, s));
    FGB_CUDA(cudaStreamSynchronize(s));
    return FGB_OK;
}
int32_t fgb_sdft_horizontal(const fgb_sdft_desc* d, int32_t u, const void* img, void* j_out, void* stream) {
    FGB_TRY(validate_sdft(d));
    if (u < 0 || u >= d->mx) return fail(FGB_EINVAL, "bin index u=" + std::to_string(u) + " outside [0, " + std::to_string(d->mx) + ")");
    std::lock_guard<std::mutex> lk(g_mu);
    cudaStream_t s = (cudaStream_t)stream;
    return d->img.dtype == FGB_F32 ? sdft_t<float>(d, u, -1, img, j_out, s) : sdft_t<double>(d, u, -1, img, j_out, s);
}

// Host-buffer bank with the D2H pipelined behind the compute: the call is cut
// into pieces (images of a batch, else frequencies of one image), each
// piece's outputs leave on a copy stream as soon as its kernels finish, so
// only the first piece's compute is exposed in front of the PCIe transfer.
static int32_t bank_host_pipelined(const fgb_bank_desc* d, const void* in_h, void* out_h) {
    Ctx& cx = ctx();
    const fgb_image& im = d->img;
    const int64_t entries = fgb_bank_entries(d);
    const int64_t hw = (int64_t)im.height * im.width;
    const size_t es = elem_size(im.dtype);
    const size_t in_b = img_bytes(im);
    const size_t out_b = (size_t)(entries * hw * im.batch) * 2 * es;
    FGB_TRY(cx.hin.ensure(in_b));
    FGB_TRY(cx.hout.ensure(out_b));
    if (!cx.copy_stream) FGB_CUDA(cudaStreamCreateWithFlags(&cx.copy_stream, cudaStreamNonBlocking));
    const bool by_image = im.batch > 1;
    const bool by_freq = !by_image && d->n_freq > 1 && d->units == nullptr;
    const bool by_units = !by_image && d->units != nullptr && d->n_units > 1;  // contiguous runs of the unit list
    const int pieces = by_image ? im.batch : (by_freq ? d->n_freq : (by_units ? std::min(d->n_units, 8) : 1));
    while ((int)cx.piece_ev.size() < pieces) {
        cudaEvent_t e;
        FGB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        cx.piece_ev.push_back(e);
    }
    cudaStream_t s = 0;
    FGB_CUDA(cudaMemcpyAsync(cx.hin.p, in_h, in_b, cudaMemcpyHostToDevice, s));
    const int64_t img_stride = im.batch > 1 ? im.batch_stride : (int64_t)im.height * im.pitch;
    const int64_t per_freq = entries / std::max(1, d->n_freq);
    std::vector<int> order(std::max(1, d->n_freq));
    for (int i = 0; i < (int)order.size(); ++i) order[i] = i;
    if (by_freq)  // smallest sigma (cheapest) first: the copy engine starts earliest
        std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return d->sigmas[x] < d->sigmas[y]; });
    for (int p = 0; p < pieces; ++p) {
        fgb_bank_desc dp = *d;
        const char* in_d = (const char*)cx.hin.p;
        int64_t out_off = 0, out_n = entries * hw * im.batch;  // complex elements
        if (by_image) {
            dp.img.batch = 1;
            in_d += (size_t)(p * img_stride) * es;
            out_off = p * entries * hw;
            out_n = entries * hw;
        } else if (by_units) {
            // compact layout: entries of units [u0, u1) follow those of units [0, u0)
            const int u0 = (int)((int64_t)d->n_units * p / pieces), u1 = (int)((int64_t)d->n_units * (p + 1) / pieces);
            fgb_bank_desc head = *d;
            head.n_units = u0;
            const int64_t before = u0 > 0 ? fgb_bank_entries(&head) : 0;
            dp.units = d->units + u0;
            dp.n_units = u1 - u0;
            const int64_t ne = fgb_bank_entries(&dp);
            if (before < 0 || ne < 0) return fail(FGB_EINVAL, "invalid unit list");
            out_off = before * hw;
            out_n = ne * hw;
        } else if (by_freq) {
            const int f = order[p];
            dp.n_freq = 1;
            dp.omegas = d->omegas + f;
            dp.sigmas = d->sigmas + f;
            out_off = f * per_freq * hw;
            out_n = per_freq * hw;
        }
        char* out_d = (char*)cx.hout.p + (size_t)out_off * 2 * es;
        FGB_TRY(im.dtype == FGB_F32 ? bank_t<float>(&dp, in_d, out_d, s) : bank_t<double>(&dp, in_d, out_d, s));
        FGB_CUDA(cudaEventRecord(cx.piece_ev[p], s));
        FGB_CUDA(cudaStreamWaitEvent(cx.copy_stream, cx.piece_ev[p], 0));
        FGB_CUDA(cudaMemcpyAsync((char*)out_h + (size_t)out_off * 2 * es, out_d, (size_t)out_n * 2 * es,
                                 cudaMemcpyDeviceToHost, cx.copy_stream));
    }
    FGB_CUDA(cudaStreamSynchronize(cx.copy_stream));
    FGB_CUDA(cudaStreamSynchronize(s));
    return FGB_OK;
}

int32_t fgb_bank_host(const fgb_bank_desc* d, const void* img_host, void* out_host) {
    FGB_TRY(validate_bank(d));
    std::lock_guard<std::mutex> lk(g_mu);
    return bank_host_pipelined(d, img_host, out_host);
}

int32_t fgb_filter_host(const fgb_filter_desc* d, const void* img_host, void* out_host) {
    FGB_TRY(validate_filter(d, false));
    std::lock_guard<std::mutex> lk(g_mu);
    const int64_t n = (int64_t)d->img.height * d->img.width * d->img.batch;
    return host_call(d->img, n, img_host, out_host, [&](void* i, void* o, cudaStream_t s) {
        return d->img.dtype == FGB_F32 ? filter_t<float>(d, 0, i, o, s) : filter_t<double>(d, 0, i, o, s);
    });
}

int32_t fgb_sdft_host(const fgb_sdft_desc* d, const void* img_host, void* out_host) {
    FGB_TRY(validate_sdft(d));
    const int64_t nb = fgb_sdft_bins(d);
    if (nb < 0) return (int32_t)nb;
    std::lock_guard<std::mutex> lk(g_mu);
    const int64_t n = nb * (int64_t)d->img.height * d->img.width * d->img.batch;
    return host_call(d->img, n, img_host, out_host, [&](void* i, void* o, cudaStream_t s) {
        return d->img.dtype == FGB_F32 ? sdft_t<float>(d, -1, -1, i, o, s) : sdft_t<double>(d, -1, -1, i, o, s);
    });
}

int32_t fgb_bank_host_planar(const fgb_bank_desc* d, const void* img_host, double* out_host, int32_t* nonfinite) {
    FGB_TRY(validate_bank(d));
    const int64_t ne = fgb_bank_entries(d);
    if (ne < 0) return (int32_t)ne;
    std::lock_guard<std::mutex> lk(g_mu);
    const int64_t plane = (int64_t)d->img.height * d->img.width;
    return host_call_planar(d->img, ne * plane * d->img.batch, plane, img_host, out_host, nonfinite,
                            [&](void* i, void* o, cudaStream_t s) {
                                return d->img.dtype == FGB_F32 ? bank_t<float>(d, i, o, s) : bank_t<double>(d, i, o, s);
                            });
}

int32_t fgb_filter_host_planar(const fgb_filter_desc* d, const void* img_host, double* out_host, int32_t* nonfinite) {
    FGB_TRY(validate_filter(d, false));
    std::lock_guard<std::mutex> lk(g_mu);
    const int64_t plane = (int64_t)d->img.height * d->img.width;
    return host_call_planar(d->img, plane * d->img.batch, plane, img_host, out_host, nonfinite,
                            [&](void* i, void* o, cudaStream_t s) {
                                return d->img.dtype == FGB_F32 ? filter_t<float>(d, 0, i, o, s)
                                                               : filter_t<double>(d, 0, i, o, s);
                            });
}

int32_t fgb_sdft_host_planar(const fgb_sdft_desc* d, const void* img_host, double* out_host, int32_t* nonfinite) {
    FGB_TRY(validate_sdft(d));
    const int64_t nb = fgb_sdft_bins(d);
    if (nb < 0) return (int32_t)nb;
    std::lock_guard<std::mutex> lk(g_mu);
    const int64_t plane = (int64_t)d->img.height * d->img.width;
    return host_call_planar(d->img, nb * plane * d->img.batch, plane, img_host, out_host, nonfinite,
                            [&](void* i, void* o, cudaStream_t s) {
                                return d->img.dtype == FGB_F32 ? sdft_t<float>(d, -1, -1, i, o, s)
                                                               : sdft_t<double>(d, -1, -1, i, o, s);
                            });
}

int32_t fgb_horizontal_stage_host(const fgb_filter_desc* d, const void* img_host, void* j_host) {
    FGB_TRY(validate_filter(d, false));
    std::lock_guard<std::mutex> lk(g_mu);
    const int64_t n = (int64_t)d->img.height * d->img.width * d->img.batch;
    return host_call(d->img, n, img_host, j_host, [&](void* i, void* o, cudaStream_t s) {
        return d->img.dtype == FGB_F32 ? filter_t<float>(d, 1, i, o, s) : filter_t<double>(d, 1, i, o, s);
    });
}

int32_t fgb_vertical_stage_host(const fgb_filter_desc* d, const void* j_host, void* out_host, int32_t conjugate) {
    FGB_TRY(validate_filter(d, true));
    std::lock_guard<std::mutex> lk(g_mu);
    const int64_t n = (int64_t)d->img.height * d->img.width * d->img.batch;
    fgb_image cim = d->img;  // complex input: twice the real element count
    cim.width *= 2;
    cim.pitch *= 2;
    cim.batch_stride *= 2;
    const int mode = conjugate ? 3 : 2;
    return host_call(cim, n, j_host, out_host, [&](void* i, void* o, cudaStream_t s) {
        return d->img.dtype == FGB_F32 ? filter_t<float>(d, mode, i, o, s) : filter_t<double>(d, mode, i, o, s);
    });
}

int32_t fgb_sdft_bin_host(const fgb_sdft_desc* d, int32_t u, int32_t v, const void* img_host, void* out_host) {
    FGB_TRY(validate_sdft(d));
    if (u < 0 || u >= d->mx) return fail(FGB_EINVAL, "bin index u=" + std::to_string(u) + " outside [0, " + std::to_string(d->mx) + ")");
    if (v < 0 || v >= d->my) return fail(FGB_EINVAL, "bin index v=" + std::to_string(v) + " outside [0, " + std::to_string(d->my) + ")");
    std::lock_guard<std::mutex> lk(g_mu);
    const int64_t n = (int64_t)d->img.height * d->img.width * d->img.batch;
    return host_call(d->img, n, img_host, out_host, [&](void* i, void* o, cudaStream_t s) {
        return d->img.dtype == FGB_F32 ? sdft_t<float>(d, u, v, i, o, s) : sdft_t<double>(d, u, v, i, o, s);
    });
}

int32_t fgb_sdft_horizontal_host(const fgb_sdft_desc* d, int32_t u, const void* img_host, void* j_host) {
    FGB_TRY(validate_sdft(d));
    if (u < 0 || u >= d->mx) return fail(FGB_EINVAL, "bin index u=" + std::to_string(u) + " outside [0, " + std::to_string(d->mx) + ")");
    std::lock_guard<std::mutex> lk(g_mu);
    const int64_t n = (int64_t)d->img.height * d->img.width * d->img.batch;
    return host_call(d->img, n, img_host, j_host, [&](void* i, void* o, cudaStream_t s) {
        return d->img.dtype == FGB_F32 ? sdft_t<float>(d, u, -1, i, o, s) : sdft_t<double>(d, u, -1, i, o, s);
    });
}

int32_t fgb_fir_gabor(const fgb_filter_desc* d, double radius, const void* img, void* out, void* stream) {
    FGB_TRY(validate_filter(d, false));
    if (radius < 3) return fail(FGB_EINVAL, "truncation radius must be at least 3 sigma");
    std::vector<cd> k;
    int h;
    fir_gabor_kernel(*d, radius, &k, &h);
    cudaStream_t s = (cudaStream_t)stream;
    const int n = 2 * h + 1;
    return d->img.dtype == FGB_F32 ? direct2d_run<float>(d->img, k, n, n, h, h, 0, img, out, s)
                                   : direct2d_run<double>(d->img, k, n, n, h, h, 0, img, out, s);
}

int32_t fgb_localized_dft(const fgb_sdft_desc* d, int32_t u, int32_t v, double radius, const void* img, void* out,
                          void* stream) {
    FGB_TRY(validate_sdft(d));
    if (u < 0 || u >= d->mx || v < 0 || v >= d->my) return fail(FGB_EINVAL, "bin indices outside the window grid");
    if (radius < 3) return fail(FGB_EINVAL, "truncation radius must be at least 3 sigma");
    std::vector<cd> k;
    int ky, kx, oy, ox, zero;
    ldft_kernel(*d, u, v, radius, &k, &ky, &kx, &oy, &ox, &zero);
    cudaStream_t s = (cudaStream_t)stream;
    return d->img.dtype == FGB_F32 ? direct2d_run<float>(d->img, k, ky, kx, oy, ox, zero, img, out, s)
                                   : direct2d_run<double>(d->img, k, ky, kx, oy, ox, zero, img, out, s);
}

int32_t fgb_fir_gabor_host(const fgb_filter_desc* d, double radius, const void* img_host, void* out_host) {
    std::lock_guard<std::mutex> lk(g_mu);
    const int64_t n = (int64_t)d->img.height * d->img.width * d->img.batch;
    return host_call(d->img, n, img_host, out_host, [&](void* i, void* o, cudaStream_t s) {
        return fgb_fir_gabor(d, radius, i, o, s);
    });
}

int32_t fgb_localized_dft_host(const fgb_sdft_desc* d, int32_t u, int32_t v, double radius, const void* img_host,
                               void* out_host) {
    std::lock_guard<std::mutex> lk(g_mu);
    const int64_t n = (int64_t)d->img.height * d->img.width * d->img.batch;
    return host_call(d->img, n, img_host, out_host, [&](void* i, void* o, cudaStream_t s) {
        return fgb_localized_dft(d, u, v, radius, i, o, s);
    });
}

int32_t fgb_gbnk_write_device(const char* path, const double* params, int32_t n_entries, int32_t height, int32_t width,
                              int32_t dtype, const void* dev_entries, int32_t sdft, void* stream) {
    if (!path || !params || !dev_entries) return fail(FGB_EINVAL, "null argument");
    if (n_entries < 1) return fail(FGB_EINVAL, "container must hold at least one entry");
    if (height < 1 || width < 1) return fail(FGB_EINVAL, "image dimensions must be at least 1x1");
    std::string err;
    const int rc = gbnk_write_device(path, params, n_entries, height, width, dtype, dev_entries, sdft,
                                     (cudaStream_t)stream, &err);
    if (rc == -1) return fail(FGB_EINVAL, err);
    if (rc == -2) return fail(FGB_ECUDA, err);
    return FGB_OK;
}

int32_t fgb_stream_synchronize(void* stream) {
    FGB_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    return FGB_OK;
}

void fgb_profile_enable(int32_t on) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_prof = on != 0;
}

int64_t fgb_launch_count(void) { return g_launches; }

int32_t fgb_profile_read(fgb_prof_entry* out, int32_t cap) {
    std::lock_guard<std::mutex> lk(g_mu);
    std::vector<fgb_prof_entry> agg;
    for (ProfRec& r : g_prof_pending) {
        FGB_CUDA(cudaEventSynchronize(r.e1));
        float ms = 0.f;
        FGB_CUDA(cudaEventElapsedTime(&ms, r.e0, r.e1));
        fgb_prof_entry* e = nullptr;
        for (auto& a : agg)
            if (std::strncmp(a.name, r.name.c_str(), sizeof(a.name) - 1) == 0) e = &a;
        if (!e) {
            agg.push_back(fgb_prof_entry{});
            e = &agg.back();
            std::strncpy(e->name, r.name.c_str(), sizeof(e->name) - 1);
        }
        e->launches += 1;
        e->ms += ms;
        e->flops += r.flops;
        e->bytes += r.bytes;
        g_event_pool.push_back(r.e0);
        g_event_pool.push_back(r.e1);
    }
    g_prof_pending.clear();
    const int n = std::min<int>((int)agg.size(), cap);
    for (int i = 0; i < n; ++i) out[i] = agg[i];
    return (int32_t)agg.size();
}

double fgb_probe_fp32_tflops(void) { return probe_fma_tflops<float>(); }
double fgb_probe_fp64_tflops(void) { return probe_fma_tflops<double>(); }
double fgb_probe_fma(int32_t dtype, int32_t mode) {
    if (mode == 0) return dtype == FGB_F64 ? probe_fma_tflops<double>() : probe_fma_tflops<float>();
    if (mode >= 4) return dtype == FGB_F64 ? -1.0 : probe_ffma2_tflops(mode);
    return dtype == FGB_F64 ? probe_fma_reg_tflops<double>(mode) : probe_fma_reg_tflops<float>(mode);
}

void fgb_release_caches(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_ctx.clear();
}

}  // extern "C"
