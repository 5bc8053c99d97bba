// Kernel launch interfaces (internal to libfgb200).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>
#include <cstdlib>

#include "common.cuh"

namespace fgb {

// A/B experiment knobs, read from the environment once
// per process -- never per launch.
struct Knobs {
    bool col1, col_smem_taps, row_smem_taps, no_realj, sdft_unfused, prof_detail, iir64;
    int col_mode;  // -1 = cost model
    int col_seg;   // 0 = cost model
};
inline const Knobs& knobs() {
    static const Knobs k = [] {
        auto on = [](const char* n) { return std::getenv(n) != nullptr; };
        auto num = [](const char* n, int d) { const char* e = std::getenv(n); return e ? std::atoi(e) : d; };
        return Knobs{on("FGB_COL1"), on("FGB_COL_SMEM_TAPS"), on("FGB_ROW_SMEM_TAPS"), on("FGB_NO_REALJ"),
                     on("FGB_SDFT_UNFUSED"), on("FGB_PROF_DETAIL"), on("FGB_IIR64"), num("FGB_COL_MODE", -1),
                     num("FGB_COL_SEG", 0)};
    }();
    return k;
}

// ---- K1: symmetric-FIR row pass (row_fir.cu) ------------------------------
template <typename T> struct RowArgs {
    const T* img;          // real input, batch 0
    cx_t<T>* dst_base;
    int64_t pitch;         // elements
    int64_t img_bstride;   // elements
    int64_t out_bstride;   // complex elements between images in dst planes
    const T* weights;      // device weight pool
    int H, W;
    int hp;                // half-width padded to a multiple of the row R
    int batch;
    // fp32 split-fp16 output for the tensor-core column pass (ColUArgs): hi plane at the job's
    // dst, lo plane j16_plane u32 later, row y at (y + jpad) * W, edge rows replicated into the pads
    int j16, jpad;
    int64_t j16_plane;
    const unsigned* maxbits;
};
template <typename T, int CAP> struct RowWParam { T w[CAP > 0 ? CAP : 1]; };
template <typename T> struct RowWCap {
    static constexpr int kSmall = 4096 / (int)sizeof(T);           // 4 KB
    static constexpr int kLarge = (30 * 1024) / (int)sizeof(T);    // 30 KB
};
template <typename T> size_t row_sym_smem(int hp, int nd, bool taps_in_smem);
template <typename T> int row_sym_pad(int h);
// pw_host: the group's [(hp+1)][NDP][2] tap table (kernel-parameter path) or nullptr
template <typename T>
cudaError_t launch_row_sym(const RowArgs<T>& a, const RowGroup<T>& g, const T* pw_host, cudaStream_t s);

// ---- K2: column pass with two real kernels (col_fir.cu) ------------------
template <typename T> struct ColArgs {
    const ColJob<T>* jobs;   // device array [njobs]
    const cx_t<T>* weights;  // device weight pool of (ka, kb) pairs
    const cx_t<T>* src_base;
    cx_t<T>* dst_base;
    int64_t src_bstride;     // complex elements between images of src planes
    int64_t dst_bstride;     // complex elements between images of dst planes
    int H, W;
    int t0;                  // first tap offset (taps t0 .. t0+nt-1)
    int nt;                  // number of taps
    int zero_boundary;       // 0 = replicate rows, 1 = zero outside [0, H)
    int njobs;
    int batch;
    int seg;                 // rows per CTA segment (set by launch_col)
    int col2;                // fp32: two columns per thread (set by launch_col)
};
// Tap pairs passed as kernel parameters (constant bank), packed per job:
// w[job * nt + q].  Two capacity tiers keep the parameter block small.
template <typename T, int CAP> struct ColWParam { cx_t<T> w[CAP > 0 ? CAP : 1]; };
template <typename T> struct ColWCap {
    static constexpr int kSmall = 2048 / (int)sizeof(cx_t<T>) * 2;            // 4 KB
    static constexpr int kLarge = (31 * 1024) / (int)sizeof(cx_t<T>);         // 31 KB
};
// Launch all jobs (same tap range/length) in one grid.  pw_host: the launch's
// packed tap pairs (nullptr = read them from `weights` through shared memory).
template <typename T> cudaError_t launch_col(const ColArgs<T>& a, const cx_t<T>* pw_host, cudaStream_t s);
template <typename T> size_t col_smem(int nt, int groups);

// ---- K2u: column pass on the tensor cores (col_umma.cu, fp32 build) ------
// J of the jobs lives in split-fp16 planes: per job slot (hpw complex elements from
// ws, hpw = (H + 2 jpad) * W) a hi plane then a lo plane of half2 (re, im) rows,
// jpad replicate rows above and below the image rows (written by the row kernel).
// J is scaled by 2^jscale_exp(max|f| bits of the image), the taps of a job by 2^wexp.
struct ColUArgs {
    const ColJob<float>* jobs;  // modes 1 / 2 only (X; X + conj(Y); no phase)
    const float2* weights;      // (ka, kb) tap pool, taps -h .. h at jobs[j].wofs
    float2* dst_base;
    int64_t dst_bstride;
    const unsigned* maxbits;    // per image of the chunk
    int64_t ws_img_c;           // complex elements between images in the workspace
    int64_t hpw;                // complex elements per J slot = (H + 2 jbuf) * W
    int H, W, h, njobs, batch;
    int jbuf;                   // replicate rows above / below the image rows in the J planes
    int jpad, K;                // set by the launcher (jpad = h rounded up to 16 <= jbuf)
    int nstrips, nchunks, ch_tiles;
    int dbg;                    // set by the launcher from FGB_UMMA_DBG (ablation only)
    int64_t hw;                 // H * W (set by the launcher): output planes are [plane][H][W] complex
    int64_t dst_planes;         // planes reachable from dst_base (the TMA store map spans them)
};
int col_umma_jpad(int h);
bool col_umma_supported(int h, int W);
size_t col_umma_smem(int h);
// ws / ws_bytes: the J region of the workspace (the tensor map spans it)
cudaError_t launch_col_umma(ColUArgs a, void* ws, int64_t ws_bytes, int sms, cudaStream_t s);
// ---- K1u: row pass on the tensor cores (row_umma.cu, fp32 build) ---------
// Reads x-padded split-fp16 image planes (launch_row_umma_prep), writes the split-fp16
// J slots of ColUArgs (rows + replicate pad rows).  jobs[j]: wofs = row taps (kr, ki)
// for t = 0..h in `weights`, wexp, dst_off[0] = the J slot (complex elements from dst_base).
struct RowUArgs {
    const ColJob<float>* jobs;
    const float2* weights;
    float2* dst_base;
    int64_t dst_bstride;        // complex elements between images (the workspace image stride)
    int64_t hpw;                // complex elements per J slot = (H + 2 jbuf) * W
    int H, W, h, njobs, batch, jbuf;
    int xbuf;                   // replicate columns left / right of the image in the prep planes
    int jpad, K, nstrips, nyb;  // set by the launcher
    int dbg;                    // FGB_UMMA_DBG (ablation only)
};
int row_umma_jpad(int h);
bool row_umma_supported(int h, int W);
size_t row_umma_fprep_bytes(int H, int W, int xbuf, int batch);
cudaError_t launch_row_umma_prep(const float* img, int64_t pitch, int64_t bstride, int H, int W, int xbuf, int batch,
                                 const unsigned* maxbits, void* fprep, cudaStream_t s);
cudaError_t launch_row_umma(RowUArgs a, const void* fprep, int sms, cudaStream_t s);
// ---- K5u: row + column passes of one frequency in one tensor-core kernel (bank_umma.cu) ----
// J stays in shared memory.  Reads the prep planes of launch_row_umma_prep (x-padded by xbuf
// >= h rounded up to 16 columns, y-padded by kBankUPadRows replicate rows); h <= 48.
constexpr int kBankUPadRows = 64;
struct BankUJob {
    int32_t rofs, cofs;         // row taps (kr, ki) t = 0..h / column taps (ka, kb) t = -h..h in `weights`
    int32_t rexp, cexp;         // tap scales 2^rexp, 2^cexp
    int64_t dst_off[2];         // F_theta, F_pi-theta (complex elements from dst_base)
    int32_t nout, pad_;
};
struct BankUArgs {
    const BankUJob* jobs;
    const float2* weights;
    float2* dst_base;
    int64_t dst_bstride;
    const unsigned* maxbits;
    int H, W, h, njobs, batch, xbuf;
    int jpc, Kc, nstrips, nchunks, ch_tiles;  // set by the launcher
    int dbg;                                  // FGB_UMMA_DBG (ablation only)
    int job_fastest;                          // unit order: directs fastest (FGB_BANKU_ORDER)
    int64_t hw;                               // H * W (set by the launcher): output planes are [plane][H][W] complex
    int64_t dst_planes;                       // planes reachable from dst_base (the TMA store map spans them)
};
bool bank_umma_supported(int h, int W);
cudaError_t launch_bank_umma(BankUArgs a, const void* fprep, int sms, cudaStream_t s);
// max|f| bits per image (memset + atomicMax)
cudaError_t launch_absmax(const float* img, int64_t pitch, int64_t bstride, int H, int W, int batch, unsigned* out,
                          int sms, cudaStream_t s);
// J scale exponent from the bits of max|f|: |f 2^e| < 2^13, so |J 2^e| < 2^13 sum|w| (= 2^13 for the
// unit-sum Gaussian) stays inside fp16; 0 for an all-zero or non-finite image
__host__ __device__ inline int jscale_exp(unsigned maxbits) {
    if (maxbits == 0u || maxbits >= 0x7f800000u) return 0;
    const int E = (int)(maxbits >> 23);
    const int x = E == 0 ? -125 : E - 126;  // max|f| < 2^x
    const int e = 13 - x;
    return e < -100 ? -100 : (e > 100 ? 100 : e);
}

// ---- transposes (transpose.cu) -------------------------------------------
// real [H][pitch] -> complex [W][H] (imag 0); complex [H][W] -> complex [W][H]
template <typename T> cudaError_t launch_transpose_real_to_cx(const T* in, int64_t pitch, int64_t in_bstride,
                                                             cx_t<T>* out, int64_t out_bstride, int H, int W,
                                                             int batch, cudaStream_t s);
template <typename T> cudaError_t launch_transpose_real(const T* in, int64_t pitch, int64_t in_bstride, T* out,
                                                       int64_t out_bstride, int H, int W, int batch, cudaStream_t s);
template <typename T> cudaError_t launch_transpose_cx(const cx_t<T>* in, int64_t in_bstride, cx_t<T>* out,
                                                     int64_t out_bstride, int H, int W, int batch, cudaStream_t s);

// ---- fused SDFT for power-of-two windows (sdft_fused.cu) ------------------
template <typename T> struct SdftFusedArgs {
    const T* img;
    int64_t pitch, img_bstride;
    cx_t<T>* out;            // [bins][H][W] (batch 0)
    int64_t out_bstride;     // complex elements between images
    const T* w;              // device: sampled Gaussian w[0..2h]
    const int32_t* heads;    // device: pair heads u to compute
    const int32_t* head_slot;// device: output slot of bin row (u,*) and (M-u,*) per head: [2*nheads]
    int nheads;
    int H, W, h;
    int batch;
};
template <typename T> cudaError_t launch_sdft_fused(const SdftFusedArgs<T>& a, int M, cudaStream_t s);
bool sdft_fused_supported(int M, int h, size_t elem);

// ---- IIR (iir.cu) ---------------------------------------------------------
// Column-direction recursive-Gaussian stage on complex planes, one thread per
// (column, job): modulate by fp64 trig tables, forward/backward 3rd-order
// recursion with fp64 state, recombine (gabor.py:135-164, sdft.py:75-131).
// Modulation pairs of a complex input (jr, ji) with (c, s) = tabm[n]:
//   pair 0: pa = jr c + ji s, pb = jr s - ji c   (Gabor direct / SDFT mirror)
//   pair 1: pa = jr c - ji s, pb = jr s + ji c   (Gabor mirror / SDFT bin)
// Recombination with (c, s) = tabr[y]:
//   Gabor: re = c Sa + s Sb, im = s Sa - c Sb;  SDFT: re = c Sa + s Sb, im = c Sb - s Sa
struct IirCoef { double B, a1, a2, a3; };
template <typename T> struct IirJob {
    int64_t src_off;         // complex elements from src_base
    int64_t tabm_off;        // [H + 2P] modulation table (true coordinate y = n - P)
    int64_t tabr_off;        // [H] recombination table
    int64_t dst_off[4];
    int8_t pair[4];
    int8_t conj[4];
    int32_t nout;
    int32_t need;            // bit 0: pair 0 used, bit 1: pair 1 used (kernel jobs: exactly one)
    int32_t sdft;
    int32_t pad_;
};
template <typename T> struct IirArgs {
    const IirJob<T>* jobs;
    const double2* tab_base;
    const void* src_base;    // T (real_in) or cx_t<T> elements
    cx_t<T>* dst_base;
    T* scratch;              // [njobs*batch][2][len+2P][lines] local forward / backward sequences
    double* state;           // [2][njobs*batch][nseg][2 planes][3][lines] segment boundary states
    const double* g;         // [seglen][3]: first row of A^(m+1)
    const float2* tab32;     // fp32 copy of the tables (same offsets as tab_base; iir32.cu)
    float* state32;          // iir32.cu: [njobs*batch][nseg][12][lines] segment states (aliases `state`)
    int* counters;           // iir32.cu: arrival counter per 32-line block and job; zero on entry, the
                             // last CTA of each block resets its own (library-owned, zeroed once)
    double Aseg[9];          // A^seglen
    double Alast[9];         // A^(length of the last segment)
    int64_t src_bstride, dst_bstride;  // per image, in source / complex elements
    int64_t src_ls, src_ss;  // source element strides per line / per sample
    int64_t dst_ls, dst_ss;  // destination strides per line / per sample
    IirCoef c;
    int len, lines, P;       // samples per line (unpadded), independent lines, pad
    int njobs, batch;
    int nseg, seglen;
    int real_in;
    int one_out;             // every job has exactly one output
};
template <typename T> cudaError_t launch_iir(const IirArgs<T>& a, cudaStream_t s);
// fp32 build: parallel-form sections in fp32, two passes + carries, no scratch
// planes (iir32.cu).  Segments of exactly kIir32M samples (nseg = ceil(L / kIir32M)).
constexpr int kIir32M = 32;
bool iir32_enabled();  // false when FGB_IIR64 is set (the fp64-state kernels of iir.cu for A/B runs)
// (q_r, Re q_c, Im q_c, c_r, Re c_c, Im c_c): poles and residues of the parallel form
void iir32_sections(const IirCoef& c, double out[6]);
cudaError_t launch_iir32(const IirArgs<float>& a, cudaStream_t s);
template <typename T> size_t iir_scratch_elems(int len, int lines, int P, int njobs, int batch);
size_t iir_state_doubles(int lines, int nseg, int njobs, int batch);

// ---- 1-D line smoothing (smooth.cu; smooth_lines gaussian.py:245-285) -----
template <typename T> struct LinesCorrArgs {
    const T* in;             // [n_lines][pitch]
    T* out;                  // [n_lines][out_pitch]
    const T* w;              // device taps w[0..nt-1] at offsets t0..t0+nt-1
    int64_t pitch, out_pitch;
    int n_lines, len, t0, nt;
    int zero_boundary;       // 0 = replicate (FIR "nearest"), 1 = zero (box)
};
template <typename T> struct LinesIirArgs {
    const T* in;
    T* out;
    double* scratch;         // [len + 2P][n_lines] forward sequence
    int64_t pitch, out_pitch;
    int n_lines, len, P;
    IirCoef c;
};
template <typename T> cudaError_t launch_lines_corr(const LinesCorrArgs<T>& a, cudaStream_t s);
template <typename T> cudaError_t launch_lines_iir(const LinesIirArgs<T>& a, cudaStream_t s);

// ---- SER on the device (ser.cu; metrics.py:63-83) -------------------------
// scratch[0..3] <- (sum tr^2, sum (ar-tr)^2, sum ti^2, sum (ai-ti)^2); scratch holds
// ser_scratch_doubles() doubles.  Deterministic (fixed-order two-pass reduction).
size_t ser_scratch_doubles();
template <typename T>
cudaError_t launch_ser(const cx_t<T>* a, const cx_t<T>* t, int64_t n, double* scratch, cudaStream_t s);

// ---- output layout conversion (gbnk.cu) -----------------------------------
// [entries][plane] interleaved complex -> [entries][2][plane] f64 (re plane,
// im plane), *nonfinite |= 1 if any value is NaN / inf.
template <typename T>
cudaError_t launch_entries_planar(const cx_t<T>* in, int64_t n, int64_t plane, double* out, int* nonfinite,
                                  cudaStream_t s);

// ---- brute-force 2-D references (bruteforce.cu) ---------------------------
template <typename T> struct Direct2DArgs {
    const T* img;
    int64_t pitch, img_bstride;
    cx_t<T>* out;
    int64_t out_bstride;
    const cx_t<T>* kern;   // [ky][kx] complex kernel (device)
    int ky, kx, oy, ox;    // input row/col = y + iy - oy, x + ix - ox
    int zero_boundary;
    int H, W, batch;
};
template <typename T> cudaError_t launch_direct2d(const Direct2DArgs<T>& a, cudaStream_t s);
template <typename T> size_t direct2d_smem(int ky, int kx);

// ---- fused small-sigma bank stage (bank_fused.cu) ------------------------
struct BankFusedOut {
    int64_t direct;  // complex elements from dst (batch 0) of F_theta
    int64_t mirror;  // of F_{pi - theta}, or -1
};
struct BankFusedArgs {
    const float* img;
    int64_t pitch, img_bstride;
    float2* dst;
    int64_t dst_bstride;
    int H, W, h, nd, batch;
    int col_w_off;               // float offset of the column taps in BankFusedW
    BankFusedOut out[kMaxND];
};
struct BankFusedW {
    static constexpr int kCap = 7168;  // floats (28 KB): row taps [(hp+1)][NDP][2], column taps [nd][ntp][2]
    float w[kCap];
};
bool bank_fused_ok(int h, int nd);
size_t bank_fused_smem(int h, int nd, int TY);
inline int bank_fused_pad(int n) { return (n + 3) & ~3; }  // row taps (hp) / column taps (ntp) in 4-tap chunks
cudaError_t launch_bank_fused(const BankFusedArgs& a, const BankFusedW& w, cudaStream_t s);

}  // namespace fgb
