/*
 * fgb200.h -- C ABI of the B200-native fastgabor hot path (libfgb200.so).
 *
 * Plain C types only (no CUDA / torch types): device buffers are passed as
 * `void*` device pointers, CUDA streams as `void*` (a cudaStream_t, NULL =
 * legacy default stream).  Every call returns FGB_OK (0) or a negative status;
 * fgb_last_error() returns a thread-local message for the last failure.
 *
 * Reference interfaces replaced (paths relative to
 * /root/reference/pkg/src/fastgabor):
 *
 *   fgb_bank            compute_bank          bank.py:90-129   (reuse = 1)
 *                       compute_bank_noreuse  bank.py:132-157  (reuse = 0)
 *   fgb_filter          gabor_filter          gabor.py:172-176
 *   fgb_horizontal_stage horizontal_stage     gabor.py:107-132
 *   fgb_vertical_stage  vertical_stage        gabor.py:167-169
 *                       vertical_stage_conjugate bank.py:68-74 (conjugate = 1)
 *   fgb_sdft            sdft_full             sdft.py:178-213
 *   fgb_sdft_bin        sdft_bin              sdft.py:169-175
 *   fgb_sdft_horizontal sdft_horizontal       sdft.py:134-150
 *   fgb_fir_gabor       fir_gabor             oracle.py:53-66   (GPU brute force)
 *   fgb_localized_dft   localized_dft         oracle.py:69-109  (GPU brute force)
 *   fgb_gbnk_write_device write_bank_container image_io.py:157-179 (device-fed)
 *   fgb_iir_coeffs      make_coeffs           gaussian.py:164-185
 *   fgb_sampled_gaussian sampled_gaussian     gaussian.py:188-195
 *   fgb_pad_radius      pad_radius            gaussian.py:198-212
 *   fgb_ser_sums        ser                   metrics.py:63-83  (device reduction)
 *   fgb_smooth_lines    smooth_lines          gaussian.py:245-285
 *                       (smooth_1d / smooth_pair_1d gaussian.py:288-302 are
 *                        one / two lines of it)
 *
 * The *_host variants take HOST buffers and do the host<->device copies
 * (through pinned staging) inside the call: they are what the reference-side
 * binding calls.
 *
 * Data layout in HBM
 *   image  : real, row-major [batch][height][pitch] (pitch in elements >= width)
 *   output : interleaved complex (float2 / double2), dense [batch][entry][height][width]
 *            bank entries in reference order (frequency-major, then k = 0..N-1,
 *            bank.py:121-128); SDFT bins in u-major order (bin = u*my + v).
 */
#ifndef FGB200_H
#define FGB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FGB_OK 0
#define FGB_EINVAL (-1)        /* bad parameter (reference raises ValueError)   */
#define FGB_ECUDA (-2)         /* CUDA runtime error                            */
#define FGB_ENOMEM (-3)        /* device / pinned allocation failed             */
#define FGB_EUNSUPPORTED (-4)  /* smoother kind not valid here (TypeError)      */
#define FGB_ENCCL (-5)         /* NCCL error (fgb_mgpu_*)                       */

#define FGB_F32 0
#define FGB_F64 1

#define FGB_SMOOTH_FIR 0  /* ExactFIR(radius)   gaussian.py:41-49 */
#define FGB_SMOOTH_IIR 1  /* RecursiveIIR()     gaussian.py:36-38 */
#define FGB_SMOOTH_BOX 2  /* Box(half_width)    gaussian.py:52-60 */

typedef struct fgb_smoother {
    int32_t kind;      /* FGB_SMOOTH_*                                      */
    int32_t box_half;  /* Box half width (kind == FGB_SMOOTH_BOX)           */
    double radius;     /* FIR truncation radius in sigmas (kind == FIR)     */
} fgb_smoother;

/* Image geometry shared by every entry point. */
typedef struct fgb_image {
    int32_t height, width;
    int64_t pitch;          /* elements between rows (>= width)             */
    int32_t batch;          /* images                                       */
    int32_t dtype;          /* FGB_F32 or FGB_F64 (input and output)        */
    int64_t batch_stride;   /* elements between images (>= height*pitch)    */
} fgb_image;

/* Filter bank (BankSpec bank.py:23-52).  sigmas[] are explicit values: the
 * host resolves the sigma = 2*pi/omega rule (bank.py:45-48). */
typedef struct fgb_bank_desc {
    fgb_image img;
    int32_t n_freq;
    int32_t orientations;     /* N, theta_k = k*pi/N                          */
    const double* omegas;     /* [n_freq] host array                          */
    const double* sigmas;     /* [n_freq] host array                          */
    fgb_smoother smoother;
    int32_t reuse;            /* 1 = compute_bank, 0 = compute_bank_noreuse   */
    /* Optional shard: a list of work units u = i*(N/2+1) + k (k <= N/2) to
     * compute (reuse mode).  NULL = all.  With a unit list the output is
     * compact: per listed unit its direct entry, then its mirror N-k when it
     * exists (bank.py:112-115). */
    const int32_t* units;
    int32_t n_units;
} fgb_bank_desc;

/* Single filter (GaborParams gabor.py:68-90); theta is normalised mod pi. */
typedef struct fgb_filter_desc {
    fgb_image img;
    double omega, theta, sigma;
    fgb_smoother smoother;
} fgb_filter_desc;

/* Localized SDFT (SdftSpec sdft.py:25-57).  sigma <= 0 selects the rule
 * floor(min(mx,my)/2)/3 (sdft.py:45-49). */
typedef struct fgb_sdft_desc {
    fgb_image img;
    int32_t mx, my;
    double sigma;
    fgb_smoother smoother;
    /* Optional shard: list of pair heads u in [0, mx/2]; each computes bins
     * (u, *) and (mx-u, *).  NULL = all bins in [mx*my] order.  With a list
     * the output is compact: per head, rows (u, 0..my-1) then (mx-u, 0..my-1)
     * when mx-u != u and u != 0. */
    const int32_t* u_heads;
    int32_t n_heads;
} fgb_sdft_desc;

/* Independent 1-D lines (smooth_lines gaussian.py:245-285): real rows of a
 * [n_lines][pitch] array, each smoothed along its length; output dense
 * [n_lines][len] of the same dtype.
 *   FGB_SMOOTH_FIR: correlation with the unit-sum sampled Gaussian (half
 *                   support max(1, ceil(radius*sigma))), replicate ("nearest")
 *                   boundary (gaussian.py:231-233);
 *   FGB_SMOOTH_IIR: replicate pad ceil(5 sigma)+2 (none with assume_padded),
 *                   forward + backward recursion with lfilter_zi steady-state
 *                   init, crop (gaussian.py:215-228); fp64 state;
 *   FGB_SMOOTH_BOX: sum over offsets [box_lo, box_hi], zero outside the line
 *                   (Box(h) = [-h, h], _AsymBox(lo, hi); gaussian.py:236-242);
 *                   smoother.box_half is ignored. */
typedef struct fgb_lines_desc {
    int32_t n_lines, len;
    int64_t pitch;            /* elements between lines (>= len)              */
    int32_t dtype;            /* FGB_F32 or FGB_F64                           */
    int32_t assume_padded;    /* IIR: caller padded already (gaussian.py:265) */
    double sigma;
    fgb_smoother smoother;
    int32_t box_lo, box_hi;
} fgb_lines_desc;

/* ---- library ----------------------------------------------------------- */
const char* fgb_last_error(void);
int32_t fgb_version(void);                  /* major*10000 + minor*100 + patch */
int32_t fgb_device_sm_count(void);

/* ---- host-side coefficient math (no GPU needed) ------------------------- */
int32_t fgb_pad_radius(const fgb_smoother* kind, double sigma);
int32_t fgb_sampled_gaussian(double sigma, double radius, double* out, int32_t cap, int32_t* half);
int32_t fgb_iir_coeffs(double sigma, double out_b_a1_a2_a3[4]);
/* The same filter in parallel form (what the fp32 kernels run): real pole q_r,
 * complex pole q_c (Im > 0), residues c_r, c_c, with
 * B / (1 + a1 z^-1 + a2 z^-2 + a3 z^-3) = c_r / (1 - q_r z^-1) + 2 Re[c_c / (1 - q_c z^-1)].
 * out = (q_r, Re q_c, Im q_c, c_r, Re c_c, Im c_c). */
int32_t fgb_iir_sections(double sigma, double out[6]);
/* Number of output entries / bins a call writes (for allocation). */
int64_t fgb_bank_entries(const fgb_bank_desc* d);
int64_t fgb_sdft_bins(const fgb_sdft_desc* d);

/* Device workspace (bytes) the library allocates for such a call (J planes,
 * IIR scratch, segment states for one chunk of images; grow-only, kept
 * across calls).  Builds and caches the call's plan; needs a CUDA device. */
int64_t fgb_bank_workspace_bytes(const fgb_bank_desc* d);
int64_t fgb_sdft_workspace_bytes(const fgb_sdft_desc* d);

/* ---- device-pointer entry points (stream ordered, async) --------------- */
int32_t fgb_bank(const fgb_bank_desc* d, const void* img, void* out, void* stream);
int32_t fgb_filter(const fgb_filter_desc* d, const void* img, void* out, void* stream);
int32_t fgb_horizontal_stage(const fgb_filter_desc* d, const void* img, void* j_out, void* stream);
int32_t fgb_vertical_stage(const fgb_filter_desc* d, const void* j_in, void* out, int32_t conjugate, void* stream);
int32_t fgb_sdft(const fgb_sdft_desc* d, const void* img, void* out, void* stream);
int32_t fgb_sdft_bin(const fgb_sdft_desc* d, int32_t u, int32_t v, const void* img, void* out, void* stream);
int32_t fgb_sdft_horizontal(const fgb_sdft_desc* d, int32_t u, const void* img, void* j_out, void* stream);
int32_t fgb_smooth_lines(const fgb_lines_desc* d, const void* lines, void* out, void* stream);

/* ---- host-buffer entry points (copies inside; synchronous) ------------- */
int32_t fgb_bank_host(const fgb_bank_desc* d, const void* img_host, void* out_host);
int32_t fgb_filter_host(const fgb_filter_desc* d, const void* img_host, void* out_host);
int32_t fgb_sdft_host(const fgb_sdft_desc* d, const void* img_host, void* out_host);
int32_t fgb_horizontal_stage_host(const fgb_filter_desc* d, const void* img_host, void* j_host);
int32_t fgb_vertical_stage_host(const fgb_filter_desc* d, const void* j_host, void* out_host, int32_t conjugate);
int32_t fgb_sdft_bin_host(const fgb_sdft_desc* d, int32_t u, int32_t v, const void* img_host, void* out_host);
int32_t fgb_sdft_horizontal_host(const fgb_sdft_desc* d, int32_t u, const void* img_host, void* j_host);
int32_t fgb_smooth_lines_host(const fgb_lines_desc* d, const void* lines_host, void* out_host);
/* Same calls returning the reference's ComplexImage layout directly:
 * [batch][entries][2][H][W] float64 (re plane, im plane per entry), converted
 * on the GPU; *nonfinite = 1 if any output value is NaN / inf (the reference
 * rejects such images, image_io.py:65-66).  Used by the Python drop-in API. */
int32_t fgb_bank_host_planar(const fgb_bank_desc* d, const void* img_host, double* out_host, int32_t* nonfinite);
int32_t fgb_filter_host_planar(const fgb_filter_desc* d, const void* img_host, double* out_host, int32_t* nonfinite);
int32_t fgb_sdft_host_planar(const fgb_sdft_desc* d, const void* img_host, double* out_host, int32_t* nonfinite);

/* ---- brute-force references (oracle.py:53-109), direct 2-D tap sums ---- */
/* fir_gabor(f, p, OracleConfig(radius)): replicate boundary.  localized_dft(f,
 * u, v, spec, OracleConfig(radius)): Gaussian (replicate) or box (zero)
 * window.  O(support^2) per pixel; validation / `compare` at full size. */
int32_t fgb_fir_gabor(const fgb_filter_desc* d, double radius, const void* img, void* out, void* stream);
int32_t fgb_localized_dft(const fgb_sdft_desc* d, int32_t u, int32_t v, double radius, const void* img, void* out,
                          void* stream);
int32_t fgb_fir_gabor_host(const fgb_filter_desc* d, double radius, const void* img_host, void* out_host);
int32_t fgb_localized_dft_host(const fgb_sdft_desc* d, int32_t u, int32_t v, double radius, const void* img_host,
                               void* out_host);

/* ---- SER on the device (metrics.py:63-83) ------------------------------ */
/* approx, truth: n interleaved complex device elements (FGB_F32 / FGB_F64).
 * out = (sum tr^2, sum (ar - tr)^2, sum ti^2, sum (ai - ti)^2) in fp64, a
 * deterministic reduction; SER(part) = 10 log10(signal / error) with the
 * reference's +inf / -inf sentinels applied by the caller.  Synchronous. */
int32_t fgb_ser_sums(const void* approx, const void* truth, int64_t n, int32_t dtype, double out[4], void* stream);

/* ---- GBNK container from device outputs (image_io.py:157-179) ---------- */
/* Writes n_entries interleaved-complex [H][W] device planes (dtype FGB_F32 /
 * FGB_F64) as float64 re/im planes with params[3*k..3*k+2] = (omega, theta,
 * sigma) or (u, v, sigma); sdft != 0 sets the SDFT flag bit.  Synchronous:
 * the D2H of entry k+1 overlaps the file write of entry k. */
int32_t fgb_gbnk_write_device(const char* path, const double* params, int32_t n_entries, int32_t height, int32_t width,
                              int32_t dtype, const void* dev_entries, int32_t sdft, void* stream);

/* ---- multi-GPU: one process per GPU, library-owned NCCL communicator ---- */
/* (replaces the reference's orientation thread pool,
 * bank.py:77-87.)  Rank 0 calls fgb_mgpu_unique_id and the host shares the
 * 128 bytes (torch.distributed / MPI / a file); every rank calls
 * fgb_mgpu_init.  The only collective is one ncclBroadcast of rank 0's input
 * image into every rank's device buffer `img` (same geometry everywhere), then
 * each rank computes its share into its own compact output:
 *   bank: the (frequency, direct k) units of fgb_mgpu_bank_units -- contiguous
 *         runs per rank from an exact linear partition over a B200-measured
 *         device-time model + local search (parallel.py:partition_units);
 *         output layout as fgb_bank_desc.units; fgb_mgpu_bank_entries gives its
 *         entry count;
 *   SDFT: the conjugate u-pair heads of fgb_mgpu_sdft_heads (layout as
 *         fgb_sdft_desc.u_heads).
 * The *_units / *_heads partition functions are host-only (no GPU, no NCCL). */
#define FGB_MGPU_ID_BYTES 128
int32_t fgb_mgpu_unique_id(unsigned char id[FGB_MGPU_ID_BYTES]);
int32_t fgb_mgpu_init(const unsigned char id[FGB_MGPU_ID_BYTES], int32_t world, int32_t rank, int32_t device);
int32_t fgb_mgpu_finalize(void);
int32_t fgb_mgpu_bank_units(const fgb_bank_desc* d, int32_t world, int32_t rank, int32_t* units, int32_t cap);
int32_t fgb_mgpu_sdft_heads(int32_t m, int32_t world, int32_t rank, int32_t* heads, int32_t cap);
int32_t fgb_mgpu_bank_entries(const fgb_bank_desc* d);
int32_t fgb_mgpu_bank(const fgb_bank_desc* d, void* img, void* out, void* stream);
int32_t fgb_mgpu_sdft(const fgb_sdft_desc* d, void* img, void* out, void* stream);
const char* fgb_mgpu_last_error(void);

/* ---- measurement ------------------------------------------------------- */
/* Live per-kernel timing: while enabled, every launch is bracketed by CUDA
 * events on its stream; fgb_profile_read synchronises them and aggregates by
 * kernel name (algorithmic flops = reference OpCounters M + A of the stage
 * work, bytes = compulsory input + output traffic). */
typedef struct fgb_prof_entry {
    char name[16];
    int64_t launches;
    double ms;
    double flops;
    double bytes;
} fgb_prof_entry;
void fgb_profile_enable(int32_t on);
int32_t fgb_profile_read(fgb_prof_entry* out, int32_t cap);
int64_t fgb_launch_count(void);      /* kernels launched by this library so far */
double fgb_probe_fp32_tflops(void);  /* FFMA peak probe (K6), TFLOP/s */
double fgb_probe_fp64_tflops(void);  /* DFMA peak probe (K6), TFLOP/s */
/* FMA probe by operand form: mode 0 immediate operands, 1 register operands
 * with a shared multiplier (operand reuse), 2 three distinct registers,
 * 3 constant-bank multiplier, 4 / 5 packed fp32x2 FFMA2 with a constant /
 * register multiplier (fp32 only). */
double fgb_probe_fma(int32_t dtype, int32_t mode);

/* ---- synchronisation helper for hosts without a CUDA binding ----------- */
int32_t fgb_stream_synchronize(void* stream);
/* Frees cached plans, workspaces and pinned staging of this process. */
void fgb_release_caches(void);

#ifdef __cplusplus
}
#endif
#endif /* FGB200_H */
