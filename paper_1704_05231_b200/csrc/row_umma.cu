// K1u: fp32-build row stage of the Gabor bank on the tensor cores (tcgen05,
// split-fp16), writing the split-fp16 J planes the column pass (col_umma.cu)
// reads.
//
// Reference semantics: horizontal_stage (gabor.py:107-132).  With the
// modulation folded into the taps, for one direct
// orientation (row phase step omega_c = omega cos theta):
//     J(y, x) = sum_{t=-h..h} w[t] e^{-i omega_c t} f[y, clamp(x+t)].
// Over a tile of 64 output columns x 128 image rows this is a banded Toeplitz
// product D (128 x 128) = Wt (128 x K) . Ft (K x 128):
//   * M row 2 xl / 2 xl + 1 = Re / Im taps of output column xl (kr[|t|],
//     sgn(t) ki[|t|]) at K column k = xl + jpad + t (zero outside the band),
//   * K = 64 + 2 jpad input columns (jpad = h rounded up to 32, so the window
//     is whole 64-column TMA boxes), read from x-padded split-fp16 image
//     planes (replicate padding: clamp() costs nothing),
//   * N = 128 image rows (the image rows are the K-major B operand).
// Precision as in col_umma.cu: f 2^e = f_hi + f_lo (the image prep kernel),
// taps 2^s = w_hi + w_lo, D = Wh Fh + Wh Fl + Wl Fh in fp32 (TMEM); the
// epilogue multiplies by 2^-s, giving J 2^e, and splits it into the hi / lo
// half2 planes.
//
// Persistent warp-specialised CTA (one per SM): warp 8 TMA producer (64-column
// x 128-row boxes of the hi and lo image planes = one 32 KB ring stage per
// 64 K columns), warp 9 TMEM allocator + MMA issuer (K/16 steps x 3 MMAs,
// M = 128, N = 128, K-major B with 128-byte swizzle), warps 0-7 epilogue
// (TMEM lane quadrant w % 4 = 16 output columns, column half w / 4 = 64 image
// rows): TMEM -> shared transpose -> hi / lo split -> row-contiguous stores,
// (the jbuf replicate pad rows are filled by jpad_fill_kernel afterwards).  Work
// unit = one tile (direct, image, 128-row block, 64-column strip), strips
// fastest; the taps of a direct are (re)built in TMEM when it changes.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kernels.h"
#include "umma.cuh"

namespace fgb {

namespace {

constexpr int kTX = 64;            // output columns per tile
constexpr int kTY = 128;           // image rows per tile (MMA N)
constexpr int kStageBytes = 32768; // 64 K columns: (hi, lo) x 128 rows x 128 B
constexpr int kStages = 5;
constexpr int kEpiWarps = 8;
constexpr int kEpiThreads = 32 * kEpiWarps;
constexpr int kTmaWarp = kEpiWarps, kMmaWarp = kEpiWarps + 1;
constexpr int kThreads = 32 * (kEpiWarps + 2);
constexpr uint32_t kAcc = 128;
constexpr int kStgPitch = 36;      // floats per staged image row: a warp's 32 M rows + 4 (conflict-free)
constexpr int kStgBytes = kEpiWarps * 32 * kStgPitch * 4;  // one [32 image rows][32 M rows] block per warp

__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + max(-126, min(127, e))) << 23); }

// Each CTA runs a contiguous range of units (consecutive strips of one row block: the
// column halo of a tile is the previous tile's, still in L2); the unit coordinates are
// decoded once and then stepped (no integer division per tile).
struct UnitIter {
    int u, u1, job, b, yb, strip;
    __device__ UnitIter(const RowUArgs& a, int nunits) {
        u = (int)((int64_t)blockIdx.x * nunits / gridDim.x);
        u1 = (int)((int64_t)(blockIdx.x + 1) * nunits / gridDim.x);
        strip = u % a.nstrips;
        int r = u / a.nstrips;
        yb = r % a.nyb;
        r /= a.nyb;
        b = r % a.batch;
        job = r / a.batch;
    }
    __device__ bool ok() const { return u < u1; }
    __device__ void next(const RowUArgs& a) {
        ++u;
        if (++strip == a.nstrips) {
            strip = 0;
            if (++yb == a.nyb) {
                yb = 0;
                if (++b == a.batch) {
                    b = 0;
                    ++job;
                }
            }
        }
    }
};

__global__ void __launch_bounds__(kThreads, 1)
    row_umma_kernel(const __grid_constant__ CUtensorMap fmap, const __grid_constant__ RowUArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint64_t full[kStages], empty[kStages], tfull[3], tempty[3], aready;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int K = a.K, kst = a.K / 64;  // ring stages per tile (K = 64 + 2 jpad, jpad a multiple of 32)
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 3; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], kEpiThreads);
        }
        mbar_init(&aready, kEpiThreads);
    }
    if (warp == kMmaWarp) umma::tmem_alloc(&tmem_base, 512);
    if (warp == kTmaWarp && lane == 0) umma::tma_prefetch_desc(&fmap);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tb = tmem_base;
    // accumulators: 3 buffers when the taps (K columns) leave room in the 512 TMEM columns, else 2
    const uint32_t nacc = (512 - K) >= 3 * (int)kAcc ? 3u : 2u;
    const uint32_t a_hi = tb + nacc * kAcc, a_lo = a_hi + (uint32_t)(K / 2);
    const int nunits = a.njobs * a.batch * a.nyb * a.nstrips;

    if (warp == kTmaWarp) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            uint32_t g = 0;
            bool run = false;
            for (UnitIter it(a, nunits); it.ok(); it.next(a)) {
                const int b = it.b, yb = it.yb, strip = it.strip;
                const int xs = strip * kTX - a.jpad + a.xbuf;  // padded-plane column of K column 0
                // consecutive strips of a row block share all but one 64-column stage: the window slides,
                // only the new stage is loaded (K / 64 times less TMA and L2 traffic than a fresh window)
                const int q0 = (run && strip > 0) ? kst - 1 : 0;
                run = true;
                for (int q = q0; q < kst; ++q, ++g) {
                    const uint32_t slot = g % (uint32_t)kStages, round = g / (uint32_t)kStages;
                    mbar_wait(&empty[slot], (round & 1u) ^ 1u);
                    uint8_t* sp = ring + slot * kStageBytes;
                    if (a.dbg & 4) {  // A/B knob: no image loads
                        umma::mbar_arrive(&full[slot]);
                        continue;
                    }
                    mbar_arrive_expect_tx(&full[slot], kStageBytes);
                    const int yr = yb * kTY + kBankUPadRows;  // padded-plane row of image row yb * kTY
                    umma::tma_load_3d(sp, &fmap, xs + 64 * q, yr, 2 * b, &full[slot]);
                    umma::tma_load_3d(sp + 16384, &fmap, xs + 64 * q, yr, 2 * b + 1, &full[slot]);
                }
            }
        }
    } else if (warp == kMmaWarp) {
        // ---------------- MMA issuer (the whole warp runs the loop; one elected lane issues) ----------------
        {
            const uint32_t idesc = umma::idesc_f16_f32(128, kTY, false, false);
            const uint64_t rdesc0 = umma::smem_desc(smem_u32(ring), 16, 1024, umma::kLayoutSw128);
            const bool do_mma = !(a.dbg & 2);  // A/B knob: no MMAs
            uint32_t gw = 0, gnext = 0, t = 0, nreload = 0;  // first ring stage of the tile's window; stages issued
            bool run = false;
            int cur = -1;
            for (UnitIter it(a, nunits); it.ok(); it.next(a), ++t) {
                const int job = it.job;
                if (run && it.strip > 0) {
                    ++gw;
                    ++gnext;
                } else {
                    gw = gnext;
                    gnext += kst;
                }
                run = true;
                if (job != cur) {
                    mbar_wait(&aready, nreload & 1u);
                    ++nreload;
                    cur = job;
                    umma::fence_after();
                }
                const uint32_t buf = t % nacc, ph = (t / nacc) & 1u;
                mbar_wait(&tempty[buf], ph ^ 1u);
                umma::fence_after();
                const uint32_t d = tb + buf * kAcc;
                // one elect region per ring stage (12 MMAs), descriptors advance by constants (K is a
                // multiple of 64): the issuing warp stays well under the MMAs' execution time
                for (int st = 0; st < kst; ++st) {
                    const uint32_t gs = gw + st;
                    const uint32_t slot = gs % (uint32_t)kStages;
                    mbar_wait(&full[slot], (gs / (uint32_t)kStages) & 1u);
                    umma::fence_after();
                    const uint64_t bh0 = rdesc0 + (uint64_t)(slot * (kStageBytes >> 4));
                    if (do_mma && umma::elect_one()) {
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            // K-major, 128-byte swizzle: K step = 32 bytes inside the swizzle atom
                            const uint64_t bh = bh0 + (uint64_t)(2 * q), bl = bh + (uint64_t)(16384 >> 4);
                            const uint32_t ah = a_hi + 8 * (4 * st + q), al = ah + (uint32_t)(K / 2);
                            umma::mma_f16_ts(d, ah, bh, idesc, (st | q) ? 1u : 0u);
                            umma::mma_f16_ts(d, ah, bl, idesc, 1u);
                            umma::mma_f16_ts(d, al, bh, idesc, 1u);
                        }
                    }
                    __syncwarp();
                }
                if (umma::elect_one()) umma::mma_commit(&tfull[buf]);
                __syncwarp();
            }
        }
        __syncwarp();
    } else {
        // ---------------- epilogue ----------------
        const int quad = warp & 3, half = warp >> 2;
        const int m = 32 * quad + lane;  // TMEM lane = M row = (output column xl = m / 2, Re / Im)
        const uint32_t lane_addr = (uint32_t)(32 * quad) << 16;
        const int xl = m >> 1, im = m & 1;
        float* stg = reinterpret_cast<float*>(ring + kStages * kStageBytes) + warp * 32 * kStgPitch;
        int cur = -1;
        uint32_t t = 0, gw = 0, gnext = 0;
        bool run = false;
        float inv_w = 1.f;
        const int H = a.H, W = a.W, jbuf = a.jbuf;
        const int64_t hpw = a.hpw;
        for (UnitIter it(a, nunits); it.ok(); it.next(a), ++t) {
            const int job = it.job, b = it.b, yb = it.yb, strip = it.strip;
            const ColJob<float>& jb = a.jobs[job];
            if (job != cur) {
                // tap row m: K column k -> t = k - jpad - xl: (kr[|t|], sgn(t) ki[|t|]) * 2^wexp
                const float2* w = a.weights + jb.wofs;
                const float wsc = pow2f(jb.wexp);
                inv_w = pow2f(-jb.wexp);
                for (int c = 16 * half; c < K / 2; c += 32) {
                    uint32_t hi[16], lo[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        float v[2];
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int tt = 2 * (c + i) + e - a.jpad - xl;
                            const int at = tt < 0 ? -tt : tt;
                            float x = 0.f;
                            if (at <= a.h) {
                                const float2 kk = w[at];
                                x = (im ? (tt < 0 ? -kk.y : kk.y) : kk.x) * wsc;
                            }
                            v[e] = x;
                        }
                        umma::split_f16x2(v[0], v[1], hi[i], lo[i]);
                    }
                    umma::tmem_st16(a_hi + lane_addr + c, hi);
                    umma::tmem_st16(a_lo + lane_addr + c, lo);
                }
                umma::tmem_st_wait();
                umma::fence_before();
                umma::mbar_arrive(&aready);
                cur = job;
            }
            uint32_t* jh = reinterpret_cast<uint32_t*>(a.dst_base + jb.dst_off[0] + (int64_t)b * a.dst_bstride);
            // write-out item of this lane: image row 8 it + (lane >> 2) of a 32-row pass, output columns
            // 16 quad + 4 cg .. + 3 (the warp's 16 columns: 64 bytes per row and plane)
            const int cg = lane & 3, rl = lane >> 2;
            const int xs = 16 * quad + 4 * cg;  // column within the strip
            const bool xok = strip * kTX + xs < W;
            const int Hp = H + 2 * jbuf;
            uint32_t* js = jh + (int64_t)strip * Hp * 64 + xs;  // strip-major plane: [strip][Hp][64]
            const uint32_t buf = t % nacc, ph = (t / nacc) & 1u;
            mbar_wait(&tfull[buf], ph);
            umma::fence_after();
            if (run && strip > 0) {
                ++gw;
                ++gnext;
            } else {
                gw = gnext;
                gnext += kst;
            }
            run = true;
            if (threadIdx.x == 0) {
                // the tile's MMAs are done (no per-stage commits): the window's oldest stage is free; all of
                // them when the next unit does not continue this run of strips
                const bool cont = it.u + 1 < it.u1 && strip + 1 < a.nstrips;
                const int nrel = cont ? 1 : kst;
                for (int q = 0; q < nrel; ++q) umma::mbar_arrive(&empty[(gw + q) % (uint32_t)kStages]);
            }
            float v[64];  // both 32-row passes of this warp's 64 image rows, one TMEM wait
#pragma unroll
            for (int j = 0; j < 4; ++j)
                umma::tmem_ld16(tb + lane_addr + buf * kAcc + 64 * half + 16 * j, *reinterpret_cast<float(*)[16]>(v + 16 * j));
            umma::tmem_ld_wait();
            umma::fence_before();
            umma::mbar_arrive(&tempty[buf]);  // accumulator drained: the MMA may reuse it
#pragma unroll
            for (int qq = 0; qq < 2; ++qq) {
                // per-warp staging [32 image rows][32 M rows (+4)]: transposed through shared memory
                __syncwarp();
#pragma unroll
                for (int j = 0; j < 32; ++j) stg[j * kStgPitch + lane] = v[32 * qq + j];
                __syncwarp();
                const int y0 = yb * kTY + 64 * half + 32 * qq + rl;
                uint32_t* pq = js + (int64_t)(y0 + jbuf) * 64;
#pragma unroll
                for (int it = 0; it < 4; ++it) {
                    const int y = y0 + 8 * it;
                    const float* sr = stg + (rl + 8 * it) * kStgPitch + 8 * cg;
                    const float4 p0 = *reinterpret_cast<const float4*>(sr);
                    const float4 p1 = *reinterpret_cast<const float4*>(sr + 4);
                    uint4 hw, lw;
                    umma::split_f16x2(p0.x * inv_w, p0.y * inv_w, hw.x, lw.x);
                    umma::split_f16x2(p0.z * inv_w, p0.w * inv_w, hw.y, lw.y);
                    umma::split_f16x2(p1.x * inv_w, p1.y * inv_w, hw.z, lw.z);
                    umma::split_f16x2(p1.z * inv_w, p1.w * inv_w, hw.w, lw.w);
                    if (y < H && xok && !(a.dbg & 1)) {
                        uint32_t* p = pq + 8 * it * 64;
                        *reinterpret_cast<uint4*>(p) = hw;
                        *reinterpret_cast<uint4*>(p + hpw) = lw;
                    }
                }
            }
        }
    }
    umma::fence_before();
    __syncthreads();
    if (warp == kMmaWarp) umma::tmem_dealloc(tb, 512);
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return (EncodeFn)p;
    }();
    return fn;
}

// image -> x- and y-padded split-fp16 planes: plane 2b = hi, 2b + 1 = lo of (f 2^e), replicate
// padding (xbuf columns, kBankUPadRows rows on each side: plane row yp = image row yp - kBankUPadRows)
__global__ void fprep_kernel(const float* __restrict__ img, int64_t pitch, int64_t bstride, int H, int W, int xbuf,
                             int Wp, const unsigned* __restrict__ maxbits, __half* __restrict__ out) {
    const int b = blockIdx.z, yp = blockIdx.y, Hq = H + 2 * kBankUPadRows;
    const int y = min(max(yp - kBankUPadRows, 0), H - 1);
    const float sc = pow2f(jscale_exp(maxbits[b]));
    const float* row = img + (int64_t)b * bstride + (int64_t)y * pitch;
    __half* hi = out + ((int64_t)(2 * b) * Hq + yp) * Wp;
    __half* lo = out + ((int64_t)(2 * b + 1) * Hq + yp) * Wp;
    // 8 output columns per thread: 16-byte stores (Wp % 8 == 0), 16-byte loads inside the image
    const bool vin = ((reinterpret_cast<uintptr_t>(row) & 15) == 0) && (xbuf & 3) == 0;
    for (int x = 8 * (blockIdx.x * blockDim.x + threadIdx.x); x < Wp; x += 8 * gridDim.x * blockDim.x) {
        float v[8];
        const int xi = x - xbuf;
        if (vin && xi >= 0 && xi + 8 <= W) {
            const float4 a = __ldg(reinterpret_cast<const float4*>(row + xi));
            const float4 c = __ldg(reinterpret_cast<const float4*>(row + xi + 4));
            v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = c.x; v[5] = c.y; v[6] = c.z; v[7] = c.w;
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = row[min(max(xi + j, 0), W - 1)];
        }
        uint4 hw, lw;
        uint32_t* ph = reinterpret_cast<uint32_t*>(&hw);
        uint32_t* pl = reinterpret_cast<uint32_t*>(&lw);
#pragma unroll
        for (int j = 0; j < 4; ++j) umma::split_f16x2(v[2 * j] * sc, v[2 * j + 1] * sc, ph[j], pl[j]);
        *reinterpret_cast<uint4*>(hi + x) = hw;
        *reinterpret_cast<uint4*>(lo + x) = lw;
    }
}

}  // namespace

int row_umma_jpad(int h) { return (h + 31) / 32 * 32; }

bool row_umma_supported(int h, int W) {
    return h >= 1 && kTX + 2 * row_umma_jpad(h) <= 256 && W % 8 == 0 && W >= kTX && encode_fn() != nullptr;
}

size_t row_umma_fprep_bytes(int H, int W, int xbuf, int batch) {
    return (size_t)batch * 2 * (H + 2 * kBankUPadRows) * (size_t)(W + 2 * xbuf) * sizeof(__half);
}

cudaError_t launch_row_umma_prep(const float* img, int64_t pitch, int64_t bstride, int H, int W, int xbuf, int batch,
                                 const unsigned* maxbits, void* fprep, cudaStream_t s) {
    const int Wp = W + 2 * xbuf;
    dim3 grid((Wp / 8 + 127) / 128, H + 2 * kBankUPadRows, batch);
    fprep_kernel<<<grid, 128, 0, s>>>(img, pitch, bstride, H, W, xbuf, Wp, maxbits, (__half*)fprep);
    return cudaGetLastError();
}

// Replicate rows of the column pass's padding: J plane rows [0, jbuf) = image row 0, rows [H + jbuf,
// H + 2 jbuf) = image row H - 1, per (job, image, plane, strip).  A separate launch after the row kernel:
// written from its epilogue by the four lanes that hold an edge row, the 2 x jbuf x 2 stores per edge
// tile made the CTAs that own a job's first / last row block stragglers (ncu: one SM 2.9 M cycles
// against 1.98 M on average).  Block = (strip, plane of job and image); thread = (row group, u32 column).
__global__ void __launch_bounds__(256) jpad_fill_kernel(const __grid_constant__ RowUArgs a) {
    const int strip = blockIdx.x, plane = blockIdx.y & 1, job = (blockIdx.y >> 1) % a.njobs, b = (blockIdx.y >> 1) / a.njobs;
    const int Hp = a.H + 2 * a.jbuf;
    uint32_t* js = reinterpret_cast<uint32_t*>(a.dst_base + a.jobs[job].dst_off[0] + (int64_t)b * a.dst_bstride) +
                   (int64_t)plane * a.hpw + (int64_t)strip * Hp * 64;
    const int x = threadIdx.x & 63, rg = threadIdx.x >> 6;
    const uint32_t top = js[(int64_t)a.jbuf * 64 + x], bot = js[(int64_t)(a.jbuf + a.H - 1) * 64 + x];
    for (int r = rg; r < a.jbuf; r += 4) {
        js[(int64_t)r * 64 + x] = top;
        js[(int64_t)(a.H + a.jbuf + r) * 64 + x] = bot;
    }
}

cudaError_t launch_row_umma(RowUArgs a, const void* fprep, int sms, cudaStream_t s) {
    EncodeFn enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    static const int dbg = std::getenv("FGB_UMMA_DBG") ? std::atoi(std::getenv("FGB_UMMA_DBG")) : 0;
    a.dbg = dbg;  // A/B ablation (1 no stores, 2 no MMAs, 4 no image loads); results are wrong when set
    a.jpad = row_umma_jpad(a.h);
    a.K = kTX + 2 * a.jpad;
    if (a.jpad > a.xbuf || a.K > 256) return cudaErrorInvalidValue;
    const int Wp = a.W + 2 * a.xbuf;
    CUtensorMap map;
    const int Hq = a.H + 2 * kBankUPadRows;
    cuuint64_t dims[3] = {(cuuint64_t)Wp, (cuuint64_t)Hq, (cuuint64_t)2 * a.batch};
    cuuint64_t strides[2] = {(cuuint64_t)Wp * 2, (cuuint64_t)Wp * 2 * Hq};
    cuuint32_t box[3] = {64, kTY, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(fprep), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        std::fprintf(stderr, "row_umma: tensor map encode failed (Wp %d H %d)\n", Wp, a.H);
        return cudaErrorInvalidValue;
    }
    a.nstrips = (a.W + kTX - 1) / kTX;
    a.nyb = (a.H + kTY - 1) / kTY;
    const int64_t units = (int64_t)a.njobs * a.batch * a.nyb * a.nstrips;
    const int grid = (int)std::min<int64_t>(units, sms);
    const size_t smem = (size_t)kStages * kStageBytes + kStgBytes + 1024;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(row_umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    row_umma_kernel<<<grid, kThreads, smem, s>>>(map, a);
    if (a.jbuf > 0 && !(a.dbg & 1)) jpad_fill_kernel<<<dim3(a.nstrips, 2 * a.njobs * a.batch), 256, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace fgb
