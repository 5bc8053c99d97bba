// K2u: fp32-build column stage of the Gabor bank on the 5th-generation tensor
// cores (tcgen05, TMEM accumulators, TMA), split-fp16 for fp32 accuracy.
//
// Reference semantics: vertical_stage + vertical_stage_conjugate
// (gabor.py:135-169, bank.py:68-74) after the row stage.  With the modulation
// folded into the taps a column job is
//     A(y) = sum_t ka[t] J[clamp(y+t)],  B(y) = sum_t kb[t] J[clamp(y+t)],
//     F_theta = A - iB,  F_{pi-theta} = conj(A + iB)
// for t in [-h, h].  Over a tile of 64 output rows this is a banded Toeplitz
// product: D (128 x 128) = Wt (128 x K) . Jt (K x 128) with
//   * M rows 2r / 2r+1 = the ka / kb taps of output row r placed at
//     K column k = r + jpad + t (zero outside the band),
//   * K = 64 + 2 jpad input rows (jpad = h rounded up to 16), read from a J
//     plane whose rows are replicate-padded by jpad on both ends (the row
//     kernel writes the pad rows), so clamp() costs nothing,
//   * N = 128 halfs of each J row = 64 complex columns (re / im interleaved:
//     the real weights multiply both components independently).
// Precision: every operand is split x = hi + lo in fp16 (round to nearest;
// |x - hi - lo| <= 2^-24 |x|), and D = Wh Jh + Wh Jl + Wl Jh accumulates in
// fp32 in tensor memory -- the dropped Wl Jl term is 2^-22 relative.  J is
// scaled by 2^e per image (e from max|f|, so |J 2^e| < 2^14 < fp16 max) and
// the taps by 2^s per job; the epilogue multiplies by 2^-(e+s) (exact).
// Measured (tools/probes/umma_probe.cu): max|err|/max|ref| 1.9e-6 at K = 256
// where a plain fp32 FMA chain gives 0.9e-6; MMA rate 2.0 PFLOP/s per GPU.
//
// Persistent warp-specialised CTA (one per SM, 512 TMEM columns):
//   warp 4   TMA producer: 16-row groups of the hi and lo J planes (4 boxes of
//            64 halfs x 16 rows, 128-byte swizzle) into a ring of slots;
//   warp 5   TMEM allocator + MMA issuer: per tile K/16 steps x 3 MMAs
//            (M = 128, N = 128, K = 16, A from TMEM, B = the ring slot);
//            consecutive tiles of a column strip share their K rows, so each
//            J row is fetched once per strip (ring slots are released 4 at a
//            time as the tile window slides by 64 rows);
//   warps 0-3 epilogue: TMEM -> registers (lane m = M row m), partner lane
//            exchange (ka row / kb row of the same output row), combine,
//            scale, streaming 16-byte stores of F_theta (even lanes) and
//            conj(A + iB) (odd lanes); they also (re)build the tap matrix in
//            TMEM (tcgen05.st) when the job changes.
// Accumulators are double-buffered (2 x 128 columns), taps hi / lo use the
// remaining K columns.  Work unit = (job, image, row chunk, 64-column strip),
// strips fastest.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kernels.h"
#include "umma.cuh"

namespace fgb {

namespace {

constexpr int kTile = 64;          // output rows per tile
constexpr int kStageBytes = 32768; // 64 J rows: (hi, lo) x 2 column blocks x 64 rows x 128 B
constexpr int kStages = 5;         // ring depth (a tile's window spans <= 4 stages)
constexpr int kEpiWarps = 8;       // two per SM sub-partition: TMEM lane quadrant w % 4, column half w / 4
constexpr int kEpiThreads = 32 * kEpiWarps;
constexpr int kTmaWarp = kEpiWarps, kMmaWarp = kEpiWarps + 1;
constexpr int kThreads = 32 * (kEpiWarps + 2);
constexpr uint32_t kAcc = 128;     // TMEM columns per accumulator
constexpr int kStgBytes = kEpiWarps * 8192;  // output staging: 2 buffers x 2 planes x 16 rows x 128 B per warp


// 2^e as a float for |e| <= 126 (exact)
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + max(-126, min(127, e))) << 23); }

__device__ __forceinline__ void unit_decode(const ColUArgs& a, int u, int& job, int& b, int& chunk, int& strip) {
    strip = u % a.nstrips;
    int r = u / a.nstrips;
    chunk = r % a.nchunks;
    r /= a.nchunks;
    b = r % a.batch;
    job = r / a.batch;
}

__device__ __forceinline__ void st_cs4(float2* p, float a, float b, float c, float d) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    col_umma_kernel(const __grid_constant__ CUtensorMap jmap, const __grid_constant__ CUtensorMap omap,
                    const __grid_constant__ ColUArgs a) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte aligned ring (128-byte swizzle atoms); offsets from smem_raw keep the shared state space
    uint8_t* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint64_t full[kStages], empty[kStages], tfull[3], tempty[3], aready;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int K = a.K, ksteps = a.K / 16, wst = (ksteps + 3) / 4;  // stages spanned by a tile's window
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
    if (warp == kTmaWarp && lane == 0) umma::tma_prefetch_desc(&jmap);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tb = tmem_base;
    // accumulators: 3 buffers when the taps (K columns) leave room in the 512 TMEM columns, else 2
    const uint32_t nacc = (512 - K) >= 3 * (int)kAcc ? 3u : 2u;
    const uint32_t a_hi = tb + nacc * kAcc, a_lo = a_hi + (uint32_t)(K / 2);
    const int nunits = a.njobs * a.batch * a.nchunks * a.nstrips;
    const int chunk_rows = a.ch_tiles * kTile;

    if (warp == kTmaWarp) {
        // ---------------- TMA producer: one 64-row stage (hi / lo x 2 column blocks) per barrier ----------------
        if (lane == 0) {
            uint32_t g = 0;  // stage counter over the CTA's units
            for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
                int job, b, chunk, strip;
                unit_decode(a, u, job, b, chunk, strip);
                const int y0 = chunk * chunk_rows;
                const int nt = min(a.ch_tiles, (a.H - y0 + kTile - 1) / kTile);
                const int Gs = nt + wst - 1;
                const int plane = (int)(2 * (((int64_t)b * a.ws_img_c + a.jobs[job].src_off) / a.hpw));

                for (int q = 0; q < Gs; ++q, ++g) {
                    const uint32_t slot = g % (uint32_t)kStages, round = g / (uint32_t)kStages;
                    mbar_wait(&empty[slot], (round & 1u) ^ 1u);
                    uint8_t* sp = ring + slot * kStageBytes;
                    if (a.dbg & 4) {  // A/B knob: no J loads
                        umma::mbar_arrive(&full[slot]);
                        continue;
                    }
                    mbar_arrive_expect_tx(&full[slot], kStageBytes);
                    const int rr = y0 + a.jbuf - a.jpad + kTile * q;  // buffer row (input row + jbuf)
                    // strip-major planes: each 64-row stage block of a strip is 16 KB contiguous
                    umma::tma_load_4d(sp, &jmap, 0, rr, strip, plane, &full[slot]);
                    umma::tma_load_4d(sp + 8192, &jmap, 64, rr, strip, plane, &full[slot]);
                    umma::tma_load_4d(sp + 16384, &jmap, 0, rr, strip, plane + 1, &full[slot]);
                    umma::tma_load_4d(sp + 24576, &jmap, 64, rr, strip, plane + 1, &full[slot]);
                }
            }
        }
    } else if (warp == kMmaWarp) {
        // ---------------- MMA issuer (the whole warp runs the loop; one elected lane issues) ----------------
        {
            const uint32_t idesc = umma::idesc_f16_f32(128, 128, false, true);
            const uint64_t rdesc0 = umma::smem_desc(smem_u32(ring), 8192, 1024, umma::kLayoutSw128);
            const bool do_mma = !(a.dbg & 2);  // A/B knob: no MMAs
            uint32_t g = 0, t = 0, nreload = 0;
            int cur = -1;
            for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
                int job, b, chunk, strip;
                unit_decode(a, u, job, b, chunk, strip);
                const int y0 = chunk * chunk_rows;
                const int nt = min(a.ch_tiles, (a.H - y0 + kTile - 1) / kTile);
                const int Gs = nt + wst - 1;
                if (job != cur) {
                    mbar_wait(&aready, nreload & 1u);
                    ++nreload;
                    cur = job;
                    umma::fence_after();
                }
                for (int i = 0; i < nt; ++i, ++t) {
                    const uint32_t buf = t % nacc, ph = (t / nacc) & 1u;
                    mbar_wait(&tempty[buf], ph ^ 1u);
                    umma::fence_after();
                    const uint32_t d = tb + buf * kAcc;
                    // K step kk = group kk of the window: stage i + kk / 4, 16-row group kk % 4.  One elect
                    // region per stage (<= 12 MMAs), descriptors advance by constants: the issuing warp must
                    // stay well under the MMAs' execution time (it was the critical path at ~60
                    // instructions per K step)
                    for (int st = 0; st < wst; ++st) {
                        const uint32_t gs = g + i + st;
                        const uint32_t slot = gs % (uint32_t)kStages;
                        mbar_wait(&full[slot], (gs / (uint32_t)kStages) & 1u);
                        umma::fence_after();
                        const uint64_t bh0 = rdesc0 + (uint64_t)(slot * (kStageBytes >> 4));
                        const int nq = ksteps - 4 * st;
                        if (do_mma && umma::elect_one()) {
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                if (q < nq) {
                                    const uint64_t bh = bh0 + (uint64_t)(128 * q), bl = bh + (uint64_t)(16384 >> 4);
                                    const uint32_t ah = a_hi + 8 * (4 * st + q), al = ah + (uint32_t)(K / 2);
                                    umma::mma_f16_ts(d, ah, bh, idesc, (st | q) ? 1u : 0u);
                                    umma::mma_f16_ts(d, ah, bl, idesc, 1u);
                                    umma::mma_f16_ts(d, al, bh, idesc, 1u);
                                }
                            }
                        }
                        __syncwarp();
                    }
                    // one commit per tile: the epilogue's first thread releases the ring stages
                    // (stage i; all the unit's remaining stages after its last tile) once it has
                    // seen this tile's accumulator complete
                    if (umma::elect_one()) umma::mma_commit(&tfull[buf]);
                    __syncwarp();
                }
                g += Gs;
            }
        }
        __syncwarp();
    } else {
        // ---------------- epilogue (warps 0-7: TMEM lanes 32 (w % 4) + 0..31, columns 64 (w / 4) + 0..63) ----------------
        const int quad = warp & 3, half = warp >> 2;
        const int m = 32 * quad + lane;  // TMEM lane = M row
        const uint32_t lane_addr = (uint32_t)(32 * quad) << 16;
        const int r = m >> 1, odd = m & 1;
        // output staging: per warp 2 buffers x (F_theta, F_pi-theta) x [16 rows][128 B] (128-byte swizzle, TMA stores)
        uint8_t* ostg = ring + kStages * kStageBytes + warp * 8192;
        int cur = -1;
        uint32_t t = 0, gst = 0;  // tiles; the producer's ring-stage counter at the start of the unit
        int wexp = 0;
        for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
            int job, b, chunk, strip;
            unit_decode(a, u, job, b, chunk, strip);
            const ColJob<float>& jb = a.jobs[job];
            if (job != cur) {
                // tap matrix row m: K column k holds (odd ? kb : ka)[t], t = k - jpad - r; the two
                // warps of a lane quadrant build alternate 16-column blocks
                const float2* w = a.weights + jb.wofs;
                wexp = jb.wexp;
                const float wsc = pow2f(wexp);
                for (int c = 16 * half; c < K / 2; c += 32) {
                    uint32_t hi[16], lo[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        float v[2];
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int tt = 2 * (c + i) + e - a.jpad - r;
                            float x = 0.f;
                            if (tt >= -a.h && tt <= a.h) {
                                const float2 kk = w[tt + a.h];
                                x = (odd ? kk.y : kk.x) * wsc;
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
            const float inv = pow2f(-(jscale_exp(a.maxbits[b]) + wexp));
            const int nout = jb.nout;
            float2* dst0 = a.dst_base + jb.dst_off[0] + (int64_t)b * a.dst_bstride;
            float2* dst1 = a.dst_base + (nout > 1 ? jb.dst_off[1] : jb.dst_off[0]) + (int64_t)b * a.dst_bstride;
            const int y0 = chunk * chunk_rows;
            const int nt = min(a.ch_tiles, (a.H - y0 + kTile - 1) / kTile);
            const int Gs = nt + wst - 1;
            const int plane0 = (int)((jb.dst_off[0] + (int64_t)b * a.dst_bstride) / a.hw);
            const int plane1 = (int)((jb.dst_off[nout > 1 ? 1 : 0] + (int64_t)b * a.dst_bstride) / a.hw);
            const int r = lane >> 1;  // output row (of the warp's 16) of this lane's M row
            for (int i = 0; i < nt; ++i, ++t) {
                const uint32_t buf = t % nacc, ph = (t / nacc) & 1u;
                mbar_wait(&tfull[buf], ph);
                umma::fence_after();
                if (threadIdx.x == 0) {  // the MMAs of this tile are done: its first stage is free
                    const int rel_end = (i == nt - 1) ? Gs : i + 1;
                    for (int q = i; q < rel_end; ++q) umma::mbar_arrive(&empty[(gst + q) % (uint32_t)kStages]);
                }
                const int ybase = y0 + i * kTile + 16 * quad;  // output row of M rows 0 / 1 of the quadrant
                float v[64];  // this warp's 64 accumulator columns, one TMEM wait
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    umma::tmem_ld16(tb + lane_addr + buf * kAcc + 64 * half + 16 * j, *reinterpret_cast<float(*)[16]>(v + 16 * j));
                umma::tmem_ld_wait();
                umma::fence_before();
                umma::mbar_arrive(&tempty[buf]);  // accumulator drained: the MMA may reuse it
#pragma unroll
                for (int qq = 0; qq < 2; ++qq) {  // 16 complex columns per pass
                    uint8_t* sb = ostg + 4096 * qq;  // pass qq -> buffer qq (two TMA store groups in flight)
                    if (lane == 0) umma::bulk_wait_read<1>();  // the store group that last read this buffer is done
                    __syncwarp();
                    // even lane: F_theta row r = A - iB (A own, B partner); odd lane: conj(A + iB) row r
                    uint8_t* rowp = sb + (odd ? 2048 : 0) + r * 128;
                    // step c: even lanes write chunk c, odd lanes chunk c ^ 4, so the two rows of a lane pair
                    // (same swizzled slot, planes 2 KB apart) land in different banks
#pragma unroll
                    for (int c = 0; c < 8; ++c) {  // 16-byte chunk = complex columns 2 ch, 2 ch + 1
                        const int ch = odd ? (c ^ 4) : c;
                        float o[4];
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int ko = 32 * qq + 4 * c + 2 * e, kx = 32 * qq + 4 * (c ^ 4) + 2 * e;
                            const float own_r = odd ? v[kx] : v[ko], own_i = odd ? v[kx + 1] : v[ko + 1];
                            // the partner's chunk is the other one of (c, c ^ 4)
                            const float pr = __shfl_xor_sync(0xffffffffu, odd ? v[ko] : v[kx], 1);
                            const float pi = __shfl_xor_sync(0xffffffffu, odd ? v[ko + 1] : v[kx + 1], 1);
                            if (!odd) {
                                o[2 * e] = (own_r + pi) * inv;
                                o[2 * e + 1] = (own_i - pr) * inv;
                            } else {
                                o[2 * e] = (pr - own_i) * inv;
                                o[2 * e + 1] = -(pi + own_r) * inv;
                            }
                        }
                        *reinterpret_cast<float4*>(rowp + ((ch ^ (r & 7)) << 4)) = make_float4(o[0], o[1], o[2], o[3]);
                    }
                    umma::fence_async_smem();
                    __syncwarp();
                    if (lane == 0 && !(a.dbg & 1)) {
                        const int xf = 2 * (strip * 64 + 32 * half + 16 * qq);  // float column
                        umma::tma_store_3d(&omap, xf, ybase, plane0, sb);
                        if (nout > 1) umma::tma_store_3d(&omap, xf, ybase, plane1, sb + 2048);
                    }
                    if (lane == 0) umma::bulk_commit();
                }
            }
            gst += Gs;
        }
        if (lane == 0) umma::bulk_wait_read<0>();  // staging reads done before the CTA exits
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

}  // namespace

int col_umma_jpad(int h) { return (h + 15) / 16 * 16; }

bool col_umma_supported(int h, int W) {
    const int K = kTile + 2 * col_umma_jpad(h);
    return h >= 1 && K <= 256 && W % 4 == 0 && W >= 64 && encode_fn() != nullptr;
}

size_t col_umma_smem(int) {
    // ring + staging + alignment slack (> 114 KB: two of these CTAs, 512 TMEM columns each, never share an SM)
    return (size_t)kStages * kStageBytes + kStgBytes + 1024;
}

cudaError_t launch_col_umma(ColUArgs a, void* ws, int64_t ws_bytes, int sms, cudaStream_t s) {
    EncodeFn enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    static const int dbg = std::getenv("FGB_UMMA_DBG") ? std::atoi(std::getenv("FGB_UMMA_DBG")) : 0;
    a.dbg = dbg;  // A/B ablation (1 no stores, 2 no MMAs, 4 no J loads); results are wrong when set
    a.jpad = col_umma_jpad(a.h);
    a.K = kTile + 2 * a.jpad;
    const int W64 = (a.W + 63) / 64 * 64;
    if (a.jpad > a.jbuf || a.hpw != (a.H + 2 * (int64_t)a.jbuf) * W64) {
        std::fprintf(stderr, "col_umma: J slot layout mismatch (jpad %d jbuf %d hpw %lld)\n", a.jpad, a.jbuf,
                     (long long)a.hpw);
        return cudaErrorInvalidValue;
    }
    const int64_t Hp = a.H + 2 * (int64_t)a.jbuf;
    // J planes: [nplanes][W64 / 64 strips][Hp][128 halfs] (hi plane, lo plane per job slot)
    const int64_t plane_bytes = a.hpw * 4;
    const int64_t nplanes = ws_bytes / plane_bytes;
    CUtensorMap map;
    cuuint64_t dims[4] = {128, (cuuint64_t)Hp, (cuuint64_t)(W64 / 64), (cuuint64_t)nplanes};
    cuuint64_t strides[3] = {256, (cuuint64_t)Hp * 256, (cuuint64_t)plane_bytes};
    cuuint32_t box[4] = {64, kTile, 1, 1};  // one 64-row stage block (one of the two column blocks) per load
    cuuint32_t estr[4] = {1, 1, 1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, ws, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS) {
        std::fprintf(stderr, "col_umma: tensor map encode failed (W %d Hp %lld planes %lld)\n", a.W, (long long)Hp,
                     (long long)nplanes);
        return cudaErrorInvalidValue;
    }
    // outputs: [plane][H][W] complex64 from dst_base, stored by TMA from the swizzled staging
    a.hw = (int64_t)a.H * a.W;
    CUtensorMap omap;
    {
        cuuint64_t od[3] = {(cuuint64_t)2 * a.W, (cuuint64_t)a.H, (cuuint64_t)a.dst_planes};
        cuuint64_t os[2] = {(cuuint64_t)a.W * 8, (cuuint64_t)a.hw * 8};
        cuuint32_t ob[3] = {32, 16, 1};
        if (a.dst_planes < 1 || (reinterpret_cast<uintptr_t>(a.dst_base) & 15) ||
            enc(&omap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, a.dst_base, od, os, ob, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
                CUDA_SUCCESS) {
            std::fprintf(stderr, "col_umma: output tensor map encode failed (W %d H %d planes %lld)\n", a.W, a.H,
                         (long long)a.dst_planes);
            return cudaErrorInvalidValue;
        }
    }
    // work units: strips x row chunks x images x jobs; enough units for an even last wave
    a.nstrips = (a.W + 63) / 64;
    const int ntiles = (a.H + kTile - 1) / kTile;
    const int64_t base = (int64_t)a.nstrips * a.batch * a.njobs;
    int nch = (int)std::min<int64_t>(std::max<int64_t>(1, (20LL * sms + base - 1) / base), std::max(1, ntiles / 8));
    a.ch_tiles = (ntiles + nch - 1) / nch;
    a.nchunks = (ntiles + a.ch_tiles - 1) / a.ch_tiles;
    const int64_t units = base * a.nchunks;
    const int grid = (int)std::min<int64_t>(units, sms);
    const size_t smem = col_umma_smem(a.h);
    static bool attr = false;
    if (!attr) {
        // the largest ring (+ alignment slack); static shared memory comes on top of it
        cudaError_t e = cudaFuncSetAttribute(col_umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)col_umma_smem(0));
        if (e != cudaSuccess) return e;
        attr = true;
    }
    col_umma_kernel<<<grid, kThreads, smem, s>>>(map, omap, a);
    return cudaGetLastError();
}

// ---- per-image max |f| (the J scale exponent) ----------------------------
// grid (row blocks, batch); threads stride the columns of their rows
// grid (blocks per image, batch); 16-byte loads when rows are 16-byte aligned (pitch % 4, W % 4)
__global__ void absmax_kernel(const float* __restrict__ img, int64_t pitch, int64_t bstride, int H, int W,
                              unsigned* __restrict__ out) {
    const float* base = img + (int64_t)blockIdx.y * bstride;
    unsigned mx = 0;
    const bool vec = (pitch & 3) == 0 && (W & 3) == 0 && ((reinterpret_cast<uintptr_t>(base) & 15) == 0);
    if (vec && pitch == W) {
        // contiguous image: one linear float4 stream, four independent loads per thread and step (a 64-bit
        // division per element made this kernel 4x slower than the read it is)
        const float4* p4 = reinterpret_cast<const float4*>(base);
        const int64_t n4 = (int64_t)H * (W >> 2), stride = (int64_t)gridDim.x * blockDim.x;
        int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        for (; i + 3 * stride < n4; i += 4 * stride) {
            const float4 a = __ldcs(p4 + i), b = __ldcs(p4 + i + stride), c = __ldcs(p4 + i + 2 * stride),
                         d = __ldcs(p4 + i + 3 * stride);
            // unsigned bit patterns order |x| and put NaN above infinity, as the scalar path does
            mx = max(mx, max(max(max(__float_as_uint(fabsf(a.x)), __float_as_uint(fabsf(a.y))),
                                 max(__float_as_uint(fabsf(a.z)), __float_as_uint(fabsf(a.w)))),
                             max(max(__float_as_uint(fabsf(b.x)), __float_as_uint(fabsf(b.y))),
                                 max(__float_as_uint(fabsf(b.z)), __float_as_uint(fabsf(b.w))))));
            mx = max(mx, max(max(max(__float_as_uint(fabsf(c.x)), __float_as_uint(fabsf(c.y))),
                                 max(__float_as_uint(fabsf(c.z)), __float_as_uint(fabsf(c.w)))),
                             max(max(__float_as_uint(fabsf(d.x)), __float_as_uint(fabsf(d.y))),
                                 max(__float_as_uint(fabsf(d.z)), __float_as_uint(fabsf(d.w))))));
        }
        for (; i < n4; i += stride) {
            const float4 v = __ldcs(p4 + i);
            mx = max(mx, max(max(__float_as_uint(fabsf(v.x)), __float_as_uint(fabsf(v.y))),
                             max(__float_as_uint(fabsf(v.z)), __float_as_uint(fabsf(v.w)))));
        }
    } else if (vec) {
        const int w4 = W >> 2;
        for (int y = blockIdx.x; y < H; y += gridDim.x) {
            const float4* row = reinterpret_cast<const float4*>(base + (int64_t)y * pitch);
            for (int x4 = threadIdx.x; x4 < w4; x4 += blockDim.x) {
                const float4 v = __ldcs(row + x4);
                mx = max(mx, max(max(__float_as_uint(fabsf(v.x)), __float_as_uint(fabsf(v.y))),
                                 max(__float_as_uint(fabsf(v.z)), __float_as_uint(fabsf(v.w)))));
            }
        }
    } else {
        for (int y = blockIdx.x; y < H; y += gridDim.x) {
            const float* row = base + (int64_t)y * pitch;
            for (int x = threadIdx.x; x < W; x += blockDim.x) mx = max(mx, __float_as_uint(fabsf(row[x])));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out + blockIdx.y, mx);
}

cudaError_t launch_absmax(const float* img, int64_t pitch, int64_t bstride, int H, int W, int batch, unsigned* out,
                          int sms, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned) * batch, s);
    if (e != cudaSuccess) return e;
    const int per = std::max(1, std::min(H, (8 * sms + batch - 1) / batch));
    absmax_kernel<<<dim3(per, batch), 512, 0, s>>>(img, pitch, bstride, H, W, out);
    return cudaGetLastError();
}

}  // namespace fgb
