// K5u: one frequency of the fp32 Gabor bank -- row AND column passes -- in one
// tensor-core kernel, J kept in shared memory (half-widths h <= 48).
//
// Reference semantics: horizontal_stage -> vertical_stage(_conjugate)
// (gabor.py:107-169, bank.py:68-74) for every direct orientation of one
// frequency, exactly as row_umma.cu + col_umma.cu compute them (DESIGN.md
// §4.1: banded Toeplitz products, split fp16, fp32 accumulation in TMEM), but
// the split-fp16 J never goes to HBM: the row pass writes each 64-row J block
// of a 64-column strip straight into a shared-memory ring in the layout the
// column MMAs read (MN-major, 128-byte swizzle), and the column pass consumes
// it.  HBM traffic per frequency: the image planes in, the outputs out.
//
// Per CTA (persistent, one per SM, 448 threads, 512 TMEM columns):
//   warp 12  TMA producer: 64-column x 64-row boxes of the x- and y-padded
//            split-fp16 image planes (2 per J block: K_r <= 128 input columns)
//   warp 13  TMEM allocator + MMA issuer, per unit in dependency order:
//            row block j (K_r / 16 steps x 2 MMAs: Wh [Fh | Fl] as one N = 128
//            MMA + Wl Fh, N = 64), then column tile j - 3 (K_c / 16 steps x
//            3 MMAs, M 128 x N 128) once blocks j - 3 .. j - 1 are in the ring
//   warps 8-11  row epilogue: D_row (TMEM, read as m8n8 fragments) -> J 2^e ->
//            fp16 hi / lo -> the ring block with stmatrix.trans (the padded
//            image rows make the column pass's replicate rows for free)
//   warps 0-7  column epilogue: D_col read as m8n8 fragments (the ka / kb rows
//            of an output row sit 8 TMEM lanes apart, so one thread holds both),
//            F_theta / F_pi-theta formed in registers (no shuffles), staged as
//            [16 rows][128 B] boxes (128-byte swizzle) and written by TMA stores
// Image chunks and J blocks are released by tcgen05.commit from the MMA warp
// (arrive when the MMAs that read them complete), so neither release waits on
// an epilogue.
// TMEM: D_col [0, 128), D_row [128, 256) (Wh Fh + Wl Fh | Wh Fl), row taps hi / lo
// [256, 256 + K_r), column taps hi / lo [384, 384 + K_c); K_r = K_c = 64 + 2 JPC,
// JPC = h rounded up to 16 (a template parameter: 16, 32 or 48).  JPC = 48 (sigma
// = 16 at radius 3: 320 tap columns) keeps a 64-column D_row and 3 MMAs per row
// K step: D_col [0, 128), D_row [128, 192), row taps [192, 352), column taps
// [352, 512) -- the 512 TMEM columns exactly.
// Work unit = (direct, 64-column strip, row chunk, image), directs fastest: the directs of a strip run at
// the same time on neighbouring CTAs and share their image reads in L2; taps are rebuilt per unit.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kernels.h"
#include "umma.cuh"

namespace fgb {

namespace {

constexpr int kT = 64;              // output columns per strip, rows per J block / column tile
constexpr int kJBytes = 32768;      // J block: (hi, lo) x 2 column blocks x 64 rows x 128 B
constexpr int kJSlots = 4;
constexpr int kIBytes = 16384;      // image chunk: (hi, lo) x 64 rows x 128 B (64 input columns)
constexpr int kISlots = 4;
constexpr int kColWarps = 8, kRowWarps = 4;
constexpr int kRowW0 = kColWarps, kTmaWarp = kColWarps + kRowWarps, kMmaWarp = kTmaWarp + 1;
constexpr int kThreads = 32 * (kMmaWarp + 1);
constexpr int kColThreads = 32 * kColWarps, kRowThreads = 32 * kRowWarps;
constexpr int kJr = 48;             // largest row / column tap padding (h <= 48); K_r = K_c = 64 + 2 JPC
constexpr uint32_t kDcol = 0, kDrow = 128;  // the tap columns follow D_row (see the kernel)
constexpr int kStgBytes = 4096;      // per column-epilogue warp: 2 buffers x [16 rows][128 B] (128-byte swizzle, TMA stores)
constexpr int kSmem = kJSlots * kJBytes + kISlots * kIBytes + kColWarps * kStgBytes + 1024;

__device__ __forceinline__ float pow2f(int e) { return __int_as_float((127 + max(-126, min(127, e))) << 23); }

struct UnitIt {
    int u, job, b, chunk, strip;
    __device__ void decode(const BankUArgs& a) {
        int r = u;
        if (a.job_fastest) {  // the directs of one (strip, chunk) run at the same time on neighbouring CTAs:
            job = r % a.njobs;  // their image reads hit L2; the taps are rebuilt per unit
            r /= a.njobs;
            strip = r % a.nstrips;
            r /= a.nstrips;
            chunk = r % a.nchunks;
            b = r / a.nchunks;
            return;
        }
        strip = r % a.nstrips;
        r /= a.nstrips;
        chunk = r % a.nchunks;
        r /= a.nchunks;
        b = r % a.batch;
        job = r / a.batch;
    }
};

template <int JPC>
__global__ void __launch_bounds__(kThreads, 1)
    bank_umma_kernel(const __grid_constant__ CUtensorMap fmap, const __grid_constant__ CUtensorMap omap,
                     const __grid_constant__ BankUArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* jring = base;
    uint8_t* iring = base + kJSlots * kJBytes;
    uint8_t* ostg_all = iring + kISlots * kIBytes;
    __shared__ uint64_t ifull[kISlots], iempty[kISlots], jfull[kJSlots], jempty[kJSlots];
    __shared__ uint64_t rfull, rempty, cfull, cempty, aready;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int Kc = kT + 2 * JPC, jpc = JPC;
    constexpr int Kr = kT + 2 * JPC;     // row K: the last image chunk contributes Kr / 16 - 4 (NCH - 1) K steps
    constexpr int NCH = (Kr + 63) / 64;  // 64-column image chunks per row block
    // JPC <= 32: D_row holds [Wh Fh + Wl Fh | Wh Fl] (128 columns, 2 MMAs per K step); JPC = 48: the taps need
    // 320 columns, so D_row is 64 columns and the row pass issues the 3 N = 64 MMAs per K step
    constexpr bool kWideRow = JPC <= 32;
    constexpr uint32_t kRtap = kDrow + (kWideRow ? 128 : 64), kCtap = kRtap + (kWideRow ? 128 : Kr);
    static_assert(kCtap + Kc <= 512, "TMEM budget");
    if (threadIdx.x == 0) {
        for (int s = 0; s < kISlots; ++s) {
            mbar_init(&ifull[s], 1);
            mbar_init(&iempty[s], 1);
        }
        for (int s = 0; s < kJSlots; ++s) {
            mbar_init(&jfull[s], kRowThreads);
            mbar_init(&jempty[s], 1);
        }
        mbar_init(&rfull, 1);
        mbar_init(&rempty, kRowThreads);
        mbar_init(&cfull, 1);
        mbar_init(&cempty, kColThreads);
        mbar_init(&aready, kColThreads + kRowThreads);
    }
    if (warp == kMmaWarp) umma::tmem_alloc(&tmem_base, 512);
    if (warp == kTmaWarp && lane == 0) umma::tma_prefetch_desc(&fmap);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tb = tmem_base;
    const int nunits = a.njobs * a.batch * a.nchunks * a.nstrips;
    const int chunk_rows = a.ch_tiles * kT;
    auto tiles_of = [&](int chunk) { return min(a.ch_tiles, (a.H - chunk * chunk_rows + kT - 1) / kT); };

    if (warp == kTmaWarp) {
        // ---------------- TMA producer: image chunks (64 columns x 64 rows, hi + lo) ----------------
        if (lane == 0) {
            uint32_t g = 0;
            for (UnitIt it{(int)blockIdx.x}; it.u < nunits; it.u += gridDim.x) {
                it.decode(a);
                const int y0 = it.chunk * chunk_rows, nb = tiles_of(it.chunk) + 2;
                const int xs = it.strip * kT - JPC + a.xbuf;
                for (int j = 0; j < nb; ++j)
                    for (int kc = 0; kc < NCH; ++kc, ++g) {
                        const uint32_t slot = g % kISlots;
                        mbar_wait(&iempty[slot], ((g / kISlots) & 1u) ^ 1u);
                        uint8_t* sp = iring + slot * kIBytes;
                        if (a.dbg & 4) {  // A/B knob: no image loads
                            umma::mbar_arrive(&ifull[slot]);
                            continue;
                        }
                        mbar_arrive_expect_tx(&ifull[slot], kIBytes);
                        // J block j = J rows y0 + 64 (j - 1) .. + 63: padded-plane rows + kPadR
                        const int row = y0 + kT * (j - 1) + kBankUPadRows;
                        umma::tma_load_3d(sp, &fmap, xs + 64 * kc, row, 2 * it.b, &ifull[slot]);
                        umma::tma_load_3d(sp + kIBytes / 2, &fmap, xs + 64 * kc, row, 2 * it.b + 1, &ifull[slot]);
                    }
            }
        }
    } else if (warp == kMmaWarp) {
        // ---------------- MMA issuer ----------------
        // The whole warp runs the loops converged; one elect.sync lane issues a block of MMAs (the 12 of an
        // image chunk / of a J block's 16-row groups) per elect region.  JPC is a template parameter and
        // the shared-memory descriptors advance by constants, so a K step costs its 3 tcgen05.mma plus a
        // few uniform adds: the issuing warp must stay well under the ~60-78 cycles an MMA executes
        // (ncu: with ~60 instructions per K step this warp was the kernel's critical path).
        {
            const uint32_t idr = umma::idesc_f16_f32(128, kT, false, false);   // row: B K-major (image rows)
            const uint32_t idr2 = umma::idesc_f16_f32(128, 2 * kT, false, false);  // row: hi rows then lo rows
            const uint32_t idc = umma::idesc_f16_f32(128, 128, false, true);   // column: B MN-major (J rows)
            const uint64_t jdesc0 = umma::smem_desc(smem_u32(jring), 8192, 1024, umma::kLayoutSw128);
            const uint64_t idesc0 = umma::smem_desc(smem_u32(iring), 16, 1024, umma::kLayoutSw128);
            const bool do_mma = !(a.dbg & 2);  // A/B knob: no MMAs
            uint32_t gb = 0, gt = 0, nreload = 0;
            uint32_t islot = 0, iphase = 0;
            int cur = -1;
            for (UnitIt it{(int)blockIdx.x}; it.u < nunits; it.u += gridDim.x) {
                it.decode(a);
                const int nt = tiles_of(it.chunk), nb = nt + 2;
                if (it.job != cur) {
                    mbar_wait(&aready, nreload & 1u);
                    ++nreload;
                    cur = it.job;
                    umma::fence_after();
                }
                const uint32_t gbase = gb;
                // column tile i = J blocks i .. i + 2 (window rows 64 i - jpc .. 64 i + 63 + jpc: 16-row groups
                // G = g0 .. g0 + ksc - 1 of the three blocks); issued three row blocks behind so the row
                // epilogue has converted its last block by then
                auto column = [&](int i) {
                    if (!(a.dbg & 16)) mbar_wait(&cempty, (gt & 1u) ^ 1u);  // 16: A/B knob, as if D_col were double-buffered
                    umma::fence_after();
#pragma unroll
                    for (int bq = 0; bq < 3; ++bq) {
                        constexpr int g0c = (kT - JPC) / 16, kscc = (kT + 2 * JPC) / 16;
                        const int q_lo = bq == 0 ? g0c : 0;
                        const int q_hi = g0c + kscc - 4 * bq < 4 ? g0c + kscc - 4 * bq : 4;
                        const uint32_t blk = gbase + i + bq;
                        const uint32_t slot = blk % kJSlots;
                        mbar_wait(&jfull[slot], (blk / kJSlots) & 1u);
                        umma::fence_after();
                        const uint64_t bh0 = jdesc0 + (uint64_t)(slot * (kJBytes >> 4));
                        if (umma::elect_one()) {
                            if (do_mma) {
#pragma unroll
                                for (int q = 0; q < 4; ++q) {
                                    if (q < q_lo || q >= q_hi) continue;
                                    const int kk = 4 * bq + q - g0c;
                                    const uint64_t bh = bh0 + (uint64_t)(128 * q), bl = bh + (uint64_t)(kJBytes >> 5);
                                    const uint32_t ah = tb + kCtap + 8 * kk, al = ah + (kT + 2 * JPC) / 2;
                                    umma::mma_f16_ts(tb + kDcol, ah, bh, idc, kk > 0 ? 1u : 0u);
                                    umma::mma_f16_ts(tb + kDcol, ah, bl, idc, 1u);
                                    umma::mma_f16_ts(tb + kDcol, al, bh, idc, 1u);
                                }
                            }
                            if (bq == 2) {
                                umma::mma_commit(&cfull);
                                // J block i is not in tile i + 1's window; after the unit's last tile, neither are
                                // i + 1, i + 2: their slots free when these MMAs complete
                                umma::mma_commit(&jempty[(gbase + i) % kJSlots]);
                                if (i == nt - 1) {
                                    umma::mma_commit(&jempty[(gbase + i + 1) % kJSlots]);
                                    umma::mma_commit(&jempty[(gbase + i + 2) % kJSlots]);
                                }
                            }
                        }
                        __syncwarp();
                    }
                    ++gt;
                };
                for (int j = 0; j < nb; ++j) {
                    // row block j -> D_row (one 128-column buffer: its drain overlaps the column tile issued
                    // in between).  Per K step: Wh . [Fh | Fl] as ONE N = 128 MMA (the lo image rows follow the
                    // hi rows in the chunk, so the B descriptor just runs on: columns 0-63 = Wh Fh, 64-127 =
                    // Wh Fl, summed by the row epilogue) + Wl . Fh (N = 64) -- an N = 64 MMA costs ~60 cycles,
                    // an N = 128 one ~78, so this is 138 instead of 180 cycles per K step
                    mbar_wait(&rempty, (gb & 1u) ^ 1u);
                    umma::fence_after();
                    const uint32_t d = tb + kDrow;
#pragma unroll
                    for (int kc = 0; kc < NCH; ++kc) {
                        mbar_wait(&ifull[islot], iphase);
                        umma::fence_after();
                        const uint64_t bh0 = idesc0 + (uint64_t)(islot * (kIBytes >> 4));
                        if (umma::elect_one()) {
                            if (do_mma) {
#pragma unroll
                                for (int q = 0; q < 4; ++q) {
                                    const int kk = 4 * kc + q;
                                    if (kk >= Kr / 16) continue;
                                    // K-major, 128-byte swizzle: K step = 32 bytes inside the swizzle atom
                                    const uint64_t bh = bh0 + (uint64_t)(2 * q);
                                    const uint32_t ah = tb + kRtap + 8 * kk, al = ah + Kr / 2;
                                    if constexpr (kWideRow) {
                                        umma::mma_f16_ts(d, ah, bh, idr2, kk > 0 ? 1u : 0u);
                                        umma::mma_f16_ts(d, al, bh, idr, 1u);
                                    } else {
                                        umma::mma_f16_ts(d, ah, bh, idr, kk > 0 ? 1u : 0u);
                                        umma::mma_f16_ts(d, ah, bh + (uint64_t)(kIBytes >> 5), idr, 1u);
                                        umma::mma_f16_ts(d, al, bh, idr, 1u);
                                    }
                                }
                            }
                            umma::mma_commit(&iempty[islot]);  // the image chunk is free once these MMAs complete
                            if (kc == NCH - 1) umma::mma_commit(&rfull);
                        }
                        __syncwarp();
                        if (++islot == kISlots) {
                            islot = 0;
                            iphase ^= 1u;
                        }
                    }
                    ++gb;
                    if (j >= 3) column(j - 3);
                }
                column(nt - 1);
            }
        }
        __syncwarp();
    } else if (warp >= kRowW0) {
        // ---------------- row epilogue (warps 8-11): D_row -> split-fp16 J block in the ring ----------------
        // The accumulator is read as m8n8 fragments (16x256b: thread t holds TMEM lanes t/4 and t/4 + 8,
        // columns 2 (t%4) + {0,1} + 8k) and written with stmatrix.trans: memory row = J row (TMEM
        // column), 16 bytes = 8 consecutive J halves (TMEM lanes) -- one instruction stores 4 swizzled
        // 8-row matrices (hi / lo x two lane octets), conflict-free.
        const int quad = warp - kRowW0;
        const int m = 32 * quad + lane;  // tap rebuild: TMEM lane = M row = J half index (2 xl + re/im)
        const uint32_t lane_addr = (uint32_t)(32 * quad) << 16;
        const int xl = m >> 1, im = m & 1;
        // stmatrix address of this thread: matrix q = lane / 8 (bit 0: lane octet +8, bit 1: lo plane),
        // row j = lane % 8 of the 8-row group; the J half index of the matrix's first column is mq
        const int sq = lane >> 3, sj = lane & 7;
        uint32_t soff[2];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const int mq = 32 * quad + 16 * hh + 8 * (sq & 1);
            soff[hh] = (uint32_t)((sq >> 1) * (kJBytes / 2) + (mq >> 6) * 8192 + sj * 128 +
                                  ((((mq & 63) >> 3) ^ sj) << 4));
        }
        const uint32_t jring_s = smem_u32(jring);
        uint32_t gb = 0;
        int cur = -1;
        float inv_r = 1.f;
        for (UnitIt it{(int)blockIdx.x}; it.u < nunits; it.u += gridDim.x) {
            it.decode(a);
            const BankUJob& jb = a.jobs[it.job];
            if (it.job != cur) {
                // row taps: M row m, K column k -> t = k - JPC - xl: (kr[|t|], sgn(t) ki[|t|]) 2^rexp
                const float2* w = a.weights + jb.rofs;
                const float wsc = pow2f(jb.rexp);
                inv_r = pow2f(-jb.rexp);
                for (int c = 0; c < Kr / 2; c += 16) {
                    uint32_t hi[16], lo[16];
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        float v[2];
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int tt = 2 * (c + q) + e - JPC - xl;
                            const int at = tt < 0 ? -tt : tt;
                            float x = 0.f;
                            if (at <= a.h) {
                                const float2 kk = w[at];
                                x = (im ? (tt < 0 ? -kk.y : kk.y) : kk.x) * wsc;
                            }
                            v[e] = x;
                        }
                        umma::split_f16x2(v[0], v[1], hi[q], lo[q]);
                    }
                    umma::tmem_st16(tb + kRtap + lane_addr + c, hi);
                    umma::tmem_st16(tb + kRtap + Kr / 2 + lane_addr + c, lo);
                }
                umma::tmem_st_wait();
                umma::fence_before();
                umma::mbar_arrive(&aready);
                cur = it.job;
            }
            const int nb = tiles_of(it.chunk) + 2;
            for (int j = 0; j < nb; ++j, ++gb) {
                mbar_wait(&rfull, gb & 1u);
                umma::fence_after();
                uint32_t v[2][32];  // J 2^(e + rexp) = Wh Fh + Wl Fh (columns 0-63) + Wh Fl (columns 64-127)
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const uint32_t ta = tb + kDrow + ((uint32_t)(32 * quad + 16 * hh) << 16);
                    umma::tmem_ld16x256b_x8(ta, v[hh]);
                    if constexpr (kWideRow) {
                        uint32_t w2[32];
                        umma::tmem_ld16x256b_x8(ta + kT, w2);
                        umma::tmem_ld_wait();
#pragma unroll
                        for (int q = 0; q < 32; ++q)
                            v[hh][q] = __float_as_uint(__uint_as_float(v[hh][q]) + __uint_as_float(w2[q]));
                    }
                }
                if constexpr (!kWideRow) umma::tmem_ld_wait();
                umma::fence_before();
                umma::mbar_arrive(&rempty);
                const uint32_t slot = gb % kJSlots;
                mbar_wait(&jempty[slot], ((gb / kJSlots) & 1u) ^ 1u);
                if (!(a.dbg & 8)) {
                    const uint32_t sbase = jring_s + slot * kJBytes;
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            uint32_t h0, l0, h1, l1;  // (J rows 8k + 2 (t%4) + {0,1}) of lanes t/4 and t/4 + 8
                            umma::split_f16x2(__uint_as_float(v[hh][4 * k]) * inv_r,
                                              __uint_as_float(v[hh][4 * k + 1]) * inv_r, h0, l0);
                            umma::split_f16x2(__uint_as_float(v[hh][4 * k + 2]) * inv_r,
                                              __uint_as_float(v[hh][4 * k + 3]) * inv_r, h1, l1);
                            umma::stmatrix_x4_trans(sbase + soff[hh] + 1024u * k, h0, h1, l0, l1);
                        }
                }
                umma::fence_async_smem();
                umma::mbar_arrive(&jfull[slot]);
            }
        }
    } else {
        // ---------------- column epilogue (warps 0-7) ----------------
        // M rows are ordered so that the ka and kb rows of an output row sit 8 TMEM lanes apart: row m =
        // 16 g + 8 odd + j holds the (odd ? kb : ka) taps of output row 8 g + j.  Read as m8n8 fragments
        // (16x256b), thread t then holds A = (lane t / 4) and B = (lane t / 4 + 8) of the SAME output row and
        // complex column (t % 4) + 4 k: F_theta = A - iB and F_pi-theta = conj(A + iB) are formed in
        // registers (no shuffles, no staging) and a thread quad stores one whole 32-byte sector per row.
        const int quad = warp & 3, half = warp >> 2;
        const int m = 32 * quad + lane;  // tap rebuild: TMEM lane = M row
        const uint32_t lane_addr = (uint32_t)(32 * quad) << 16;
        const int r = 8 * (m >> 4) + (m & 7), odd = (m >> 3) & 1;
        const int fr = lane >> 2, fc = lane & 3;
        uint8_t* ostg = ostg_all + warp * kStgBytes;
        uint32_t gt = 0, nst = 0;  // tiles, staged passes
        int cur = -1, cexp = 0;
        for (UnitIt it{(int)blockIdx.x}; it.u < nunits; it.u += gridDim.x) {
            it.decode(a);
            const BankUJob& jb = a.jobs[it.job];
            if (it.job != cur) {
                // column taps: M row m, K column k -> t = k - jpc - r: (odd ? kb : ka)[t] 2^cexp
                const float2* w = a.weights + jb.cofs;
                cexp = jb.cexp;
                const float wsc = pow2f(cexp);
                for (int c = 16 * half; c < Kc / 2; c += 32) {
                    uint32_t hi[16], lo[16];
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        float v[2];
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int tt = 2 * (c + q) + e - jpc - r;
                            float x = 0.f;
                            if (tt >= -a.h && tt <= a.h) {
                                const float2 kk = w[tt + a.h];
                                x = (odd ? kk.y : kk.x) * wsc;
                            }
                            v[e] = x;
                        }
                        umma::split_f16x2(v[0], v[1], hi[q], lo[q]);
                    }
                    umma::tmem_st16(tb + kCtap + lane_addr + c, hi);
                    umma::tmem_st16(tb + kCtap + Kc / 2 + lane_addr + c, lo);
                }
                umma::tmem_st_wait();
                umma::fence_before();
                umma::mbar_arrive(&aready);
                cur = it.job;
            }
            const float inv = pow2f(-(jscale_exp(a.maxbits[it.b]) + cexp));
            const int nout = jb.nout;
            const int xf = 2 * (it.strip * kT + 32 * half);  // first float column of this warp's half
            const int plane0 = (int)((jb.dst_off[0] + (int64_t)it.b * a.dst_bstride) / a.hw);
            const int plane1 = (int)((jb.dst_off[nout > 1 ? 1 : 0] + (int64_t)it.b * a.dst_bstride) / a.hw);
            const int y0 = it.chunk * chunk_rows, nt = tiles_of(it.chunk);
            for (int i = 0; i < nt; ++i, ++gt) {
                mbar_wait(&cfull, gt & 1u);
                umma::fence_after();
                uint32_t v[2][32];
#pragma unroll
                for (int hh = 0; hh < 2; ++hh)
                    umma::tmem_ld16x256b_x8(tb + kDcol + ((uint32_t)(32 * quad + 16 * hh) << 16) + 64 * half, v[hh]);
                umma::tmem_ld_wait();
                umma::fence_before();
                umma::mbar_arrive(&cempty);
                const int ybase = y0 + i * kT + 16 * quad;  // output row of the warp's 16-row box
                // four passes (16-column half qq x output o), each one [16 rows][128 B] box through one of the
                // warp's two staging buffers: 8 conflict-free STS.64 per thread, one TMA store (which also
                // clips the image edges); the LSU sees 2 wavefronts per 256 bytes instead of 8
#pragma unroll
                for (int ps = 0; ps < 4; ++ps) {
                    const int qq = ps >> 1, o = ps & 1;
                    if (o == 1 && nout < 2) continue;
                    uint8_t* sb = ostg + 2048 * (nst & 1u);  // buffers alternate over the passes actually stored
                    ++nst;
                    if (lane == 0 && !(a.dbg & 32)) umma::bulk_wait_read<1>();  // the store that last read this buffer is done (32: A/B knob)
                    __syncwarp();
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                        for (int kq = 0; kq < 4; ++kq) {
                            const int k = 4 * qq + kq;
                            const float ar = __uint_as_float(v[hh][4 * k]), ai = __uint_as_float(v[hh][4 * k + 1]);
                            const float br = __uint_as_float(v[hh][4 * k + 2]), bi = __uint_as_float(v[hh][4 * k + 3]);
                            const float2 f = o == 0 ? make_float2((ar + bi) * inv, (ai - br) * inv)
                                                    : make_float2((ar - bi) * inv, -(ai + br) * inv);
                            const int rb = 8 * hh + fr;
                            *reinterpret_cast<float2*>(sb + rb * 128 + (((2 * kq + (fc >> 1)) ^ (rb & 7)) << 4) + 8 * (fc & 1)) = f;
                        }
                    umma::fence_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        if (!(a.dbg & 1)) umma::tma_store_3d(&omap, xf + 32 * qq, ybase, o == 0 ? plane0 : plane1, sb);
                        umma::bulk_commit();
                    }
                }
            }
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

bool bank_umma_supported(int h, int W) {
    return h >= 1 && h <= kJr && W % 8 == 0 && W >= kT && encode_fn() != nullptr;
}

cudaError_t launch_bank_umma(BankUArgs a, const void* fprep, int sms, cudaStream_t s) {
    EncodeFn enc = encode_fn();
    if (!enc) return cudaErrorNotSupported;
    static const int dbg = std::getenv("FGB_UMMA_DBG") ? std::atoi(std::getenv("FGB_UMMA_DBG")) : 0;
    a.dbg = dbg;  // A/B ablation (1 no stores, 2 no MMAs, 4 no image loads, 8 no J conversion)
    a.jpc = (a.h + 15) / 16 * 16;
    a.Kc = kT + 2 * a.jpc;
    if (a.h > kJr || a.xbuf < a.jpc || a.Kc > kT + 2 * kJr) return cudaErrorInvalidValue;
    const int Wp = a.W + 2 * a.xbuf, Hq = a.H + 2 * kBankUPadRows;
    CUtensorMap map;
    cuuint64_t dims[3] = {(cuuint64_t)Wp, (cuuint64_t)Hq, (cuuint64_t)2 * a.batch};
    cuuint64_t strides[2] = {(cuuint64_t)Wp * 2, (cuuint64_t)Wp * 2 * Hq};
    cuuint32_t box[3] = {64, kT, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(fprep), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        std::fprintf(stderr, "bank_umma: tensor map encode failed (Wp %d Hq %d)\n", Wp, Hq);
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
            std::fprintf(stderr, "bank_umma: output tensor map encode failed (W %d H %d planes %lld)\n", a.W, a.H,
                         (long long)a.dst_planes);
            return cudaErrorInvalidValue;
        }
    }
    a.nstrips = (a.W + kT - 1) / kT;
    const int ntiles = (a.H + kT - 1) / kT;
    const int64_t basen = (int64_t)a.nstrips * a.batch * a.njobs;
    // chunks: >= 8 tiles each (2 halo J blocks per chunk), enough units for an even last wave
    const int nch = (int)std::min<int64_t>(std::max<int64_t>(1, (20LL * sms + basen - 1) / basen), std::max(1, ntiles / 8));
    a.ch_tiles = (ntiles + nch - 1) / nch;
    a.nchunks = (ntiles + a.ch_tiles - 1) / a.ch_tiles;
    const int64_t units = basen * a.nchunks;
    // unit order: directs fastest when the split-fp16 image planes do not fit L2 and the units are long enough
    // to amortise a tap rebuild per unit (config 5: DRAM reads per launch 2.5 -> 0.05 GB, launch -4 %; config 3's
    // 8-tile units on L2-resident planes lose 7 % with it); FGB_BANKU_ORDER=0 / 1 forces strips / directs fastest
    static const char* order = std::getenv("FGB_BANKU_ORDER");
    a.job_fastest = order ? std::atoi(order) : (a.ch_tiles >= 32 && (int64_t)a.batch * Hq * Wp * 4 > (96LL << 20));
    const int grid = (int)std::min<int64_t>(units, sms);
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(bank_umma_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(bank_umma_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(bank_umma_kernel<48>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    if (a.jpc == 16)
        bank_umma_kernel<16><<<grid, kThreads, kSmem, s>>>(map, omap, a);
    else if (a.jpc == 32)
        bank_umma_kernel<32><<<grid, kThreads, kSmem, s>>>(map, omap, a);
    else
        bank_umma_kernel<48><<<grid, kThreads, kSmem, s>>>(map, omap, a);
    return cudaGetLastError();
}

}  // namespace fgb
