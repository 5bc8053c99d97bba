// Shared device/host helpers for libfgb200 (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fgb {

// Complex sample type per precision: float2 for the fp32 build, double2 for
// the fp64 validation build.  Interleaved (re, im) = one 8 / 16 byte access.
template <typename T> struct cx;
template <> struct cx<float> { using type = float2; };
template <> struct cx<double> { using type = double2; };
template <typename T> using cx_t = typename cx<T>::type;

template <typename T> __host__ __device__ inline cx_t<T> mk(T a, T b) { cx_t<T> r; r.x = a; r.y = b; return r; }

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Streaming (evict-first) stores for final outputs, so the L2 keeps the
// row-pass intermediates J resident for the column pass.
__device__ __forceinline__ void st_cs(float2* p, float2 v) { __stcs(p, v); }
__device__ __forceinline__ void st_cs(double2* p, double2 v) { __stcs(p, v); }

// Asynchronous global->shared copies (LDGSTS): every thread issues all of its
// tile copies back to back, then waits once -- the tile load costs one
// memory latency instead of one per row.
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
template <int BYTES> __device__ __forceinline__ void cp_async(void* smem, const void* gmem) {
    if constexpr (BYTES == 4) cp_async4(smem, gmem);
    else if constexpr (BYTES == 8) cp_async8(smem, gmem);
    else cp_async16(smem, gmem);
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Bulk (non-tensor) async copies global -> shared completing on an mbarrier:
// one instruction moves a contiguous run (multiple of 16 bytes, 16-byte aligned).
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// (the suspend-time hint parks the waiting warps instead of spinning on issue slots)
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// Output descriptor of one column job (one J source, up to 4 outputs).
//   X = A - iB, Y = A + iB with A = sum ka[t] J[y+t], B = sum kb[t] J[y+t];
//   out_o = phase_o * (conj_o ? conj(base_o) : base_o)
// Plans are immutable and cached: jobs hold element offsets relative to the
// per-call base pointers carried in the launch arguments.
template <typename T> struct ColJob {
    int64_t src_off;         // complex elements from src_base (batch 0)
    int64_t dst_off[4];      // complex elements from dst_base (batch 0)
    T phase_re[4], phase_im[4];
    int32_t wofs;            // offset (in taps) into the weight pool
    int32_t nout;
    int8_t base[4];          // 0 = X, 1 = Y
    int8_t conj[4];
    int32_t has_b;           // kb != 0 (0 for the theta = 0 / v = 0 jobs: A only)
    int32_t mode;            // epilogue: 0 generic, 1 Gabor X only, 2 Gabor X + conj(Y) (no phase)
    int32_t realj;           // fp32 kernel, mode 1: J is real to ~1e-12 (theta = pi/2: the row phase step
                             // omega cos(theta) ~ 1e-17), so A and B read only Re J (half the FMAs)
    int32_t wexp;            // tensor-core column pass: taps scaled by 2^wexp (|scaled| < 2^10)
};

// Row job group: up to kMaxND jobs sharing one input row and one symmetric
// tap range [-h, h]:  J_k = phase_k * sum_t (kr_k[|t|] + i sgn(t) ki_k[|t|]) f[x+t]
constexpr int kMaxND = 8;
template <typename T> struct RowGroup {
    int64_t dst_off[kMaxND]; // complex elements from dst_base
    T phase_re[kMaxND], phase_im[kMaxND];
    int32_t wofs;            // offset (in T units) of the [(hp+1)][NDP][2] table
    int32_t nd;
    int32_t has_phase;
    int32_t last_real;       // fp32: the last job's J is real to <= 1e-12 |J| (theta = pi/2, row phase step
                             // omega cos(theta) ~ 1e-17): its taps accumulate Re J only (scalar FFMA)
};

}  // namespace fgb
