// Probe: write-only HBM bandwidth on B200 by store flavour and address pattern.
// Every bank kernel of this repo is bounded by its output stream (8 B per
// px*filter, 43 GB per config-5 step), so the write-only ceiling -- not the
// copy bandwidth -- is what the output stores can reach.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        tools/probes/write_probe.cu -o tools/probes/write_probe
//
// mode 0 st.global.v4 (default policy)      mode 1 st.global.cs.v4 (streaming)
// mode 2 st.global.wt.v4                     mode 3 st.global.L2::cache_hint evict_first
// mode 4 cp.async.bulk shared -> global (16 KB per CTA and step)
// mode 5 st.global.cs.v4, tile pattern: 512-byte row segments at a 64 KB pitch,
//        64 rows x 2 planes per tile (the column epilogues' pattern)
// mode 6 st.global.cs.v2, tile pattern by thread quads (32-byte sectors)
// mode 7 cp.async.bulk shared -> global, tile pattern (512 B per row and copy)
// mode 8 cudaMemsetAsync
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            std::exit(1);                                                                  \
        }                                                                                  \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int MODE> __global__ void __launch_bounds__(256) wr_linear(float4* dst, size_t n16) {
    const float4 v = make_float4(1.f, 2.f, 3.f, (float)blockIdx.x);
    uint64_t pol = 0;
    if (MODE == 3) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
    // each CTA writes contiguous 4 KB blocks, grid-stride
    for (size_t i = (size_t)blockIdx.x * 256 + threadIdx.x; i < n16; i += (size_t)gridDim.x * 256) {
        float4* p = dst + i;
        if (MODE == 0) asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};\n" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
        if (MODE == 1) asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};\n" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
        if (MODE == 2) asm volatile("st.global.wt.v4.f32 [%0], {%1,%2,%3,%4};\n" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
        if (MODE == 3)
            asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;\n" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
                         : "memory");
    }
}

__global__ void __launch_bounds__(256) wr_bulk(uint8_t* dst, size_t nbytes) {
    __shared__ __align__(128) uint8_t buf[16384];
    for (int i = threadIdx.x; i < 16384 / 4; i += 256) reinterpret_cast<float*>(buf)[i] = (float)i;
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        int inflight = 0;
        for (size_t o = (size_t)blockIdx.x * 16384; o + 16384 <= nbytes; o += (size_t)gridDim.x * 16384) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst + o), "r"(smem_u32(buf)), "r"(16384) : "memory");
            asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
            if (++inflight >= 8) asm volatile("cp.async.bulk.wait_group.read 7;\n" ::: "memory");
        }
        asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    }
}

// tile pattern: planes of H x W complex64 (W = 8192: 64 KB rows); a tile = 64 rows x 64 complex (512 B) x 2 planes;
// CTA c takes tiles c, c + grid, ... with strips fastest (as the column kernels)
template <int MODE> __global__ void __launch_bounds__(256) wr_tiles(uint8_t* dst, int nplanes, int H, int W) {
    __shared__ __align__(128) uint8_t buf[8192];
    const int nstrips = W / 64, ntr = H / 64;
    const size_t rowb = (size_t)W * 8, planeb = rowb * H;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (MODE == 7) {
        for (int i = threadIdx.x; i < 2048; i += 256) reinterpret_cast<float*>(buf)[i] = (float)i;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();
    }
    const int ntiles = (nplanes / 2) * ntr * nstrips;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int strip = t % nstrips, tr = (t / nstrips) % ntr, pp = t / (nstrips * ntr);
        uint8_t* base = dst + (size_t)(2 * pp) * planeb + (size_t)(tr * 64) * rowb + (size_t)strip * 512;
        if (MODE == 5) {
            // warp w: rows 8 w .. 8 w + 7; per instruction 4 rows x 128 B... here: lane -> 16 B of a 512-B row
            for (int r = 0; r < 8; ++r)
                for (int pl = 0; pl < 2; ++pl) {
                    uint8_t* p = base + pl * planeb + (size_t)(8 * warp + r) * rowb + lane * 16;
                    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};\n" ::"l"(p), "f"(1.f), "f"(2.f), "f"(3.f), "f"((float)t) : "memory");
                }
        } else if (MODE == 6) {
            // thread quads write 32-byte sectors: warp w rows 8 w + lane / 4, 16 steps of 32 B across the 512-B row
            for (int k = 0; k < 16; ++k)
                for (int pl = 0; pl < 2; ++pl) {
                    uint8_t* p = base + pl * planeb + (size_t)(8 * warp + (lane >> 2)) * rowb + k * 32 + (lane & 3) * 8;
                    asm volatile("st.global.cs.v2.f32 [%0], {%1,%2};\n" ::"l"(p), "f"(1.f), "f"((float)t) : "memory");
                }
        } else {
            if (lane == 0) {
                for (int r = 0; r < 8; ++r)
                    for (int pl = 0; pl < 2; ++pl) {
                        uint8_t* p = base + pl * planeb + (size_t)(8 * warp + r) * rowb;
                        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(p), "r"(smem_u32(buf + 512 * (r & 7))), "r"(512)
                                     : "memory");
                    }
                asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 4;\n" ::: "memory");
            }
        }
    }
    if (MODE == 7 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

int main(int argc, char** argv) {
    const size_t nbytes = (size_t)8 << 30;  // 16 planes of 8192 x 8192 complex64
    uint8_t* d;
    CK(cudaMalloc(&d, nbytes));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int ctas_list[3] = {148, 592, 1184};
    for (int mode = 0; mode <= 8; ++mode)
        for (int ci = 0; ci < 3; ++ci) {
            const int ctas = ctas_list[ci];
            if (mode == 8 && ci > 0) continue;
            auto run = [&] {
                switch (mode) {
                    case 0: wr_linear<0><<<ctas, 256>>>((float4*)d, nbytes / 16); break;
                    case 1: wr_linear<1><<<ctas, 256>>>((float4*)d, nbytes / 16); break;
                    case 2: wr_linear<2><<<ctas, 256>>>((float4*)d, nbytes / 16); break;
                    case 3: wr_linear<3><<<ctas, 256>>>((float4*)d, nbytes / 16); break;
                    case 4: wr_bulk<<<ctas, 256>>>(d, nbytes); break;
                    case 5: wr_tiles<5><<<ctas, 256>>>(d, 16, 8192, 8192); break;
                    case 6: wr_tiles<6><<<ctas, 256>>>(d, 16, 8192, 8192); break;
                    case 7: wr_tiles<7><<<ctas, 256>>>(d, 16, 8192, 8192); break;
                    case 8: CK(cudaMemsetAsync(d, 1, nbytes)); break;
                }
            };
            run();
            CK(cudaDeviceSynchronize());
            CK(cudaEventRecord(e0));
            for (int r = 0; r < 3; ++r) run();
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            CK(cudaGetLastError());
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            std::printf("mode %d ctas %4d: %.3f ms per 8 GiB, %.0f GB/s\n", mode, ctas, ms / 3, nbytes / (ms / 3) / 1e6);
        }
    (void)argc;
    (void)argv;
    return 0;
}
