// GBNK container writer fed from device buffers.
//
// Format (image_io.py:157-212 of the reference): b"GBNK", <IIII (version | SDFT
// flag bit 24, width, height, count), then per entry <ddd params followed by
// the real and the imaginary planes as little-endian float64 [H][W].
// The device outputs are interleaved complex (float2/double2); each entry is
// split into two f64 planes by a small kernel, copied to one of two pinned
// staging buffers (async, one stream) and written to the file while the next
// entry is converted and copied.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>

#include "common.cuh"
#include "kernels.h"

namespace fgb {

namespace {

template <typename T>
__global__ void planar_f64(const cx_t<T>* in, int64_t n, double* re, double* im) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const cx_t<T> v = in[i];
        re[i] = (double)v.x;
        im[i] = (double)v.y;
    }
}

// [entries][H*W] interleaved complex -> [entries][2][H*W] f64 planes (re then
// im per entry, the reference's ComplexImage layout) + a non-finite flag.
template <typename T>
__global__ void entries_planar_f64(const cx_t<T>* in, int64_t n, int64_t plane, double* out, int* nonfinite) {
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const cx_t<T> v = in[i];
        const int64_t e = i / plane, q = i - e * plane;
        const double re = (double)v.x, im = (double)v.y;
        __stcs(out + 2 * e * plane + q, re);
        __stcs(out + (2 * e + 1) * plane + q, im);
        bad |= !(isfinite(re) && isfinite(im));
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1);
}

}  // namespace

template <typename T>
cudaError_t launch_entries_planar(const cx_t<T>* in, int64_t n, int64_t plane, double* out, int* nonfinite,
                                  cudaStream_t s) {
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>((n + threads - 1) / threads, 148 * 16);
    entries_planar_f64<T><<<blocks, threads, 0, s>>>(in, n, plane, out, nonfinite);
    return cudaGetLastError();
}
template cudaError_t launch_entries_planar<float>(const float2*, int64_t, int64_t, double*, int*, cudaStream_t);
template cudaError_t launch_entries_planar<double>(const double2*, int64_t, int64_t, double*, int*, cudaStream_t);

// Returns 0 on success, -1 on I/O failure, -2 on CUDA failure (message in *err).
int gbnk_write_device(const char* path, const double* params, int n_entries, int H, int W, int dtype,
                      const void* dev_entries, int sdft, cudaStream_t s, std::string* err) {
    const int64_t plane = (int64_t)H * W;
    FILE* fh = std::fopen(path, "wb");
    if (!fh) {
        *err = std::string("cannot open ") + path;
        return -1;
    }
    const uint32_t hdr[4] = {(uint32_t)(1u | (sdft ? (1u << 24) : 0u)), (uint32_t)W, (uint32_t)H, (uint32_t)n_entries};
    bool ok = std::fwrite("GBNK", 1, 4, fh) == 4 && std::fwrite(hdr, 4, 4, fh) == 4;
    double* dstage = nullptr;
    double* hstage[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    auto cuda_fail = [&](cudaError_t e) {
        *err = std::string("CUDA: ") + cudaGetErrorString(e);
        return -2;
    };
    int rc = 0;
    cudaError_t e = cudaMalloc(&dstage, 2 * plane * sizeof(double) * 2);
    if (e != cudaSuccess) rc = cuda_fail(e);
    for (int i = 0; i < 2 && rc == 0; ++i) {
        e = cudaMallocHost(&hstage[i], 2 * plane * sizeof(double));
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
        if (e != cudaSuccess) rc = cuda_fail(e);
    }
    auto flush = [&](int k, int buf) {  // wait for entry k's copy, write params + planes
        if (cudaEventSynchronize(ev[buf]) != cudaSuccess) return false;
        const double* pr = params + 3 * (size_t)k;
        return std::fwrite(pr, 8, 3, fh) == 3 &&
               std::fwrite(hstage[buf], sizeof(double), 2 * plane, fh) == (size_t)(2 * plane);
    };
    const int threads = 256, blocks = (int)std::min<int64_t>((plane + threads - 1) / threads, 148 * 16);
    for (int k = 0; k < n_entries && rc == 0 && ok; ++k) {
        const int buf = k & 1;
        double* d = dstage + (size_t)buf * 2 * plane;
        if (dtype == 0) {
            planar_f64<float><<<blocks, threads, 0, s>>>((const float2*)dev_entries + (size_t)k * plane, plane, d, d + plane);
        } else {
            planar_f64<double><<<blocks, threads, 0, s>>>((const double2*)dev_entries + (size_t)k * plane, plane, d,
                                                          d + plane);
        }
        if (k >= 2) ok = flush(k - 2, buf);  // this staging buffer's previous entry is on disk before reuse
        e = cudaMemcpyAsync(hstage[buf], d, 2 * plane * sizeof(double), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaEventRecord(ev[buf], s);
        if (e != cudaSuccess) rc = cuda_fail(e);
    }
    for (int k = std::max(0, n_entries - 2); k < n_entries && rc == 0 && ok; ++k) ok = flush(k, k & 1);
    if (!ok && rc == 0) {
        *err = std::string("write failed: ") + path;
        rc = -1;
    }
    if (std::fclose(fh) != 0 && rc == 0) {
        *err = std::string("close failed: ") + path;
        rc = -1;
    }
    for (int i = 0; i < 2; ++i) {
        if (hstage[i]) cudaFreeHost(hstage[i]);
        if (ev[i]) cudaEventDestroy(ev[i]);
    }
    if (dstage) cudaFree(dstage);
    return rc;
}

}  // namespace fgb
