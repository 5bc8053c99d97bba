// Tiled transposes used by the side routes that run a row stage through the
// column kernels (box window, IIR row pass, the My < Mx SDFT route of
// sdft.py:185-195).  32x32 tiles through padded shared memory.
#include "common.cuh"
#include "kernels.h"

namespace fgb {

namespace {

template <typename T>
__global__ void tr_real_cx(const T* in, int64_t pitch, int64_t ibs, cx_t<T>* out, int64_t obs, int H, int W) {
    __shared__ T t[32][33];
    const int b = blockIdx.z;
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
    in += (size_t)b * ibs;
    out += (size_t)b * obs;
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        int y = y0 + j, x = x0 + threadIdx.x;
        if (y < H && x < W) t[j][threadIdx.x] = in[(size_t)y * pitch + x];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        int x = x0 + j, y = y0 + threadIdx.x;  // out[x][y]
        if (y < H && x < W) out[(size_t)x * H + y] = mk<T>(t[threadIdx.x][j], T(0));
    }
}

template <typename T>
__global__ void tr_real(const T* in, int64_t pitch, int64_t ibs, T* out, int64_t obs, int H, int W) {
    __shared__ T t[32][33];
    const int b = blockIdx.z;
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
    in += (size_t)b * ibs;
    out += (size_t)b * obs;
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        int y = y0 + j, x = x0 + threadIdx.x;
        if (y < H && x < W) t[j][threadIdx.x] = in[(size_t)y * pitch + x];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        int x = x0 + j, y = y0 + threadIdx.x;
        if (y < H && x < W) out[(size_t)x * H + y] = t[threadIdx.x][j];
    }
}

template <typename T>
__global__ void tr_cx(const cx_t<T>* in, int64_t ibs, cx_t<T>* out, int64_t obs, int H, int W) {
    __shared__ cx_t<T> t[32][33];
    const int b = blockIdx.z;
    const int x0 = blockIdx.x * 32, y0 = blockIdx.y * 32;
    in += (size_t)b * ibs;
    out += (size_t)b * obs;
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        int y = y0 + j, x = x0 + threadIdx.x;
        if (y < H && x < W) t[j][threadIdx.x] = in[(size_t)y * W + x];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        int x = x0 + j, y = y0 + threadIdx.x;
        if (y < H && x < W) out[(size_t)x * H + y] = t[threadIdx.x][j];
    }
}

}  // namespace

template <typename T>
cudaError_t launch_transpose_real_to_cx(const T* in, int64_t pitch, int64_t ibs, cx_t<T>* out, int64_t obs, int H,
                                        int W, int batch, cudaStream_t s) {
    dim3 grid((W + 31) / 32, (H + 31) / 32, batch);
    tr_real_cx<T><<<grid, dim3(32, 8), 0, s>>>(in, pitch, ibs, out, obs, H, W);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_transpose_real(const T* in, int64_t pitch, int64_t ibs, T* out, int64_t obs, int H, int W,
                                  int batch, cudaStream_t s) {
    dim3 grid((W + 31) / 32, (H + 31) / 32, batch);
    tr_real<T><<<grid, dim3(32, 8), 0, s>>>(in, pitch, ibs, out, obs, H, W);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_transpose_cx(const cx_t<T>* in, int64_t ibs, cx_t<T>* out, int64_t obs, int H, int W, int batch,
                                cudaStream_t s) {
    dim3 grid((W + 31) / 32, (H + 31) / 32, batch);
    tr_cx<T><<<grid, dim3(32, 8), 0, s>>>(in, ibs, out, obs, H, W);
    return cudaGetLastError();
}

template cudaError_t launch_transpose_real_to_cx<float>(const float*, int64_t, int64_t, float2*, int64_t, int, int, int,
                                                        cudaStream_t);
template cudaError_t launch_transpose_real_to_cx<double>(const double*, int64_t, int64_t, double2*, int64_t, int, int,
                                                         int, cudaStream_t);
template cudaError_t launch_transpose_real<float>(const float*, int64_t, int64_t, float*, int64_t, int, int, int,
                                                  cudaStream_t);
template cudaError_t launch_transpose_real<double>(const double*, int64_t, int64_t, double*, int64_t, int, int, int,
                                                   cudaStream_t);
template cudaError_t launch_transpose_cx<float>(const float2*, int64_t, float2*, int64_t, int, int, int, cudaStream_t);
template cudaError_t launch_transpose_cx<double>(const double2*, int64_t, double2*, int64_t, int, int, int,
                                                 cudaStream_t);

}  // namespace fgb
