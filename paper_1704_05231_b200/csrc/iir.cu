// K4: recursive-Gaussian (RecursiveIIR) column stage, fp64 recursion state.
//
// Restates gaussian.py:215-228 (_iir_lines with assume_padded: the stage
// already replicate-padded by P = ceil(5 sigma)+2, gaussian.py:211) inside
// the modulate / smooth / recombine stage of gabor.py:135-164 and
// sdft.py:75-131:
//   forward : y[n] = B z[n] - a1 y[n-1] - a2 y[n-2] - a3 y[n-3],
//             y[-1] = y[-2] = y[-3] = z[0]  (lfilter_zi * x[0] steady state)
//   backward: u[n] = B y[n] - a1 u[n+1] - a2 u[n+2] - a3 u[n+3],
//             u[L] = u[L+1] = u[L+2] = y[L-1]
// The recursion must run in fp64 (an fp32 recursion
// misses 1e-5 by up to 125x at sigma=32); the forward sequence is parked in
// a scratch plane of the storage type T (coalesced: thread = column).
// Row stages run through this kernel on a transposed image.
#include "common.cuh"
#include "kernels.h"

namespace fgb {

namespace {

constexpr int kIirThreads = 128;

template <typename T>
__global__ void __launch_bounds__(kIirThreads) iir_col_kernel(IirArgs<T> a) {
    const int x = blockIdx.x * kIirThreads + threadIdx.x;
    const int jb = blockIdx.y % a.njobs;
    const int b = blockIdx.y / a.njobs;
    if (x >= a.W) return;
    const IirJob<T>& job = a.jobs[jb];
    const int H = a.H, W = a.W, P = a.P;
    const int L = H + 2 * P;
    const cx_t<T>* src = a.src_base + job.src_off + (size_t)b * a.src_bstride + x;
    const double2* tabm = a.tab_base + job.tabm_off;
    const double2* tabr = a.tab_base + job.tabr_off;
    T* sc = a.scratch + (size_t)blockIdx.y * 4 * L * W + x;
    const size_t plane = (size_t)L * W;
    const bool n0 = job.need & 1, n1 = (job.need >> 1) & 1;
    const double B = a.c.B, a1 = a.c.a1, a2 = a.c.a2, a3 = a.c.a3;

    // ---- forward sweep over the replicate-padded column ----
    double p[4][3];  // planes: 0 = pair0.a, 1 = pair0.b, 2 = pair1.a, 3 = pair1.b
    double z[4];
    {
        const cx_t<T> v = src[0];  // clamp(-P) = row 0
        const double2 cs = tabm[0];
        const double jr = v.x, ji = v.y;
        z[0] = jr * cs.x + ji * cs.y;
        z[1] = jr * cs.y - ji * cs.x;
        z[2] = jr * cs.x - ji * cs.y;
        z[3] = jr * cs.y + ji * cs.x;
#pragma unroll
        for (int q = 0; q < 4; ++q) p[q][0] = p[q][1] = p[q][2] = z[q];
    }
#pragma unroll 2
    for (int n = 0; n < L; ++n) {
        const int yy = clampi(n - P, 0, H - 1);
        const cx_t<T> v = src[(size_t)yy * W];
        const double2 cs = tabm[n];
        const double jr = v.x, ji = v.y;
        z[0] = jr * cs.x + ji * cs.y;
        z[1] = jr * cs.y - ji * cs.x;
        z[2] = jr * cs.x - ji * cs.y;
        z[3] = jr * cs.y + ji * cs.x;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if ((q < 2 && !n0) || (q >= 2 && !n1)) continue;
            const double t = fma(B, z[q], -(a2 * p[q][1] + a3 * p[q][2]));
            const double yv = fma(-a1, p[q][0], t);
            p[q][2] = p[q][1];
            p[q][1] = p[q][0];
            p[q][0] = yv;
            sc[q * plane + (size_t)n * W] = (T)yv;
        }
    }
    // ---- backward sweep, recombination on the cropped rows ----
    double u[4][3];
#pragma unroll
    for (int q = 0; q < 4; ++q) u[q][0] = u[q][1] = u[q][2] = p[q][0];
    const size_t ob = (size_t)b * a.dst_bstride + x;
    for (int n = L - 1; n >= 0; --n) {
        double s[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if ((q < 2 && !n0) || (q >= 2 && !n1)) { s[q] = 0.0; continue; }
            const double yv = (n == L - 1) ? p[q][0] : (double)sc[q * plane + (size_t)n * W];
            const double t = fma(B, yv, -(a2 * u[q][1] + a3 * u[q][2]));
            const double uv = fma(-a1, u[q][0], t);
            u[q][2] = u[q][1];
            u[q][1] = u[q][0];
            u[q][0] = uv;
            s[q] = uv;
        }
        const int yo = n - P;
        if (yo < 0 || yo >= H) continue;
        const double2 cs = tabr[yo];
        for (int o = 0; o < job.nout; ++o) {
            const int pr = job.pair[o];
            const double sa = s[2 * pr], sb = s[2 * pr + 1];
            double re = cs.x * sa + cs.y * sb;
            double im = job.sdft ? (cs.x * sb - cs.y * sa) : (cs.y * sa - cs.x * sb);
            if (job.conj[o]) im = -im;
            a.dst_base[job.dst_off[o] + ob + (size_t)yo * W] = mk<T>((T)re, (T)im);
        }
    }
}

}  // namespace

template <typename T> size_t iir_scratch_elems(int H, int W, int P, int njobs, int batch) {
    return (size_t)njobs * batch * 4 * (size_t)(H + 2 * P) * W;
}

template <typename T> cudaError_t launch_iir_col(const IirArgs<T>& a, cudaStream_t s) {
    dim3 grid((a.W + kIirThreads - 1) / kIirThreads, a.njobs * a.batch);
    iir_col_kernel<T><<<grid, kIirThreads, 0, s>>>(a);
    return cudaGetLastError();
}

template size_t iir_scratch_elems<float>(int, int, int, int, int);
template size_t iir_scratch_elems<double>(int, int, int, int, int);
template cudaError_t launch_iir_col<float>(const IirArgs<float>&, cudaStream_t);
template cudaError_t launch_iir_col<double>(const IirArgs<double>&, cudaStream_t);

}  // namespace fgb
