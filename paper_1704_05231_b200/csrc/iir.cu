// K4: recursive-Gaussian (RecursiveIIR) column stage, fp64 recursion state,
// segment-parallel.
//
// Restates gaussian.py:215-228 (_iir_lines with assume_padded: the stage
// already replicate-padded by P = ceil(5 sigma)+2, gaussian.py:211) inside
// the modulate / smooth / recombine stage of gabor.py:135-164 and
// sdft.py:75-131:
//   forward : y[n] = B z[n] - a1 y[n-1] - a2 y[n-2] - a3 y[n-3],
//             y[-1] = y[-2] = y[-3] = z[0]  (lfilter_zi * x[0] steady state)
//   backward: u[n] = B y[n] - a1 u[n+1] - a2 u[n+2] - a3 u[n+3],
//             u[L] = u[L+1] = u[L+2] = y[L-1]
// The recursion runs in fp64 (an fp32 recursion misses 1e-5 by up to 125x
// at sigma = 32).
//
// Parallelisation is EXACT (no warm-up approximation): each column is cut
// into NS segments.  A segment runs its recursion from a zero state; with
// the companion matrix A = [[-a1,-a2,-a3],[1,0,0],[0,1,0]] the true output is
//     y[a+m] = y_loc[a+m] + g_m . s_in,   g_m = first row of A^(m+1),
// where s_in is the true 3-sample state entering the segment, and the states
// chain as s_out = s_loc_end + A^len s_in (a 3x3 scan over segments).  The
// backward pass is the same recursion on reversed indices.  Three kernels:
//   fwd  : modulate, local forward recursion -> y_loc (storage type), end states
//   bwd  : carry-in, correct y, local backward recursion -> u_loc, start states
//   out  : carry-in, correct u, recombine -> outputs
#include "common.cuh"
#include "kernels.h"

namespace fgb {

namespace {

constexpr int kIirTX = 32;
constexpr int kIirU = 3;  // samples per load batch

__device__ __forceinline__ void mat3_apply(const double* A, const double* s, double* o) {
    o[0] = A[0] * s[0] + A[1] * s[1] + A[2] * s[2];
    o[1] = A[3] * s[0] + A[4] * s[1] + A[5] * s[2];
    o[2] = A[6] * s[0] + A[7] * s[1] + A[8] * s[2];
}

template <typename T>
__device__ __forceinline__ void modulate(const IirJob<T>& job, cx_t<T> v, double2 cs, double* z) {
    const double jr = v.x, ji = v.y;
    z[0] = jr * cs.x + ji * cs.y;  // pair 0
    z[1] = jr * cs.y - ji * cs.x;
    z[2] = jr * cs.x - ji * cs.y;  // pair 1
    z[3] = jr * cs.y + ji * cs.x;
}

__device__ __forceinline__ bool plane_used(int need, int q) { return (need >> (q >> 1)) & 1; }

// ---- pass 1: modulate + zero-state forward recursion per segment ----
template <typename T>
__global__ void __launch_bounds__(128) iir_fwd(IirArgs<T> a) {
    const int x = blockIdx.x * kIirTX + threadIdx.x;
    const int seg = blockIdx.y * blockDim.y + threadIdx.y;
    const int jb = blockIdx.z % a.njobs;
    const int b = blockIdx.z / a.njobs;
    if (x >= a.W || seg >= a.nseg) return;
    const IirJob<T>& job = a.jobs[jb];
    const int H = a.H, W = a.W, P = a.P, L = H + 2 * P;
    const int n0 = seg * a.seglen, n1 = min(L, n0 + a.seglen);
    const cx_t<T>* src = a.src_base + job.src_off + (size_t)b * a.src_bstride + x;
    const double2* tabm = a.tab_base + job.tabm_off;
    T* sc = a.scratch + (size_t)blockIdx.z * 4 * L * W + x;
    const size_t plane = (size_t)L * W;
    const double B = a.c.B, a1 = a.c.a1, a2 = a.c.a2, a3 = a.c.a3;
    const int need = job.need;
    double p[4][3];
    double z[4];
    if (seg == 0) {  // the reference's steady-state init on the first padded sample
        modulate<T>(job, src[0], tabm[0], z);
#pragma unroll
        for (int q = 0; q < 4; ++q) p[q][0] = p[q][1] = p[q][2] = z[q];
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) p[q][0] = p[q][1] = p[q][2] = 0.0;
    }
    // kIirU input samples are loaded before the dependent recursion consumes
    // them (the stores into scratch would otherwise keep the compiler from
    // hoisting the next loads: one load in flight per thread)
    for (int nb = n0; nb < n1; nb += kIirU) {
        cx_t<T> v[kIirU];
#pragma unroll
        for (int u = 0; u < kIirU; ++u)
            if (nb + u < n1) v[u] = src[(size_t)clampi(nb + u - P, 0, H - 1) * W];
#pragma unroll
        for (int u = 0; u < kIirU; ++u) {
            const int n = nb + u;
            if (n >= n1) break;
            modulate<T>(job, v[u], tabm[n], z);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (!plane_used(need, q)) continue;
                const double t = fma(B, z[q], -(a2 * p[q][1] + a3 * p[q][2]));
                const double yv = fma(-a1, p[q][0], t);
                p[q][2] = p[q][1];
                p[q][1] = p[q][0];
                p[q][0] = yv;
                sc[q * plane + (size_t)n * W] = (T)yv;
            }
        }
    }
    // local end state (y[end], y[end-1], y[end-2]) per plane
    double* st = a.state + (((size_t)blockIdx.z * a.nseg + seg) * 12) * W + x;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int k = 0; k < 3; ++k) st[(size_t)(q * 3 + k) * W] = p[q][k];
}

// ---- pass 2: forward carry + correction, zero-state backward recursion ----
template <typename T>
__global__ void __launch_bounds__(128) iir_bwd(IirArgs<T> a) {
    const int x = blockIdx.x * kIirTX + threadIdx.x;
    const int seg = blockIdx.y * blockDim.y + threadIdx.y;
    const int jb = blockIdx.z % a.njobs;
    if (x >= a.W || seg >= a.nseg) return;
    const IirJob<T>& job = a.jobs[jb];
    const int H = a.H, W = a.W, P = a.P, L = H + 2 * P;
    const int n0 = seg * a.seglen, n1 = min(L, n0 + a.seglen);
    T* sc = a.scratch + (size_t)blockIdx.z * 4 * L * W + x;
    const size_t plane = (size_t)L * W;
    const double B = a.c.B, a1 = a.c.a1, a2 = a.c.a2, a3 = a.c.a3;
    const int need = job.need;
    double* st_all = a.state + ((size_t)blockIdx.z * a.nseg * 12) * W + x;
    // true state entering this segment: scan the local end states of segments < seg
    double s_in[4][3];
#pragma unroll
    for (int q = 0; q < 4; ++q) s_in[q][0] = s_in[q][1] = s_in[q][2] = 0.0;
    for (int j = 0; j < seg; ++j) {
        const double* sj = st_all + (size_t)j * 12 * W;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            double o[3];
            mat3_apply(a.Aseg, s_in[q], o);  // segments < last are full length
#pragma unroll
            for (int k = 0; k < 3; ++k) s_in[q][k] = o[k] + sj[(size_t)(q * 3 + k) * W];
        }
    }
    // backward local recursion from the segment end, on the corrected forward output
    double u[4][3];
    if (seg == a.nseg - 1) {  // u[L..L+2] = y[L-1] (true value)
        const int m = n1 - 1 - n0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double yl = plane_used(need, q) ? (double)sc[q * plane + (size_t)(n1 - 1) * W] : 0.0;
            const double* g = a.g + 3 * m;
            const double yv = seg == 0 ? yl : yl + g[0] * s_in[q][0] + g[1] * s_in[q][1] + g[2] * s_in[q][2];
            u[q][0] = u[q][1] = u[q][2] = yv;
        }
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) u[q][0] = u[q][1] = u[q][2] = 0.0;
    }
    for (int nb = n1 - 1; nb >= n0; nb -= kIirU) {
        T ys[kIirU][4];
#pragma unroll
        for (int u = 0; u < kIirU; ++u)
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (nb - u >= n0 && plane_used(need, q)) ys[u][q] = sc[q * plane + (size_t)(nb - u) * W];
#pragma unroll
        for (int uu = 0; uu < kIirU; ++uu) {
            const int n = nb - uu;
            if (n < n0) break;
            const double* g = a.g + 3 * (n - n0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (!plane_used(need, q)) continue;
                const double yl = (double)ys[uu][q];
                const double yv = seg == 0 ? yl : yl + g[0] * s_in[q][0] + g[1] * s_in[q][1] + g[2] * s_in[q][2];
                const double t = fma(B, yv, -(a2 * u[q][1] + a3 * u[q][2]));
                const double uv = fma(-a1, u[q][0], t);
                u[q][2] = u[q][1];
                u[q][1] = u[q][0];
                u[q][0] = uv;
                sc[q * plane + (size_t)n * W] = (T)uv;
            }
        }
    }
    // local start state (u[start], u[start+1], u[start+2]) -> the backward half of the state buffer
    double* st = st_all + ((size_t)a.njobs * a.batch * a.nseg * 12) * W + (size_t)seg * 12 * W;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int k = 0; k < 3; ++k) st[(size_t)(q * 3 + k) * W] = u[q][k];
}

// ---- pass 3: backward carry + correction, recombination, outputs ----
template <typename T>
__global__ void __launch_bounds__(128) iir_out(IirArgs<T> a) {
    const int x = blockIdx.x * kIirTX + threadIdx.x;
    const int seg = blockIdx.y * blockDim.y + threadIdx.y;
    const int jb = blockIdx.z % a.njobs;
    const int b = blockIdx.z / a.njobs;
    if (x >= a.W || seg >= a.nseg) return;
    const IirJob<T>& job = a.jobs[jb];
    const int H = a.H, W = a.W, P = a.P, L = H + 2 * P;
    const int n0 = seg * a.seglen, n1 = min(L, n0 + a.seglen);
    if (n1 <= P || n0 >= P + H) return;  // nothing of this segment survives the crop
    T* sc = a.scratch + (size_t)blockIdx.z * 4 * L * W + x;
    const size_t plane = (size_t)L * W;
    const double* st_all = a.state + ((size_t)a.njobs * a.batch * a.nseg * 12) * W +
                           ((size_t)blockIdx.z * a.nseg * 12) * W + x;
    // true state entering this segment from above: scan local start states of segments > seg
    double t_in[4][3];
#pragma unroll
    for (int q = 0; q < 4; ++q) t_in[q][0] = t_in[q][1] = t_in[q][2] = 0.0;
    for (int j = a.nseg - 1; j > seg; --j) {
        const double* sj = st_all + (size_t)j * 12 * W;
        const double* A = (j == a.nseg - 1) ? a.Alast : a.Aseg;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            double o[3];
            mat3_apply(A, t_in[q], o);
#pragma unroll
            for (int k = 0; k < 3; ++k) t_in[q][k] = o[k] + sj[(size_t)(q * 3 + k) * W];
        }
    }
    const bool last = seg == a.nseg - 1;
    const double2* tabr = a.tab_base + job.tabr_off;
    const size_t ob = (size_t)b * a.dst_bstride + x;
    const int lo = max(n0, P), hi = min(n1, P + H);
    const int need = job.need;
    for (int nb = lo; nb < hi; nb += kIirU) {
      T us[kIirU][4];
#pragma unroll
      for (int u = 0; u < kIirU; ++u)
#pragma unroll
          for (int q = 0; q < 4; ++q)
              if (nb + u < hi && plane_used(need, q)) us[u][q] = sc[q * plane + (size_t)(nb + u) * W];
#pragma unroll
      for (int uu = 0; uu < kIirU; ++uu) {
        const int n = nb + uu;
        if (n >= hi) break;
        const double* g = a.g + 3 * (n1 - 1 - n);
        double sv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (!plane_used(need, q)) { sv[q] = 0.0; continue; }
            const double ul = (double)us[uu][q];
            sv[q] = last ? ul : ul + g[0] * t_in[q][0] + g[1] * t_in[q][1] + g[2] * t_in[q][2];
        }
        const int yo = n - P;
        const double2 cs = tabr[yo];
        for (int o = 0; o < job.nout; ++o) {
            const int pr = job.pair[o];
            const double sa = sv[2 * pr], sb = sv[2 * pr + 1];
            double re = cs.x * sa + cs.y * sb;
            double im = job.sdft ? (cs.x * sb - cs.y * sa) : (cs.y * sa - cs.x * sb);
            if (job.conj[o]) im = -im;
            a.dst_base[job.dst_off[o] + ob + (size_t)yo * W] = mk<T>((T)re, (T)im);
        }
      }
    }
}

}  // namespace

template <typename T> size_t iir_scratch_elems(int H, int W, int P, int njobs, int batch) {
    return (size_t)njobs * batch * 4 * (size_t)(H + 2 * P) * W;
}

size_t iir_state_doubles(int W, int nseg, int njobs, int batch) { return 2 * (size_t)njobs * batch * nseg * 12 * W; }

template <typename T> cudaError_t launch_iir_col(const IirArgs<T>& a, cudaStream_t s) {
    const int SY = 4;  // segments per block (blockDim.y)
    dim3 block(kIirTX, SY);
    dim3 grid((a.W + kIirTX - 1) / kIirTX, (a.nseg + SY - 1) / SY, a.njobs * a.batch);
    iir_fwd<T><<<grid, block, 0, s>>>(a);
    iir_bwd<T><<<grid, block, 0, s>>>(a);
    iir_out<T><<<grid, block, 0, s>>>(a);
    return cudaGetLastError();
}

template size_t iir_scratch_elems<float>(int, int, int, int, int);
template size_t iir_scratch_elems<double>(int, int, int, int, int);
template cudaError_t launch_iir_col<float>(const IirArgs<float>&, cudaStream_t);
template cudaError_t launch_iir_col<double>(const IirArgs<double>&, cudaStream_t);

}  // namespace fgb
