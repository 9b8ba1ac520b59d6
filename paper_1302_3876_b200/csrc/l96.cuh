// l96.cuh — Lorenz-96 ensemble forecast (models/lorenz96.py:31-49).
//
//   dx_i/dt = (x_{i+1} - x_{i-2}) x_{i-1} - x_i + F   (indices cyclic), RK4 step dt.
//
// Every ensemble member (column of the row-major [Ns][N] ensemble) evolves
// independently, so a CTA owns MB whole columns and keeps their rings in
// shared memory for all steps of the window (one launch per forecast, no
// grid-wide synchronisation).  Rings too long for shared memory take the
// per-stage global-memory kernel (4 launches per step).
//
// The arithmetic is the reference's operation by operation, each rounded
// separately (explicit __d*_rn intrinsics, no FMA contraction):
//   k      = (((x[i+1] - x[i-2]) * x[i-1]) - x[i]) + F
//   stage  = x + (0.5 dt) k          (x + dt k3 for the last stage)
//   x_new  = x + (dt / 6) (((k1 + 2 k2) + 2 k3) + k4)
// so the GPU forecast is bit-identical to numpy's.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace enkf {

constexpr int L96_THREADS = 512;
constexpr size_t L96_SMEM_MAX = 200 * 1024;

__device__ __forceinline__ double l96_tendency(double xp1, double xm2, double xm1, double x, double forcing) {
  return __dadd_rn(__dsub_rn(__dmul_rn(__dsub_rn(xp1, xm2), xm1), x), forcing);
}

__device__ __forceinline__ int64_t l96_wrap(int64_t i, int64_t ns) { return i < 0 ? i + ns : (i >= ns ? i - ns : i); }

// Record the first (step, member) whose state became non-finite: the
// reference checks after every step and reports the first bad column
// (lorenz96.py:52-58).  status->bad_index holds ~key maximised, key =
// step << 32 | member, so 0 means "none" with zero-initialised status.
__device__ __forceinline__ void l96_flag_divergence(DevStatus* st, int step, int member) {
  const unsigned long long key = ((unsigned long long)(unsigned)step << 32) | (unsigned)member;
  atomicMax(reinterpret_cast<unsigned long long*>(&st->bad_index), ~key);
  atomicOr(&st->flags, FLAG_DIVERGED);
}

// Shared-memory path: CTA = MB members; 4 rings of Ns x MB doubles
// (x, two stage buffers, accumulator), member-interleaved ([i][m]).
__global__ void __launch_bounds__(L96_THREADS)
l96_rk4_smem_kernel(const double* __restrict__ X, double* __restrict__ Xout, int64_t ns, int n, int mb_max,
                    double half_dt, double dt, double dt6, double forcing, int nsteps, DevStatus* st) {
  extern __shared__ double l96sm[];
  const int j0 = blockIdx.x * mb_max;
  const int mb = min(mb_max, n - j0);
  const int64_t len = ns * mb;
  double* x = l96sm;
  double* sa = x + len;
  double* sb = sa + len;
  double* acc = sb + len;
  for (int64_t e = threadIdx.x; e < len; e += blockDim.x) {
    const int64_t i = e / mb;
    const int m = (int)(e - i * mb);
    x[e] = X[i * n + j0 + m];
  }
  __syncthreads();
  for (int step = 0; step < nsteps; ++step) {
    // stage s reads `src` (x, sa, sb, sa) and writes the next stage input to `dst`
    const double* src = x;
    double* dst = sa;
#pragma unroll 1
    for (int s = 0; s < 4; ++s) {
      for (int64_t e = threadIdx.x; e < len; e += blockDim.x) {
        const int64_t i = e / mb;
        const int m = (int)(e - i * mb);
        const double k = l96_tendency(src[l96_wrap(i + 1, ns) * mb + m], src[l96_wrap(i - 2, ns) * mb + m],
                                      src[l96_wrap(i - 1, ns) * mb + m], src[e], forcing);
        if (s == 0) {
          acc[e] = k;
          dst[e] = __dadd_rn(x[e], __dmul_rn(half_dt, k));
        } else if (s == 1 || s == 2) {
          acc[e] = __dadd_rn(acc[e], __dmul_rn(2.0, k));
          dst[e] = __dadd_rn(x[e], __dmul_rn(s == 1 ? half_dt : dt, k));
        } else {
          acc[e] = __dadd_rn(acc[e], k);
        }
      }
      __syncthreads();
      src = dst;
      dst = (dst == sa) ? sb : sa;
    }
    bool bad = false;
    int bad_m = 0x7fffffff;
    for (int64_t e = threadIdx.x; e < len; e += blockDim.x) {
      const double v = __dadd_rn(x[e], __dmul_rn(dt6, acc[e]));
      x[e] = v;
      if (!isfinite(v)) {
        bad = true;
        bad_m = min(bad_m, j0 + (int)(e % mb));
      }
    }
    if (bad) l96_flag_divergence(st, step, bad_m);
    __syncthreads();
  }
  for (int64_t e = threadIdx.x; e < len; e += blockDim.x) {
    const int64_t i = e / mb;
    const int m = (int)(e - i * mb);
    Xout[i * n + j0 + m] = x[e];
  }
}

// Register path (rings of at most L96R_THREADS * PT points per CTA): as the
// shared-memory path, but a thread owns PT fixed points of the member-interleaved
// ring ([i][m]: the neighbours of element e are e + mb, e - mb, e - 2 mb, cyclic, so
// no index division) and keeps their x, accumulator and current stage value in
// registers; shared memory holds only what neighbours read (x and two stage rings).
// Stage 3 writes no ring, so the step's final update follows it without a barrier:
// 4 barriers per RK4 step.  Same operations in the same order: bit-identical.
constexpr int L96R_THREADS = 1024;
template <int PT>
__global__ void __launch_bounds__(L96R_THREADS)
l96_rk4_reg_kernel(const double* __restrict__ X, double* __restrict__ Xout, int ns, int n, int mb_max,
                   double half_dt, double dt, double dt6, double forcing, int nsteps, DevStatus* st) {
  extern __shared__ double l96sm[];
  const int j0 = blockIdx.x * mb_max;
  const int mb = min(mb_max, n - j0);
  const int len = ns * mb;
  double* xs = l96sm;       // x ring (stage 0 reads neighbours here)
  double* sa = xs + len;
  double* sb = sa + len;
  double xr[PT], ar[PT], cur[PT];
  int gidx[PT];  // element e = (i, m) -> global offset i n + j0 + m
#pragma unroll
  for (int t = 0; t < PT; ++t) {
    const int e = threadIdx.x + t * L96R_THREADS;
    xr[t] = 0.0;
    ar[t] = 0.0;
    gidx[t] = -1;
    if (e < len) {
      const int i = e / mb, m = e - i * mb;
      gidx[t] = i * n + j0 + m;
      xr[t] = X[(int64_t)gidx[t]];
      xs[e] = xr[t];
    }
    cur[t] = xr[t];
  }
  __syncthreads();
  const int o1 = mb, o2 = 2 * mb;
  for (int step = 0; step < nsteps; ++step) {
    const double* src = xs;
    double* dst = sa;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
#pragma unroll
      for (int t = 0; t < PT; ++t) {
        const int e = threadIdx.x + t * L96R_THREADS;
        if (e < len) {
          const int ep1 = e + o1 >= len ? e + o1 - len : e + o1;
          const int em1 = e - o1 < 0 ? e - o1 + len : e - o1;
          const int em2 = e - o2 < 0 ? e - o2 + len : e - o2;
          const double k = l96_tendency(src[ep1], src[em2], src[em1], cur[t], forcing);
          if (s == 0) {
            ar[t] = k;
            cur[t] = __dadd_rn(xr[t], __dmul_rn(half_dt, k));
            dst[e] = cur[t];
          } else if (s == 1 || s == 2) {
            ar[t] = __dadd_rn(ar[t], __dmul_rn(2.0, k));
            cur[t] = __dadd_rn(xr[t], __dmul_rn(s == 1 ? half_dt : dt, k));
            dst[e] = cur[t];
          } else {
            ar[t] = __dadd_rn(ar[t], k);
          }
        }
      }
      if (s < 3) __syncthreads();
      src = dst;
      dst = (dst == sa) ? sb : sa;
    }
    bool bad = false;
    int bad_m = 0x7fffffff;
#pragma unroll
    for (int t = 0; t < PT; ++t) {
      const int e = threadIdx.x + t * L96R_THREADS;
      if (e < len) {
        const double v = __dadd_rn(xr[t], __dmul_rn(dt6, ar[t]));
        xr[t] = v;
        cur[t] = v;
        xs[e] = v;
        if (!isfinite(v)) {
          bad = true;
          bad_m = min(bad_m, j0 + e % mb);
        }
      }
    }
    if (bad) l96_flag_divergence(st, step, bad_m);
    __syncthreads();  // x ring complete; every thread is past stage 3's reads of sa
  }
#pragma unroll
  for (int t = 0; t < PT; ++t)
    if (gidx[t] >= 0) Xout[(int64_t)gidx[t]] = xr[t];
}

// Global-memory path, one RK4 stage per launch over all (i, j).
//   s = 0: k1 from x;   acc = k1;          out = x + (dt/2) k1
//   s = 1: k2 from in;  acc += 2 k2;       out = x + (dt/2) k2
//   s = 2: k3 from in;  acc += 2 k3;       out = x + dt k3
//   s = 3: k4 from in;  acc += k4;         xnew = x + (dt/6) acc (written to `out`)
__global__ void l96_stage_kernel(const double* __restrict__ x, const double* __restrict__ in,
                                 double* __restrict__ acc, double* __restrict__ out, int64_t ns, int n, int s,
                                 double half_dt, double dt, double dt6, double forcing, int step, DevStatus* st) {
  const int64_t total = ns * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / n;
    const int j = (int)(e - i * n);
    const double k = l96_tendency(in[l96_wrap(i + 1, ns) * n + j], in[l96_wrap(i - 2, ns) * n + j],
                                  in[l96_wrap(i - 1, ns) * n + j], in[e], forcing);
    if (s == 0) {
      acc[e] = k;
      out[e] = __dadd_rn(x[e], __dmul_rn(half_dt, k));
    } else if (s < 3) {
      acc[e] = __dadd_rn(acc[e], __dmul_rn(2.0, k));
      out[e] = __dadd_rn(x[e], __dmul_rn(s == 1 ? half_dt : dt, k));
    } else {
      const double v = __dadd_rn(x[e], __dmul_rn(dt6, __dadd_rn(acc[e], k)));
      out[e] = v;
      if (!isfinite(v)) l96_flag_divergence(st, step, j);
    }
  }
}

// Covariance inflation (enkf.py:123-135): mean + alpha (x - mean) per row, the
// reference's operation order (no FMA contraction).  Warp per row; X may alias Xout.
__global__ void inflate_kernel(const double* __restrict__ X, double* __restrict__ Xout, int64_t ns, int n,
                               double alpha) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= ns) return;
  double s = 0.0;
  for (int c = lane; c < n; c += 32) s += X[row * n + c];
  const double mean = __ddiv_rn(warp_sum(s), (double)n);
  for (int c = lane; c < n; c += 32)
    Xout[row * n + c] = __dadd_rn(mean, __dmul_rn(alpha, __dsub_rn(X[row * n + c], mean)));
}

// Row means of the ensemble (diagnostics of the cycled driver: the forecast
// and analysis ensemble means the reference's cycle_error uses).  Warp per row.
__global__ void row_mean_kernel(const double* __restrict__ X, double* __restrict__ out, int64_t ns, int n) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= ns) return;
  double s = 0.0;
  for (int c = lane; c < n; c += 32) s += X[row * n + c];
  s = warp_sum(s);
  if (lane == 0) out[row] = s / (double)n;
}

}  // namespace enkf
