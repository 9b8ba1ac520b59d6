// tiny.cuh — the whole analysis step (enkf.py:167-192) in ONE CTA for desk-scale
// problems (the reference's CPU-runnable config 1 and the lorenz-small preset:
// 40 states, 20 members).  At that size the multi-kernel path is launch- and
// setup-bound (Gram, reduce, levels and anomaly kernels: ~60 us of GPU time
// for ~30 KFLOP); here one launch does, in shared memory:
//   V = (X[idx] - mean)/sqrt(N-1), D = Y - X[idx]      (enkf.py:82-120)
//   Gamma = [V'R^-1 V | V'R^-1 D]                        (level 0, sherman.py:149-154)
//   the N Sherman-Morrison levels on Gamma, den_k and the singular guard of
//   sherman.py:171-174 (the same reduced recursion as ism_levels_kernel)
//   T = I + (A - 1 colmean(A)')/sqrt(N-1), A = V'Z;  X^A = X T
// with the input checks of the Gram pass (index order / range, r > 0, finite
// observed rows and Y).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "enkf_kernels.cuh"

namespace enkf {

constexpr int TINY_THREADS = 256;
constexpr int TINY_MAX_N = 64;
constexpr int64_t TINY_MAX_OBS = 512;
constexpr int64_t TINY_MAX_STATE_ELEMS = 1 << 16;  // n_state * n

__host__ __device__ inline int64_t tiny_smem_doubles(int64_t n_obs, int n) {
  return 2 * n_obs * n /*V, D*/ + 2 * (int64_t)n * n /*Gamma*/ + 4 * (int64_t)n /*pivot row, col*/ +
         n_obs /*1/r*/ + (int64_t)n * n /*T*/ + n /*colmean*/ + (TINY_THREADS / 32) * (int64_t)n /*row bufs*/ + 8;
}
__host__ inline bool tiny_eligible(int64_t n_state, int64_t n_obs, int n) {
  return n >= 2 && n <= TINY_MAX_N && n_obs >= 1 && n_obs <= TINY_MAX_OBS && n_state * n <= TINY_MAX_STATE_ELEMS &&
         tiny_smem_doubles(n_obs, n) * 8 <= 200 * 1024;
}

__global__ void __launch_bounds__(TINY_THREADS, 1)
analysis_tiny_kernel(const double* __restrict__ X, const double* __restrict__ Y, const int64_t* __restrict__ idx,
                     const double* __restrict__ r, double* __restrict__ XA, int64_t n_state, int64_t n_obs, int n,
                     double root, DevStatus* __restrict__ status) {
  extern __shared__ __align__(16) double tsm[];
  const int nobs = (int)n_obs, n2 = 2 * n;
  double* Vs = tsm;                  // [nobs][n]
  double* Ds = Vs + nobs * n;        // [nobs][n]
  double* G = Ds + nobs * n;         // [n][2n]
  double* prow = G + n * n2;         // [2n]  Gamma[k][.] of the current level
  double* pcol = prow + n2;          // [n]   Gamma[.][k]
  double* rinv = pcol + 2 * n;       // [nobs]
  double* Ts = rinv + nobs;          // [n][n]
  double* cm = Ts + n * n;           // [n]
  double* rowb = cm + n;             // [warps][n] one state row per warp (XA may alias X)
  __shared__ int sflags;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = TINY_THREADS / 32;
  if (tid == 0) sflags = 0;
  __syncthreads();
  int flags = 0;
  // ---- V, D rows and the checks (warp per observation row)
  for (int j = warp; j < nobs; j += nwarps) {
    const int64_t src = idx ? idx[j] : j;
    bool ok = true;
    if (idx) {
      if (j > 0 && idx[j - 1] >= src) flags |= FLAG_IDX_ORDER;
      if (src < 0 || src >= n_state) { flags |= FLAG_IDX_RANGE; ok = false; }
    }
    const double rv = r[j];
    if (!isfinite(rv)) flags |= FLAG_NONFINITE;
    else if (!(rv > 0.0)) flags |= FLAG_R_NONPOS;
    double s = 0.0;
    for (int c = lane; c < n; c += 32) s += ok ? X[src * n + c] : 0.0;
    const double mean = warp_sum(s) / (double)n;
    for (int c = lane; c < n; c += 32) {
      const double xv = ok ? X[src * n + c] : 0.0, yv = Y[(int64_t)j * n + c];
      if (!isfinite(xv) || !isfinite(yv)) flags |= FLAG_NONFINITE;
      Vs[j * n + c] = (xv - mean) / root;
      Ds[j * n + c] = yv - xv;
    }
    if (lane == 0) rinv[j] = 1.0 / rv;
  }
  if (flags) atomicOr(&sflags, flags);
  __syncthreads();
  if (sflags) {
    if (tid == 0) atomicOr(&status->flags, sflags);
    return;
  }
  // ---- level-0 Gram [V'R^-1 V | V'R^-1 D]
  for (int e = tid; e < n * n2; e += TINY_THREADS) {
    const int i = e / n2, c = e - i * n2;
    const double* w = c < n ? Vs + c : Ds + (c - n);
    double s = 0.0;
    for (int j = 0; j < nobs; ++j) s = fma(Vs[j * n + i] * rinv[j], w[j * n], s);
    G[e] = s;
  }
  __syncthreads();
  // ---- the N levels: den_k = 1 + Gamma[k][k]; Gamma[i][c] -= Gamma[i][k] Gamma[k][c] / den_k
  //      for the V'V columns c > k and all V'D columns
  for (int k = 0; k < n; ++k) {
    for (int c = tid; c < n2; c += TINY_THREADS) prow[c] = G[k * n2 + c];
    for (int i = tid; i < n; i += TINY_THREADS) pcol[i] = G[i * n2 + k];
    __syncthreads();
    const double dk = 1.0 + prow[k];
    if (fabs(dk) < kSingularTol) {
      if (tid == 0 && !(atomicOr(&status->flags, FLAG_SINGULAR) & FLAG_SINGULAR)) {
        status->level = k + 1;
        status->den = dk;
      }
      return;  // uniform
    }
    const double inv = 1.0 / dk;
    const int ncol = n2 - (k + 1);
    for (int e = tid; e < n * ncol; e += TINY_THREADS) {
      const int i = e / ncol, c = k + 1 + (e - i * ncol);
      G[i * n2 + c] -= pcol[i] * (prow[c] * inv);
    }
    __syncthreads();
  }
  // ---- T = I + (A - 1 colmean(A)') / sqrt(N-1), A = V'D block of Gamma
  for (int c = tid; c < n; c += TINY_THREADS) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += G[i * n2 + n + c];
    cm[c] = s / (double)n;
  }
  __syncthreads();
  for (int e = tid; e < n * n; e += TINY_THREADS) {
    const int i = e / n, c = e - i * n;
    Ts[e] = (i == c ? 1.0 : 0.0) + (G[i * n2 + n + c] - cm[c]) / root;
  }
  __syncthreads();
  // ---- X^A = X T, warp per state row: the row is read into shared memory before any
  //      of it is written, so XA may alias X
  double* rb = rowb + warp * n;
  for (int64_t row = warp; row < n_state; row += nwarps) {
    for (int c = lane; c < n; c += 32) rb[c] = X[row * n + c];
    __syncwarp();
    for (int c = lane; c < n; c += 32) {
      double s = 0.0;
      for (int k2 = 0; k2 < n; ++k2) s = fma(rb[k2], Ts[k2 * n + c], s);
      XA[row * n + c] = s;
    }
    __syncwarp();
  }
}

}  // namespace enkf
