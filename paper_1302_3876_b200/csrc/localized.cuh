// localized.cuh — localized analysis (enkf.py:193-199):
//
//   X^A = X + (Delta o (S V')) Z,   S = member_deviations(X), V = H S,
//   Z = W^-1 (Y - H X) from the ISM solve (the same Gram -> levels -> Z pass
//   as enkf_ism_solve_f64).
//
// The Ns x Nobs matrix S V' is never formed in HBM: one CTA owns TI state rows,
// keeps their deviations in shared memory and streams the observation rows in
// chunks of TJ: P = S_blk V_chunk' (TI x TJ, K = N), Q = Delta o P, then
// acc += Q Z_chunk (TI x N) in registers.  Delta is either read from memory
// (the reference's dense `localization` argument) or evaluated on the fly as
// the cyclic taper of influence_matrix_cyclic (enkf.py:138-164), which makes
// the localized step matrix-free.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace enkf {

constexpr int LOC_TI = 32;       // state rows per CTA
constexpr int LOC_TJ = 32;       // observation rows per chunk
constexpr int LOC_THREADS = 256;

__host__ __device__ inline size_t localized_smem_bytes(int n) {
  const size_t ld = (size_t)n + 1;
  return sizeof(double) * ((LOC_TI + 2 * LOC_TJ) * ld + (size_t)LOC_TI * (LOC_TJ + 1));
}

// V_k = (X[idx_k] - mean) / sqrt(N-1) (enkf.py:82-92 then :59), D_k = Y_k - X[idx_k]
// (enkf.py:114-120), with the SelectionOperator checks (enkf.py:36-58).  Warp per row.
__global__ void obs_rows_kernel(const double* __restrict__ X, const double* __restrict__ Y,
                                const int64_t* __restrict__ idx, double* __restrict__ V,
                                double* __restrict__ D, int64_t n_obs, int64_t n_state, int n,
                                double root, DevStatus* status) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n_obs) return;
  const int64_t src = idx ? idx[row] : row;
  int flags = 0;
  if (src < 0 || src >= n_state) flags |= FLAG_IDX_RANGE;
  if (idx && row > 0 && idx[row - 1] >= src) flags |= FLAG_IDX_ORDER;
  if (flags) {
    if (lane == 0) atomicOr(&status->flags, flags);
    for (int c = lane; c < n; c += 32) V[row * n + c] = D[row * n + c] = 0.0;
    return;
  }
  const double* x = X + src * n;
  double s = 0.0;
  for (int c = lane; c < n; c += 32) s += x[c];
  const double mean = warp_sum(s) / (double)n;
  for (int c = lane; c < n; c += 32) {
    V[row * n + c] = (x[c] - mean) / root;
    D[row * n + c] = Y[row * n + c] - x[c];
  }
}

// MODE 0: Delta dense [n_state][n_obs] in memory.  MODE 1: Delta_ij =
// exp(-d(i, p_j) / scale), d the cyclic distance min(|i-p|, Ns-|i-p|) and p_j
// the state index of observation j (idx, or j for the identity operator).
template <int MODE>
__global__ void __launch_bounds__(LOC_THREADS)
localized_update_kernel(const double* __restrict__ X, const double* __restrict__ V,
                        const double* __restrict__ Z, const double* __restrict__ delta,
                        const int64_t* __restrict__ idx, double scale, double* __restrict__ XA,
                        int64_t n_state, int64_t n_obs, int n, double root) {
  extern __shared__ double lsm[];
  const int ld = n + 1;
  double* Ss = lsm;                     // [TI][ld] deviations of this CTA's state rows
  double* Vs = Ss + LOC_TI * ld;        // [TJ][ld]
  double* Zs = Vs + LOC_TJ * ld;        // [TJ][ld]
  double* Qs = Zs + LOC_TJ * ld;        // [TI][TJ+1]  Delta o (S V')
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t i0 = (int64_t)blockIdx.x * LOC_TI;

  // S rows (4 per warp)
  for (int a = 0; a < LOC_TI / 8; ++a) {
    const int i = warp * (LOC_TI / 8) + a;
    const int64_t gi = i0 + i;
    if (gi < n_state) {
      const double* x = X + gi * n;
      double s = 0.0;
      for (int c = lane; c < n; c += 32) s += x[c];
      const double mean = warp_sum(s) / (double)n;
      for (int c = lane; c < n; c += 32) Ss[i * ld + c] = (x[c] - mean) / root;
    } else {
      for (int c = lane; c < n; c += 32) Ss[i * ld + c] = 0.0;
    }
  }

  const int pi = (tid >> 4) * 2, pj = (tid & 15) * 2;  // this thread's 2x2 block of P
  const int rg = warp * 4;                             // this thread's 4 output rows
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[a][q] = 0.0;

  for (int64_t j0 = 0; j0 < n_obs; j0 += LOC_TJ) {
    __syncthreads();  // previous chunk's Vs/Zs/Qs are consumed (and Ss is written)
    for (int e = tid; e < LOC_TJ * n; e += LOC_THREADS) {
      const int j = e / n, c = e - j * n;
      const bool ok = j0 + j < n_obs;
      Vs[j * ld + c] = ok ? V[(j0 + j) * n + c] : 0.0;
      Zs[j * ld + c] = ok ? Z[(j0 + j) * n + c] : 0.0;
    }
    __syncthreads();
    double p00 = 0.0, p01 = 0.0, p10 = 0.0, p11 = 0.0;
    for (int m = 0; m < n; ++m) {
      const double s0 = Ss[pi * ld + m], s1 = Ss[(pi + 1) * ld + m];
      const double v0 = Vs[pj * ld + m], v1 = Vs[(pj + 1) * ld + m];
      p00 = fma(s0, v0, p00);
      p01 = fma(s0, v1, p01);
      p10 = fma(s1, v0, p10);
      p11 = fma(s1, v1, p11);
    }
    const double pv[2][2] = {{p00, p01}, {p10, p11}};
#pragma unroll
    for (int a = 0; a < 2; ++a) {
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int64_t gi = i0 + pi + a, gj = j0 + pj + b;
        double dl = 0.0;
        if (gi < n_state && gj < n_obs) {
          if (MODE == 0) {
            dl = delta[gi * n_obs + gj];
          } else {
            const int64_t p = idx ? idx[gj] : gj;
            int64_t dist = gi > p ? gi - p : p - gi;
            if (n_state - dist < dist) dist = n_state - dist;
            dl = exp(-(double)dist / scale);
          }
        }
        Qs[(pi + a) * (LOC_TJ + 1) + pj + b] = dl * pv[a][b];
      }
    }
    __syncthreads();
#pragma unroll 4
    for (int j = 0; j < LOC_TJ; ++j) {
      double z[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = lane + 32 * q;
        z[q] = c < n ? Zs[j * ld + c] : 0.0;
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const double qv = Qs[(rg + a) * (LOC_TJ + 1) + j];
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[a][q] = fma(qv, z[q], acc[a][q]);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int64_t gi = i0 + rg + a;
    if (gi >= n_state) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = lane + 32 * q;
      if (c < n) XA[gi * n + c] = X[gi * n + c] + acc[a][q];
    }
  }
}

}  // namespace enkf
