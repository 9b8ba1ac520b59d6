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

// ---------------------------------------------------------------------------
// FP64 tensor-core (DMMA m8n8k4) form of the localized update, NP = N rounded up
// to 8.  CTA = 64 state rows, 8 warps; observation chunks of 32 rows are
// double-buffered with cp.async.  Per chunk, warp w owns state rows 8w..8w+7:
//   P = S_blk V_chunk'  (its 8 x 32 slab, K = NP: 4 DMMA tiles per k-step)
//   Q = Delta o P       (-> shared memory)
//   acc += Q Z_chunk    (its 8 x NP slab, K = 32: NP/8 DMMA tiles per k-step)
// The shared-memory row stride padded_ld (== 4 mod 16 doubles) keeps every
// fragment load conflict-free.
constexpr int LD_TI = 64;
constexpr int LD_TJ = 32;
constexpr int LD_THREADS = 256;

__host__ __device__ inline size_t localized_dmma_smem_bytes(int np) {
  const size_t ld = (size_t)padded_ld(np), ldq = (size_t)padded_ld(LD_TJ);
  return sizeof(double) * (LD_TI * ld + 2 * 2 * LD_TJ * ld + LD_TI * ldq);
}

template <int NP, int MODE>
__global__ void __launch_bounds__(LD_THREADS)
localized_update_dmma_kernel(const double* __restrict__ X, const double* __restrict__ V,
                             const double* __restrict__ Z, const double* __restrict__ delta,
                             const int64_t* __restrict__ idx, double scale, double* __restrict__ XA,
                             int64_t n_state, int64_t n_obs, int n, double root) {
  extern __shared__ __align__(16) double dsm[];
  const int ld = padded_ld(NP), ldq = padded_ld(LD_TJ);
  double* Ss = dsm;                          // [64][ld]
  double* Vb = Ss + LD_TI * ld;              // [2][32][ld]
  double* Zb = Vb + 2 * LD_TJ * ld;          // [2][32][ld]
  double* Qs = Zb + 2 * LD_TJ * ld;          // [64][ldq]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t i0 = (int64_t)blockIdx.x * LD_TI;
  const int64_t nchunks = (n_obs + LD_TJ - 1) / LD_TJ;

  // zero the padding columns n..NP-1 of every V/Z buffer (loads never write them)
  for (int e = tid; e < 2 * 2 * LD_TJ * (NP - n); e += LD_THREADS) {
    const int row = e / (NP - n), c = n + e % (NP - n);
    Vb[row * ld + c] = 0.0;  // Vb and Zb are contiguous: rows 0..127 cover both
  }
  auto issue = [&](int64_t ch) {
    const int b = (int)(ch & 1);
    double* vs = Vb + b * LD_TJ * ld;
    double* zs = Zb + b * LD_TJ * ld;
    for (int e = tid; e < LD_TJ * n; e += LD_THREADS) {
      const int j = e / n, c = e - j * n;
      const int64_t gj = ch * LD_TJ + j;
      const bool ok = gj < n_obs;
      cp_async8(vs + j * ld + c, V + (ok ? gj : 0) * n + c, ok);
      cp_async8(zs + j * ld + c, Z + (ok ? gj : 0) * n + c, ok);
    }
  };
  if (nchunks > 0) issue(0);
  cp_async_commit();

  // S rows of this CTA (8 per warp), zero outside the state and in the padding
  for (int a = 0; a < LD_TI / 8; ++a) {
    const int i = warp * (LD_TI / 8) + a;
    const int64_t gi = i0 + i;
    double s = 0.0;
    if (gi < n_state)
      for (int c = lane; c < n; c += 32) s += X[gi * n + c];
    const double mean = warp_sum(s) / (double)n;
    for (int c = lane; c < NP; c += 32)
      Ss[i * ld + c] = (gi < n_state && c < n) ? (X[gi * n + c] - mean) / root : 0.0;
  }

  constexpr int NT = NP / 8;
  double acc[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
  const int fr = lane >> 2, fk = lane & 3;  // fragment row (m or n) and k of this lane
  const int mrow = 8 * warp + fr;           // this lane's A-fragment state row

  for (int64_t ch = 0; ch < nchunks; ++ch) {
    if (ch + 1 < nchunks) issue(ch + 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();  // chunk ch (and, at ch == 0, S and the padding) visible
    const int b = (int)(ch & 1);
    const double* vs = Vb + b * LD_TJ * ld;
    const double* zs = Zb + b * LD_TJ * ld;
    // P = S V' for rows 8w..8w+7, obs 0..31
    double p[4][2];
#pragma unroll
    for (int t = 0; t < 4; ++t) p[t][0] = p[t][1] = 0.0;
#pragma unroll 4
    for (int k0 = 0; k0 < NP; k0 += 4) {
      const double a = Ss[mrow * ld + k0 + fk];
#pragma unroll
      for (int t = 0; t < 4; ++t) dmma884(p[t][0], p[t][1], a, vs[(8 * t + fr) * ld + k0 + fk]);
    }
    // Q = Delta o P -> Qs (element (8w + fr, 8t + 2fk + e))
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int jj = 8 * t + 2 * fk + e;
        const int64_t gi = i0 + mrow, gj = ch * LD_TJ + jj;
        double dl = 0.0;
        if (gi < n_state && gj < n_obs) {
          if (MODE == 0) {
            dl = delta[gi * n_obs + gj];
          } else {
            const int64_t pj = idx ? idx[gj] : gj;
            int64_t dist = gi > pj ? gi - pj : pj - gi;
            if (n_state - dist < dist) dist = n_state - dist;
            dl = exp(-(double)dist / scale);
          }
        }
        Qs[mrow * ldq + jj] = dl * p[t][e];
      }
    __syncwarp();  // a warp reads back only its own 8 rows of Q
    // acc += Q Z for rows 8w..8w+7, members 0..NP-1
#pragma unroll
    for (int k0 = 0; k0 < LD_TJ; k0 += 4) {
      const double a = Qs[mrow * ldq + k0 + fk];
#pragma unroll
      for (int t = 0; t < NT; ++t) dmma884(acc[t][0], acc[t][1], a, zs[(k0 + fk) * ld + 8 * t + fr]);
    }
    __syncthreads();  // buffer b is refilled by the load issued in the next iteration
  }
  cp_async_wait<0>();
  // X^A = X + acc (element (8w + fr, 8t + 2fk + e))
  const int64_t gi = i0 + mrow;
  if (gi < n_state) {
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * t + 2 * fk + e;
        if (c < n) XA[gi * n + c] = X[gi * n + c] + acc[t][e];
      }
  }
}

}  // namespace enkf
