// enkf_kernels.cuh — sm_100a kernels of the EnKF analysis step
// (iterative Sherman-Morrison, arXiv 1302.3876).
//
// The reference path (enkf.py:167-192 -> sherman.py:157-214) is re-organised
// for B200 as three kernels over HBM plus one on-chip kernel:
//
//   gram_kernel      one streaming pass over the observed rows: gathers X[idx]
//                    rows (K2), removes the row mean and scales (K1), forms
//                    D = Y - HX (K3) and level 0 R^-1 (K4) on the fly in
//                    registers, and accumulates the level-0 Gram
//                    [V'R^-1 V | V'R^-1 D] with FP64 DMMA (mma.sync m8n8k4).
//                    These are exactly the dot products v_k'u / v_k'col of every
//                    Sherman-Morrison level (K5/K8), taken before any update.
//   gram_reduce      fixed-order sum of the per-CTA partials (deterministic).
//   ism_levels       the N Sherman-Morrison levels (sherman.py:164-187: den_k,
//                    singular guard, rank-one composition) applied to the
//                    N x 2N Gram in shared memory: reduced coordinates, the
//                    same rank-one sequence on v_i'W_k^-1 x instead of on the
//                    Nobs x 2N panel.  Ends with A = V'Z (enkf.py:192, K10).
//   rowgemm          the anomaly update X^A = X T, T = I + (I - 11'/N) A/sqrt(N-1)
//                    (enkf.py:192, K11), and Z = (D - V A) R^-1 for solve_sherman;
//                    T / A stationary in registers, rows streamed through a
//                    4-stage cp.async ring, FP64 DMMA.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace enkf {

struct DevStatus {
  int flags;        // ENKF_FLAG_* bits
  int level;        // first singular level (1-based)
  double den;       // its denominator
  long long bad_index;  // first offending obs row for index errors (or -1)
};

enum : int {
  FLAG_NONFINITE = 1,
  FLAG_R_NONPOS = 2,
  FLAG_IDX_ORDER = 4,
  FLAG_IDX_RANGE = 8,
  FLAG_SINGULAR = 16,
};

constexpr double kSingularTol = 1e-14;  // sherman.py:51

// ---------------------------------------------------------------------------
// PTX helpers
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Shared-memory row stride (in doubles) for a row of `n` values: >= n, even,
// and == 4 (mod 16) so the DMMA fragment pattern (row = lane&3 or lane>>2,
// col = the other) hits 16 distinct 8-byte banks per half-warp.
__host__ __device__ inline int padded_ld(int n) {
  int ld = (n + 15) / 16 * 16 + 4;
  return ld;
}

// ---------------------------------------------------------------------------
// Gram pass.
//   ANALYSIS: rows x = X[idx[i]] (or X[i]), y = Y[i]; v = x - mean(x),
//             Gram_raw = sum_i (v_i / r_i) [v_i | y_i - x_i]'
//             (the 1/sqrt(N-1) scalings are applied in gram_reduce).
//   SOLVE:    rows v = V[i], d = D[i]; Gram = sum_i (v_i / r_i) [v_i | d_i]'.
// Grid: x = column block of the 2N Gram columns (64 each), y = row block of
// the N Gram rows (128 each), z = split of the observation rows.
constexpr int G_BM = 128;
constexpr int G_BN = 64;
constexpr int G_RT = 16;
constexpr int G_STAGES = 3;
constexpr int G_THREADS = 256;

template <bool ANALYSIS, bool VEC16>
__global__ void __launch_bounds__(G_THREADS, 2)
gram_kernel(const double* __restrict__ X, const double* __restrict__ Y,
            const int64_t* __restrict__ idx, const double* __restrict__ r,
            int64_t n_state, int64_t n_obs, int n, int ld, int64_t rows_per_split,
            double* __restrict__ partial, DevStatus* __restrict__ status) {
  extern __shared__ __align__(16) double gsm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n0 = blockIdx.x * G_BN;   // first Gram column of this CTA (over 2n)
  const int m0 = blockIdx.y * G_BM;   // first Gram row (over n)
  const int split = blockIdx.z;
  const bool needY = (n0 + G_BN > n);
  const bool checker = (blockIdx.x == gridDim.x - 1) && (blockIdx.y == 0);
  const int64_t row_begin = (int64_t)split * rows_per_split;
  int64_t row_end = row_begin + rows_per_split;
  if (row_end > n_obs) row_end = n_obs;

  const int stage_elems = G_RT * ld;
  double* xs = gsm;                                   // [S][RT][ld]
  double* ys = xs + G_STAGES * stage_elems;           // [S][RT][ld] (if needY)
  double* meanv = ys + (needY ? G_STAGES * stage_elems : 0);  // [S][RT]
  double* rinvv = meanv + G_STAGES * G_RT;                     // [S][RT]

  const int64_t nrows = row_end > row_begin ? row_end - row_begin : 0;
  const int nstages = (int)((nrows + G_RT - 1) / G_RT);

  auto load_stage = [&](int t) {
    if (t >= nstages) return;
    const int buf = t % G_STAGES;
    double* xb = xs + buf * stage_elems;
    double* yb = ys + buf * stage_elems;
    for (int rr = warp; rr < G_RT; rr += G_THREADS / 32) {
      const int64_t g = row_begin + (int64_t)t * G_RT + rr;
      bool valid = g < row_end;
      int64_t src = g;
      if (ANALYSIS && valid && idx != nullptr) {
        src = idx[g];
        if (src < 0 || src >= n_state) valid = false;  // flagged by the checker
      }
      const double* xrow = X + (valid ? src : 0) * (int64_t)n;
      const double* yrow = Y + (valid ? g : 0) * (int64_t)n;
      if (VEC16) {
        for (int c = 2 * lane; c < n; c += 64) {
          cp_async16(xb + rr * ld + c, xrow + c, valid);
          if (needY) cp_async16(yb + rr * ld + c, yrow + c, valid);
        }
      } else {
        for (int c = lane; c < n; c += 32) {
          cp_async8(xb + rr * ld + c, xrow + c, valid);
          if (needY) cp_async8(yb + rr * ld + c, yrow + c, valid);
        }
      }
    }
  };

  // Per-lane column roles (constant over the whole pass).
  const int wm = warp & 3, wn = warp >> 2;
  int acol[4];
  bool aval[4];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    acol[mt] = m0 + wm * 32 + mt * 8 + (lane >> 2);
    aval[mt] = acol[mt] < n;
  }
  int bcol[4], bkind[4];  // kind 0: v column, 1: d column, 2: zero
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) {
    int c = n0 + wn * 32 + nt * 8 + (lane >> 2);
    if (c < n) { bkind[nt] = 0; bcol[nt] = c; }
    else if (c < 2 * n) { bkind[nt] = 1; bcol[nt] = c - n; }
    else { bkind[nt] = 2; bcol[nt] = 0; }
  }

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < G_STAGES - 1; ++s) { load_stage(s); cp_async_commit(); }

  int local_flags = 0;
  for (int t = 0; t < nstages; ++t) {
    cp_async_wait<G_STAGES - 2>();
    __syncthreads();
    load_stage(t + G_STAGES - 1);
    cp_async_commit();

    const int buf = t % G_STAGES;
    const double* xb = xs + buf * stage_elems;
    const double* yb = ys + buf * stage_elems;
    // Row statistics (and input checks on the checker CTA).
    for (int rr = warp; rr < G_RT; rr += G_THREADS / 32) {
      const int64_t g = row_begin + (int64_t)t * G_RT + rr;
      const bool valid = g < row_end;
      double s = 0.0;
      if (ANALYSIS) {
        for (int c = lane; c < n; c += 32) s += xb[rr * ld + c];
        s = warp_sum(s);
      }
      if (checker && valid) {
        bool bad = false;
        for (int c = lane; c < n; c += 32) {
          bad |= !isfinite(xb[rr * ld + c]);
          if (needY) bad |= !isfinite(yb[rr * ld + c]);
        }
        if (__any_sync(0xffffffffu, bad)) local_flags |= FLAG_NONFINITE;
        if (lane == 0) {
          const double rv = r[g];
          if (!isfinite(rv)) local_flags |= FLAG_NONFINITE;
          else if (!(rv > 0.0)) local_flags |= FLAG_R_NONPOS;
          if (ANALYSIS && idx != nullptr) {
            const int64_t iv = idx[g];
            if (iv < 0 || iv >= n_state) local_flags |= FLAG_IDX_RANGE;
            if (g > 0 && idx[g - 1] >= iv) local_flags |= FLAG_IDX_ORDER;
          }
        }
      }
      if (lane == 0) {
        meanv[buf * G_RT + rr] = ANALYSIS ? s / (double)n : 0.0;
        rinvv[buf * G_RT + rr] = valid ? 1.0 / r[g] : 0.0;
      }
    }
    __syncthreads();

    // DMMA over the stage: k = observation row.
#pragma unroll
    for (int ks = 0; ks < G_RT / 4; ++ks) {
      const int row = ks * 4 + (lane & 3);
      const double mu = meanv[buf * G_RT + row];
      const double ri = rinvv[buf * G_RT + row];
      const double* xr = xb + row * ld;
      const double* yr = yb + row * ld;
      double a[4], b[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        double v = aval[mt] ? xr[acol[mt]] : 0.0;
        if (ANALYSIS) v -= mu;
        a[mt] = aval[mt] ? v * ri : 0.0;
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        double v;
        if (bkind[nt] == 0) {
          v = xr[bcol[nt]];
          if (ANALYSIS) v -= mu;
        } else if (bkind[nt] == 1) {
          v = yr[bcol[nt]];
          if (ANALYSIS) v -= xr[bcol[nt]];
        } else {
          v = 0.0;
        }
        b[nt] = v;
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma884(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
    }
  }
  cp_async_wait<0>();

  if (checker) {
    if (local_flags) atomicOr(&status->flags, local_flags);
  }

  // Epilogue: this CTA's (128 x 64) block of the split's partial Gram.
  double* out = partial + (int64_t)split * n * (2 * n);
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int gi = m0 + wm * 32 + mt * 8 + (lane >> 2);
    if (gi >= n) continue;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int gc = n0 + wn * 32 + nt * 8 + 2 * (lane & 3);
      if (gc + 1 < 2 * n) {
        *reinterpret_cast<double2*>(out + (int64_t)gi * 2 * n + gc) =
            make_double2(acc[mt][nt][0], acc[mt][nt][1]);
      } else if (gc < 2 * n) {
        out[(int64_t)gi * 2 * n + gc] = acc[mt][nt][0];
      }
    }
  }
}

// Fixed-order reduction of the split partials; scale V'R^-1V by s_vv and
// V'R^-1D by s_vd (1/(N-1) and 1/sqrt(N-1) in analysis mode).
__global__ void gram_reduce(const double* __restrict__ partial, int splits, int n,
                            double s_vv, double s_vd, double* __restrict__ gram) {
  const int64_t count = (int64_t)n * 2 * n;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= count) return;
  double s = 0.0;
  for (int k = 0; k < splits; ++k) s += partial[(int64_t)k * count + e];
  const int col = (int)(e % (2 * n));
  gram[e] = s * (col < n ? s_vv : s_vd);
}

// ---------------------------------------------------------------------------
// The N Sherman-Morrison levels on the Gram (one CTA, shared memory).
// Gamma_k[i][c] = v_i' W_k^-1 g_c with W_k = R + sum_{j<=k} v_j v_j':
//   den_k = 1 + Gamma_{k-1}[k][k]                       (sherman.py:172)
//   |den_k| < 1e-14  ->  SingularUpdateError(k+1, den_k) (sherman.py:173-174)
//   Gamma_k[i][c] = Gamma_{k-1}[i][c] - Gamma_{k-1}[i][k] Gamma_{k-1}[k][c] / den_k
// for every later column c (the rank-one update col -= h_k (v_k'col) of
// sherman.py:182-187/208-214 seen through v_i').  The V'V block is symmetric at
// every level and is kept packed (upper triangle); after N levels the V'D block
// is A = V'Z.
__host__ __device__ inline int64_t levels_smem_doubles(int n) {
  return (int64_t)n * (n + 1) / 2 + (int64_t)n * n + 3 * (int64_t)n + 8;
}

__global__ void __launch_bounds__(1024, 1)
ism_levels_kernel(const double* __restrict__ gram, int n, double cscale,
                  double* __restrict__ A, double* __restrict__ T,
                  double* __restrict__ den_out, DevStatus* __restrict__ status) {
  extern __shared__ __align__(16) double lsm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  double* vv = lsm;                               // packed: p(i,c) = c(c+1)/2 + i, i <= c
  double* vd = vv + (int64_t)n * (n + 1) / 2;     // [n][n]
  double* pc = vd + (int64_t)n * n;               // pivot column Gamma[.][k]
  double* q = pc + n;                             // scaled pivot row: [0,n) V part, [n,2n) D part
  auto P = [](int i, int c) { return c * (c + 1) / 2 + i; };

  const int n2 = 2 * n;
  for (int e = tid; e < n * n2; e += blockDim.x) {
    const int i = e / n2, c = e - i * n2;
    const double g = gram[e];
    if (c < n) {
      if (i <= c) vv[P(i, c)] = g;
    } else {
      vd[i * n + (c - n)] = g;
    }
  }
  __syncthreads();

  for (int k = 0; k < n; ++k) {
    const double dk = 1.0 + vv[P(k, k)];
    if (fabs(dk) < kSingularTol) {
      if (tid == 0) {
        if (!(atomicOr(&status->flags, FLAG_SINGULAR) & FLAG_SINGULAR)) {
          status->level = k + 1;
          status->den = dk;
        }
      }
      return;
    }
    if (tid == 0 && den_out) den_out[k] = dk;
    const double inv = 1.0 / dk;
    for (int i = tid; i < n; i += blockDim.x) pc[i] = (i <= k) ? vv[P(i, k)] : vv[P(k, i)];
    for (int c = tid; c < n2; c += blockDim.x) {
      if (c < n) q[c] = (c > k) ? vv[P(k, c)] * inv : 0.0;
      else q[c] = vd[k * n + (c - n)] * inv;
    }
    __syncthreads();
    for (int c = k + 1 + warp; c < n; c += nwarps) {
      const double qc = q[c];
      double* col = vv + P(0, c);
      for (int i = lane; i <= c; i += 32) col[i] -= pc[i] * qc;
    }
    for (int i = warp; i < n; i += nwarps) {
      const double pi = pc[i];
      double* row = vd + i * n;
      for (int c = lane; c < n; c += 32) row[c] -= pi * q[n + c];
    }
    __syncthreads();
  }

  // A = V'Z; T = I + cscale (A - 1 colmean(A)').
  for (int e = tid; e < n * n; e += blockDim.x) A[e] = vd[e];
  if (T != nullptr) {
    for (int c = tid; c < n; c += blockDim.x) {
      double s = 0.0;
      for (int i = 0; i < n; ++i) s += vd[i * n + c];
      pc[c] = s / (double)n;
    }
    __syncthreads();
    for (int e = tid; e < n * n; e += blockDim.x) {
      const int i = e / n, c = e - i * n;
      T[e] = (i == c ? 1.0 : 0.0) + cscale * (vd[e] - pc[c]);
    }
  }
}

// ---------------------------------------------------------------------------
// Row-streaming GEMM with the small N x N operand stationary in registers.
//   MODE 0 (anomaly):  out[i] = P[i] @ Q                (P = X, Q = T)
//   MODE 1 (Z pass):   out[i] = (C[i] - P[i] @ Q) / r_i  (P = V, C = D, Q = A)
// NP = N rounded up (multiple of 8, <= 128).  CTA = 8 warps; warp w owns the
// 8-column output tiles {w, w+8}; a 32-row tile is 4 DMMA m-tiles.
constexpr int R_ROWS = 32;
constexpr int R_STAGES = 4;
constexpr int R_THREADS = 256;

template <int NP, int MODE, bool VEC16>
__global__ void __launch_bounds__(R_THREADS, 1)
rowgemm_kernel(const double* __restrict__ P, const double* __restrict__ Q,
               const double* __restrict__ C, const double* __restrict__ r,
               double* __restrict__ out, int64_t n_rows, int n, int ld) {
  constexpr int KT = NP / 4;             // k-steps
  constexpr int NTT = NP / 8;            // 8-column output tiles
  constexpr int NTW = (NTT + 7) / 8;     // tiles per warp
  extern __shared__ __align__(16) double rsm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int stage_elems = R_ROWS * ld;

  // Stationary operand: b[ks][j] = Q[4ks + (lane&3)][8 (warp + 8j) + (lane>>2)].
  double b[KT][NTW];
#pragma unroll
  for (int ks = 0; ks < KT; ++ks)
#pragma unroll
    for (int j = 0; j < NTW; ++j) {
      const int k = 4 * ks + (lane & 3);
      const int col = 8 * (warp + 8 * j) + (lane >> 2);
      b[ks][j] = (k < n && col < n && warp + 8 * j < NTT) ? Q[k * n + col] : 0.0;
    }

  // Zero the K padding columns once (loads never touch them).
  for (int e = tid; e < R_STAGES * R_ROWS; e += blockDim.x)
    for (int c = n; c < ld; ++c) rsm[e * ld + c] = 0.0;

  const int64_t ntiles = (n_rows + R_ROWS - 1) / R_ROWS;
  auto load_tile = [&](int64_t tile, int buf) {
    if (tile >= ntiles) return;
    double* dst = rsm + buf * stage_elems;
    for (int rr = warp; rr < R_ROWS; rr += R_THREADS / 32) {
      const int64_t g = tile * R_ROWS + rr;
      const bool valid = g < n_rows;
      const double* src = P + (valid ? g : 0) * (int64_t)n;
      if (VEC16) {
        for (int c = 2 * lane; c < n; c += 64) cp_async16(dst + rr * ld + c, src + c, valid);
      } else {
        for (int c = lane; c < n; c += 32) cp_async8(dst + rr * ld + c, src + c, valid);
      }
    }
  };

  int64_t tile = blockIdx.x;
  const int64_t step = gridDim.x;
#pragma unroll
  for (int s = 0; s < R_STAGES - 1; ++s) { load_tile(tile + s * step, s); cp_async_commit(); }

  for (int64_t it = 0; tile < ntiles; ++it, tile += step) {
    cp_async_wait<R_STAGES - 2>();
    __syncthreads();
    load_tile(tile + (R_STAGES - 1) * step, (int)((it + R_STAGES - 1) % R_STAGES));
    cp_async_commit();

    const double* ps = rsm + (int)(it % R_STAGES) * stage_elems;
    double acc[4][NTW][2];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int j = 0; j < NTW; ++j) acc[mt][j][0] = acc[mt][j][1] = 0.0;

    if (warp < NTT) {
#pragma unroll
      for (int ks = 0; ks < KT; ++ks) {
        double a[4];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) a[mt] = ps[(mt * 8 + (lane >> 2)) * ld + 4 * ks + (lane & 3)];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int j = 0; j < NTW; ++j) dmma884(acc[mt][j][0], acc[mt][j][1], a[mt], b[ks][j]);
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int64_t g = tile * R_ROWS + mt * 8 + (lane >> 2);
        if (g >= n_rows) continue;
#pragma unroll
        for (int j = 0; j < NTW; ++j) {
          if (warp + 8 * j >= NTT) continue;
          const int col = 8 * (warp + 8 * j) + 2 * (lane & 3);
          double o0 = acc[mt][j][0], o1 = acc[mt][j][1];
          if (MODE == 1) {
            const double rv = r[g];
            if (col < n) o0 = (C[g * n + col] - o0) / rv;
            if (col + 1 < n) o1 = (C[g * n + col + 1] - o1) / rv;
          }
          double* dst = out + g * (int64_t)n + col;
          if (VEC16 && col + 1 < n) {
            *reinterpret_cast<double2*>(dst) = make_double2(o0, o1);
          } else {
            if (col < n) dst[0] = o0;
            if (col + 1 < n) dst[1] = o1;
          }
        }
      }
    }
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// Row-local helpers (enkf.py:82-92, :114-120).  One warp per row.
__global__ void deviations_kernel(const double* __restrict__ X, double* __restrict__ S,
                                  int64_t n_rows, int n, double root) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n_rows) return;
  const double* x = X + row * n;
  double s = 0.0;
  for (int c = lane; c < n; c += 32) s += x[c];
  const double mean = warp_sum(s) / (double)n;
  for (int c = lane; c < n; c += 32) S[row * n + c] = (x[c] - mean) / root;
}

__global__ void innovations_kernel(const double* __restrict__ X, const double* __restrict__ Y,
                                   const int64_t* __restrict__ idx, double* __restrict__ D,
                                   int64_t n_obs, int n) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n_obs) return;
  const int64_t src = idx ? idx[row] : row;
  for (int c = lane; c < n; c += 32) D[row * n + c] = Y[row * n + c] - X[src * n + c];
}

}  // namespace enkf
