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
  FLAG_DIVERGED = 32,  // Lorenz-96 forecast became non-finite (bad_index = ~(step << 32 | member))
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


// ---- mbarrier / bulk-copy (TMA engine) helpers ------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// try_wait with a suspend-time hint: a waiting warp sleeps in hardware until
// the phase completes (or the hint expires) instead of spinning on issue slots.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      " @!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x100000u)
      : "memory");
}
// Bulk (non-tensor) TMA copy global -> shared, completion counted on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
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


// ---------------------------------------------------------------------------
// Warp-specialised Gram pass (even N, 16-byte aligned rows): the production
// kernel.  One CTA per SM computes a 128 x 128 block (column block `cb` of the
// 2N Gram columns) over a contiguous range of observation rows:
//   warp 8  (loader)      : idx/r for RT rows, one bulk TMA copy per gathered
//                           X row (and Y row), completion on load_full[slot]
//   warps 9-10 (transform): row mean, 1/r, input checks; in place
//                           A operand w = (x - mean)/r, B operand [s | d]
//   warps 0-7 (DMMA)      : 64 x 32 warp tiles, m8n8k4 FP64 DMMA over the
//                           stage's rows (k = observation row)
// Stages are recycled through load_full / op_full / op_empty mbarriers.
constexpr int W_RT = 16;       // observation rows per stage
constexpr int W_STAGES = 4;
constexpr int W_MMA_WARPS = 8;
constexpr int W_XFORM_WARPS = 3;
constexpr int W_THREADS = 32 * (W_MMA_WARPS + 1 + W_XFORM_WARPS);
constexpr int W_TILE = 128;    // Gram block edge

__host__ __device__ inline size_t gram_ws_smem_bytes(int ld) {
  return (size_t)W_STAGES * 3 * W_RT * ld * sizeof(double)   // x, y, B buffers
         + (size_t)W_STAGES * W_RT * (sizeof(double) + sizeof(int))  // rinv, valid
         + 3 * W_STAGES * sizeof(uint64_t) + 64;
}

template <bool ANALYSIS>
__global__ void __launch_bounds__(W_THREADS, 1)
gram_ws_kernel(const double* __restrict__ X, const double* __restrict__ Y,
               const int64_t* __restrict__ idx, const double* __restrict__ r,
               int64_t n_state, int64_t n_obs, int n, int ld, int ctas_per_block,
               int64_t rows_per_cta, double* __restrict__ partial, DevStatus* __restrict__ status) {
  extern __shared__ __align__(128) unsigned char wsm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cb = blockIdx.x / ctas_per_block;       // Gram column block
  const int part = blockIdx.x % ctas_per_block;     // row range
  const int nb = (2 * n + W_TILE - 1) / W_TILE;
  const int col0 = cb * W_TILE;
  const bool needY = (col0 + W_TILE > n);           // block touches D columns
  const bool checker = (cb == nb - 1);
  const int64_t row_begin = (int64_t)part * rows_per_cta;
  const int64_t row_end = row_begin + rows_per_cta < n_obs ? row_begin + rows_per_cta : n_obs;
  const int nstages = row_end > row_begin ? (int)((row_end - row_begin + W_RT - 1) / W_RT) : 0;

  const int stage_elems = W_RT * ld;
  double* xb = reinterpret_cast<double*>(wsm);
  double* yb = xb + W_STAGES * stage_elems;
  double* bb = yb + W_STAGES * stage_elems;
  double* rinv_s = bb + W_STAGES * stage_elems;
  int* valid_s = reinterpret_cast<int*>(rinv_s + W_STAGES * W_RT);
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(valid_s + W_STAGES * W_RT) + 15) & ~uintptr_t(15));
  uint64_t* load_full = bars;
  uint64_t* op_full = bars + W_STAGES;
  uint64_t* op_empty = bars + 2 * W_STAGES;

  if (tid == 0) {
    for (int i = 0; i < W_STAGES; ++i) {
      mbar_init(&load_full[i], 1);
      mbar_init(&op_full[i], 32 * W_XFORM_WARPS);
      mbar_init(&op_empty[i], 32 * W_MMA_WARPS);
    }
    fence_mbar_init();
  }
  // zero the padding columns of every buffer once (operands beyond n stay 0)
  for (int e = tid; e < 3 * W_STAGES * W_RT; e += blockDim.x)
    for (int c = n; c < ld; ++c) xb[(size_t)e * ld + c] = 0.0;
  __syncthreads();

  if (warp == W_MMA_WARPS) {
    // ------------------------------------------------------------- loader
    // idx / r of stage t+1 are fetched before waiting for the slot of stage t
    int flags = 0;
    auto fetch = [&](int t, bool& valid, int64_t& src, double& rv, int64_t& prev) {
      const int64_t g = row_begin + (int64_t)t * W_RT + lane;
      valid = t < nstages && lane < W_RT && g < row_end;
      src = g;
      rv = 1.0;
      prev = -1;
      if (valid) {
        rv = r[g];
        if (ANALYSIS && idx != nullptr) {
          src = idx[g];
          if (checker && g > 0) prev = idx[g - 1];
        }
      }
    };
    bool nvalid;
    int64_t nsrc, nprev;
    double nrv;
    fetch(0, nvalid, nsrc, nrv, nprev);
    for (int t = 0; t < nstages; ++t) {
      const int slot = t % W_STAGES;
      bool valid = nvalid;
      const int64_t src = nsrc, prev = nprev, g = row_begin + (int64_t)t * W_RT + lane;
      const double rv = nrv;
      fetch(t + 1, nvalid, nsrc, nrv, nprev);
      if (valid) {
        if (ANALYSIS && idx != nullptr) {
          if (checker && g > 0 && prev >= src) flags |= FLAG_IDX_ORDER;
          if (src < 0 || src >= n_state) { flags |= FLAG_IDX_RANGE; valid = false; }
        }
        if (checker) {
          if (!isfinite(rv)) flags |= FLAG_NONFINITE;
          else if (!(rv > 0.0)) flags |= FLAG_R_NONPOS;
        }
      }
      if (t >= W_STAGES) mbar_wait(&op_empty[slot], ((t / W_STAGES) - 1) & 1);
      fence_proxy_async();
      if (lane < W_RT) {
        rinv_s[slot * W_RT + lane] = valid ? 1.0 / rv : 0.0;
        valid_s[slot * W_RT + lane] = valid ? 1 : 0;
      }
      const unsigned vmask = __ballot_sync(0xffffffffu, valid);
      const uint32_t row_bytes = (uint32_t)n * 8u;
      const uint32_t total = (uint32_t)__popc(vmask) * row_bytes * (needY ? 2u : 1u);
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&load_full[slot], total);
      __syncwarp();
      if (valid) {
        bulk_g2s(xb + slot * stage_elems + lane * ld, X + src * (int64_t)n, row_bytes, &load_full[slot]);
        if (needY) bulk_g2s(yb + slot * stage_elems + lane * ld, Y + g * (int64_t)n, row_bytes, &load_full[slot]);
      }
    }
    flags |= __shfl_xor_sync(0xffffffffu, flags, 16);
    flags |= __shfl_xor_sync(0xffffffffu, flags, 8);
    flags |= __shfl_xor_sync(0xffffffffu, flags, 4);
    flags |= __shfl_xor_sync(0xffffffffu, flags, 2);
    flags |= __shfl_xor_sync(0xffffffffu, flags, 1);
    if (lane == 0 && flags) atomicOr(&status->flags, flags);
    return;
  }

  if (warp > W_MMA_WARPS) {
    // ---------------------------------------------------------- transforms
    // Each warp handles rows tw, tw + 3, ... two at a time (independent
    // load -> shuffle-reduce -> scale chains in flight).
    const int tw = warp - W_MMA_WARPS - 1;
    const double inv_n = 1.0 / (double)n;
    // a block is "pure" when all of its 128 columns are V columns or all are
    // D columns of one aligned 128-wide slice (n == 128)
    const bool pure = (n == W_TILE);
    const bool pure_d = pure && col0 >= n;
    int flags = 0;
    constexpr int CPL = (W_TILE + 31) / 32;  // columns per lane (4 for n <= 128)
    for (int t = 0; t < nstages; ++t) {
      const int slot = t % W_STAGES;
      mbar_wait(&load_full[slot], (t / W_STAGES) & 1);
      double* xs = xb + slot * stage_elems;
      double* ys = yb + slot * stage_elems;
      double* bs = bb + slot * stage_elems;
      if (pure) {
        // Pure block (all V or all D columns, n == 128 in practice): lane owns
        // columns {2l, 2l+1, 64+2l, 65+2l}; 16-byte shared accesses; input
        // checks folded into the row sums (a non-finite entry makes them
        // non-finite).
        for (int r0 = tw; r0 < W_RT; r0 += 2 * W_XFORM_WARPS) {
          const int r1 = r0 + W_XFORM_WARPS;
          const bool has1 = r1 < W_RT;
          double2 xv[2][2], yv[2][2];
          double sx[2], sy[2], ri[2];
          bool valid[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int rr = u ? (has1 ? r1 : r0) : r0;
            valid[u] = valid_s[slot * W_RT + rr] != 0;
            ri[u] = rinv_s[slot * W_RT + rr];
            const double* xr = xs + rr * ld;
            const double* yr = ys + rr * ld;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              xv[u][h] = *reinterpret_cast<const double2*>(xr + 64 * h + 2 * lane);
              yv[u][h] = pure_d ? *reinterpret_cast<const double2*>(yr + 64 * h + 2 * lane) : make_double2(0.0, 0.0);
            }
            sx[u] = (xv[u][0].x + xv[u][0].y) + (xv[u][1].x + xv[u][1].y);
            sy[u] = (yv[u][0].x + yv[u][0].y) + (yv[u][1].x + yv[u][1].y);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            sx[0] += __shfl_xor_sync(0xffffffffu, sx[0], o);
            sx[1] += __shfl_xor_sync(0xffffffffu, sx[1], o);
            if (checker) {
              sy[0] += __shfl_xor_sync(0xffffffffu, sy[0], o);
              sy[1] += __shfl_xor_sync(0xffffffffu, sy[1], o);
            }
          }
          if (checker && ((valid[0] && !(isfinite(sx[0]) && isfinite(sy[0]))) ||
                          (has1 && valid[1] && !(isfinite(sx[1]) && isfinite(sy[1])))))
            flags |= FLAG_NONFINITE;
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            if (u == 1 && !has1) break;
            const int rr = u ? r1 : r0;
            const double mu = ANALYSIS ? sx[u] * inv_n : 0.0;
            const double rs = valid[u] ? ri[u] : 0.0;
            double* xr = xs + rr * ld;
            double* br = bs + rr * ld;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const double2 xx = xv[u][h];
              const double2 yy = yv[u][h];
              const double s0 = xx.x - mu, s1 = xx.y - mu;
              *reinterpret_cast<double2*>(xr + 64 * h + 2 * lane) =
                  valid[u] ? make_double2(s0 * rs, s1 * rs) : make_double2(0.0, 0.0);
              double2 b;
              if (pure_d) b = ANALYSIS ? make_double2(yy.x - xx.x, yy.y - xx.y) : yy;
              else b = ANALYSIS ? make_double2(s0, s1) : xx;
              if (!valid[u]) b = make_double2(0.0, 0.0);
              *reinterpret_cast<double2*>(br + 64 * h + 2 * lane) = b;
            }
          }
        }
      } else
      for (int r0 = tw; r0 < W_RT; r0 += 2 * W_XFORM_WARPS) {
        const int r1 = r0 + W_XFORM_WARPS;
        const bool has1 = r1 < W_RT;
        double xv[2][CPL], bx[2][CPL], by[2][CPL], sum[2] = {0.0, 0.0};
        bool valid[2];
        double ri[2];
        bool bad = false;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int rr = u ? r1 : r0;
          valid[u] = (u == 0 || has1) && valid_s[slot * W_RT + rr] != 0;
          ri[u] = (u == 0 || has1) ? rinv_s[slot * W_RT + rr] : 0.0;
          const double* xr = xs + rr * ld;
          const double* yr = ys + rr * ld;
#pragma unroll
          for (int q = 0; q < CPL; ++q) {
            const int c = lane + 32 * q;
            xv[u][q] = (valid[u] && c < n) ? xr[c] : 0.0;
            sum[u] += xv[u][q];
            if (checker && valid[u] && c < n) bad |= !isfinite(xv[u][q]) || !isfinite(yr[c]);
            const int gc = col0 + c;
            bx[u][q] = 0.0;
            by[u][q] = 0.0;
            if (valid[u]) {
              if (gc < n) bx[u][q] = xr[gc];
              else if (gc < 2 * n) { bx[u][q] = xr[gc - n]; by[u][q] = yr[gc - n]; }
            }
          }
        }
        if (checker && __any_sync(0xffffffffu, bad)) flags |= FLAG_NONFINITE;
        double mean[2] = {0.0, 0.0};
        if (ANALYSIS) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            sum[0] += __shfl_xor_sync(0xffffffffu, sum[0], o);
            sum[1] += __shfl_xor_sync(0xffffffffu, sum[1], o);
          }
          mean[0] = sum[0] * inv_n;
          mean[1] = sum[1] * inv_n;
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (u == 1 && !has1) break;
          const int rr = u ? r1 : r0;
          double* xr = xs + rr * ld;
#pragma unroll
          for (int q = 0; q < CPL; ++q) {
            const int c = lane + 32 * q;
            if (c < n) xr[c] = valid[u] ? (xv[u][q] - mean[u]) * ri[u] : 0.0;  // A operand (w)
            const int gc = col0 + c;
            double b = 0.0;
            if (valid[u]) {
              if (gc < n) b = ANALYSIS ? bx[u][q] - mean[u] : bx[u][q];
              else if (gc < 2 * n) b = ANALYSIS ? by[u][q] - bx[u][q] : by[u][q];
            }
            bs[rr * ld + c] = b;
          }
        }
      }
      fence_proxy_async();  // generic writes of this slot precede its next TMA refill
      mbar_arrive(&op_full[slot]);
    }
    if (flags) atomicOr(&status->flags, flags);
    return;
  }

  // ------------------------------------------------------------------ DMMA
  const int wm = warp & 1, wn = warp >> 1;   // 64-row x 32-col warp tiles
  const bool active = (64 * wm < n) && (col0 + 32 * wn < 2 * n);
  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int arow = lane & 3, acol = 64 * wm + (lane >> 2), bcol = 32 * wn + (lane >> 2);
  for (int t = 0; t < nstages; ++t) {
    const int slot = t % W_STAGES;
    mbar_wait(&op_full[slot], (t / W_STAGES) & 1);
    if (active) {
      const double* as = xb + slot * stage_elems;
      const double* bsm = bb + slot * stage_elems;
#pragma unroll
      for (int ks = 0; ks < W_RT / 4; ++ks) {
        const int row = 4 * ks + arow;
        double a[8], b[4];
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) a[mt] = as[row * ld + acol + 8 * mt];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) b[nt] = bsm[row * ld + bcol + 8 * nt];
#pragma unroll
        for (int mt = 0; mt < 8; ++mt)
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) dmma884(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
      }
    }
    mbar_arrive(&op_empty[slot]);
  }
  // partial tile [blockIdx.x][128][128]
  double* out = partial + (size_t)blockIdx.x * W_TILE * W_TILE;
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
    const int i = 64 * wm + 8 * mt + (lane >> 2);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int j = 32 * wn + 8 * nt + 2 * (lane & 3);
      *reinterpret_cast<double2*>(out + i * W_TILE + j) = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
    }
  }
}


// ---------------------------------------------------------------------------
// N == 128 specialisation of the warp-specialised Gram pass (configs 4/5).
// The two 128-column blocks are pure: block 0 = V'R^-1 V, block 1 = V'R^-1 D.
// Transform warps only form s = x - mean (in place) and, for block 1,
// d = y - x (in place): 1-2 FP64 ops per element, 4 rows in flight.  The
// 1/r_i weight is applied by the DMMA warps to the B fragment they load
// (k = observation row), so no separate operand buffer exists and the ring is
// 6 stages deep.  Rationale: transform-side DADDs share the FP64 pipe with
// DMMA, so their count and dependency depth bound the whole pass.
constexpr int P_STAGES = 6;
// gram128 DMMA warps: 8 (64x32 warp tiles) or 16 (32x32 tiles: more warps to hide the
// fragment-load latency, and the V'V block skips 6 of 16 tiles below the diagonal)
#ifndef G128_MW
#define G128_MW 8
#endif
constexpr int G128_MMA_WARPS = G128_MW;
constexpr int P_XFORM = 4;  // gram128: transform warps 8..11 (warp 8 also loads)
__host__ __device__ inline size_t gram128_smem_bytes(int ld) {
  return (size_t)P_STAGES * 2 * W_RT * ld * sizeof(double)
         + (size_t)P_STAGES * W_RT * (sizeof(double) + sizeof(int))
         + 3 * P_STAGES * sizeof(uint64_t) + 64;
}

// The V'V block is symmetric: its CTAs skip the two strictly-lower 64 x 32
// warp tiles (25 % less DMMA work), and get proportionally more rows each
// (cpb_vv CTAs for V'V, cpb_vd for V'D, chosen by the host to balance).
template <bool ANALYSIS>
__global__ void __launch_bounds__(32 * (G128_MW + 4), 1)
gram128_kernel(const double* __restrict__ X, const double* __restrict__ Y,
               const int64_t* __restrict__ idx, const double* __restrict__ r,
               int64_t n_state, int64_t n_obs, int ld, int cpb_vv, int64_t rows_vv,
               int64_t rows_vd, double* __restrict__ partial, DevStatus* __restrict__ status,
               const int* __restrict__ gate = nullptr) {
  // gate (the int8 Gram's overflow flag): run only as its FP64 fallback
  if (gate != nullptr && *gate == 0) return;
  constexpr int n = 128;
  extern __shared__ __align__(128) unsigned char psm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool dblk = (int)blockIdx.x >= cpb_vv;   // false: V'V block, true: V'D block
  const int part = dblk ? (int)blockIdx.x - cpb_vv : (int)blockIdx.x;
  const int64_t rows_per_cta = dblk ? rows_vd : rows_vv;
  const bool checker = dblk;
  const int64_t row_begin = (int64_t)part * rows_per_cta;
  const int64_t row_end = row_begin + rows_per_cta < n_obs ? row_begin + rows_per_cta : n_obs;
  const int nstages = row_end > row_begin ? (int)((row_end - row_begin + W_RT - 1) / W_RT) : 0;

  const int stage_elems = W_RT * ld;
  double* xb = reinterpret_cast<double*>(psm);
  double* yb = xb + P_STAGES * stage_elems;
  double* rinv_s = yb + P_STAGES * stage_elems;
  int* valid_s = reinterpret_cast<int*>(rinv_s + P_STAGES * W_RT);
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(valid_s + P_STAGES * W_RT) + 15) & ~uintptr_t(15));
  uint64_t* load_full = bars;
  uint64_t* op_full = bars + P_STAGES;
  uint64_t* op_empty = bars + 2 * P_STAGES;

  if (tid == 0) {
    for (int i = 0; i < P_STAGES; ++i) {
      mbar_init(&load_full[i], 1);
      mbar_init(&op_full[i], 32 * P_XFORM);
      mbar_init(&op_empty[i], 32 * G128_MMA_WARPS);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp >= G128_MMA_WARPS) {
    // ------------------------------------------------- transforms (+ loader)
    // Warps 8..11 transform rows tw, tw+4, tw+8, tw+12 of each stage; warp 8
    // also streams the rows in (idx/r prefetched one stage ahead, one bulk TMA
    // copy per gathered X row and per Y row), S-1 stages ahead of the DMMA warps.
    const int tw = warp - G128_MMA_WARPS;
    const double inv_n = 1.0 / 128.0;
    int flags = 0;
    // loader state (warp 8 only)
    bool nvalid = false;
    int64_t nsrc = 0, nprev = -1;
    double nrv = 1.0;
    auto fetch = [&](int t, bool& valid, int64_t& src, double& rv, int64_t& prev) {
      const int64_t g = row_begin + (int64_t)t * W_RT + lane;
      valid = t < nstages && lane < W_RT && g < row_end;
      src = g;
      rv = 1.0;
      prev = -1;
      if (valid) {
        rv = r[g];
        if (ANALYSIS && idx != nullptr) {
          src = idx[g];
          if (checker && g > 0) prev = idx[g - 1];
        }
      }
    };
    auto issue = [&](int u) {  // stream stage u (its slot's previous stage already consumed)
      const int slot = u % P_STAGES;
      bool valid = nvalid;
      const int64_t src = nsrc, prev = nprev, g = row_begin + (int64_t)u * W_RT + lane;
      const double rv = nrv;
      fetch(u + 1, nvalid, nsrc, nrv, nprev);
      if (valid) {
        if (ANALYSIS && idx != nullptr) {
          if (checker && g > 0 && prev >= src) flags |= FLAG_IDX_ORDER;
          if (src < 0 || src >= n_state) { flags |= FLAG_IDX_RANGE; valid = false; }
        }
        if (checker) {
          if (!isfinite(rv)) flags |= FLAG_NONFINITE;
          else if (!(rv > 0.0)) flags |= FLAG_R_NONPOS;
        }
      }
      fence_proxy_async();
      if (lane < W_RT) {
        rinv_s[slot * W_RT + lane] = valid ? 1.0 / rv : 0.0;
        valid_s[slot * W_RT + lane] = valid ? 1 : 0;
      }
      const unsigned vmask = __ballot_sync(0xffffffffu, valid);
      const uint32_t row_bytes = (uint32_t)n * 8u;
      const uint32_t total = (uint32_t)__popc(vmask) * row_bytes * (dblk ? 2u : 1u);
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&load_full[slot], total);
      __syncwarp();
      if (valid) {
        bulk_g2s(xb + slot * stage_elems + lane * ld, X + src * (int64_t)n, row_bytes, &load_full[slot]);
        if (dblk) bulk_g2s(yb + slot * stage_elems + lane * ld, Y + g * (int64_t)n, row_bytes, &load_full[slot]);
      }
    };
    if (tw == 0) {
      fetch(0, nvalid, nsrc, nrv, nprev);
      for (int u = 0; u < P_STAGES - 1 && u < nstages; ++u) issue(u);
    }
    constexpr int RPI = W_RT / P_XFORM;  // 4 rows per warp per stage, all in flight
    for (int t = 0; t < nstages; ++t) {
      const int slot = t % P_STAGES;
      mbar_wait(&load_full[slot], (t / P_STAGES) & 1);
      double* xs = xb + slot * stage_elems;
      double* ys = yb + slot * stage_elems;
      {
        const int base = tw;
        double2 xv[RPI][2], yv[RPI][2];
        double sx[RPI], sy[RPI];
        bool valid[RPI];
#pragma unroll
        for (int u = 0; u < RPI; ++u) {
          const int rr = base + u * P_XFORM;
          valid[u] = valid_s[slot * W_RT + rr] != 0;
          const double* xr = xs + rr * ld;
          const double* yr = ys + rr * ld;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            xv[u][h] = valid[u] ? *reinterpret_cast<const double2*>(xr + 64 * h + 2 * lane) : make_double2(0.0, 0.0);
            yv[u][h] = (dblk && valid[u]) ? *reinterpret_cast<const double2*>(yr + 64 * h + 2 * lane)
                                          : make_double2(0.0, 0.0);
          }
          sx[u] = (xv[u][0].x + xv[u][0].y) + (xv[u][1].x + xv[u][1].y);
          if (checker) {  // non-finite inputs: integer test of the exponent bits (no FP64 work)
            uint32_t ex = 0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const uint32_t e0 = (uint32_t)__double2hiint(xv[u][h].x), e1 = (uint32_t)__double2hiint(xv[u][h].y);
              const uint32_t e2 = (uint32_t)__double2hiint(yv[u][h].x), e3 = (uint32_t)__double2hiint(yv[u][h].y);
              ex |= ((e0 & 0x7ff00000u) == 0x7ff00000u) | ((e1 & 0x7ff00000u) == 0x7ff00000u) |
                    ((e2 & 0x7ff00000u) == 0x7ff00000u) | ((e3 & 0x7ff00000u) == 0x7ff00000u);
            }
            if (ex) flags |= FLAG_NONFINITE;
          }
        }
        (void)sy;
        if (ANALYSIS) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int u = 0; u < RPI; ++u) sx[u] += __shfl_xor_sync(0xffffffffu, sx[u], o);
        }
#pragma unroll
        for (int u = 0; u < RPI; ++u) {
          const int rr = base + u * P_XFORM;
          const double mu = ANALYSIS ? sx[u] * inv_n : 0.0;
          double* xr = xs + rr * ld;
          double* yr = ys + rr * ld;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double2 xx = xv[u][h];
            *reinterpret_cast<double2*>(xr + 64 * h + 2 * lane) =
                ANALYSIS ? make_double2(xx.x - mu, xx.y - mu) : xx;
            if (dblk) {
              const double2 yy = yv[u][h];
              *reinterpret_cast<double2*>(yr + 64 * h + 2 * lane) =
                  ANALYSIS ? make_double2(yy.x - xx.x, yy.y - xx.y) : yy;
            }
          }
        }
      }
      fence_proxy_async();
      mbar_arrive(&op_full[slot]);
      if (tw == 0) {
        const int u = t + P_STAGES - 1;  // reuses the slot of stage t-1
        if (u < nstages) {
          if (t >= 1) mbar_wait(&op_empty[(t - 1) % P_STAGES], ((t - 1) / P_STAGES) & 1);
          issue(u);
        }
      }
    }
    if (tw == 0) {
      flags |= __shfl_xor_sync(0xffffffffu, flags, 16);
      flags |= __shfl_xor_sync(0xffffffffu, flags, 8);
      flags |= __shfl_xor_sync(0xffffffffu, flags, 4);
      flags |= __shfl_xor_sync(0xffffffffu, flags, 2);
      flags |= __shfl_xor_sync(0xffffffffu, flags, 1);
    }
    if (flags) atomicOr(&status->flags, flags);
    return;
  }

// ------------------------------------------------------------------ DMMA
  constexpr int TM = G128_MMA_WARPS == 16 ? 32 : 64;  // warp tile rows (cols are 32)
  constexpr int MT = TM / 8;
  constexpr int WMN = 128 / TM;                        // warp tiles per column
  const int wm = warp % WMN, wn = warp / WMN;
  // V'V is symmetric: tiles strictly below the diagonal are not computed
  const bool active = dblk || (TM * wm < 32 * wn + 32);
  double acc[MT][4][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int arow = lane & 3, acol = TM * wm + (lane >> 2), bcol = 32 * wn + (lane >> 2);
  for (int t = 0; t < nstages; ++t) {
    const int slot = t % P_STAGES;
    mbar_wait(&op_full[slot], (t / P_STAGES) & 1);
    const double* as = xb + slot * stage_elems;
    const double* bsm = (dblk ? yb : xb) + slot * stage_elems;
#pragma unroll
    for (int ks = 0; ks < (active ? W_RT / 4 : 0); ++ks) {
      const int row = 4 * ks + arow;
      const double ri = rinv_s[slot * W_RT + row];
      double a[MT], b[4];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) a[mt] = as[row * ld + acol + 8 * mt];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) b[nt] = bsm[row * ld + bcol + 8 * nt] * ri;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma884(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
    }
    mbar_arrive(&op_empty[slot]);
  }
  double* out = partial + (size_t)blockIdx.x * W_TILE * W_TILE;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int i = TM * wm + 8 * mt + (lane >> 2);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int j = 32 * wn + 8 * nt + 2 * (lane & 3);
      *reinterpret_cast<double2*>(out + i * W_TILE + j) = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
    }
  }
}


// Fixed-order reduction for gram128: V'V entries (upper triangle computed,
// lower mirrored) from the cpb_vv V'V CTAs, V'D entries from the V'D CTAs.
__global__ void gram128_reduce(const double* __restrict__ partial, int cpb_vv, int cpb_vd,
                               double s_vv, double s_vd, double* __restrict__ gram,
                               const int* __restrict__ gate = nullptr) {
  if (gate != nullptr && *gate == 0) return;
  constexpr int n = 128;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * 2 * n) return;
  const int i = e / (2 * n), c = e % (2 * n);
  double s = 0.0;
  if (c < n) {
    const int a = i <= c ? i : c, b = i <= c ? c : i;  // upper-triangle source
    const double* src = partial + a * W_TILE + b;
    for (int k = 0; k < cpb_vv; ++k) s += src[(size_t)k * W_TILE * W_TILE];
    gram[e] = s * s_vv;
  } else {
    const double* src = partial + (size_t)cpb_vv * W_TILE * W_TILE + i * W_TILE + (c - n);
    for (int k = 0; k < cpb_vd; ++k) s += src[(size_t)k * W_TILE * W_TILE];
    gram[e] = s * s_vd;
  }
}

// Fixed-order reduction of the warp-specialised partial tiles into the Gram.
// CTA = 32 entries x GWR_SPLIT partial ranges: warp s sums its contiguous range of
// partials for 32 consecutive entries (coalesced), then thread (s = 0) adds the
// GWR_SPLIT range sums in order.  (One thread per entry summing all partials
// serially was latency-bound: 14.5 us at N = 64 for 8 MB.)
constexpr int GWR_SPLIT = 8;
__global__ void __launch_bounds__(32 * GWR_SPLIT)
gram_ws_reduce(const double* __restrict__ partial, int n, int ctas_per_block,
               double s_vv, double s_vd, double* __restrict__ gram) {
  __shared__ double part[GWR_SPLIT][32];
  const int lane = threadIdx.x & 31, sp = threadIdx.x >> 5;
  const int64_t e = blockIdx.x * (int64_t)32 + lane;
  const int64_t count = (int64_t)n * 2 * n;
  const bool live = e < count;
  const int i = live ? (int)(e / (2 * n)) : 0, c = live ? (int)(e % (2 * n)) : 0;
  const int cb = c / W_TILE, j = c % W_TILE;
  const double* src = partial + (size_t)cb * ctas_per_block * W_TILE * W_TILE + i * W_TILE + j;
  const int per = (ctas_per_block + GWR_SPLIT - 1) / GWR_SPLIT;
  const int k_lo = sp * per, k_hi = min(ctas_per_block, k_lo + per);
  double s = 0.0;
  if (live)
    for (int k = k_lo; k < k_hi; ++k) s += src[(size_t)k * W_TILE * W_TILE];
  part[sp][lane] = s;
  __syncthreads();
  if (sp == 0 && live) {
    double t = part[0][lane];
#pragma unroll
    for (int q = 1; q < GWR_SPLIT; ++q) t += part[q][lane];
    gram[e] = t * (c < n ? s_vv : s_vd);
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
// The N Sherman-Morrison levels on the Gram (one CTA of 1024 threads).
// Gamma_k[i][c] = v_i' W_k^-1 g_c with W_k = R + sum_{j<=k} v_j v_j':
//   den_k = 1 + Gamma_{k-1}[k][k]                       (sherman.py:172)
//   |den_k| < 1e-14  ->  SingularUpdateError(k+1, den_k) (sherman.py:173-174)
//   Gamma_k[i][c] = Gamma_{k-1}[i][c] - Gamma_{k-1}[i][k] Gamma_{k-1}[k][c] / den_k
// for every later column c (the rank-one update col -= h_k (v_k'col) of
// sherman.py:182-187/208-214 seen through v_i').  The V'V block is symmetric at
// every level: it is kept packed (upper triangle) in shared memory, and its
// column k doubles as the pivot row (pc).  The V'D block (A = V'Z after the
// last level) lives in registers: warp w owns rows 4w..4w+3, lane l owns
// columns 4l..4l+3.  Pivot data for level k+1 is written by the threads that
// produce it during level k (double-buffered), so each level costs one barrier.
__host__ __device__ inline int64_t levels_vv_doubles(int n) {
  const int64_t packed = (int64_t)n * (n + 1) / 2;
  return packed > 32 * (int64_t)n ? packed : 32 * (int64_t)n;  // also holds the column partials
}
__host__ __device__ inline int64_t levels_smem_doubles(int n) {
  return levels_vv_doubles(n) + 4 * (int64_t)n + 8;
}

__global__ void __launch_bounds__(1024, 1)
ism_levels_kernel(const double* __restrict__ gram, int n, double cscale,
                  double* __restrict__ A, double* __restrict__ T,
                  double* __restrict__ den_out, DevStatus* __restrict__ status) {
  extern __shared__ __align__(16) double lsm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* vv = lsm;                               // packed: p(i,c) = c(c+1)/2 + i, i <= c
  double* pcb = vv + levels_vv_doubles(n);        // [2][n] pivot column Gamma[.][k]
  double* qdb = pcb + 2 * n;                      // [2][n] pivot row of V'D: Gamma[k][n + c]
  double* dinv = qdb + 2 * n;                     // [2]: 1/den of the current / next level
  auto P = [](int i, int c) { return c * (c + 1) / 2 + i; };
  const int n2 = 2 * n;

  // V'D block in registers.
  double vd[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = 4 * warp + a, c = 4 * lane + b;
      vd[a][b] = (i < n && c < n) ? gram[(int64_t)i * n2 + n + c] : 0.0;
    }
  for (int e = tid; e < n * n; e += blockDim.x) {
    const int i = e / n, c = e - i * n;
    if (i <= c) vv[P(i, c)] = gram[(int64_t)i * n2 + c];
  }
  // level-0 pivot data: pc[i] = Gamma[i][0] = Gamma[0][i]; qd = V'D row 0
  for (int i = tid; i < n; i += blockDim.x) {
    pcb[i] = gram[i];
    qdb[i] = gram[n + i];
  }
  if (tid == 0) dinv[0] = 1.0 / (1.0 + gram[0]);
  __syncthreads();

  for (int k = 0; k < n; ++k) {
    const int cur = k & 1, nxt = cur ^ 1;
    const double* pc = pcb + cur * n;
    const double* qd = qdb + cur * n;
    double* pcn = pcb + nxt * n;
    double* qdn = qdb + nxt * n;
    const double dk = 1.0 + pc[k];
    if (fabs(dk) < kSingularTol) {
      if (tid == 0 && !(atomicOr(&status->flags, FLAG_SINGULAR) & FLAG_SINGULAR)) {
        status->level = k + 1;
        status->den = dk;
      }
      return;  // uniform: every thread read the same dk
    }
    if (tid == 0 && den_out) den_out[k] = dk;
    const double inv = dinv[cur];  // 1/dk, computed once by the producer of pc[k]
    // V'V: columns c > k, rows i <= c.
#pragma unroll 1
    for (int c = k + 1 + warp; c < n; c += 32) {
      const double qc = pc[c] * inv;
      double* col = vv + P(0, c);
#pragma unroll 1
      for (int i = lane; i <= c; i += 32) {
        const double val = col[i] - pc[i] * qc;
        col[i] = val;
        if (c == k + 1) {                         // column k+1, rows <= k+1
          pcn[i] = val;
          if (i == c) dinv[nxt] = 1.0 / (1.0 + val);
        } else if (i == k + 1) {
          pcn[c] = val;                           // row k+1 = column k+1 by symmetry
        }
      }
    }
    // V'D: all rows, all columns (registers).
    double qs[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int c = 4 * lane + b;
      qs[b] = c < n ? qd[c] * inv : 0.0;
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int i = 4 * warp + a;
      const double pr = i < n ? pc[i] : 0.0;
#pragma unroll
      for (int b = 0; b < 4; ++b) vd[a][b] -= pr * qs[b];
    }
    if ((k + 1) >> 2 == warp) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
        if (4 * warp + a == k + 1) {
#pragma unroll
          for (int b = 0; b < 4; ++b)
            if (4 * lane + b < n) qdn[4 * lane + b] = vd[a][b];
        }
    }
    __syncthreads();
  }

  // A = V'Z; T = I + cscale (A - 1 colmean(A)').
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = 4 * warp + a, c = 4 * lane + b;
      if (i < n && c < n) A[i * n + c] = vd[a][b];
    }
  if (T != nullptr) {
    // column means in a fixed order: per-warp partial over its 4 rows, then
    // a serial sum over warps
    double* cpart = vv;  // the packed V'V block is dead now; it holds >= 32 n doubles
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int c = 4 * lane + b;
      if (c < n) cpart[warp * n + c] = vd[0][b] + vd[1][b] + vd[2][b] + vd[3][b];
    }
    __syncthreads();
    double* cm = pcb;
    for (int c = tid; c < n; c += blockDim.x) {
      double s = 0.0;
      for (int w = 0; w < 32; ++w) s += cpart[w * n + c];
      cm[c] = s / (double)n;
    }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int i = 4 * warp + a, c = 4 * lane + b;
        if (i < n && c < n) T[i * n + c] = (i == c ? 1.0 : 0.0) + cscale * (vd[a][b] - cm[c]);
      }
  }
}

// ---------------------------------------------------------------------------
// Blocked form of the N Sherman-Morrison levels (production): levels are taken
// LB at a time.  For a block K = {k0..k0+b-1}, applying its b rank-one levels
// to every later column c equals (Woodbury, W -> W + V_K V_K')
//     Gamma[:, c] -= Gamma[:, K] (I + Gamma[K, K])^-1 Gamma[K, c],
// and the sequential den_k of the block are exactly the LDL' pivots of
// I + Gamma[K, K] (same values, same guard, same 1-based level).  One CTA:
// gather P = Gamma[:, K], R = Gamma[K, trailing] -> one thread factors the
// LB x LB block -> Q = M^-1 R column-parallel -> rank-b update of the trailing
// V'V (packed, smem) and of V'D (registers).  4 barriers per block instead of
// 1 per level.
constexpr int LB = 8;
// profiling only (-DLV_TRACE_ON): clock64 stamps of thread 0 per block and phase
__device__ long long g_lv_trace[20][6];
#ifdef LV_TRACE_ON
#define LV_TRACE(blk, ph) do { if (threadIdx.x == 0) g_lv_trace[(blk)][(ph)] = clock64(); } while (0)
#else
#define LV_TRACE(blk, ph) do { } while (0)
#endif
#ifndef LV_SERIAL_LDL
#define LV_SERIAL_LDL 1  // pivot-block LDL' by one thread in registers (0: the warp-shuffle form; an
                         // in-place shared-memory form was measured 1.4x slower over the kernel)
#endif
#ifndef LV_THREADS
#define LV_THREADS 512  // 128 registers per thread: the 1024-thread form spilled (ncu: STL in the trailing update)
#endif

__host__ __device__ inline int64_t levels_blk_smem_doubles(int n) {
  // (V'D lives in registers and leaves through them: no [n][n] buffer, so the kernel
  // leaves ~140 KiB of the SM's 256 KiB to L1, where the fragments that do not fit
  // in registers live)
  return levels_vv_doubles(n) + (int64_t)LB * n /*PT*/ + (int64_t)LB * 2 * n /*R/Q*/ + (int64_t)LB * LB /*L*/ +
         2 * LB /*D, 1/D*/ + 4 * (int64_t)n /*column partials*/ + n /*colmean*/ + 16;
}

__global__ void __launch_bounds__(LV_THREADS, 1)
ism_levels_blocked_kernel(const double* __restrict__ gram, int n, double cscale,
                          double* __restrict__ A, double* __restrict__ T,
                          double* __restrict__ den_out, DevStatus* __restrict__ status) {
  extern __shared__ __align__(16) double bsm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nthr = blockDim.x, nwarps = nthr >> 5;
  double* vv = bsm;                                  // packed upper V'V: p(i,c) = c(c+1)/2 + i
  double* PT = vv + levels_vv_doubles(n);            // [LB][n]   Gamma[i][k0+j] at PT[j][i]
  double* RQ = PT + LB * n;                          // [LB][2n]  R, then Q = M^-1 R
  double* Lm = RQ + LB * 2 * n;                      // [LB][LB]  unit lower factor
  double* Dm = Lm + LB * LB;                         // [LB]      pivots
  double* cpart = Dm + 2 * LB;                       // [4][n]    column partial sums (epilogue)
  double* cm = cpart + 4 * n;                        // [n]       column means (epilogue)
  int* fail = reinterpret_cast<int*>(cm + n);
  auto P = [](int i, int c) { return c * (c + 1) / 2 + i; };
  const int n2 = 2 * n;

  for (int e = tid; e < n * n; e += nthr) {
    const int i = e / n, c = e - i * n;
    if (i <= c) vv[P(i, c)] = gram[(int64_t)i * n2 + c];
  }
  // V'D lives in DMMA accumulator fragments: warp w owns the 32 x 32 tile (rows
  // 32(w&3).., cols 32(w>>2)..), 4 x 4 m8n8 tiles; lane holds (row fr, cols 2fk, 2fk+1)
  static_assert(LV_THREADS == 512, "the V'D register tiling assumes 16 warps");
  const int wm = warp & 3, wn = warp >> 2, fr = lane >> 2, fk = lane & 3;
  double vdr[4][4][2];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = 32 * wm + 8 * mt + fr, c = 32 * wn + 8 * nt + 2 * fk + e;
        vdr[mt][nt][e] = (i < n && c < n) ? gram[(int64_t)i * n2 + n + c] : 0.0;
      }
  for (int e = tid; e < LB * LB; e += nthr) Lm[e] = 0.0;  // rows of a short last block stay finite
  if (tid == 0) *fail = 0;
  __syncthreads();

  for (int k0 = 0; k0 < n; k0 += LB) {
    const int b = (n - k0) < LB ? (n - k0) : LB;
    const int c0 = k0 + b;  // first trailing V'V column
    LV_TRACE(k0 / LB, 0);
    // ---- 1. gather P = Gamma[:, K], R = Gamma[K, trailing] (M = I + Gamma[K, K] is in PT)
    for (int e = tid; e < b * n; e += nthr) {
      const int j = e / n, i = e - j * n, k = k0 + j;
      PT[j * n + i] = (i <= k) ? vv[P(i, k)] : vv[P(k, i)];
      if (i >= c0) RQ[j * n2 + i] = vv[P(k, i)];
    }
    // the block's V'D rows k0..k0+b-1 (R, V'D part) straight from the owning fragments
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int i = 32 * wm + 8 * mt + fr;
      if (i >= k0 && i < k0 + b) {
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int c = 32 * wn + 8 * nt + 2 * fk + e;
            if (c < n) RQ[(i - k0) * n2 + n + c] = vdr[mt][nt][e];
          }
      }
    }
    __syncthreads();
    LV_TRACE(k0 / LB, 1);
    // ---- 2. LDL' of M = I + Gamma[K, K] (the block's den_k), one warp in
    //         registers: lane l holds entries l and l+32 of the row-major 8x8
    //         block; column j is broadcast by shuffles at step j.  Dm = den,
    //         Dm[LB + j] = 1/den (one reciprocal per pivot), Lm unit lower.
#if LV_SERIAL_LDL
    // one thread, the whole b x b block in registers (the shuffle-based warp form
    // spent ~4K cycles per block in dependent shuffle rounds)
    if (tid == 0) {
      double m[LB][LB];
#pragma unroll
      for (int r = 0; r < LB; ++r)
#pragma unroll
        for (int c = 0; c <= r; ++c)
          m[r][c] = (r < b && c < b) ? (r == c ? 1.0 : 0.0) + PT[c * n + k0 + r] : 0.0;
      bool sing = false;
#pragma unroll
      for (int jj = 0; jj < LB; ++jj) {
        if (jj >= b || sing) break;
        const double d = m[jj][jj];
        if (fabs(d) < kSingularTol) {
          if (!(atomicOr(&status->flags, FLAG_SINGULAR) & FLAG_SINGULAR)) {
            status->level = k0 + jj + 1;
            status->den = d;
          }
          *fail = 1;
          sing = true;
          break;
        }
        const double dinv = 1.0 / d;
        Dm[jj] = d;
        Dm[LB + jj] = dinv;
        if (den_out) den_out[k0 + jj] = d;
#pragma unroll
        for (int r = jj + 1; r < LB; ++r) {
          if (r < b) Lm[r * LB + jj] = m[r][jj] * dinv;
#pragma unroll
          for (int c = jj + 1; c <= r; ++c) m[r][c] -= m[r][jj] * m[c][jj] * dinv;
        }
      }
    }
#else
    if (warp == 0) {
      double m[2];
      int er[2], ec[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e = lane + 32 * h;
        er[h] = e >> 3;
        ec[h] = e & 7;
        m[h] = (er[h] < b && ec[h] < b) ? (er[h] == ec[h] ? 1.0 : 0.0) + PT[ec[h] * n + k0 + er[h]] : 0.0;
      }
#pragma unroll
      for (int j = 0; j < LB; ++j) {
        if (j >= b) break;
        // pivot M[j][j] lives at e = 9j
        const double d = __shfl_sync(0xffffffffu, (9 * j) < 32 ? m[0] : m[1], (9 * j) & 31);
        if (fabs(d) < kSingularTol) {
          if (lane == 0) {
            if (!(atomicOr(&status->flags, FLAG_SINGULAR) & FLAG_SINGULAR)) {
              status->level = k0 + j + 1;
              status->den = d;
            }
            *fail = 1;
          }
          break;
        }
        const double dinv = 1.0 / d;
        if (lane == 0) {
          Dm[j] = d;
          Dm[LB + j] = dinv;
          if (den_out) den_out[k0 + j] = d;
        }
        // column j: M[r][j] at e = 8r + j -> lane (8r+j)&31, slot (8r+j)>>5
        double colr[2], colc[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int er_ = 8 * er[h] + j, ec_ = 8 * ec[h] + j;
          const double v0 = __shfl_sync(0xffffffffu, m[0], er_ & 31);
          const double v1 = __shfl_sync(0xffffffffu, m[1], er_ & 31);
          colr[h] = (er_ >> 5) ? v1 : v0;
          const double w0 = __shfl_sync(0xffffffffu, m[0], ec_ & 31);
          const double w1 = __shfl_sync(0xffffffffu, m[1], ec_ & 31);
          colc[h] = (ec_ >> 5) ? w1 : w0;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (ec[h] == j && er[h] > j && er[h] < b) Lm[er[h] * LB + j] = m[h] * dinv;
          if (er[h] > j && ec[h] > j) m[h] -= colr[h] * colc[h] * dinv;
        }
      }
    }
#endif
    __syncthreads();
    if (*fail) return;  // uniform
    LV_TRACE(k0 / LB, 2);
    // ---- 3. Q = M^-1 R, one trailing column per thread
    const int nv = n - c0;  // trailing V'V columns
    for (int t = tid; t < nv + n; t += nthr) {
      const int col = (t < nv) ? (c0 + t) : (n + (t - nv));
      double y[LB];
#pragma unroll
      for (int j = 0; j < LB; ++j) y[j] = (j < b) ? RQ[j * n2 + col] : 0.0;
#pragma unroll
      for (int j = 0; j < LB; ++j)
#pragma unroll
        for (int m = 0; m < j; ++m) y[j] -= Lm[j * LB + m] * y[m];
#pragma unroll
      for (int j = 0; j < LB; ++j) y[j] = (j < b) ? y[j] * Dm[LB + j] : 0.0;
#pragma unroll
      for (int j = LB - 1; j >= 0; --j)
#pragma unroll
        for (int m = j + 1; m < LB; ++m) y[j] -= Lm[m * LB + j] * y[m];
#pragma unroll
      for (int j = 0; j < LB; ++j)
        if (j < b) RQ[j * n2 + col] = y[j];
    }
    __syncthreads();
    LV_TRACE(k0 / LB, 3);
    // ---- 4. rank-b update of the trailing V'V (warp per column) and all of V'D
#pragma unroll 1
    for (int c = c0 + warp; c < n; c += nwarps) {
      double q[LB];
#pragma unroll
      for (int j = 0; j < LB; ++j) q[j] = (j < b) ? RQ[j * n2 + c] : 0.0;
      double* col = vv + P(0, c);
#pragma unroll 1
      for (int i = lane; i <= c; i += 32) {
        double acc = col[i];
#pragma unroll
        for (int j = 0; j < LB; ++j) acc -= PT[j * n + i] * q[j];  // q[j] = 0 for j >= b
        col[i] = acc;
      }
    }
    // V'D -= P Q on the FP64 tensor pipe (DMMA m8n8k4, two k-steps of the rank-b
    // update; A = -P from PT, B = Q from RQ, zero beyond b and n)
#pragma unroll
    for (int ks = 0; ks < LB / 4; ++ks) {
      const int j = 4 * ks + fk;
      double a[4], bq[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int i = 32 * wm + 8 * mt + fr;
        a[mt] = (j < b && i < n) ? -PT[j * n + i] : 0.0;
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int c = 32 * wn + 8 * nt + fr;
        bq[nt] = (j < b && c < n) ? RQ[j * n2 + n + c] : 0.0;
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma884(vdr[mt][nt][0], vdr[mt][nt][1], a[mt], bq[nt]);
    }
    __syncthreads();
  }

  LV_TRACE(16, 0);
  // A = V'Z straight from the fragments; T = I + cscale (A - 1 colmean(A)'), the column
  // sums in a fixed order: per warp over its 32 rows (fragment rows, then shuffles
  // over the 8 row lanes), then the 4 row blocks in order
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int c = 32 * wn + 8 * nt + 2 * fk + e;
      double cs = 0.0;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int i = 32 * wm + 8 * mt + fr;
        if (i < n && c < n) {
          A[i * n + c] = vdr[mt][nt][e];
          cs += vdr[mt][nt][e];
        }
      }
      cs += __shfl_xor_sync(0xffffffffu, cs, 4);
      cs += __shfl_xor_sync(0xffffffffu, cs, 8);
      cs += __shfl_xor_sync(0xffffffffu, cs, 16);
      if (fr == 0 && c < n) cpart[wm * n + c] = cs;
    }
  if (T != nullptr) {
    __syncthreads();
    for (int c = tid; c < n; c += nthr) cm[c] = (((cpart[c] + cpart[n + c]) + cpart[2 * n + c]) + cpart[3 * n + c]) / (double)n;
    __syncthreads();
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = 32 * wm + 8 * mt + fr, c = 32 * wn + 8 * nt + 2 * fk + e;
          if (i < n && c < n) T[i * n + c] = (i == c ? 1.0 : 0.0) + cscale * (vdr[mt][nt][e] - cm[c]);
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


// TMA-fed row GEMM (even N, 16-byte aligned rows): the production anomaly-
// update / Z-pass kernel.  Thread 0 streams 32-row tiles of P into a 4-slot
// ring with one bulk TMA copy per row (mbarrier full/empty pairs), refilling a
// slot as soon as all 8 warps have released it; the warps keep the N x N
// operand Q stationary in registers (no producer warp, so each thread keeps
// the full 255-register budget) and run the m8n8k4 FP64 DMMA, releasing each
// slot before their epilogue stores.
template <int NP, int MODE>
__global__ void __launch_bounds__(R_THREADS, 1)
rowgemm_ws_kernel(const double* __restrict__ P, const double* __restrict__ Q,
                  const double* __restrict__ C, const double* __restrict__ r,
                  double* __restrict__ out, int64_t n_rows, int n, int ld) {
  constexpr int KT = NP / 4;
  constexpr int NTT = NP / 8;
  constexpr int NTW = (NTT + 7) / 8;
  extern __shared__ __align__(128) unsigned char rwsm[];
  double* ring = reinterpret_cast<double*>(rwsm);
  const int stage_elems = R_ROWS * ld;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + R_STAGES * stage_elems);
  uint64_t* empty = full + R_STAGES;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t ntiles = (n_rows + R_ROWS - 1) / R_ROWS;
  const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if (tid == 0) {
    for (int i = 0; i < R_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], R_THREADS);
    }
    fence_mbar_init();
  }
  for (int e = tid; e < R_STAGES * R_ROWS; e += blockDim.x)
    for (int c = n; c < ld; ++c) ring[(size_t)e * ld + c] = 0.0;
  __syncthreads();

  // issue the bulk copies of local tile `it` (thread 0 only)
  auto issue = [&](int64_t it) {
    const int slot = (int)(it % R_STAGES);
    if (it >= R_STAGES) mbar_wait(&empty[slot], (uint32_t)(((it / R_STAGES) - 1) & 1));
    fence_proxy_async();
    const int64_t tile = blockIdx.x + it * gridDim.x;
    const int64_t g0 = tile * R_ROWS;
    const int rows = (int)(n_rows - g0 < R_ROWS ? n_rows - g0 : R_ROWS);
    const uint32_t row_bytes = (uint32_t)n * 8u;
    mbar_arrive_expect_tx(&full[slot], (uint32_t)rows * row_bytes);
    for (int rr = 0; rr < rows; ++rr)
      bulk_g2s(ring + slot * stage_elems + rr * ld, P + (g0 + rr) * (int64_t)n, row_bytes, &full[slot]);
  };
  if (tid == 0)
    for (int64_t it = 0; it < R_STAGES - 1 && it < my_tiles; ++it) issue(it);

  double b[KT][NTW];
#pragma unroll
  for (int ks = 0; ks < KT; ++ks)
#pragma unroll
    for (int j = 0; j < NTW; ++j) {
      const int k = 4 * ks + (lane & 3);
      const int col = 8 * (warp + 8 * j) + (lane >> 2);
      b[ks][j] = (k < n && col < n && warp + 8 * j < NTT) ? Q[k * n + col] : 0.0;
    }

  for (int64_t it = 0; it < my_tiles; ++it) {
    if (tid == 0 && it + R_STAGES - 1 < my_tiles) issue(it + R_STAGES - 1);
    const int slot = (int)(it % R_STAGES);
    mbar_wait(&full[slot], (uint32_t)((it / R_STAGES) & 1));
    const int64_t tile = blockIdx.x + it * gridDim.x;
    const double* ps = ring + slot * stage_elems;
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
    }
    mbar_arrive(&empty[slot]);
    if (warp < NTT) {
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int64_t g = tile * R_ROWS + mt * 8 + (lane >> 2);
        if (g >= n_rows) continue;
#pragma unroll
        for (int j = 0; j < NTW; ++j) {
          if (warp + 8 * j >= NTT) continue;
          const int col = 8 * (warp + 8 * j) + 2 * (lane & 3);
          if (col >= n) continue;
          double o0 = acc[mt][j][0], o1 = acc[mt][j][1];
          if (MODE == 1) {
            const double rv = r[g];
            const double2 cv = *reinterpret_cast<const double2*>(C + g * n + col);
            o0 = (cv.x - o0) / rv;
            o1 = (cv.y - o1) / rv;
          }
          *reinterpret_cast<double2*>(out + g * (int64_t)n + col) = make_double2(o0, o1);
        }
      }
    }
  }
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
