// levels_cluster.cuh — the N Sherman-Morrison levels (sherman.py:164-187, the
// reduced-coordinate recursion of DESIGN §3) on a cluster of LC_CTAS CTAs instead
// of one SM.  Same blocked algorithm and arithmetic order as
// ism_levels_blocked_kernel (8 levels per block: LDL' of the 8 x 8 pivot block,
// Q = M^-1 R, rank-8 update of the trailing V'V triangle and of all of V'D), with
// the update work split over the cluster:
//  * CTA r owns the V'V columns c = r (mod LC_CTAS) (packed, rows 0..c, in its shared
//    memory) and a band of lc_w(n) V'D columns, held as DMMA accumulator fragments in
//    its registers (8 warps: 4 row blocks of 32 x 2 column halves);
//  * every CTA factors the (identical) pivot block itself, solves Q for its own
//    columns and updates them;
//  * the next block's pivot columns P = Gamma[:, K'] are pushed by the owners of the
//    entries into every CTA's P buffer through distributed shared memory, then one
//    cluster barrier per block.  The P buffer is triple-buffered: a CTA still reads
//    P(blk) in its V'D update after it has arrived at block blk's barrier, and a faster
//    CTA that has passed that barrier pushes P(blk + 2) during block blk + 1 — into a
//    third buffer, so no push can land in a buffer that is still being read.
// CTA 0 reports the singular guard / den_k; A and T leave straight from the
// fragments (column means in a fixed order).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "enkf_kernels.cuh"

namespace enkf {

constexpr int LC_CTAS = 4;
constexpr int LC_THREADS = 256;

__host__ __device__ inline int lc_w(int n) { return n <= 64 ? 16 : 32; }  // V'D columns per CTA
__host__ __device__ inline int lc_cols(int n, int r) { return n > r ? (n - 1 - r) / LC_CTAS + 1 : 0; }
// packed offset of own column m (c = LC_CTAS m + r): sum_{m' < m} (LC_CTAS m' + r + 1)
__host__ __device__ inline int lc_off(int m, int r) { return LC_CTAS * m * (m - 1) / 2 + m * (r + 1); }
// packed size of the largest CTA's V'V share
__host__ __device__ inline int lc_vv_doubles(int n) {
  int mx = 0;
  for (int r = 0; r < LC_CTAS; ++r) {
    const int v = lc_off(lc_cols(n, r), r);
    mx = v > mx ? v : mx;
  }
  return (mx + 1) & ~1;
}
__host__ __device__ inline int64_t levels_cluster_smem_doubles(int n) {
  const int mmax = lc_cols(n, 0);
  return (int64_t)lc_vv_doubles(n) + 3 * LB * (int64_t)n /*PT x3*/ + LB * (int64_t)(mmax + 1) /*Rv/Qv*/ +
         LB * 32 /*Rd/Qd*/ + LB * LB /*L*/ + 2 * LB /*D, 1/D*/ + 4 * 32 /*column partials*/ + 32 /*colmean*/ + 8;
}

__device__ __forceinline__ uint32_t lc_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t lc_mapa(const void* p, uint32_t cta) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p), out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(out) : "r"(a), "r"(cta));
  return out;
}
__device__ __forceinline__ void lc_st_remote(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void lc_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__global__ void __launch_bounds__(LC_THREADS, 1)
ism_levels_cluster_kernel(const double* __restrict__ gram, int n, double cscale, double* __restrict__ A,
                          double* __restrict__ T, double* __restrict__ den_out, DevStatus* __restrict__ status) {
  extern __shared__ __align__(16) double csm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = (int)lc_rank();
  const int n2 = 2 * n;
  const int mown = lc_cols(n, r), mmax = lc_cols(n, 0);
  const int w = lc_w(n), cd0 = r * w;  // V'D columns [cd0, cd0 + w) of this CTA
  double* vv = csm;                                        // own V'V columns, packed
  double* PTb = vv + lc_vv_doubles(n);                     // [3][LB][n] pivot columns, triple-buffered
  double* Rv = PTb + 3 * LB * n;                           // [LB][mmax + 1] R, then Q (own V'V columns)
  double* Rd = Rv + LB * (mmax + 1);                       // [LB][32]       R, then Q (own V'D columns)
  double* Lm = Rd + LB * 32;                               // [LB][LB]
  double* Dm = Lm + LB * LB;                               // [2 LB]
  double* cpart = Dm + 2 * LB;                             // [4][32]
  double* cm = cpart + 4 * 32;                             // [32]
  int* fail = reinterpret_cast<int*>(cm + 32);
  const int rv_ld = mmax + 1;

  // own V'V columns (upper triangle of the Gram's V'V block)
  for (int m = 0; m < mown; ++m) {
    const int c = LC_CTAS * m + r;
    for (int i = tid; i <= c; i += LC_THREADS) vv[lc_off(m, r) + i] = gram[(int64_t)i * n2 + c];
  }
  // the first block's pivot columns, from the Gram (symmetric)
  for (int e = tid; e < LB * n; e += LC_THREADS) {
    const int j = e / n, i = e - j * n;
    PTb[e] = (j < n) ? (i <= j ? gram[(int64_t)i * n2 + j] : gram[(int64_t)j * n2 + i]) : 0.0;
    PTb[LB * n + e] = 0.0;  // rows of a short last block are never pushed: keep them finite
    PTb[2 * LB * n + e] = 0.0;
  }
  // V'D fragments: warp (wm, wn) owns rows 32 wm.., columns cd0 + (w/2) wn + 8 nt
  const int wm = warp & 3, wn = warp >> 2, fr = lane >> 2, fk = lane & 3;
  const int ntn = w / 16;  // n-tiles per warp (1 or 2)
  double vdr[4][2][2];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = 32 * wm + 8 * mt + fr, c = cd0 + (w / 2) * wn + 8 * nt + 2 * fk + e;
        vdr[mt][nt][e] = (nt < ntn && i < n && c < n) ? gram[(int64_t)i * n2 + n + c] : 0.0;
      }
  for (int e = tid; e < LB * LB; e += LC_THREADS) Lm[e] = 0.0;  // rows of a short block stay finite
  if (tid == 0) *fail = 0;
  __syncthreads();
  lc_cluster_sync();  // every CTA's buffers initialised before any remote store

  // R = Gamma[K, own trailing columns] for the block K = [kk0, kk0 + bb): rows of the own
  // V'V columns and of the own V'D fragments
  auto gather = [&](int kk0, int bb, int cc0) {
    for (int e = tid; e < bb * mown; e += LC_THREADS) {
      const int j = e / mown, m = e - j * mown, c = LC_CTAS * m + r;
      if (c >= cc0) Rv[j * rv_ld + m] = vv[lc_off(m, r) + kk0 + j];
    }
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int i = 32 * wm + 8 * mt + fr;
      if (i >= kk0 && i < kk0 + bb) {
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int cl = (w / 2) * wn + 8 * nt + 2 * fk + e;
            if (nt < ntn) Rd[(i - kk0) * 32 + cl] = vdr[mt][nt][e];
          }
      }
    }
  };
  gather(0, n < LB ? n : LB, n < LB ? n : LB);
  __syncthreads();

  for (int k0 = 0, blk = 0; k0 < n; k0 += LB, ++blk) {
    const int b = (n - k0) < LB ? (n - k0) : LB;
    const int c0 = k0 + b;
    const double* PT = PTb + (blk % 3) * LB * n;
    double* PTn = PTb + ((blk + 1) % 3) * LB * n;
    if (r == 0) LV_TRACE(blk, 0);
    // (1. R for this block was gathered at the end of the previous one)
    // ---- 2. LDL' of M = I + Gamma[K, K] (every CTA the same), one thread in registers
    if (r == 0) LV_TRACE(blk, 1);
    if (tid == 0) {
      double m[LB][LB];
#pragma unroll
      for (int rr = 0; rr < LB; ++rr)
#pragma unroll
        for (int c = 0; c <= rr; ++c)
          m[rr][c] = (rr < b && c < b) ? (rr == c ? 1.0 : 0.0) + PT[c * n + k0 + rr] : 0.0;
      bool sing = false;
#pragma unroll
      for (int jj = 0; jj < LB; ++jj) {
        if (jj >= b || sing) break;
        const double d = m[jj][jj];
        if (fabs(d) < kSingularTol) {
          if (r == 0 && !(atomicOr(&status->flags, FLAG_SINGULAR) & FLAG_SINGULAR)) {
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
        if (den_out && r == 0) den_out[k0 + jj] = d;
#pragma unroll
        for (int rr = jj + 1; rr < LB; ++rr) {
          if (rr < b) Lm[rr * LB + jj] = m[rr][jj] * dinv;
#pragma unroll
          for (int c = jj + 1; c <= rr; ++c) m[rr][c] -= m[rr][jj] * m[c][jj] * dinv;
        }
      }
    }
    __syncthreads();
    if (r == 0) LV_TRACE(blk, 2);
    if (*fail) return;  // uniform across the cluster: every CTA factors the same block
    // ---- 3. Q = M^-1 R, one own column per thread (V'V trailing, then V'D)
    for (int t = tid; t < mown + w; t += LC_THREADS) {
      double* col;
      int ld;
      if (t < mown) {
        if (LC_CTAS * t + r < c0) continue;
        col = Rv + t;
        ld = rv_ld;
      } else {
        if (cd0 + (t - mown) >= n) continue;
        col = Rd + (t - mown);
        ld = 32;
      }
      double y[LB];
#pragma unroll
      for (int j = 0; j < LB; ++j) y[j] = (j < b) ? col[j * ld] : 0.0;
#pragma unroll
      for (int j = 0; j < LB; ++j)
#pragma unroll
        for (int mm = 0; mm < j; ++mm) y[j] -= Lm[j * LB + mm] * y[mm];
#pragma unroll
      for (int j = 0; j < LB; ++j) y[j] = (j < b) ? y[j] * Dm[LB + j] : 0.0;
#pragma unroll
      for (int j = LB - 1; j >= 0; --j)
#pragma unroll
        for (int mm = j + 1; mm < LB; ++mm) y[j] -= Lm[mm * LB + j] * y[mm];
#pragma unroll
      for (int j = 0; j < LB; ++j)
        if (j < b) col[j * ld] = y[j];
    }
    __syncthreads();
    if (r == 0) LV_TRACE(blk, 3);
    // ---- 4. rank-b update of the own trailing V'V columns (warp per column) and V'D
#pragma unroll 1
    for (int m = warp; m < mown; m += LC_THREADS / 32) {
      const int c = LC_CTAS * m + r;
      if (c < c0) continue;
      double q[LB];
#pragma unroll
      for (int j = 0; j < LB; ++j) q[j] = (j < b) ? Rv[j * rv_ld + m] : 0.0;
      double* col = vv + lc_off(m, r);
#pragma unroll 1
      for (int i = lane; i <= c; i += 32) {
        double acc = col[i];
#pragma unroll
        for (int j = 0; j < LB; ++j) acc -= PT[j * n + i] * q[j];  // q[j] = 0 for j >= b
        col[i] = acc;
      }
    }
    if (c0 < n) {
      __syncthreads();  // own V'V columns updated
      if (r == 0) LV_TRACE(blk, 4);
      // ---- 5. push the next block's pivot columns Gamma[:, c0..c0+b'-1] to every CTA:
      //      the owner of column c writes Gamma[c0+j][c] (c >= c0 + j) and, for a pivot
      //      column c = c0 + j, its rows 0..c-1 as well
      const int bn = (n - c0) < LB ? (n - c0) : LB;
      for (int m = warp; m < mown; m += LC_THREADS / 32) {
        const int c = LC_CTAS * m + r;
        if (c < c0) continue;
        const double* col = vv + lc_off(m, r);
        const bool pivot = c < c0 + bn;
        const int nrow = pivot ? c + 1 : 0;  // full column for a pivot column
        // items: (j, row c0 + j) for j < bn with c0 + j <= c, then the pivot column rows
        const int nj = (c - c0 + 1) < bn ? (c - c0 + 1) : bn;
        for (int it = lane; it < LC_CTAS * (nj + nrow); it += 32) {
          const int dst = it % LC_CTAS, e = it / LC_CTAS;
          int j, i;
          double v;
          if (e < nj) {
            j = e;
            i = c;
            v = col[c0 + e];
          } else {
            j = c - c0;
            i = e - nj;
            if (i == c) continue;  // the diagonal entry is item j = c - c0 above
            v = col[i];
          }
          lc_st_remote(lc_mapa(PTn + j * n + i, (uint32_t)dst), v);
        }
      }
      if (r == 0) LV_TRACE(blk, 5);
      // the cluster barrier in two halves: arrive (release: the pushes) now, wait after
      // the V'D update and the next block's gather, which overlap its latency
      asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    }
#pragma unroll
    for (int ks = 0; ks < LB / 4; ++ks) {
      const int j = 4 * ks + fk;
      double a[4], bq[2];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int i = 32 * wm + 8 * mt + fr;
        a[mt] = (j < b && i < n) ? -PT[j * n + i] : 0.0;
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int cl = (w / 2) * wn + 8 * nt + fr;
        bq[nt] = (nt < ntn && j < b && cd0 + cl < n) ? Rd[j * 32 + cl] : 0.0;
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
          if (nt < ntn) dmma884(vdr[mt][nt][0], vdr[mt][nt][1], a[mt], bq[nt]);
    }
    if (c0 >= n) break;
    __syncthreads();  // Q (Rd) read by every warp's DMMA before the next gather overwrites it
    {
      const int bn = (n - c0) < LB ? (n - c0) : LB;
      gather(c0, bn, c0 + bn);
    }
    __syncthreads();
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }

  // ---- A = V'Z from the fragments; T = I + cscale (A - 1 colmean(A)') for the own columns
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int cl = (w / 2) * wn + 8 * nt + 2 * fk + e, c = cd0 + cl;
      double cs = 0.0;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int i = 32 * wm + 8 * mt + fr;
        if (nt < ntn && i < n && c < n) {
          A[i * n + c] = vdr[mt][nt][e];
          cs += vdr[mt][nt][e];
        }
      }
      cs += __shfl_xor_sync(0xffffffffu, cs, 4);
      cs += __shfl_xor_sync(0xffffffffu, cs, 8);
      cs += __shfl_xor_sync(0xffffffffu, cs, 16);
      if (fr == 0 && nt < ntn) cpart[wm * 32 + cl] = cs;
    }
  if (T != nullptr) {
    __syncthreads();
    for (int cl = tid; cl < w; cl += LC_THREADS)
      cm[cl] = (((cpart[cl] + cpart[32 + cl]) + cpart[64 + cl]) + cpart[96 + cl]) / (double)n;
    __syncthreads();
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = 32 * wm + 8 * mt + fr, cl = (w / 2) * wn + 8 * nt + 2 * fk + e, c = cd0 + cl;
          if (nt < ntn && i < n && c < n) T[i * n + c] = (i == c ? 1.0 : 0.0) + cscale * (vdr[mt][nt][e] - cm[cl]);
        }
  }
}

}  // namespace enkf
