// gram_i8.cuh — the level-0 Gram [S'R^-1 S | S'R^-1 D] on the 5th-generation tensor
// cores (N == 128, analysis mode), by exact byte-digit products (the scheme of
// anomaly_i8.cuh, SURVEY §8 rows a9/a10 and the Gram pass of DESIGN §3).
//
//   S = X[idx] - rowmean, D = Y - X[idx], rho = 1/r (sherman.py:149-154, enkf.py:82-120)
//   P = sqrt(rho) S, Q = sqrt(rho) D  ->  Gamma = P'[P | Q]
//   (the reduce applies 1/(N-1) and 1/sqrt(N-1)).
//
// Two kernels:
//  * gram_i8_slice_kernel (HBM-bound): per 32-row block of observations, gathers
//    X[idx], forms P and Q in FP64, rounds every column c onto one power-of-two
//    scale 2^(47-e_c) (e_c from a sampled pre-pass with 2 bits of headroom), cuts
//    the 48-bit integers into six BALANCED byte digits (V + 0x808080808080, then
//    byte ^ 0x80: |digit| <= 128) and writes them as ready-made UMMA operand
//    images: per block, [P planes 6 x 4 KiB | Q planes 6 x 4 KiB], each plane
//    128 members x 32 K-bytes, K-major with the 32-byte swizzle.  An element
//    outside its column scale (heavy tail, non-finite) raises the overflow flag.
//  * gram_i8_mma_ls_kernel (the MMA pass): pure TMA -> tcgen05 pipeline.  CTAs come
//    in groups of 4 over the same observation blocks and split the 26 digit pairs
//    (p + q <= 8) by level l = p + q: each owns all 256 output columns [P'P | P'Q] for
//    two levels (two 256-column int32 accumulators = all of TMEM) and issues one
//    N = 256 kind::i8 MMA per pair with A = P_p and B = [P_q ; Q_q] from shared memory;
//    every 512 blocks (16384 rows, where the int32 levels are still exact) 4 flush
//    warps fold the levels into the fp64 partial.  No FP64 arithmetic runs next to the
//    MMAs (on B200 it stalls the tensor pipe, anomaly_i8.cuh).
// (One-kernel forms that keep the images in L2 were built and measured slower.)
// Any overflow -> the FP64 DMMA Gram (gram128_kernel, gated on the flag, same
// stream) recomputes the Gram: no host round trip, same results contract.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace enkf {

constexpr int G8_N = 128;
constexpr int G8_KB = 32;        // observation rows per digit block (one MMA k-step)
constexpr int G8_ND = 6;         // digits per value
// digit pairs p + q <= 8 (1-based digit index): 26 pairs, levels 2..8 (g8ls_level)
constexpr int G8_FLUSH_BLOCKS = 512;  // 16384 rows per int32 accumulation period
constexpr int G8_PLANE = G8_N * G8_KB;            // 4 KiB: one plane, 128 members x 32 B
constexpr int G8_BLOCK_BYTES = 2 * G8_ND * G8_PLANE;  // 48 KiB per 32-row block (P and Q)
constexpr int G8_SAMPLE = 16;    // pre-pass samples every 16th observation row at least ...
constexpr int64_t G8_SAMPLES_MAX = 1 << 17;  // ... and at most ~128K rows (sparser for large n_obs)
__host__ __device__ inline int64_t g8_sample_stride(int64_t n_obs) {
  int64_t st = G8_SAMPLE;
  while ((n_obs + st - 1) / st > G8_SAMPLES_MAX) st *= 2;
  return st;
}
constexpr int G8_HEADROOM = 2;   // scale exponent headroom (bits) over the sampled max
constexpr int G8_SLICE_THREADS = 256;
#ifndef G8_SLICE_CTAS_PER_SM
#define G8_SLICE_CTAS_PER_SM 2   // the resident count: a grid of one full wave
#endif
constexpr int G8_VLD = 2 * G8_N + 1;  // slice-kernel staging row stride (uint64)

__host__ __device__ inline size_t gram_i8_slice_smem_bytes() {
  return (size_t)G8_KB * G8_VLD * 8 + 2 * G8_N * 8 /*scales*/;
}

// UMMA smem descriptor: K-major, SWIZZLE_32B (8-row atoms of 32-byte rows, 256 B apart)
__device__ __forceinline__ uint64_t umma_desc_sw32(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(256 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)6 << 61;  // SWIZZLE_32B
  return d;
}
__device__ __forceinline__ void umma_i8_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 2^(47 - e - headroom) for a column whose sampled max|.| has IEEE bits b
__device__ __forceinline__ double g8_scale(unsigned long long b) { return pow2(47 - exp_above(b) - G8_HEADROOM); }

__device__ __forceinline__ double g8_sqrt_rho(double rv) { return sqrt(1.0 / rv); }

// Column maxima over every g8_sample_stride(n_obs)-th observation row (16th, or
// sparser so that ~128K rows are sampled): |P| (128) then |Q| (128),
// as IEEE bit patterns (monotone for non-negative values).
__global__ void __launch_bounds__(256) gram_i8_scales_kernel(const double* __restrict__ X,
                                                             const double* __restrict__ Y,
                                                             const int64_t* __restrict__ idx,
                                                             const double* __restrict__ r, int64_t n_state,
                                                             int64_t n_obs, unsigned long long* __restrict__ cmax) {
  __shared__ unsigned long long red[2 * G8_N];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < 2 * G8_N; e += blockDim.x) red[e] = 0ull;
  __syncthreads();
  double mp[4] = {0, 0, 0, 0}, mq[4] = {0, 0, 0, 0};
  const int64_t stride = g8_sample_stride(n_obs);
  const int64_t nsamp = (n_obs + stride - 1) / stride;
  // 4 samples per warp in flight (independent idx -> row loads)
  constexpr int U = 4;
  const int64_t wstride = (int64_t)gridDim.x * 8;
  for (int64_t s0 = blockIdx.x * 8 + warp; s0 < nsamp; s0 += U * wstride) {
    int64_t src[U], k[U];
    double rv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t sidx = s0 + u * wstride;
      k[u] = sidx * stride;
      src[u] = -1;
      rv[u] = 0.0;
      if (sidx < nsamp) {
        src[u] = idx ? idx[k[u]] : k[u];
        rv[u] = r[k[u]];
      }
    }
    double xv[U][4], yv[U][4];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      // invalid samples (bad index, r <= 0, non-finite r) are skipped: flagged by the slice kernel
      ok[u] = src[u] >= 0 && src[u] < n_state && rv[u] > 0.0 && isfinite(rv[u]);
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        xv[u][m] = ok[u] ? X[src[u] * G8_N + lane + 32 * m] : 0.0;
        yv[u][m] = ok[u] ? Y[k[u] * G8_N + lane + 32 * m] : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double mean = warp_sum((xv[u][0] + xv[u][1]) + (xv[u][2] + xv[u][3])) * (1.0 / G8_N);
      const double sr = ok[u] ? g8_sqrt_rho(rv[u]) : 0.0;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        mp[m] = fmax(mp[m], fabs(sr * (xv[u][m] - mean)));
        mq[m] = fmax(mq[m], fabs(sr * (yv[u][m] - xv[u][m])));
      }
    }
  }
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int c = lane + 32 * m;
    atomicMax(&red[c], (unsigned long long)__double_as_longlong(mp[m]));
    atomicMax(&red[G8_N + c], (unsigned long long)__double_as_longlong(mq[m]));
  }
  __syncthreads();
  for (int e = tid; e < 2 * G8_N; e += blockDim.x)
    if (red[e]) atomicMax(&cmax[e], red[e]);
}

// sqrt(1/r) of every observation row, once (thread per row), with the checks of r
// (sherman.py:96-101: finite, positive).  The slice pass then loads the result instead
// of evaluating the FP64 divide and square root in every warp for its 4 rows — a
// quarter of that pass's instructions, which at the power-capped SM clock is what
// bounds it.  Same function on the same input: bit-identical digits.
__global__ void gram_i8_sqrt_rho_kernel(const double* __restrict__ r, int64_t n_obs, double* __restrict__ sr,
                                        DevStatus* __restrict__ status) {
  int flags = 0;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n_obs; g += (int64_t)gridDim.x * blockDim.x) {
    const double rv = r[g];
    if (!isfinite(rv)) flags |= FLAG_NONFINITE;
    else if (!(rv > 0.0)) flags |= FLAG_R_NONPOS;
    sr[g] = g8_sqrt_rho(rv);
  }
  flags = __reduce_or_sync(0xffffffffu, flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(&status->flags, flags);
}

// ---------------------------------------------------------------------------
// Slicing of one 32-row block by 8 warps (256 threads, slicer thread index st).
// Phase 1 (warp w: rows 4w..4w+3 of the block, lane: members lane + 32j): the
// biased 48-bit integers V + 0x808080808080 of P and Q into shared memory
// vals[row][256].  Phase 2 (lanes 0-15 / 16-31: 16 members, K-chunk 0 / 1): 16
// rows of one member -> 6 planes x 16 bytes, one 16-byte store per plane; a warp
// writes 16 whole 32-byte plane rows (512 contiguous bytes) of the 48 KiB image
// `out`.  `sync` is the slicers' barrier (between the phases, and after phase 2
// so vals can be reused).
template <class Sync>
__device__ __forceinline__ void g8_slice_block(const double* __restrict__ X, const double* __restrict__ Y,
                                               const int64_t* __restrict__ idx, const double* __restrict__ sqrt_rho,
                                               int64_t n_state, int64_t n_obs, int64_t blk, int st,
                                               const double (&sp)[4], const double (&sq)[4],
                                               unsigned long long* vals, unsigned char* __restrict__ out,
                                               int& flags, int& ovf, Sync sync) {
  const double kMagicB = 6755399441055744.0 + (double)0x808080808080ull;  // 1.5 2^52 + the digit bias
  const int lane = st & 31, warp = st >> 5;
  // ---- phase 1
  const int64_t g0 = blk * G8_KB + 4 * warp;
  int64_t src[4];
  double rv[4];
  bool valid[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t g = g0 + u;
    valid[u] = g < n_obs;
    src[u] = g;
    rv[u] = 1.0;
    if (valid[u]) {
      rv[u] = sqrt_rho[g];  // sqrt(1/r[g]) (gram_i8_sqrt_rho_kernel, which also checked r)
      if (idx) {
        src[u] = idx[g];
        if (lane == 0 && g > 0 && idx[g - 1] >= src[u]) flags |= FLAG_IDX_ORDER;
        if (src[u] < 0 || src[u] >= n_state) {
          flags |= FLAG_IDX_RANGE;
          valid[u] = false;
        }
      }
    }
  }
  double xv[4][4], yv[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      xv[u][j] = valid[u] ? __ldcs(X + src[u] * G8_N + lane + 32 * j) : 0.0;
      yv[u][j] = valid[u] ? __ldcs(Y + (g0 + u) * G8_N + lane + 32 * j) : 0.0;
    }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const double mean = warp_sum((xv[u][0] + xv[u][1]) + (xv[u][2] + xv[u][3])) * (1.0 / G8_N);
    const double sr = valid[u] ? rv[u] : 0.0;
    unsigned long long* vrow = vals + (4 * warp + u) * G8_VLD;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      // V = round(v 2^(47-e)): fma(v, sc, 1.5 2^52 + bias) holds V + bias in the low 51
      // bits of its mantissa (bias and 1.5 2^52 are even integers and the sum stays in
      // [2^52, 2^53), so the rounding is the rounding of v sc alone): the low word is
      // the low word of V + bias, the high word minus 0x43380000 its high word.  The six
      // balanced digits represent V iff V + bias lies in [0, 2^48): anything else (|V|
      // near or above 2^47, non-finite inputs) sets the overflow flag.
      const double tp = fma(sr * (xv[u][j] - mean), sp[j], kMagicB);
      const double tq = fma(sr * (yv[u][j] - xv[u][j]), sq[j], kMagicB);
      const uint32_t hp = (uint32_t)__double2hiint(tp) - 0x43380000u, hq = (uint32_t)__double2hiint(tq) - 0x43380000u;
      ovf |= (hp >= 0x10000u) | (hq >= 0x10000u);
      vrow[lane + 32 * j] = (unsigned long long)hp << 32 | (uint32_t)__double2loint(tp);
      vrow[G8_N + lane + 32 * j] = (unsigned long long)hq << 32 | (uint32_t)__double2loint(tq);
    }
  }
  sync();
  // ---- phase 2: two passes of 128 (member, chunk) items per warp-half
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    const int m = 128 * pass + 16 * warp + (lane & 15);  // 0..255: P members, then Q
    const int ck = lane >> 4;                            // K chunk: rows 16ck..16ck+15
    uint32_t w[G8_ND][4];
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      uint32_t vlo[4], vhi[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const unsigned long long v = vals[(16 * ck + 4 * q4 + u) * G8_VLD + m];
        vlo[u] = (uint32_t)v;
        vhi[u] = (uint32_t)(v >> 32);
      }
      // plane p (1..6) = byte (6-p) of the biased value, ^ 0x80; 4 rows per word
      auto two_planes = [&](const uint32_t (&x)[4], uint32_t bi, uint32_t bj, uint32_t& wi, uint32_t& wj) {
        const uint32_t sel = bi | ((bi + 4u) << 4) | (bj << 8) | ((bj + 4u) << 12);
        const uint32_t A = __byte_perm(x[0], x[1], sel);
        const uint32_t B = __byte_perm(x[2], x[3], sel);
        wi = __byte_perm(A, B, 0x5410) ^ 0x80808080u;
        wj = __byte_perm(A, B, 0x7632) ^ 0x80808080u;
      };
      two_planes(vhi, 1u, 0u, w[0][q4], w[1][q4]);
      two_planes(vlo, 3u, 2u, w[2][q4], w[3][q4]);
      two_planes(vlo, 1u, 0u, w[4][q4], w[5][q4]);
    }
    const int mm = m & (G8_N - 1);
    const size_t off = (size_t)(m >= G8_N ? G8_ND * G8_PLANE : 0) + (size_t)mm * 32 +
                       (size_t)((ck ^ ((mm >> 2) & 1)) << 4);
#pragma unroll
    for (int p = 0; p < G8_ND; ++p)
      *reinterpret_cast<uint4*>(out + off + (size_t)p * G8_PLANE) = make_uint4(w[p][0], w[p][1], w[p][2], w[p][3]);
  }
  sync();
}

// Slice pass of the (default) two-kernel form: every 32-row block -> its
// operand image in HBM.
#ifndef G8_SLICE_MINB
#define G8_SLICE_MINB 1
#endif
__global__ void __launch_bounds__(G8_SLICE_THREADS, G8_SLICE_MINB)
gram_i8_slice_kernel(const double* __restrict__ X, const double* __restrict__ Y, const int64_t* __restrict__ idx,
                     const double* __restrict__ sqrt_rho, const unsigned long long* __restrict__ cmax, int64_t n_state,
                     int64_t n_obs, int64_t n_blocks, unsigned char* __restrict__ planes, int* __restrict__ overflow,
                     DevStatus* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char g8s_raw[];
  unsigned long long* vals = reinterpret_cast<unsigned long long*>(g8s_raw);  // [32][G8_VLD]
  double* scl = reinterpret_cast<double*>(vals + G8_KB * G8_VLD);              // [256]
  const int tid = threadIdx.x, lane = tid & 31;
  for (int c = tid; c < 2 * G8_N; c += G8_SLICE_THREADS) scl[c] = g8_scale(cmax[c]);
  __syncthreads();
  double sp[4], sq[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    sp[j] = scl[lane + 32 * j];
    sq[j] = scl[G8_N + lane + 32 * j];
  }
  int flags = 0, ovf = 0;
  for (int64_t blk = blockIdx.x; blk < n_blocks; blk += gridDim.x)
    g8_slice_block(X, Y, idx, sqrt_rho, n_state, n_obs, blk, tid, sp, sq, vals, planes + (size_t)blk * G8_BLOCK_BYTES,
                   flags, ovf, [] { __syncthreads(); });
  flags = __reduce_or_sync(0xffffffffu, flags);
  ovf = __reduce_or_sync(0xffffffffu, ovf);
  if (lane == 0) {
    if (flags) atomicOr(&status->flags, flags);
    if (ovf) atomicOr(overflow, 1);
  }
}

// ---------------------------------------------------------------------------
// Level-split MMA pass (the product MMA pass; an earlier column-split form with
// N = 64 MMAs and A in TMEM was measured slower and removed).  The 4 CTAs
// of a group split the
// digit pairs by level l = p + q instead of by output column: CTA r owns the level
// set G8LS_SETS[r] ({7}, {8, 2}, {6, 3}, {5, 4}: 6, 6, 7, 7 pairs) for all 256
// output columns [P'P | P'Q], in two 256-column int32 accumulators (all of TMEM).
// Each pair is ONE N = 256 MMA with A = P_p and B = [P_q ; Q_q] straight from
// shared memory (the producer lays each block's planes out as P_1 Q_1 P_2 Q_2 ...,
// so one 256-row K-major descriptor spans P_q and Q_q): no tcgen05.cp, 4x the math
// per instruction of a column split (tools/probe/g8_levelsplit_probe.cu: N = 256
// from shared memory runs at the 128-cycle math floor).  The flush folds the CTA's
// two levels into its fp64 partial [group][r][256 columns][128 members]
// (read-modify-write in global memory, coalesced across a warp's members);
// gram_i8_ls_reduce sums groups and level sets in a fixed order.
constexpr int G8LS_NST = 4;                        // 48 KiB stages
constexpr int G8LS_STAGE = 2 * G8_ND * G8_PLANE;   // P_1 Q_1 ... P_6 Q_6
constexpr int G8LS_THREADS = 6 * 32;
constexpr int G8LS_LEAD = 48;                      // max blocks a CTA runs ahead of its group
__host__ __device__ constexpr size_t gram_i8_ls_smem_bytes() {
  return (size_t)G8LS_NST * G8LS_STAGE + (2 * G8LS_NST + 2) * 8 + 16 + 1024;
}
__device__ __forceinline__ uint32_t idesc_g8_n256() {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
// level set of CTA r: first and second level (p + q), 0 = none
__device__ __forceinline__ int g8ls_level(int r, int k) {
  const int a[4] = {7, 8, 6, 5}, b[4] = {0, 2, 3, 4};
  return k == 0 ? a[r] : b[r];
}

__global__ void __launch_bounds__(G8LS_THREADS, 1)
gram_i8_mma_ls_kernel(const unsigned char* __restrict__ planes, const unsigned long long* __restrict__ cmax,
                      int64_t n_blocks, int64_t blocks_per_group, double* __restrict__ partial,
                      const int* __restrict__ overflow, int* __restrict__ progress /* [groups][4], zeroed */) {
  if (*overflow) return;  // the FP64 fallback computes the Gram
  extern __shared__ __align__(1024) unsigned char g8sm_raw[];
  unsigned char* sm = g8sm_raw + ((1024u - (smem_u32(g8sm_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + G8LS_NST * G8LS_STAGE);
  uint64_t* sfull = bars;
  uint64_t* sempty = bars + G8LS_NST;
  uint64_t* afull = bars + 2 * G8LS_NST;
  uint64_t* aempty = afull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + 1);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = blockIdx.x & 3;
  const int64_t grp = blockIdx.x >> 2;
  const int64_t b0 = grp * blocks_per_group;
  const int64_t b1 = b0 + blocks_per_group < n_blocks ? b0 + blocks_per_group : n_blocks;
  const int64_t nblk = b1 > b0 ? b1 - b0 : 0;
  const int lv0 = g8ls_level(r, 0), lv1 = g8ls_level(r, 1);

  if (tid == 0) {
    for (int i = 0; i < G8LS_NST; ++i) {
      mbar_init(&sfull[i], 1);
      mbar_init(&sempty[i], 1);
    }
    mbar_init(afull, 1);
    mbar_init(aempty, 128);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(512u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  constexpr uint32_t tmem = 0;
  if (tid == 0 && *tmem_slot != 0u) __trap();

  if (warp == 0) {
    // ---- producer: the block's 12 planes, interleaved P_1 Q_1 P_2 Q_2 ...
    //      The 4 CTAs of a group carry 6, 6, 7, 7 pairs per block; the producer of a
    //      CTA that runs ahead waits (bounded: a hint, never a correctness barrier)
    //      until the group's slowest CTA is within G8LS_LEAD blocks, so each image is
    //      read from DRAM once and served from L2 to the other three.
    if (lane == 0) {
      const volatile int* gp = progress + grp * 4;
      int known = 0;  // last group minimum read: poll (~1-2 us of L2 latency) only when needed
      for (int64_t k = 0; k < nblk; ++k) {
        const int slot = (int)(k % G8LS_NST);
        if ((int)k - G8LS_LEAD > known) {
          int spin = 0;
          for (; spin < (1 << 16); ++spin) {
            known = min(min(gp[0], gp[1]), min(gp[2], gp[3]));
            if (known >= (int)k - G8LS_LEAD) break;
            __nanosleep(256);
          }
          // a group member that is not co-resident (SM-limited contexts, MPS, another
          // persistent kernel) would make every later block time out: after one
          // timeout, pacing is off for the rest of the kernel
          if (spin == (1 << 16)) known = 0x7fffffff;
        }
        if (k >= G8LS_NST) mbar_wait(&sempty[slot], (uint32_t)(((k / G8LS_NST) - 1) & 1));
        unsigned char* st = sm + slot * G8LS_STAGE;
        const unsigned char* src = planes + (size_t)(b0 + k) * G8_BLOCK_BYTES;
        mbar_arrive_expect_tx(&sfull[slot], (uint32_t)G8LS_STAGE);
#pragma unroll
        for (int d = 0; d < G8_ND; ++d) {
          bulk_g2s(st + 2 * d * G8_PLANE, src + d * G8_PLANE, (uint32_t)G8_PLANE, &sfull[slot]);
          bulk_g2s(st + (2 * d + 1) * G8_PLANE, src + (G8_ND + d) * G8_PLANE, (uint32_t)G8_PLANE, &sfull[slot]);
        }
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer: one N = 256 MMA per digit pair of the CTA's level set
    const uint32_t sbase = smem_u32(sm);
    const uint32_t idesc = idesc_g8_n256();
    for (int64_t k = 0; k < nblk; ++k) {
      const int slot = (int)(k % G8LS_NST);
      const bool first_in_period = (k % G8_FLUSH_BLOCKS) == 0;
      if (first_in_period && k > 0) mbar_wait(aempty, (uint32_t)(((k / G8_FLUSH_BLOCKS) - 1) & 1));
      mbar_wait(&sfull[slot], (uint32_t)((k / G8LS_NST) & 1));
      tc_fence_after();
      const uint32_t st = sbase + (uint32_t)(slot * G8LS_STAGE);
      bool fresh0 = first_in_period, fresh1 = first_in_period;
#pragma unroll
      for (int p = 1; p <= G8_ND; ++p) {
        const int q0 = lv0 - p, q1 = lv1 - p;
        if (q0 >= 1 && q0 <= G8_ND) {
          umma_i8_ss(tmem, umma_desc_sw32(st + (uint32_t)(2 * (p - 1) * G8_PLANE)),
                     umma_desc_sw32(st + (uint32_t)(2 * (q0 - 1) * G8_PLANE)), idesc, fresh0 ? 0u : 1u);
          fresh0 = false;
        }
        if (lv1 && q1 >= 1 && q1 <= G8_ND) {
          umma_i8_ss(tmem + 256u, umma_desc_sw32(st + (uint32_t)(2 * (p - 1) * G8_PLANE)),
                     umma_desc_sw32(st + (uint32_t)(2 * (q1 - 1) * G8_PLANE)), idesc, fresh1 ? 0u : 1u);
          fresh1 = false;
        }
      }
      umma_commit_elect(&sempty[slot]);
      if ((k % G8_FLUSH_BLOCKS) == G8_FLUSH_BLOCKS - 1 || k == nblk - 1) umma_commit_elect(afull);
      if (lane == 0) *(volatile int*)(progress + grp * 4 + r) = (int)(k + 1);
      __syncwarp();
    }
    if (lane == 0) *(volatile int*)(progress + grp * 4 + r) = 0x7fffffff;  // done: never the minimum
  } else {
    // ---- flush: thread = member i = TMEM lane; columns in chunks of 8
    const int quad = warp & 3;
    const int i = 32 * quad + lane;
    const int64_t nper = (nblk + G8_FLUSH_BLOCKS - 1) / G8_FLUSH_BLOCKS;
    double* prow = partial + (size_t)blockIdx.x * (2 * G8_N) * G8_N + i;  // column j at prow[j * G8_N]
    // level l weighs 256^(8 - l) in units of level 8 (g8_combine's convention)
    const double w0 = pow2(8 * (8 - lv0)), w1 = lv1 ? pow2(8 * (8 - lv1)) : 0.0;
    for (int j = 0; j < 2 * G8_N; ++j) prow[(size_t)j * G8_N] = 0.0;
    for (int64_t pd = 0; pd < nper; ++pd) {
      mbar_wait(afull, (uint32_t)(pd & 1));
      tc_fence_after();
      for (int cg = 0; cg < 2 * G8_N / 8; ++cg) {
        uint32_t v0[8], v1[8];
        tmem_ld8(tmem + ((uint32_t)(32 * quad) << 16) + (uint32_t)(8 * cg), v0);
        tmem_ld8(tmem + ((uint32_t)(32 * quad) << 16) + 256u + (uint32_t)(8 * cg), v1);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 8; ++c)
          prow[(size_t)(8 * cg + c) * G8_N] += fma((double)(int)v1[c], w1, (double)(int)v0[c] * w0);
      }
      tc_fence_before();
      mbar_arrive(aempty);
    }
    // scales: 2^(e_i + f_j - 62) = 2^32 / (sc_i sc_j): each operand carries 2^(47 - e - 2),
    // the level weights are in units of level 8 = 2^-62 of the combined scale
    const double ai = 4294967296.0 / g8_scale(cmax[i]);
    for (int j = 0; j < 2 * G8_N; ++j) prow[(size_t)j * G8_N] *= ai / g8_scale(cmax[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512u) : "memory");
  }
}

// Gram from the level-split partials [group][set][256][128]: fixed-order sum over
// groups and the 4 level sets; V'V from its upper triangle (exactly symmetric).
__global__ void gram_i8_ls_reduce(const double* __restrict__ partial, int ngroups, double s_vv, double s_vd,
                                  const int* __restrict__ overflow, double* __restrict__ gram) {
  if (*overflow) return;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= G8_N * 2 * G8_N) return;
  const int i = e / (2 * G8_N), c = e % (2 * G8_N);
  int a = i, b = c;
  if (c < G8_N && i > c) { a = c; b = i; }
  const double* src = partial + (size_t)b * G8_N + a;
  double s = 0.0;
  for (int g = 0; g < ngroups; ++g)
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) s += src[((size_t)g * 4 + rr) * G8_N * 2 * G8_N];
  gram[e] = s * (c < G8_N ? s_vv : s_vd);
}

}  // namespace enkf
