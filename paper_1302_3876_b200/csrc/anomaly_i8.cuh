// anomaly_i8.cuh — X^A = X + X C on the 5th-generation tensor cores (N == 128).
//
// The anomaly update (enkf.py:192, x + s @ A, K11) is an Ns x 128 x 128 fp64
// product.  B200 has no fp64 tcgen05 kind, so the product is evaluated
// EXACTLY in integer arithmetic on byte "digits" (Ozaki-style splitting) and
// rounded once at the end:
//   row i of X  : e_i with max|X_i.| < 2^e_i,  V_ik = round(X_ik 2^(47-e_i))  (48-bit)
//   column j of C: f_j with max|C_.j| < 2^f_j, W_kj = round(C_kj 2^(47-f_j))
//   V = sum_p d_p 256^(6-p), W = sum_q c_q 256^(6-q), p,q = 1..6 two's-complement
//   bytes (p = 1 signed, the rest unsigned).  X C ~= 2^(e_i+f_j-94) sum_{p+q<=8}
//   256^(12-p-q) (D_p C_q)_ij with every D_p C_q an exact int32 tcgen05.mma
//   (kind::i8, K = 128 -> |acc| < 2^26).  26 digit pairs, 7 levels l = p+q.
// Truncation (p+q > 8) and the input roundings give |error| ~ 1e-13 relative
// to max|X^A| on the config inputs (tests compare against the FP64 DMMA path
// and the oracle).
//
// Layout: the 6 digit planes of C^T (M = 128 output columns x K = 128) stay in
// TMEM for the whole kernel (A operand, 6 x 32 columns); X-row digit planes
// (B operand, N = 16 rows per MMA, K-major, 128B swizzle) are produced by 4
// slicer warps into a 2-deep smem ring; the accumulators (7 levels x 16
// columns) are double-buffered in TMEM; 4 epilogue warps (thread = output
// column = TMEM lane) recombine the 7 int32 levels exactly in int64, round to
// fp64, add X and store.  One elected thread issues the MMAs.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace enkf {

constexpr int I8_N = 128;         // ensemble size handled by this kernel
constexpr int I8_TILE = 64;       // X rows per tile
constexpr int I8_CHUNK = 16;      // rows per MMA (N of the instruction)
constexpr int I8_ND = 6;          // byte digits per value
constexpr int I8_LMAX = 8;        // keep digit pairs with p + q <= 8
constexpr int I8_NLEV = I8_LMAX - 1;  // levels 2..8
constexpr int I8_SLICE_WARPS = 4;
constexpr int I8_EPI_WARPS = 8;   // two per TMEM lane quadrant, each half of a chunk's rows
constexpr int I8_THREADS = (I8_SLICE_WARPS + I8_EPI_WARPS + 2) * 32;  // + MMA warp + TMA warp
constexpr int I8_STAGE_BYTES = I8_TILE * I8_N * 8;     // raw X tile (64 KiB)
constexpr int I8_PLANE_BYTES = I8_TILE * 128;          // 8 KiB per digit plane
constexpr int I8_XBUF_BYTES = I8_ND * I8_PLANE_BYTES;  // 48 KiB per tile buffer
// TMEM columns: C planes at [0, 192); accumulators buffer b, level l at
// 192 + b*112 + (l-2)*16
constexpr uint32_t I8_TMEM_COLS = 512;
constexpr int I8_ACC0 = I8_ND * 32;
constexpr int I8_ACCBUF = I8_NLEV * I8_CHUNK;

__host__ __device__ inline size_t anomaly_i8_smem_bytes() {
  return 1024 /*align slack*/ + 2 * (size_t)I8_XBUF_BYTES + 2 * (size_t)I8_STAGE_BYTES +
         2 * I8_TILE * sizeof(int) + 256;
}

// ---- tcgen05 helpers ---------------------------------------------------------
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row atoms 1024 B apart.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr & 0x3FFFF) >> 4);         // start address
  d |= (uint64_t)1 << 16;                              // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;                    // SBO: 8-row atom stride
  d |= (uint64_t)1 << 46;                              // descriptor version (sm100)
  d |= (uint64_t)2 << 61;                              // SWIZZLE_128B
  return d;
}

// Instruction descriptor: kind::i8, D = s32, A/B K-major, M = 128, N = I8_CHUNK.
__device__ __forceinline__ uint32_t idesc_i8(bool a_signed, bool b_signed) {
  uint32_t d = 0;
  d |= 2u << 4;                                        // c_format = S32
  d |= (a_signed ? 1u : 0u) << 7;                      // a_format
  d |= (b_signed ? 1u : 0u) << 10;                     // b_format
  d |= (uint32_t)(I8_CHUNK >> 3) << 17;                // n_dim
  d |= (uint32_t)(128 >> 4) << 24;                     // m_dim
  return d;
}

// Issued by the whole (converged) warp; one elected lane executes the MMA, so
// the operands stay warp-uniform (uniform registers, no per-lane waterfall).
__device__ __forceinline__ void umma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
      "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tmem_st1(uint32_t taddr, uint32_t v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};\n" ::"r"(taddr), "r"(v) : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// exponent e with |v| < 2^e for the largest |v| (from the IEEE bits of max|v|)
__device__ __forceinline__ int exp_above(uint64_t absbits) {
  if (absbits == 0) return 0;
  return (int)((absbits >> 52) & 0x7ff) - 1022;
}
// 2^k as a double (exact; falls back to ldexp outside the normal range)
__device__ __forceinline__ double pow2(int k) {
  if (k < -1022 || k > 1023) return ldexp(1.0, k);
  return __longlong_as_double((long long)(k + 1023) << 52);
}
constexpr int I8_NONFINITE = 0x7fff;  // row exponent marker: the row holds inf/nan
// round(x * 2^s) as int64 for |x 2^s| < 2^51, via the 1.5*2^52 magic constant
__device__ __forceinline__ long long round_scaled(double x, double scale) {
  const double magic = 6755399441055744.0;  // 1.5 * 2^52
  return __double_as_longlong(fma(x, scale, magic)) - __double_as_longlong(magic);
}
// exact int64 -> double for |v| < 2^51
__device__ __forceinline__ double i64_to_f64_exact(long long v) {
  const double magic = 6755399441055744.0;
  return __longlong_as_double(v + __double_as_longlong(magic)) - magic;
}
// byte b (0 = least significant) of the 48-bit two's-complement value v
__device__ __forceinline__ uint32_t byte_of(long long v, int b) { return (uint32_t)(v >> (8 * b)) & 0xffu; }

// ---- the kernel ------------------------------------------------------------------
// Roles (14 warps):  0-3 slicers, 4-11 epilogue (two per TMEM lane quadrant),
// 12 MMA issuer (also owns TMEM), 13 TMA producer.  Per 64-row tile:
//   producer : one bulk TMA copy of the contiguous X tile -> stage[buf]
//   slicers  : stage[buf] -> 6 byte-digit planes (K-major, 128B swizzle) + row exponents
//   MMA      : 4 chunks x 26 digit pairs x 4 k-steps of tcgen05.mma kind::i8
//   epilogue : TMEM -> exact int64 recombination -> fp64, + X (from stage[buf]) -> X^A
__global__ void __launch_bounds__(I8_THREADS, 1)
anomaly_i8_kernel(const double* __restrict__ X, const double* __restrict__ C /* = T */,
                  double* __restrict__ XA, int64_t n_rows, int dbg) {
  // dbg (profiling only): bit0 skip MMAs, bit1 skip slicing, bit2 skip epilogue math/IO
  extern __shared__ __align__(1024) unsigned char i8sm_raw[];
  unsigned char* i8sm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(i8sm_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* xdig = i8sm;                                            // [2][6][64][128 B]
  double* stage = reinterpret_cast<double*>(xdig + 2 * I8_XBUF_BYTES);  // [2][64][128]
  int* rexp = reinterpret_cast<int*>(stage + 2 * I8_TILE * I8_N);       // [2][64]
  uint64_t* bars = reinterpret_cast<uint64_t*>(rexp + 2 * I8_TILE);
  uint64_t* sfull = bars;        // [2] TMA -> slicers/epilogue       (count 1 + tx)
  uint64_t* sempty = bars + 2;   // [2] slicers+epilogue -> producer  (count slicer+epi threads)
  uint64_t* xfull = bars + 4;    // [2] slicers -> MMA                (count slicer threads)
  uint64_t* xempty = bars + 6;   // [2] MMA commit -> slicers         (count 1)
  uint64_t* afull = bars + 8;    // [2] MMA commit -> epilogue        (count 1)
  uint64_t* aempty = bars + 10;  // [2] epilogue -> MMA               (count epi threads)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  constexpr int EPI0 = I8_SLICE_WARPS;                 // first epilogue warp
  constexpr int MMAW = I8_SLICE_WARPS + I8_EPI_WARPS;  // MMA warp
  constexpr int TMAW = MMAW + 1;                       // producer warp
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t ntiles = (n_rows + I8_TILE - 1) / I8_TILE;
  const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sfull[i], 1);
      mbar_init(&sempty[i], 32 * (I8_SLICE_WARPS + I8_EPI_WARPS));
      mbar_init(&xfull[i], 32 * I8_SLICE_WARPS);
      mbar_init(&xempty[i], 1);
      mbar_init(&afull[i], 1);
      mbar_init(&aempty[i], 32 * I8_EPI_WARPS);
    }
    fence_mbar_init();
  }
  if (warp == MMAW) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(I8_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // One CTA per SM owns all 512 columns, so the allocation starts at lane 0,
  // column 0: a compile-time TMEM base keeps every MMA operand uniform.
  constexpr uint32_t tmem = 0;
  if (tid == 0 && *tmem_slot != 0u) __trap();

  if (warp == TMAW) {
    // ---- producer: one bulk copy per tile (the tile's rows are contiguous) -----
    if (lane == 0) {
      for (int64_t it = 0; it < my_tiles; ++it) {
        const int buf = (int)(it & 1);
        const int64_t tile = blockIdx.x + it * gridDim.x;
        if (it >= 2) mbar_wait(&sempty[buf], (uint32_t)(((it >> 1) - 1) & 1));
        fence_proxy_async();
        const int64_t g0 = tile * I8_TILE;
        const int rows = (int)(n_rows - g0 < I8_TILE ? n_rows - g0 : I8_TILE);
        const uint32_t bytes = (uint32_t)rows * I8_N * 8u;
        mbar_arrive_expect_tx(&sfull[buf], bytes);
        double* dst = stage + buf * I8_TILE * I8_N;
        const double* src = X + g0 * I8_N;
        for (uint32_t off = 0; off < bytes; off += 16384u) {
          const uint32_t len = bytes - off < 16384u ? bytes - off : 16384u;
          bulk_g2s(reinterpret_cast<unsigned char*>(dst) + off, reinterpret_cast<const unsigned char*>(src) + off,
                   len, &sfull[buf]);
        }
      }
    }
  } else if (warp >= EPI0 && warp < MMAW) {
    // ---- epilogue warps: thread = output column j = TMEM lane ------------------
    const int quad = warp & 3;            // TMEM lane quadrant this warp may access
    const int half = (warp - EPI0) >> 2;  // which 8 rows of each 16-row chunk
    const int j = 32 * quad + lane;
    // C^T digit planes into TMEM (A operand), column scale f_j
    // C = T - I (T = I + (I - 11'/N) A / sqrt(N-1) from the levels kernel)
    auto cval = [&](int k) { return C[k * I8_N + j] - (k == j ? 1.0 : 0.0); };
    uint64_t cmax = 0;
    for (int k = 0; k < I8_N; ++k) {
      const uint64_t b = (uint64_t)__double_as_longlong(cval(k)) & 0x7fffffffffffffffull;
      cmax = b > cmax ? b : cmax;
    }
    const int fj = exp_above(cmax);
    if (half == 0) {
      const double cscale = pow2(47 - fj);
#pragma unroll 1
      for (int p = 0; p < I8_ND; ++p) {
#pragma unroll 1
        for (int w = 0; w < 32; ++w) {
          uint32_t word = 0;
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const long long v = round_scaled(cval(4 * w + b), cscale);
            word |= byte_of(v, 5 - p) << (8 * b);
          }
          tmem_st1(tmem + ((uint32_t)(32 * quad) << 16) + (uint32_t)(32 * p + w), word);
        }
      }
      tmem_st_wait();
    }
    tc_fence_before();
    asm volatile("bar.sync 1, 288;\n" ::: "memory");  // C planes are in TMEM before the first MMA
    int chunk_ctr = 0;
    for (int64_t it = 0; it < my_tiles; ++it) {
      const int buf = (int)(it & 1);
      const int64_t tile = blockIdx.x + it * gridDim.x;
      mbar_wait(&sfull[buf], (uint32_t)((it >> 1) & 1));  // raw X of the tile is in smem
      mbar_wait(&xfull[buf], (uint32_t)((it >> 1) & 1));  // and the slicers' row exponents
      const double* xs = stage + buf * I8_TILE * I8_N;
      for (int c = 0; c < I8_TILE / I8_CHUNK; ++c, ++chunk_ctr) {
        const int ab = chunk_ctr & 1;
        const int r0 = c * I8_CHUNK + 8 * half;  // first tile row of this thread's 8
        const int64_t g0 = tile * I8_TILE + r0;
        mbar_wait(&afull[ab], (uint32_t)((chunk_ctr >> 1) & 1));
        tc_fence_after();
        if (dbg & 4) {
          tc_fence_before();
          mbar_arrive(&aempty[ab]);
          continue;
        }
        const uint32_t tbase = tmem + ((uint32_t)(32 * quad) << 16) +
                               (uint32_t)(I8_ACC0 + ab * I8_ACCBUF + 8 * half);
        uint32_t v[I8_NLEV][8];
#pragma unroll
        for (int l = 0; l < I8_NLEV; ++l) tmem_ld8(tbase + (uint32_t)(l * I8_CHUNK), v[l]);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&aempty[ab]);  // accumulators copied out: the MMA may reuse them
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          // levels 2..4 -> hi, 5..8 -> lo (exact int64); X C = 2^(e+f-94) (hi 2^64 + lo 2^32)
          const long long hi = ((long long)(int)v[0][r] << 16) + ((long long)(int)v[1][r] << 8) +
                               (long long)(int)v[2][r];
          const long long lo = ((long long)(int)v[3][r] << 24) + ((long long)(int)v[4][r] << 16) +
                               ((long long)(int)v[5][r] << 8) + (long long)(int)v[6][r];
          const int64_t g = g0 + r;
          if (g < n_rows) {
            const int e = rexp[buf * I8_TILE + r0 + r];
            const double xc = fma(i64_to_f64_exact(hi), pow2(e + fj - 30), i64_to_f64_exact(lo) * pow2(e + fj - 62));
            XA[g * I8_N + j] = (e == I8_NONFINITE) ? __longlong_as_double(0x7ff8000000000000ll)
                                                    : xs[(r0 + r) * I8_N + j] + xc;
          }
        }
      }
      mbar_arrive(&sempty[buf]);
    }
  } else if (warp == MMAW) {
    // ---- MMA issuer ---------------------------------------------------------------
    asm volatile("bar.sync 1, 288;\n" ::: "memory");
    tc_fence_after();
    const uint32_t xbase = smem_u32(xdig);
    int chunk_ctr = 0;
    for (int64_t it = 0; it < my_tiles; ++it) {
      const int buf = (int)(it & 1);
      mbar_wait(&xfull[buf], (uint32_t)((it >> 1) & 1));
      tc_fence_after();
      for (int c = 0; c < I8_TILE / I8_CHUNK; ++c, ++chunk_ctr) {
        const int ab = chunk_ctr & 1;
        if (chunk_ctr >= 2) mbar_wait(&aempty[ab], (uint32_t)(((chunk_ctr >> 1) - 1) & 1));
        tc_fence_after();
        if (!(dbg & 1)) {
          const uint32_t dacc = tmem + (uint32_t)(I8_ACC0 + ab * I8_ACCBUF);
          const uint64_t desc0 = umma_desc_sw128(xbase + (uint32_t)(buf * I8_XBUF_BYTES + c * I8_CHUNK * 128));
          // all 26 digit pairs x 4 k-steps, fully unrolled: (p, q, ks) are
          // compile-time, so each MMA is one descriptor add + UTCIMMA
#pragma unroll
          for (int p = 1; p <= I8_ND; ++p) {
#pragma unroll
            for (int q = 1; q <= I8_ND; ++q) {
              if (p + q > I8_LMAX) continue;
              const int l = p + q;
              // first pair of level l in this (p, q) order overwrites the accumulator
              const bool first = (p == 1) || (l > I8_ND + 1 && p == l - I8_ND);
              const uint32_t idesc = idesc_i8(q == 1, p == 1);  // A = C digits (q), B = X digits (p)
#pragma unroll
              for (int ks = 0; ks < 4; ++ks) {
                const uint64_t bdesc = desc0 + (uint64_t)(((p - 1) * I8_PLANE_BYTES + 32 * ks) >> 4);
                const uint32_t atm = tmem + (uint32_t)(32 * (q - 1) + 8 * ks);
                umma_i8_ts(dacc + (uint32_t)((l - 2) * I8_CHUNK), atm, bdesc, idesc, (first && ks == 0) ? 0u : 1u);
              }
            }
          }
        }
        umma_commit_elect(&afull[ab]);
        __syncwarp();
      }
      umma_commit_elect(&xempty[buf]);
      __syncwarp();
    }
  } else {
    // ---- slicer warps: rows 16w .. 16w+15 of each tile, from the smem stage ----
    for (int64_t it = 0; it < my_tiles; ++it) {
      const int buf = (int)(it & 1);
      mbar_wait(&sfull[buf], (uint32_t)((it >> 1) & 1));
      if (it >= 2) mbar_wait(&xempty[buf], (uint32_t)(((it >> 1) - 1) & 1));
      unsigned char* planes = xdig + buf * I8_XBUF_BYTES;
      const double* xs = stage + buf * I8_TILE * I8_N;
      if (!(dbg & 2)) {
#pragma unroll 4
        for (int rr = 0; rr < I8_TILE / I8_SLICE_WARPS; ++rr) {
          const int r = (I8_TILE / I8_SLICE_WARPS) * warp + rr;
          const double2 a0 = *reinterpret_cast<const double2*>(xs + r * I8_N + 4 * lane);
          const double2 a1 = *reinterpret_cast<const double2*>(xs + r * I8_N + 4 * lane + 2);
          const double xv[4] = {a0.x, a0.y, a1.x, a1.y};
          uint64_t m = 0;
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const uint64_t ab = (uint64_t)__double_as_longlong(xv[b]) & 0x7fffffffffffffffull;
            m = ab > m ? ab : m;
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const uint64_t other = __shfl_xor_sync(0xffffffffu, m, o);
            m = other > m ? other : m;
          }
          // a non-finite row cannot be split; its digits are zeroed and the
          // epilogue writes NaN for the whole row (what x T gives in fp64)
          const bool finite_row = ((m >> 52) & 0x7ff) != 0x7ff;
          const int e = finite_row ? exp_above(m) : I8_NONFINITE;
          const double scale = finite_row ? pow2(47 - e) : 0.0;
          long long v[4];
#pragma unroll
          for (int b = 0; b < 4; ++b) v[b] = round_scaled(xv[b], scale);
          // K-major, 128B-swizzled row r: 16-byte chunk (lane/4) ^ (r%8), word lane%4
          const uint32_t off = (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + (((lane >> 2) ^ (r & 7)) << 4) +
                                          ((lane & 3) << 2));
#pragma unroll
          for (int p = 0; p < I8_ND; ++p) {
            const int bi = 5 - p;
            const uint32_t word = byte_of(v[0], bi) | (byte_of(v[1], bi) << 8) | (byte_of(v[2], bi) << 16) |
                                  (byte_of(v[3], bi) << 24);
            *reinterpret_cast<uint32_t*>(planes + p * I8_PLANE_BYTES + off) = word;
          }
          if (lane == 0) rexp[buf * I8_TILE + r] = e;
        }
      }
      fence_proxy_async();
      mbar_arrive(&xfull[buf]);
      mbar_arrive(&sempty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == MMAW) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(I8_TMEM_COLS)
                 : "memory");
  }
}

}  // namespace enkf
