// gram_i8.cuh — the level-0 Gram [S'R^-1 S | S'R^-1 D] on the 5th-generation tensor
// cores (N == 128, analysis mode), by exact byte-digit products (the scheme of
// anomaly_i8.cuh, SURVEY §8 rows a9/a10 and the Gram pass of DESIGN §3).
//
//   S = X[idx] - rowmean, D = Y - X[idx], rho = 1/r (sherman.py:149-154, enkf.py:82-120)
//   Gamma = S' diag(rho) [S | D]          (the reduce applies 1/(N-1), 1/sqrt(N-1))
//
// Operands: A = S (M = 128 members), B = rho*S or rho*D (N = 64 columns per CTA),
// K = observation rows.  Every column c gets one power-of-two scale 2^(47-e_c)
// (e_c from a sampled pre-pass with a 4x headroom); the 48-bit integers are cut
// into six BALANCED byte digits (V + 0x808080808080, then byte ^ 0x80), so each
// int8 product is |.| <= 2^14 and a level (<= 7 pairs) grows by <= 2^16.8 per row:
// the int32 TMEM accumulators are exact for 16384 rows, after which the flush
// warps add the levels (fp64) into an L2-resident partial and the next period
// restarts the accumulators.  An element outside the sampled scale (heavy
// tails) raises a device flag and the FP64 DMMA Gram (gram128_kernel, gated on
// that flag) recomputes the Gram in the same stream: no host round trip.
//
// CTAs come in groups of 4 over the same observation rows (adjacent blockIdx,
// co-resident, so the row gathers of the 3 followers hit L2): CTA q of a group
// owns B columns [64q, 64q+64) of [rho S | rho D].
//
// Roles (14 warps): 0-7 slicers, 8-11 flush (TMEM lane quadrants), 12 producer
// (bulk-TMA row gathers), 13 MMA issuer.  FP64 arithmetic is kept to the
// transforms: on B200 it shares the tensor datapath (anomaly_i8.cuh).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace enkf {

constexpr int G8_N = 128;
constexpr int G8_NS = 64;        // B columns per CTA
constexpr int G8_KB = 32;        // observation rows per digit block (one MMA k-step)
constexpr int G8_SUB = 16;       // rows per TMA stage
constexpr int G8_NST = 6;        // stage ring depth
constexpr int G8_ND = 6;
constexpr int G8_LMAX = 8;
constexpr int G8_NLEV = G8_LMAX - 1;
constexpr int G8_FLUSH_BLOCKS = 512;  // 16384 rows per int32 accumulation period
constexpr int G8_SW = 8;         // slicer warps
constexpr int G8_THREADS = (G8_SW + 4 + 2) * 32;  // + 4 flush warps + producer + MMA
constexpr int G8_XLD = 130;      // stage row strides (doubles): 16-byte aligned rows
constexpr int G8_YLD = 66;
constexpr int G8_APLANE = G8_N * G8_KB;    // 4 KiB: one A digit plane (128 rows x 32 B)
constexpr int G8_BPLANE = G8_NS * G8_KB;   // 2 KiB
constexpr int G8_DIGBUF = G8_ND * (G8_APLANE + G8_BPLANE);  // 36 KiB
constexpr int G8_SPB = G8_KB / G8_SUB;  // stages per digit block (2): slicer team t owns sub-block t
constexpr int G8_STAGE = (G8_SUB * G8_XLD + G8_SUB * G8_YLD + G8_SUB) * 8;
constexpr int G8_SAMPLE = 16;    // pre-pass samples every 16th observation row
constexpr int G8_HEADROOM = 2;   // scale exponent headroom (bits) over the sampled max

__host__ __device__ inline size_t gram_i8_smem_bytes() {
  return 1024 + 2 * (size_t)G8_DIGBUF + G8_NST * (size_t)G8_STAGE + G8_NST * G8_SUB * 8 /*means*/ +
         (G8_N + G8_NS) * 8 /*scales*/ + 64 * 8 /*barriers*/;
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
// kind::i8, D = s32, both operands signed (balanced digits), K-major, M = 128, N = 64
__device__ __forceinline__ uint32_t idesc_g8() {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(G8_NS >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
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

// rho = 1/r with the r checks of _validate_system (sherman.py:100-107); padded with 0.
__global__ void rinv_kernel(const double* __restrict__ r, double* __restrict__ rinv, int64_t n_obs, int64_t n_pad,
                            DevStatus* status) {
  int flags = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n_pad; k += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    if (k < n_obs) {
      const double rv = r[k];
      if (!isfinite(rv)) flags |= FLAG_NONFINITE;
      else if (!(rv > 0.0)) flags |= FLAG_R_NONPOS;
      else v = 1.0 / rv;
    }
    rinv[k] = v;
  }
  if (flags) atomicOr(&status->flags, flags);
}

// Column maxima over every G8_SAMPLE-th observation row: |S| (128), rho|S| (128),
// rho|D| (128), as IEEE bit patterns (monotone for non-negative values).
__global__ void __launch_bounds__(256) gram_i8_scales_kernel(const double* __restrict__ X,
                                                             const double* __restrict__ Y,
                                                             const int64_t* __restrict__ idx,
                                                             const double* __restrict__ rinv, int64_t n_state,
                                                             int64_t n_obs, unsigned long long* __restrict__ cmax) {
  __shared__ unsigned long long red[3 * G8_N];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < 3 * G8_N; e += blockDim.x) red[e] = 0ull;
  __syncthreads();
  double ma[4] = {0, 0, 0, 0}, mbs[4] = {0, 0, 0, 0}, mbd[4] = {0, 0, 0, 0};
  const int64_t nsamp = (n_obs + G8_SAMPLE - 1) / G8_SAMPLE;
  for (int64_t sidx = blockIdx.x * 8 + warp; sidx < nsamp; sidx += (int64_t)gridDim.x * 8) {
    const int64_t k = sidx * G8_SAMPLE;
    const int64_t src = idx ? idx[k] : k;
    if (src < 0 || src >= n_state) continue;  // flagged by the main kernel
    const double rho = rinv[k];
    double xv[4], yv[4], s = 0.0;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      xv[m] = X[src * G8_N + lane + 32 * m];
      yv[m] = Y[k * G8_N + lane + 32 * m];
      s += xv[m];
    }
    const double mean = warp_sum(s) * (1.0 / G8_N);
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const double sv = fabs(xv[m] - mean), dv = fabs(yv[m] - xv[m]);
      ma[m] = fmax(ma[m], sv);
      mbs[m] = fmax(mbs[m], rho * sv);
      mbd[m] = fmax(mbd[m], rho * dv);
    }
  }
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int c = lane + 32 * m;
    atomicMax(&red[c], (unsigned long long)__double_as_longlong(ma[m]));
    atomicMax(&red[G8_N + c], (unsigned long long)__double_as_longlong(mbs[m]));
    atomicMax(&red[2 * G8_N + c], (unsigned long long)__double_as_longlong(mbd[m]));
  }
  __syncthreads();
  for (int e = tid; e < 3 * G8_N; e += blockDim.x)
    if (red[e]) atomicMax(&cmax[e], red[e]);
}

// Profiling-only trace (CTA 0, -DG8_TRACE_ON): [stage][event] %globaltimer:
// 0 producer issued, 1 slicer saw data, 2 means done, 3 digits stored; [block][8+]: 8 MMA start, 9 MMA issued
constexpr int G8_TRACE_N = 512;
__device__ unsigned long long g_g8_trace[G8_TRACE_N][12];
#ifdef G8_TRACE_ON
#define G8_TRACE(i, ev) \
  do { if (blockIdx.x == 0 && (i) < G8_TRACE_N) g_g8_trace[(i)][(ev)] = gtime(); } while (0)
#else
#define G8_TRACE(i, ev) do { } while (0)
#endif

__global__ void __launch_bounds__(G8_THREADS, 1)
gram_i8_kernel(const double* __restrict__ X, const double* __restrict__ Y, const int64_t* __restrict__ idx,
               const double* __restrict__ rinv, const unsigned long long* __restrict__ cmax, int64_t n_state,
               int64_t n_obs, int64_t rows_per_group, double* __restrict__ partial, int* __restrict__ overflow,
               DevStatus* __restrict__ status, uint32_t uz /* = 0 */) {
  extern __shared__ __align__(1024) unsigned char g8sm_raw[];
  unsigned char* sm = g8sm_raw + ((1024u - (smem_u32(g8sm_raw) & 1023u)) & 1023u);
  unsigned char* dig = sm;                                         // [2][A 6x128x64 | B 6x64x64]
  unsigned char* stg = dig + 2 * G8_DIGBUF;                        // [NST][x | y | rho]
  double* means = reinterpret_cast<double*>(stg + G8_NST * G8_STAGE);  // [NST][16]
  double* ascale = means + G8_NST * G8_SUB;                         // [128] 2^(47-e_i)
  double* bscale = ascale + G8_N;                                   // [64]
  uint64_t* bars = reinterpret_cast<uint64_t*>(bscale + G8_NS);
  uint64_t* sfull = bars;                 // [NST] producer -> slicers (tx)
  uint64_t* sempty = bars + G8_NST;       // [NST] slicers -> producer
  uint64_t* dfull = bars + 2 * G8_NST;    // [2] slicers -> MMA
  uint64_t* dempty = dfull + 2;           // [2] MMA commit -> slicers
  uint64_t* afull = dempty + 2;           // [1] MMA commit -> flush
  uint64_t* aempty = afull + 1;           // [1] flush -> MMA
  uint32_t* vmask = reinterpret_cast<uint32_t*>(aempty + 1);  // [NST] valid rows of a stage
  uint32_t* tmem_slot = vmask + 4;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = blockIdx.x & 3;  // B column quarter: 0,1 -> rho S, 2,3 -> rho D
  const int64_t grp = blockIdx.x >> 2;
  const int64_t row0 = grp * rows_per_group;
  const int64_t row1 = row0 + rows_per_group < n_obs ? row0 + rows_per_group : n_obs;
  const int64_t nrows = row1 > row0 ? row1 - row0 : 0;
  const int64_t nblk = (nrows + G8_KB - 1) / G8_KB;
  const int64_t nstage = nblk * G8_SPB;  // whole blocks: rows past the end are zero digits
  const bool dslice = q >= 2;

  if (tid == 0) {
    for (int i = 0; i < G8_NST; ++i) {
      mbar_init(&sfull[i], 1);
      mbar_init(&sempty[i], 32 * G8_SW / G8_SPB);  // one slicer team per stage
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&dfull[i], 32 * G8_SW);
      mbar_init(&dempty[i], 1);
    }
    mbar_init(afull, 1);
    mbar_init(aempty, 128);  // the 4 flush warps
    fence_mbar_init();
  }
  // column scales from the sampled maxima (G8_HEADROOM bits above them)
  for (int c = tid; c < G8_N + G8_NS; c += G8_THREADS) {
    const unsigned long long b = c < G8_N ? cmax[c] : cmax[G8_N * (dslice ? 2 : 1) + 64 * (q & 1) + (c - G8_N)];
    const int e = exp_above(b) + G8_HEADROOM;
    const double sc = pow2(47 - e);
    if (c < G8_N) ascale[c] = sc; else bscale[c - G8_N] = sc;
  }
  constexpr int FLW = G8_SW, PRODW = G8_SW + 4, MMAW = G8_SW + 5;
  if (warp == MMAW) {
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

  if (warp == PRODW) {
    // ---- producer: bulk-TMA gathers of 16 observation rows per stage ------------
    // idx of the next stage is read one stage ahead, so its global-load latency
    // overlaps the wait for a free slot.
    int flags = 0;
    auto fetch = [&](int64_t st, bool& valid, int64_t& src) {
      const int64_t g = row0 + st * G8_SUB + lane;
      valid = lane < G8_SUB && g < row1;
      src = g;
      if (valid && idx) {
        src = idx[g];
        const int64_t prev = g > 0 ? idx[g - 1] : -1;
        if (prev >= src) flags |= FLAG_IDX_ORDER;
        if (src < 0 || src >= n_state) { flags |= FLAG_IDX_RANGE; valid = false; }
      }
    };
    bool nvalid;
    int64_t nsrc;
    fetch(0, nvalid, nsrc);
    for (int64_t st = 0; st < nstage; ++st) {
      const int slot = (int)(st % G8_NST);
      const bool valid = nvalid;
      const int64_t src = nsrc, g = row0 + st * G8_SUB + lane;
      if (st + 1 < nstage) fetch(st + 1, nvalid, nsrc);
      if (st >= G8_NST) mbar_wait(&sempty[slot], (uint32_t)(((st / G8_NST) - 1) & 1));
      const unsigned vm = __ballot_sync(0xffffffffu, valid);
      unsigned char* base = stg + slot * G8_STAGE;
      double* xs = reinterpret_cast<double*>(base);
      double* ys = xs + G8_SUB * G8_XLD;
      double* rs = ys + G8_SUB * G8_YLD;
      if (vm != 0xffffu) {  // rows past the end (or with a bad index) become zero rows
        for (int rr = 0; rr < G8_SUB; ++rr) {
          if ((vm >> rr) & 1u) continue;
          for (int c = lane; c < G8_XLD; c += 32) xs[rr * G8_XLD + c] = 0.0;
          for (int c = lane; c < G8_YLD; c += 32) ys[rr * G8_YLD + c] = 0.0;
        }
        __syncwarp();
      }
      fence_proxy_async();
      if (lane == 0) {
        vmask[slot] = vm;
        const uint32_t bytes = (uint32_t)__popc(vm) * (1024u + (dslice ? 512u : 0u)) + 128u;
        mbar_arrive_expect_tx(&sfull[slot], bytes);
        bulk_g2s(rs, rinv + (row0 + st * G8_SUB), 128u, &sfull[slot]);
        G8_TRACE(st, 0);
      }
      __syncwarp();
      if (valid) {
        bulk_g2s(xs + lane * G8_XLD, X + src * G8_N, 1024u, &sfull[slot]);
        if (dslice) bulk_g2s(ys + lane * G8_YLD, Y + g * G8_N + 64 * (q - 2), 512u, &sfull[slot]);
      }
    }
    flags = __reduce_or_sync(0xffffffffu, flags);
    if (lane == 0 && flags) atomicOr(&status->flags, flags);
  } else if (warp < G8_SW) {
    // ---- slicers ---------------------------------------------------------------------
    int ovf = 0;
    const int mi = lane & 7, w = lane >> 3;  // transposed phase: column mi of a group of 8, row quad w
    constexpr int TW = G8_SW / G8_SPB;       // warps per team
    const int team = warp / TW, tw = warp % TW;
    // team t takes stages t, t+2, ...: sub-block t of every digit block, so the two
    // teams slice two stages at once
    for (int64_t st = team; st < nstage; st += G8_SPB) {
      const int slot = (int)(st % G8_NST);
      const int64_t blk = st / G8_SPB;
      const int sb = (int)(st % G8_SPB);
      const int dbuf = (int)(blk & 1);
      mbar_wait(&sfull[slot], (uint32_t)((st / G8_NST) & 1));
      if (blk >= 2) mbar_wait(&dempty[dbuf], (uint32_t)(((blk >> 1) - 1) & 1));
      if (warp == 0 && lane == 0) G8_TRACE(st, 1);
      const double* xs = reinterpret_cast<const double*>(stg + slot * G8_STAGE);
      const double* ys = xs + G8_SUB * G8_XLD;
      const double* rs = ys + G8_SUB * G8_YLD;
      double* mn = means + slot * G8_SUB;
      // row means (invalid rows were zero-filled by the producer): 4 rows per warp
#pragma unroll
      for (int u = 0; u < G8_SUB / TW; ++u) {
        const int row = (G8_SUB / TW) * tw + u;
        double s = 0.0;
#pragma unroll
        for (int m = 0; m < 4; ++m) s += xs[row * G8_XLD + lane + 32 * m];
        s = warp_sum(s);
        if (lane == 0) mn[row] = s * (1.0 / G8_N);
      }
      asm volatile("bar.sync %0, %1;\n" ::"r"(2 + team), "n"(32 * TW) : "memory");
      if (warp == 0 && lane == 0) G8_TRACE(st, 2);
      unsigned char* da = dig + dbuf * G8_DIGBUF;
      unsigned char* db = da + G8_ND * G8_APLANE;
      double mr[4], rr4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        mr[u] = mn[4 * w + u];
        rr4[u] = rs[4 * w + u];
      }
      // 24 groups of 8 columns (16 of A, 8 of B), 6 per warp of the team, 3 in flight
#pragma unroll 2
      for (int gi = 0; gi < 24 / TW; ++gi) {
        const int cgi = tw + TW * gi;
        const bool isA = cgi < 16;
        const int col = isA ? 8 * cgi + mi : 8 * (cgi - 16) + mi;  // A member i, or B column j (0..63)
        const double sc = isA ? ascale[col] : bscale[col];
        uint32_t vlo[4], vhi[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int row = 4 * w + u;
          double v;
          if (isA) {
            v = xs[row * G8_XLD + col] - mr[u];
          } else if (!dslice) {
            v = rr4[u] * (xs[row * G8_XLD + 64 * q + col] - mr[u]);
          } else {
            v = rr4[u] * (ys[row * G8_YLD + col] - xs[row * G8_XLD + 64 * (q - 2) + col]);
          }
          // V = round(v 2^(47-e)): fma(v, sc, 1.5 2^52) holds V in its low 51 bits; the
          // high word minus 0x43380000 is floor(V / 2^32), in [-2^15, 2^15) iff |V| < 2^47
          // (out of range, non-finite included -> overflow flag -> FP64 fallback, which
          // also reports non-finite inputs)
          const double t = fma(v, sc, 6755399441055744.0);
          const int hs = __double2hiint(t) - 0x43380000;
          ovf |= (uint32_t)(hs + 0x8000) >= 0x10000u;
          // balanced digits: bytes of V + 0x808080808080, each ^ 0x80
          const unsigned long long vb =
              ((unsigned long long)(uint32_t)hs << 32 | (uint32_t)__double2loint(t)) + 0x808080808080ull;
          vlo[u] = (uint32_t)vb;
          vhi[u] = (uint32_t)(vb >> 32);
        }
        // plane p (1..6) = byte (6-p) of the 48-bit value, 4 rows per word
        auto two_planes = [&](uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3, uint32_t bi, uint32_t bj,
                              uint32_t& wi, uint32_t& wj) {
          const uint32_t sel = bi | ((bi + 4u) << 4) | (bj << 8) | ((bj + 4u) << 12);
          const uint32_t A = __byte_perm(x0, x1, sel);
          const uint32_t B = __byte_perm(x2, x3, sel);
          wi = __byte_perm(A, B, 0x5410) ^ 0x80808080u;
          wj = __byte_perm(A, B, 0x7632) ^ 0x80808080u;
        };
        uint32_t wd[G8_ND];
        two_planes(vhi[0], vhi[1], vhi[2], vhi[3], 1u, 0u, wd[0], wd[1]);
        two_planes(vlo[0], vlo[1], vlo[2], vlo[3], 3u, 2u, wd[2], wd[3]);
        two_planes(vlo[0], vlo[1], vlo[2], vlo[3], 1u, 0u, wd[4], wd[5]);
        // K-major SWIZZLE_32B: row = col (32 B), 16-byte chunk sb ^ ((col >> 2) & 1), word w
        const uint32_t off = (uint32_t)(col * 32 + ((sb ^ ((col >> 2) & 1)) << 4) + 4 * w);
        unsigned char* pb = isA ? da : db;
        const int pstride = isA ? G8_APLANE : G8_BPLANE;
#pragma unroll
        for (int p = 0; p < G8_ND; ++p) *reinterpret_cast<uint32_t*>(pb + p * pstride + off) = wd[p];
      }
      fence_proxy_async();
      if (warp == 0 && lane == 0) G8_TRACE(st, 3);
      mbar_arrive(&sempty[slot]);
      mbar_arrive(&dfull[dbuf]);  // both teams (one sub-block each) complete a block
    }
    ovf = __reduce_or_sync(0xffffffffu, ovf);
    if (lane == 0 && ovf) atomicOr(overflow, 1);
  } else if (warp == MMAW) {
    // ---- MMA issuer ------------------------------------------------------------------
    const uint32_t dbase = smem_u32(dig);
    const uint32_t idesc = uz + idesc_g8();
    for (int64_t blk = 0; blk < nblk; ++blk) {
      const int dbuf = (int)(blk & 1);
      const int64_t period = blk / G8_FLUSH_BLOCKS;
      const bool first_in_period = (blk % G8_FLUSH_BLOCKS) == 0;
      if (first_in_period && period > 0) mbar_wait(aempty, (uint32_t)((period - 1) & 1));
      mbar_wait(&dfull[dbuf], (uint32_t)((blk >> 1) & 1));
      tc_fence_after();
      if (lane == 0) G8_TRACE(blk, 8);
      const uint32_t abuf = dbase + (uint32_t)(dbuf * G8_DIGBUF);
      const uint32_t bbuf = abuf + (uint32_t)(G8_ND * G8_APLANE);
#pragma unroll
      for (int p = 1; p <= G8_ND; ++p) {
#pragma unroll
        for (int qq = 1; qq <= G8_ND; ++qq) {
          if (p + qq > G8_LMAX) continue;
          const int l = p + qq;
          const bool first = first_in_period && ((p == 1) || (l > G8_ND + 1 && p == l - G8_ND));
          const uint64_t ad = umma_desc_sw32(abuf + (uint32_t)((p - 1) * G8_APLANE));
          const uint64_t bd = umma_desc_sw32(bbuf + (uint32_t)((qq - 1) * G8_BPLANE));
#ifndef G8_SKIP_MMA
          umma_i8_ss(uz + tmem + (uint32_t)((l - 2) * G8_NS), ad, bd, idesc, first ? 0u : 1u);
#endif
        }
      }
      umma_commit_elect(&dempty[dbuf]);
      if (lane == 0) G8_TRACE(blk, 9);
      if ((blk % G8_FLUSH_BLOCKS) == G8_FLUSH_BLOCKS - 1 || blk == nblk - 1) umma_commit_elect(afull);
      __syncwarp();
    }
  } else if (warp >= FLW && warp < FLW + 4) {
    // ---- flush: thread = member i = TMEM lane; fold the 7 levels into the fp64 partial
    const int quad = warp & 3;
    const int i = 32 * quad + lane;
    const int64_t nper = (nblk + G8_FLUSH_BLOCKS - 1) / G8_FLUSH_BLOCKS;
    double* prow = partial + ((size_t)blockIdx.x * G8_N + i) * G8_NS;
    // Gamma_ij = 2^(e_i + f_j - 94) sum_l 256^(12-l) D_l = (hi 2^32 + lo) 2^(e_i+f_j-62),
    // and 2^(47-e) = sc  ->  2^(e_i+f_j-62) = 2^32 / (sc_i sc_j)
    const double ai = 4294967296.0 / ascale[i];
    for (int64_t pd = 0; pd < nper; ++pd) {
      mbar_wait(afull, (uint32_t)(pd & 1));
      tc_fence_after();
#pragma unroll 1
      for (int cg = 0; cg < G8_NS / 8; ++cg) {
        uint32_t v[G8_NLEV][8];
#pragma unroll
        for (int l = 0; l < G8_NLEV; ++l)
          tmem_ld8(tmem + ((uint32_t)(32 * quad) << 16) + (uint32_t)(l * G8_NS + 8 * cg), v[l]);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const double hi = fma((double)(int)v[0][c], 65536.0, fma((double)(int)v[1][c], 256.0, (double)(int)v[2][c]));
          const double lo = fma((double)(int)v[3][c], 16777216.0,
                                fma((double)(int)v[4][c], 65536.0, fma((double)(int)v[5][c], 256.0, (double)(int)v[6][c])));
          const int j = 8 * cg + c;
          const double val = fma(hi, 4294967296.0, lo) * (ai / bscale[j]);
          prow[j] = (pd == 0 ? 0.0 : prow[j]) + val;
        }
      }
      tc_fence_before();
      mbar_arrive(aempty);
    }
    if (nper == 0)
      for (int j = 0; j < G8_NS; ++j) prow[j] = 0.0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == MMAW) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512u) : "memory");
  }
}

// Gram from the per-CTA partials [group][quarter][128][64]: fixed-order sum over
// groups; the V'V block from its upper triangle (exactly symmetric); scales
// s_vv = 1/(N-1), s_vd = 1/sqrt(N-1).  Skipped when the FP64 fallback ran.
__global__ void gram_i8_reduce(const double* __restrict__ partial, int ngroups, double s_vv, double s_vd,
                               const int* __restrict__ overflow, double* __restrict__ gram) {
  if (*overflow) return;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= G8_N * 2 * G8_N) return;
  const int i = e / (2 * G8_N), c = e % (2 * G8_N);
  int qq, a, b;
  if (c < G8_N) {
    a = i <= c ? i : c;
    b = i <= c ? c : i;
    qq = b >> 6;
  } else {
    a = i;
    b = c - G8_N;
    qq = 2 + (b >> 6);
  }
  const double* src = partial + ((size_t)qq * G8_N + a) * G8_NS + (b & 63);
  double s = 0.0;
  for (int g = 0; g < ngroups; ++g) s += src[(size_t)g * 4 * G8_N * G8_NS];
  gram[e] = s * (c < G8_N ? s_vv : s_vd);
}

}  // namespace enkf
