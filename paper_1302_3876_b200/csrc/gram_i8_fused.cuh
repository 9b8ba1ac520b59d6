// gram_i8_fused.cuh — the int8 tensor-core Gram (gram_i8.cuh) as ONE persistent
// kernel: slicing and the level-split MMAs overlap on the same SMs and the byte-digit
// operand images never reach DRAM (the two-kernel form writes every 32-row block's
// 48 KiB image to HBM and reads it back: 26 GB of the Gram's 44 GB of DRAM traffic at
// config 5, against 17.3 GB compulsory).
//
// Groups of 4 CTAs (one per SM, cooperative launch: all co-resident) own a range of
// 32-row observation blocks.  CTA q of a group:
//  * slices the blocks t = q (mod 4) of its group into a per-group ring of GFL_RING
//    images in global memory, small enough to stay in L2 (37 x 32 x 48 KiB = 57 MiB),
//    written directly in the level-split layout [P_1 Q_1 P_2 Q_2 ... P_6 Q_6];
//  * consumes EVERY image of the group through one 48 KiB bulk TMA copy per block and
//    issues the N = 256 kind::i8 MMAs of its level set (G8LS_SETS, as
//    gram_i8_mma_ls_kernel: A = P_p and B = [P_q ; Q_q] straight from shared memory),
//    accumulating two levels x 256 columns in TMEM; 4 flush warps fold them into the
//    fp64 partial every G8_FLUSH_BLOCKS blocks.
// Cross-CTA hand-off through the ring (acquire/release flags in global memory):
//   slicer  : wait consumed[slot] >= 4 * (t / RING) (previous occupant read by all 4),
//             write the image; team barrier; leader: fence + release ready[slot] = t + 1
//   consumer: acquire ready[slot] >= k + 1; fence.proxy.async; bulk copy into a stage;
//             the MMA issuer, once the copy has landed: consumed[slot] += 1 (release)
// Every spin is bounded (a deadlock traps instead of hanging the GPU).
//
// Slicing (2 teams of 4 warps, thread = member mm of P and Q): per 16-row half-block
// the loader warp bulk-copies the X[idx] rows into a staging ring and checks the
// indices; the team forms the row means and sqrt(1/r), then per row
//   P: fma(sqrt(rho) (x - mean), 2^s_p, 1.5 2^52 + bias)
//   Q: fma(sqrt(rho) (y - x),    2^s_q, 1.5 2^52 + bias)
// whose low 51 bits hold V + 0x808080808080 (balanced digits, as gram_i8_slice_kernel);
// 16 rows of one member give its 16-byte K-chunk of all 12 planes.  The level-split
// MMA issuer needs one instruction per 128 tensor cycles, so it keeps its issue slots
// next to the slicers (the earlier column-split fused form, 26 MMAs per block, did not).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "gram_i8.cuh"

namespace enkf {

#ifndef GFL_RING_DEF
#define GFL_RING_DEF 32
#endif
constexpr int GFL_RING = GFL_RING_DEF;  // images per group ring (37 x 32 x 48 KiB = 57 MiB of L2)
#ifndef GFL_NST_DEF
#define GFL_NST_DEF 3
#endif
#ifndef GFL_TEAMS_DEF
#define GFL_TEAMS_DEF 2
#endif
constexpr int GFL_NST = GFL_NST_DEF;  // MMA smem stages (48 KiB each)
constexpr int GFL_HB = 16;        // rows per slicer half-block
constexpr int GFL_TEAMS = GFL_TEAMS_DEF;  // slicer teams of 4 warps; a team slices whole blocks
constexpr int GFL_NHB = 2 * GFL_TEAMS;  // staging depth (half-blocks the loader runs ahead)
constexpr int GFL_XST = GFL_HB * G8_N * 8;       // 16 KiB: X rows of a half-block
constexpr int GFL_STG = GFL_XST + GFL_HB * 8;    // + r of its rows
constexpr int GFL_SLW = 4 * GFL_TEAMS;           // slicer warps 0..7
constexpr int GFL_LDW = GFL_SLW, GFL_MPW = GFL_SLW + 1, GFL_MMAW = GFL_SLW + 2, GFL_FLW0 = GFL_SLW + 3;
constexpr int GFL_THREADS = (GFL_SLW + 7) * 32;  // + loader, producer, issuer, 4 flush
constexpr long long GFL_SPIN_LIMIT = 1ll << 26;  // seconds of polling: a deadlock traps instead of hanging

__host__ __device__ inline size_t gram_i8_fused_smem_bytes() {
  return 1024 + (size_t)GFL_NST * G8LS_STAGE + GFL_NHB * (size_t)GFL_STG + 2 * G8_N * 8 /*scales*/ +
         GFL_NHB * GFL_HB * 8 * 2 /*mean, sr*/ + GFL_NHB * GFL_HB * 4 /*valid*/ + 64 * 8 /*barriers*/;
}

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_release_gpu(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// poll until *p >= target (bounded; trap on a deadlock).  Relaxed polls (an acquire
// load invalidates the whole L1 on every try: CCTL.IVALL), then one acquire fence.
__device__ __forceinline__ void gfl_wait_geq(const int* p, int target) {
  long long spins = 0;
  while (ld_relaxed_gpu(p) < target) {
    __nanosleep(32);
    if (++spins > GFL_SPIN_LIMIT) __trap();
  }
  asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
}

// profiling only (-DGFL_TRACE_ON): %globaltimer stamps of the roles of group 0
// (CTAs 0-3) for its first GFL_TRACE_BLOCKS blocks, read by enkf_debug_gfl_trace
constexpr int GFL_TRACE_BLOCKS = 512;
__device__ unsigned long long g_gfl_trace[4][GFL_TRACE_BLOCKS][6];
#ifdef GFL_TRACE_ON
#define GFL_TRACE(k, ev)                                                                   \
  do {                                                                                     \
    if (blockIdx.x < 4 && (k) < GFL_TRACE_BLOCKS) {                                        \
      unsigned long long _t;                                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                               \
      g_gfl_trace[blockIdx.x][(k)][(ev)] = _t;                                             \
    }                                                                                      \
  } while (0)
#else
#define GFL_TRACE(k, ev) do { } while (0)
#endif

__global__ void __launch_bounds__(GFL_THREADS, 1)
gram_i8_fused_kernel(const double* __restrict__ X, const double* __restrict__ Y, const int64_t* __restrict__ idx,
                     const double* __restrict__ r, const unsigned long long* __restrict__ cmax, int64_t n_state,
                     int64_t n_obs, int64_t n_blocks, int64_t blocks_per_group, unsigned char* __restrict__ ring,
                     int* __restrict__ ready, int* __restrict__ consumed, double* __restrict__ partial,
                     int* __restrict__ overflow, DevStatus* __restrict__ status) {
  extern __shared__ __align__(1024) unsigned char gfsm_raw[];
  unsigned char* sm = gfsm_raw + ((1024u - (smem_u32(gfsm_raw) & 1023u)) & 1023u);
  unsigned char* stages = sm;                                             // [NST][48 KiB]
  double* stg = reinterpret_cast<double*>(stages + GFL_NST * G8LS_STAGE);  // [NHB][X 16x128 | r 16]
  double* scl = stg + GFL_NHB * (GFL_STG / 8);                            // [256]
  double* rmean = scl + 2 * G8_N;                                         // [NHB][16]
  double* rsr = rmean + GFL_NHB * GFL_HB;                                 // [NHB][16]
  int* rvalid = reinterpret_cast<int*>(rsr + GFL_NHB * GFL_HB);           // [NHB][16]
  uint64_t* bars = reinterpret_cast<uint64_t*>(rvalid + GFL_NHB * GFL_HB);
  uint64_t* sfull = bars;                   // [NST] producer -> issuer (tx)
  uint64_t* sempty = bars + GFL_NST;        // [NST] issuer commit -> producer
  uint64_t* afull = bars + 2 * GFL_NST;     // issuer commit -> flush
  uint64_t* aempty = afull + 1;             // flush -> issuer
  uint64_t* hfull = aempty + 1;             // [NHB] loader -> slicers (tx)
  uint64_t* hempty = hfull + GFL_NHB;       // [NHB] slicers -> loader
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hempty + GFL_NHB);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = blockIdx.x & 3;
  const int64_t grp = blockIdx.x >> 2;
  const int64_t b0 = grp * blocks_per_group;
  const int64_t b1 = b0 + blocks_per_group < n_blocks ? b0 + blocks_per_group : n_blocks;
  const int64_t nblk = b1 > b0 ? b1 - b0 : 0;
  unsigned char* gring = ring + (size_t)grp * GFL_RING * G8LS_STAGE;
  int* gready = ready + grp * GFL_RING;
  int* gcons = consumed + grp * GFL_RING;
  const int lv0 = g8ls_level(q, 0), lv1 = g8ls_level(q, 1);

  if (tid == 0) {
    for (int i = 0; i < GFL_NST; ++i) {
      mbar_init(&sfull[i], 1);
      mbar_init(&sempty[i], 1);
    }
    mbar_init(afull, 1);
    mbar_init(aempty, 128);
    for (int i = 0; i < GFL_NHB; ++i) {
      mbar_init(&hfull[i], 1);
      mbar_init(&hempty[i], 128);  // one team
    }
    fence_mbar_init();
  }
  for (int c = tid; c < 2 * G8_N; c += GFL_THREADS) scl[c] = g8_scale(cmax[c]);
  if (warp == GFL_MMAW) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(512u)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  constexpr uint32_t tmem = 0;  // one CTA per SM owns all 512 columns
  if (tid == 0 && *tmem_slot != 0u) __trap();

  // this CTA slices blocks t = q, q + 4, ... of its group (team k: every GFL_TEAMS-th
  // of them), as two 16-row halves each
  const int64_t my_blocks = nblk > q ? (nblk - 1 - q) / 4 + 1 : 0;
  const int64_t my_halves = 2 * my_blocks;

  if (warp == GFL_LDW) {
    // ---- loader: X[idx] rows (one bulk copy per row) and r of each half-block, in the
    // order the teams consume them (half hh = 2 j + h of the CTA's j-th block)
    int flags = 0;
    auto fetch = [&](int64_t hh, int64_t& src, int64_t& prev, double& rv) {
      const int64_t t = q + 4 * (hh >> 1);
      const int64_t g = (b0 + t) * G8_KB + GFL_HB * (hh & 1) + lane;
      src = -1;
      prev = -1;
      rv = 1.0;
      if (hh < my_halves && lane < GFL_HB && g < n_obs) {
        rv = r[g];
        src = g;
        if (idx) {
          src = idx[g];
          if (g > 0) prev = idx[g - 1];
        }
      }
    };
    int64_t nsrc, nprev;
    double nrv;
    fetch(0, nsrc, nprev, nrv);
    for (int64_t hh = 0; hh < my_halves; ++hh) {
      const int buf = (int)(hh % GFL_NHB);
      const int64_t t = q + 4 * (hh >> 1);
      const int64_t g = (b0 + t) * G8_KB + GFL_HB * (hh & 1) + lane;
      int64_t src = nsrc;
      const int64_t prev = nprev;
      const double rv = nrv;
      fetch(hh + 1, nsrc, nprev, nrv);
      bool valid = lane < GFL_HB && g < n_obs;
      if (valid && idx) {
        if (g > 0 && prev >= src) flags |= FLAG_IDX_ORDER;
        if (src < 0 || src >= n_state) {
          flags |= FLAG_IDX_RANGE;
          valid = false;
        }
      }
      if (hh >= GFL_NHB) mbar_wait(&hempty[buf], (uint32_t)(((hh / GFL_NHB) - 1) & 1));
      double* xs = stg + buf * (GFL_STG / 8);
      double* rs = xs + GFL_XST / 8;
      if (lane < GFL_HB) {
        rvalid[buf * GFL_HB + lane] = valid ? 1 : 0;
        rs[lane] = rv;
      }
      const unsigned vmask = __ballot_sync(0xffffffffu, valid);
      const int nx = __popc(vmask);
      if (nx < GFL_HB) {  // rows with no data (past the end, bad index) become exact zeros
        for (int rr = 0; rr < GFL_HB; ++rr)
          if (!((vmask >> rr) & 1u))
            for (int c = lane; c < G8_N; c += 32) xs[rr * G8_N + c] = 0.0;
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&hfull[buf], (uint32_t)nx * 1024u);
      __syncwarp();
      if (valid) bulk_g2s(xs + lane * G8_N, X + src * G8_N, 1024u, &hfull[buf]);
    }
    flags = __reduce_or_sync(0xffffffffu, flags);
    if (lane == 0 && flags) atomicOr(&status->flags, flags);
  } else if (warp < GFL_SLW) {
    // ---- slicers: team k takes the CTA's blocks j = k (mod GFL_TEAMS), both halves
    const int team = warp >> 2, mm = tid & 127, tw = warp & 3;
    const double scp = scl[mm], scq = scl[G8_N + mm];
    int flags = 0, ovf = 0;
    // 1.5 2^52 + bias: fma(v, sc, kMagicB) holds V + 0x808080808080 in its low 51 bits
    const double kMagicB = 6755399441055744.0 + (double)0x808080808080ull;
    auto two_planes = [](const uint32_t (&x)[4], uint32_t bi, uint32_t bj, uint32_t& wi, uint32_t& wj) {
      const uint32_t sel = bi | ((bi + 4u) << 4) | (bj << 8) | ((bj + 4u) << 12);
      const uint32_t A = __byte_perm(x[0], x[1], sel);
      const uint32_t B = __byte_perm(x[2], x[3], sel);
      wi = __byte_perm(A, B, 0x5410) ^ 0x80808080u;
      wj = __byte_perm(A, B, 0x7632) ^ 0x80808080u;
    };
    // the team's halves in order: i -> block j = team + GFL_TEAMS (i >> 1), half i & 1
    const int64_t my_team_blocks = my_blocks > team ? (my_blocks - 1 - team) / GFL_TEAMS + 1 : 0;
    const int64_t nhalf = 2 * my_team_blocks;
    auto half_row0 = [&](int64_t i) { return (b0 + q + 4 * (team + GFL_TEAMS * (i >> 1))) * G8_KB + GFL_HB * (i & 1); };
    // Y of a half straight from global memory into registers, one half ahead: the
    // next half's loads are issued as soon as this half's Q digits are formed, so
    // their latency overlaps the P digits, the staging wait and the row means
    double yv[GFL_HB];
    if (nhalf > 0) {
      const int64_t g0 = half_row0(0);
#pragma unroll
      for (int k = 0; k < GFL_HB; ++k) yv[k] = (g0 + k < n_obs) ? __ldcs(Y + (g0 + k) * G8_N + mm) : 0.0;
    }
    for (int64_t i = 0; i < nhalf; ++i) {
      const int64_t j = team + GFL_TEAMS * (i >> 1);
      const int h = (int)(i & 1);
      const int64_t t = q + 4 * j;
      const int slot = (int)(t % GFL_RING);
      unsigned char* img = gring + (size_t)slot * G8LS_STAGE;
      if (h == 0) {
        if (mm == 0) GFL_TRACE(j, 0);
        if (t >= GFL_RING) {  // the slot's previous image must be consumed by all 4 CTAs
          if (mm == 0) gfl_wait_geq(gcons + slot, 4 * (int)(t / GFL_RING));
          asm volatile("bar.sync %0, 128;\n" ::"r"(2 + team) : "memory");
        }
        if (mm == 0) GFL_TRACE(j, 1);
      }
      const int64_t hh = 2 * j + h;  // the loader's half index
      const int buf = (int)(hh % GFL_NHB);
      mbar_wait(&hfull[buf], (uint32_t)((hh / GFL_NHB) & 1));
      const double* xs = stg + buf * (GFL_STG / 8);
      const double* rs = xs + GFL_XST / 8;
      // step A: row means (warp tw: rows 4tw..4tw+3), sqrt(1/r) (warp 0, lane = row)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int row = 4 * tw + u;
        double sx = (xs[row * G8_N + lane] + xs[row * G8_N + lane + 32]) +
                    (xs[row * G8_N + lane + 64] + xs[row * G8_N + lane + 96]);
        sx = warp_sum(sx);
        if (lane == 0) rmean[buf * GFL_HB + row] = sx * (1.0 / G8_N);
      }
      if (tw == 0 && lane < GFL_HB) {
        double srv = 0.0;  // invalid rows (bad index, past the end) contribute exact zeros
        if (rvalid[buf * GFL_HB + lane] != 0) {
          const double rv = rs[lane];
          if (!isfinite(rv)) flags |= FLAG_NONFINITE;
          else if (!(rv > 0.0)) flags |= FLAG_R_NONPOS;
          srv = g8_sqrt_rho(rv);
        }
        rsr[buf * GFL_HB + lane] = srv;
      }
      asm volatile("bar.sync %0, 128;\n" ::"r"(2 + team) : "memory");
      // step B: 16 rows -> the 16-byte chunk h of member mm's row in all 12 planes,
      // Q first (it frees yv for the next half's loads), then P
      // (x is re-read from the staging buffer in each pass rather than held in 16
      // registers: the slicers live at the 128-register cap of this 15-warp CTA)
      const size_t off = (size_t)mm * 32 + (size_t)((h ^ ((mm >> 2) & 1)) << 4);
#pragma unroll
      for (int pq = 1; pq >= 0; --pq) {
        uint32_t w[G8_ND][4];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          uint32_t vlo[4], vhi[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int row = 4 * q4 + u;
            // the slice pass's exact arithmetic (gram_i8_slice_kernel): the two Gram
            // forms agree bit for bit
            const double sr = rsr[buf * GFL_HB + row];
            const double xv = xs[row * G8_N + mm];
            const double d = pq == 0 ? xv - rmean[buf * GFL_HB + row] : yv[row] - xv;
#ifdef GFL_NO_FP64  // timing experiment only (wrong digits): the slicers without FP64 arithmetic
            const double tv = __hiloint2double(0x43380000 + (__double2hiint(xv) & 0xff),
                                               __double2loint(xv) ^ __double2loint(yv[row]) ^ row);
            (void)sr; (void)d;
#else
            const double tv = fma(sr * d, pq == 0 ? scp : scq, kMagicB);
#endif
            const uint32_t hv = (uint32_t)__double2hiint(tv) - 0x43380000u;
            ovf |= hv >= 0x10000u;  // V + bias outside [0, 2^48): |V| too large, or non-finite
            vlo[u] = (uint32_t)__double2loint(tv);
            vhi[u] = hv;
          }
          two_planes(vhi, 1u, 0u, w[0][q4], w[1][q4]);
          two_planes(vlo, 3u, 2u, w[2][q4], w[3][q4]);
          two_planes(vlo, 1u, 0u, w[4][q4], w[5][q4]);
        }
        // level-split layout: plane p of P at 2p, of Q at 2p + 1 (x 4 KiB)
        unsigned char* base = img + (size_t)pq * G8_PLANE + off;
#pragma unroll
        for (int p = 0; p < G8_ND; ++p)
          *reinterpret_cast<uint4*>(base + (size_t)(2 * p) * G8_PLANE) = make_uint4(w[p][0], w[p][1], w[p][2], w[p][3]);
        if (pq == 1 && i + 1 < nhalf) {  // prefetch the next half's Y
          const int64_t g1 = half_row0(i + 1);
#pragma unroll
          for (int k = 0; k < GFL_HB; ++k) yv[k] = (g1 + k < n_obs) ? __ldcs(Y + (g1 + k) * G8_N + mm) : 0.0;
        }
      }
      mbar_arrive(&hempty[buf]);  // staging read: the loader may refill it
      if (h == 1) {
        // publish the block: the team's stores precede its barrier; the leader's
        // gpu-scope fence orders them before the release of ready[slot]
        asm volatile("bar.sync %0, 128;\n" ::"r"(2 + team) : "memory");
        if (mm == 0) {
          __threadfence();
          fence_proxy_async_global();
          st_release_gpu(gready + slot, (int)t + 1);
          GFL_TRACE(j, 2);
        }
      }
    }
    flags = __reduce_or_sync(0xffffffffu, flags);
    ovf = __reduce_or_sync(0xffffffffu, ovf);
    if (lane == 0) {
      if (flags) atomicOr(&status->flags, flags);
      if (ovf) atomicOr(overflow, 1);
    }
  } else if (warp == GFL_MPW) {
    // ---- MMA producer: ring image -> smem stage (one 48 KiB bulk copy) ---------------
    // (the MMA issuer releases each ring slot once its copy has landed, so the
    // producer never waits on a copy: up to GFL_NST copies in flight).  Readiness is
    // checked for up to 32 blocks at once (lane i: block k + i) with relaxed loads
    // and one acquire fence per batch: a per-block acquire poll costs an L2 round
    // trip plus a fence (~1 us) on the producer's critical path.
    int64_t avail = -1;  // every block <= avail is known to be published
    long long spins = 0;
    for (int64_t k = 0; k < nblk; ++k) {
      const int st = (int)(k % GFL_NST);
      const int slot = (int)(k % GFL_RING);
      if (k >= GFL_NST) mbar_wait(&sempty[st], (uint32_t)(((k / GFL_NST) - 1) & 1));
      GFL_TRACE(k, 3);
      while (k > avail) {
        const int64_t kk = k + lane;
        const bool ok = kk >= nblk || (lane < GFL_RING && ld_relaxed_gpu(gready + (int)(kk % GFL_RING)) >= (int)kk + 1);
        const unsigned ball = __ballot_sync(0xffffffffu, ok);
        const int run = ball == 0xffffffffu ? 32 : __ffs(~ball) - 1;  // leading published blocks
        if (run > 0) {
          avail = k + run - 1;
          asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
        } else {
          __nanosleep(32);
          if (++spins > GFL_SPIN_LIMIT) __trap();
        }
      }
      GFL_TRACE(k, 4);
      if (lane == 0) {
        fence_proxy_async_global();
        mbar_arrive_expect_tx(&sfull[st], (uint32_t)G8LS_STAGE);
        bulk_g2s(stages + st * G8LS_STAGE, gring + (size_t)slot * G8LS_STAGE, (uint32_t)G8LS_STAGE, &sfull[st]);
      }
      __syncwarp();
    }
  } else if (warp == GFL_MMAW) {
    // ---- MMA issuer: one N = 256 MMA per digit pair of the CTA's level set
    const uint32_t sbase = smem_u32(stages);
    const uint32_t idesc = idesc_g8_n256();
    for (int64_t k = 0; k < nblk; ++k) {
      const int slot = (int)(k % GFL_NST);
      const bool first_in_period = (k % G8_FLUSH_BLOCKS) == 0;
      if (first_in_period && k > 0) mbar_wait(aempty, (uint32_t)(((k / G8_FLUSH_BLOCKS) - 1) & 1));
      mbar_wait(&sfull[slot], (uint32_t)((k / GFL_NST) & 1));
      if (lane == 0) GFL_TRACE(k, 5);
      // the image is in shared memory: its ring slot may be refilled
      if (lane == 0) red_add_release_gpu(gcons + (int)(k % GFL_RING), 1);
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
      __syncwarp();
    }
  } else if (warp >= GFL_FLW0) {
    // ---- flush: thread = member i = TMEM lane; columns in chunks of 8 (as gram_i8_mma_ls_kernel)
    const int quad = warp & 3;
    const int i = 32 * quad + lane;
    const int64_t nper = (nblk + G8_FLUSH_BLOCKS - 1) / G8_FLUSH_BLOCKS;
    double* prow = partial + (size_t)blockIdx.x * (2 * G8_N) * G8_N + i;  // column j at prow[j * G8_N]
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
    const double ai = 4294967296.0 / scl[i];
    for (int j = 0; j < 2 * G8_N; ++j) prow[(size_t)j * G8_N] *= ai / scl[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == GFL_MMAW) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512u) : "memory");
  }
}

}  // namespace enkf
