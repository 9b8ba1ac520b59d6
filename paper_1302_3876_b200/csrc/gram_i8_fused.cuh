// gram_i8_fused.cuh — the int8 tensor-core Gram (gram_i8.cuh) as ONE persistent
// kernel: slicing and MMAs overlap, and the operand images never reach DRAM.
// Opt-in (ENKF_GRAM=i8fused): correct and tested, but measured slower than the
// two-kernel form (config 5: 13.2 vs 11.8 ms alone, 21.1 vs 21.8 steps/s in the
// power-capped step): the MMA issuer shares its SM's issue slots with 12 slicer
// warps and reaches 26 % tensor activity (61 % in gram_i8_mma_kernel), while the
// slicers mostly wait for ring slots.
//
// The two-kernel form writes every 32-row block's 48 KiB operand image to HBM
// (12.8 GB at config 5) and reads it back (12.9 GB); under B200's ~1 kW power
// cap that traffic is paid for in clock.  Here the 4 CTAs of a group
// slice their group's blocks themselves (CTA q slices blocks t = q mod 4) into a
// per-group ring of GF_RING images in global memory, small enough to stay in L2
// (37 groups x 32 x 48 KiB = 57 MiB), and all 4 consume every image of the ring
// through bulk TMA exactly as gram_i8_mma_kernel does.  Cross-CTA hand-off:
//   slicer  : wait consumed[slot] >= 4 * (t / RING)   (previous occupant read by all 4)
//             write the image; barrier; thread 0: fence + release -> ready[slot] = t + 1
//   consumer: acquire ready[slot] >= t + 1; fence.proxy.async; bulk copy;
//             once the copy has landed: consumed[slot] += 1 (release)
// All CTAs must be co-resident (one per SM): the kernel is launched cooperatively,
// and every spin is bounded (a hang becomes a trap, not a stuck GPU).
//
// Roles (19 warps): 0-11 slicers in 3 teams of 4 warps (a team takes every third
// 16-row half-block; thread = one member of P and Q; Y values read straight from
// global memory), 12 slice loader (bulk TMA of a half-block's X[idx] rows, and r,
// into a 4-deep staging ring), 13 MMA producer, 14 MMA issuer (owns TMEM), 15-18
// flush.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "gram_i8.cuh"

namespace enkf {

constexpr int GF_RING = 32;       // images per group ring (37 x 32 x 48 KiB = 57 MiB of L2)
constexpr int GF_NST = 4;         // MMA smem stages
constexpr int GF_HB = 16;         // rows per slicer half-block
constexpr int GF_TEAMS = 3;       // slicer teams of 4 warps
constexpr int GF_THREADS = (4 * GF_TEAMS + 7) * 32;
constexpr int GF_NHB = 4;        // staging depth (half-blocks the loader runs ahead)
constexpr int GF_XST = GF_HB * G8_N * 8;       // 16 KiB: X rows of a half-block
constexpr int GF_STG = GF_XST + GF_HB * 8;     // + r of its rows
constexpr long long GF_SPIN_LIMIT = 1ll << 24;  // ~10-20 s of polling: a deadlock traps instead of hanging

__host__ __device__ inline size_t gram_i8_fused_smem_bytes() {
  return 1024 + (size_t)GF_NST * G8_STAGE + GF_NHB * (size_t)GF_STG + 2 * G8_N * 8 /*scales*/ +
         GF_NHB * GF_HB * 8 * 2 /*mean, sr*/ + GF_NHB * GF_HB * 4 /*valid*/ + GF_RING * 4 /*halfdone*/ +
         64 * 8 /*barriers*/;
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
// poll until *p >= target (bounded; trap on a deadlock)
__device__ __forceinline__ void gf_wait_geq(const int* p, int target) {
  long long spins = 0;
  while (ld_acquire_gpu(p) < target) {
    __nanosleep(64);
    if (++spins > GF_SPIN_LIMIT) __trap();
  }
}

__global__ void __launch_bounds__(GF_THREADS, 1)
gram_i8_fused_kernel(const double* __restrict__ X, const double* __restrict__ Y, const int64_t* __restrict__ idx,
                     const double* __restrict__ r, const unsigned long long* __restrict__ cmax, int64_t n_state,
                     int64_t n_obs, int64_t n_blocks, int64_t blocks_per_group, unsigned char* __restrict__ ring,
                     int* __restrict__ ready, int* __restrict__ consumed, double* __restrict__ partial,
                     int* __restrict__ overflow, DevStatus* __restrict__ status, uint32_t uz /* = 0 */) {
  extern __shared__ __align__(1024) unsigned char gfsm_raw[];
  unsigned char* sm = gfsm_raw + ((1024u - (smem_u32(gfsm_raw) & 1023u)) & 1023u);
  unsigned char* stages = sm;                                        // [GF_NST][G8_STAGE]
  double* stg = reinterpret_cast<double*>(stages + GF_NST * G8_STAGE);  // [NHB][X 16x128 | r 16]
  double* scl = stg + GF_NHB * (GF_STG / 8);                         // [256]
  double* rmean = scl + 2 * G8_N;                                    // [NHB][16]
  double* rsr = rmean + GF_NHB * GF_HB;                              // [NHB][16]
  int* rvalid = reinterpret_cast<int*>(rsr + GF_NHB * GF_HB);        // [NHB][16]
  int* halfdone = rvalid + GF_NHB * GF_HB;                           // [RING] halves written
  uint64_t* bars = reinterpret_cast<uint64_t*>(halfdone + GF_RING);
  uint64_t* sfull = bars;                  // [NST] MMA producer -> issuer (tx)
  uint64_t* sempty = bars + GF_NST;        // [NST] issuer commit -> producer
  uint64_t* afull = bars + 2 * GF_NST;     // issuer commit -> flush
  uint64_t* aempty = afull + 1;            // flush -> issuer
  uint64_t* hfull = aempty + 1;            // [NHB] slice loader -> slicers (tx)
  uint64_t* hempty = hfull + GF_NHB;       // [NHB] slicers -> slice loader
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hempty + GF_NHB);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = blockIdx.x & 3;
  const int64_t grp = blockIdx.x >> 2;
  const int64_t b0 = grp * blocks_per_group;
  const int64_t b1 = b0 + blocks_per_group < n_blocks ? b0 + blocks_per_group : n_blocks;
  const int64_t nblk = b1 > b0 ? b1 - b0 : 0;
  const bool qslice = q >= 2;
  unsigned char* gring = ring + (size_t)grp * GF_RING * G8_BLOCK_BYTES;
  int* gready = ready + grp * GF_RING;
  int* gcons = consumed + grp * GF_RING;
  constexpr int SLW = 4 * GF_TEAMS, LDW = SLW, MPW = SLW + 1, MMAW = SLW + 2, FLW0 = SLW + 3;

  if (tid == 0) {
    for (int i = 0; i < GF_NST; ++i) {
      mbar_init(&sfull[i], 1);
      mbar_init(&sempty[i], 1);
    }
    mbar_init(afull, 1);
    mbar_init(aempty, 128);
    for (int i = 0; i < GF_NHB; ++i) {
      mbar_init(&hfull[i], 1);
      mbar_init(&hempty[i], 128);  // one team
    }
    fence_mbar_init();
  }
  for (int c = tid; c < 2 * G8_N; c += GF_THREADS) scl[c] = g8_scale(cmax[c]);
  for (int c = tid; c < GF_RING; c += GF_THREADS) halfdone[c] = 0;
  if (warp == MMAW) {
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

  // this CTA slices blocks t = q, q + 4, ... of its group, two 16-row halves each
  const int64_t my_blocks = nblk > q ? (nblk - 1 - q) / 4 + 1 : 0;
  const int64_t my_halves = 2 * my_blocks;

  if (warp == LDW) {
    // ---- slice loader: X[idx] rows (one bulk copy per row) and r of a half-block.
    // idx, idx[g-1] and r of the next half are loaded one iteration ahead, so their
    // latency overlaps the wait for a free staging buffer and the bulk copies.
    int flags = 0;
    auto fetch = [&](int64_t hh, int64_t& src, int64_t& prev, double& rv) {
      const int64_t t = q + 4 * (hh >> 1);
      const int64_t g = (b0 + t) * G8_KB + GF_HB * (hh & 1) + lane;
      src = -1;
      prev = -1;
      rv = 1.0;
      if (hh < my_halves && lane < GF_HB && g < n_obs) {
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
      const int buf = (int)(hh % GF_NHB);
      const int64_t t = q + 4 * (hh >> 1);
      const int64_t g0 = (b0 + t) * G8_KB + GF_HB * (hh & 1);
      const int64_t g = g0 + lane;
      int64_t src = nsrc;
      const int64_t prev = nprev;
      const double rv = nrv;
      fetch(hh + 1, nsrc, nprev, nrv);
      bool valid = lane < GF_HB && g < n_obs;
      if (valid && idx) {
        if (g > 0 && prev >= src) flags |= FLAG_IDX_ORDER;
        if (src < 0 || src >= n_state) {
          flags |= FLAG_IDX_RANGE;
          valid = false;
        }
      }
      if (hh >= GF_NHB) mbar_wait(&hempty[buf], (uint32_t)(((hh / GF_NHB) - 1) & 1));
      double* xs = stg + buf * (GF_STG / 8);
      double* rs = xs + GF_XST / 8;
      if (lane < GF_HB) {
        rvalid[buf * GF_HB + lane] = valid ? 1 : 0;
        rs[lane] = rv;  // plain loads (a bulk copy needs 16-byte multiples)
      }
      const unsigned vmask = __ballot_sync(0xffffffffu, valid);
      const int nx = __popc(vmask);
      if (nx < GF_HB) {  // rows with no data (past the end, bad index) become exact zeros
        for (int rr = 0; rr < GF_HB; ++rr)
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
  } else if (warp < SLW) {
    // ---- slicers: GF_TEAMS teams of 4 warps; team k takes half-blocks hh = k mod
    // GF_TEAMS.  Thread = member mm of P AND Q for the 16 rows of its half.
    const int team = warp >> 2, tt = tid & 127, tw = warp & 3;
    const int mm = tt;
    const double scp = scl[mm], scq = scl[G8_N + mm];
    int flags = 0, ovf = 0;
    // 1.5 2^52 + bias: fma(v, sc, kMagicB) holds V + 0x808080808080 in its low 51 bits
    const double kMagicB = 6755399441055744.0 + (double)0x808080808080ull;
    for (int64_t hh = team; hh < my_halves; hh += GF_TEAMS) {
      const int buf = (int)(hh % GF_NHB), h = (int)(hh & 1);
      const int64_t t = q + 4 * (hh >> 1);
      const int slot = (int)(t % GF_RING);
      const int64_t g0 = (b0 + t) * G8_KB + GF_HB * h;
      unsigned char* img = gring + (size_t)slot * G8_BLOCK_BYTES;
      // Y of the 16 rows straight from global memory, issued first (latency overlaps
      // the waits and step A)
      double yv[GF_HB];
#pragma unroll
      for (int k = 0; k < GF_HB; ++k) yv[k] = (g0 + k < n_obs) ? __ldcs(Y + (g0 + k) * G8_N + mm) : 0.0;
      if (t >= GF_RING) {  // the slot's previous image must be consumed by all 4 CTAs
        if (tt == 0) gf_wait_geq(gcons + slot, 4 * (int)(t / GF_RING));
        asm volatile("bar.sync %0, 128;\n" ::"r"(2 + team) : "memory");
      }
      mbar_wait(&hfull[buf], (uint32_t)((hh / GF_NHB) & 1));
      const double* xs = stg + buf * (GF_STG / 8);
      const double* rs = xs + GF_XST / 8;
      // step A: row means (warp tw: rows 4tw..4tw+3), sqrt(1/r) (warp 0 of the team, lane = row)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int row = 4 * tw + u;
        double sx = (xs[row * G8_N + lane] + xs[row * G8_N + lane + 32]) +
                    (xs[row * G8_N + lane + 64] + xs[row * G8_N + lane + 96]);
        sx = warp_sum(sx);
        if (lane == 0) rmean[buf * GF_HB + row] = sx * (1.0 / G8_N);
      }
      if (tw == 0 && lane < GF_HB) {
        double srv = 0.0;  // invalid rows (bad index, past the end) contribute exact zeros
        if (rvalid[buf * GF_HB + lane] != 0) {
          const double rv = rs[lane];
          if (!isfinite(rv)) flags |= FLAG_NONFINITE;
          else if (!(rv > 0.0)) flags |= FLAG_R_NONPOS;
          srv = g8_sqrt_rho(rv);
        }
        rsr[buf * GF_HB + lane] = srv;
      }
      asm volatile("bar.sync %0, 128;\n" ::"r"(2 + team) : "memory");
      // step B: 16 rows -> the 16-byte chunk h of member mm's row in all 6 P and 6 Q planes
      double xr[GF_HB];
#pragma unroll
      for (int k = 0; k < GF_HB; ++k) xr[k] = xs[k * G8_N + mm];
      const size_t off = (size_t)mm * 32 + (size_t)((h ^ ((mm >> 2) & 1)) << 4);
#pragma unroll
      for (int pq = 0; pq < 2; ++pq) {
        uint32_t w[G8_ND][4];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          uint32_t vlo[4], vhi[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int row = 4 * q4 + u;
            const double sr = rsr[buf * GF_HB + row];
            const double d = pq == 0 ? xr[row] - rmean[buf * GF_HB + row] : yv[row] - xr[row];
            const double tv = fma(sr * d, pq == 0 ? scp : scq, kMagicB);
            const uint32_t hv = (uint32_t)__double2hiint(tv) - 0x43380000u;
            ovf |= hv >= 0x10000u;  // V + bias outside [0, 2^48): |V| too large, or non-finite
            vlo[u] = (uint32_t)__double2loint(tv);
            vhi[u] = hv;
          }
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
        unsigned char* base = img + (pq == 0 ? 0 : G8_ND * G8_PLANE) + off;
#pragma unroll
        for (int p = 0; p < G8_ND; ++p)
          *reinterpret_cast<uint4*>(base + (size_t)p * G8_PLANE) = make_uint4(w[p][0], w[p][1], w[p][2], w[p][3]);
      }
      mbar_arrive(&hempty[buf]);  // staging read: the loader may refill it
      // publish the block once both halves (two teams) are written: the team's stores
      // precede its barrier; the team leader's gpu-scope fence orders them before its
      // shared-memory count, the second leader fences again and releases ready[slot]
      asm volatile("bar.sync %0, 128;\n" ::"r"(2 + team) : "memory");
      if (tt == 0) {
        __threadfence();
        if (atomicAdd(&halfdone[slot], 1) == 1) {
          halfdone[slot] = 0;
          fence_proxy_async_global();
          __threadfence();
          st_release_gpu(gready + slot, (int)t + 1);
        }
      }
    }
    flags = __reduce_or_sync(0xffffffffu, flags);
    ovf = __reduce_or_sync(0xffffffffu, ovf);
    if (lane == 0) {
      if (flags) atomicOr(&status->flags, flags);
      if (ovf) atomicOr(overflow, 1);
    }
  } else if (warp == MPW) {
    // ---- MMA producer: ring image -> smem stage ---------------------------------
    if (lane == 0) {
      const uint32_t bytes = (uint32_t)(G8_ND * G8_PLANE + (qslice ? G8_ND * G8_BSL : 0));
      for (int64_t k = 0; k < nblk; ++k) {
        const int st = (int)(k % GF_NST);
        const int slot = (int)(k % GF_RING);
        if (k >= GF_NST) mbar_wait(&sempty[st], (uint32_t)(((k / GF_NST) - 1) & 1));
        gf_wait_geq(gready + slot, (int)k + 1);
        fence_proxy_async_global();
        unsigned char* dst = stages + st * G8_STAGE;
        const unsigned char* src = gring + (size_t)slot * G8_BLOCK_BYTES;
        mbar_arrive_expect_tx(&sfull[st], bytes);
        bulk_g2s(dst, src, (uint32_t)(G8_ND * G8_PLANE), &sfull[st]);
        if (qslice) {
#pragma unroll
          for (int p = 0; p < G8_ND; ++p)
            bulk_g2s(dst + G8_ND * G8_PLANE + p * G8_BSL, src + G8_ND * G8_PLANE + p * G8_PLANE + (q - 2) * G8_BSL,
                     (uint32_t)G8_BSL, &sfull[st]);
        }
        // the previous image is in shared memory: its ring slot may be refilled
        if (k >= 1) {
          mbar_wait(&sfull[(k - 1) % GF_NST], (uint32_t)(((k - 1) / GF_NST) & 1));
          red_add_release_gpu(gcons + (int)((k - 1) % GF_RING), 1);
        }
      }
      if (nblk >= 1) {
        mbar_wait(&sfull[(nblk - 1) % GF_NST], (uint32_t)(((nblk - 1) / GF_NST) & 1));
        red_add_release_gpu(gcons + (int)((nblk - 1) % GF_RING), 1);
      }
    }
  } else if (warp == MMAW) {
    // ---- MMA issuer (as gram_i8_mma_kernel, A planes from TMEM) -------------------
    const uint32_t sbase = smem_u32(stages);
    for (int64_t k = 0; k < nblk; ++k) {
      const int st = (int)(k % GF_NST);
      const bool first_in_period = (k % G8_FLUSH_BLOCKS) == 0;
      if (first_in_period && k > 0) mbar_wait(aempty, (uint32_t)(((k / G8_FLUSH_BLOCKS) - 1) & 1));
      mbar_wait(&sfull[st], (uint32_t)((k / GF_NST) & 1));
      tc_fence_after();
      const uint32_t abuf = sbase + (uint32_t)(st * G8_STAGE);
      const uint32_t bbuf = qslice ? abuf + (uint32_t)(G8_ND * G8_PLANE) : abuf + (uint32_t)(q * G8_BSL);
      const uint32_t bstride = qslice ? (uint32_t)G8_BSL : (uint32_t)G8_PLANE;
      g8_issue_block(uz, abuf, bbuf, bstride, first_in_period);
      umma_commit_elect(&sempty[st]);
      if ((k % G8_FLUSH_BLOCKS) == G8_FLUSH_BLOCKS - 1 || k == nblk - 1) umma_commit_elect(afull);
      __syncwarp();
    }
  } else if (warp >= FLW0) {
    // ---- flush: thread = member i = TMEM lane; the 7 levels into the fp64 partial
    const int quad = warp & 3;
    const int i = 32 * quad + lane;
    const int64_t nper = (nblk + G8_FLUSH_BLOCKS - 1) / G8_FLUSH_BLOCKS;
    double* prow = partial + ((size_t)blockIdx.x * G8_N + i) * G8_NS;
    const double ai = 4294967296.0 / scl[i];
    const double* bsc = scl + (qslice ? G8_N + 64 * (q - 2) : 64 * q);
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
          const int j = 8 * cg + c;
          const double val = g8_combine(v, c) * (ai / bsc[j]);
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

}  // namespace enkf
