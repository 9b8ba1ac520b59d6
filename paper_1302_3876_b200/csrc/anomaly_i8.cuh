// anomaly_i8.cuh — X^A = X T on the 5th-generation tensor cores (N == 128).
//
// The anomaly update (enkf.py:192, x + s @ A) is evaluated as X^A = X T with
// T = I + (I - 11'/N) A / sqrt(N-1) (ism_levels writes T), an Ns x 128 x 128 fp64
// product.  B200 has no fp64 tcgen05 kind, so the product is evaluated EXACTLY in
// integer arithmetic on byte "digits" (Ozaki-style splitting) and rounded once:
//   row i of X : e_i with max|X_i.| < 2^e_i,  V_ik = round(X_ik 2^(47-e_i))  (48-bit)
//   all of T   : ONE power-of-two scale f,    W_kj = round(T_kj 2^(47-f))
//   V = sum_p d_p 256^(6-p), W = sum_q c_q 256^(6-q), p,q = 1..6 two's-complement
//   bytes (p = 1 signed, the rest unsigned).  X T ~= 2^(e_i+f-94) sum_{p+q<=8}
//   256^(12-p-q) (D_p C_q)_ij with every D_p C_q an exact int32 tcgen05.mma
//   (kind::i8, K = 128 -> |acc| < 2^26): 26 digit pairs, 7 levels l = p + q.
// Truncation (p+q > 8) and the input roundings give ~7e-14 relative to max|X^A|
// (tests compare against the FP64 DMMA path and the oracle).
//
// Roles (14 warps): a TMA warp bulk-copies each contiguous 32-row X
// tile into a 4-deep smem ring; 4 slicer warps form the row exponents and the six
// X digit planes (B operand, N = 16 rows per MMA, K-major, 128B swizzle) and
// release the stage at once (the epilogue never reads X); the six digit planes of
// T^T stay in TMEM for the whole kernel (A operand, 192 columns); one elected
// thread issues the 208 MMAs of a tile into double-buffered TMEM accumulators
// (7 levels x 16 columns); 8 epilogue warps (thread = output column = TMEM lane)
// combine the 7 int32 levels in INTEGER arithmetic into one int64, convert once
// (the only rounding) and scale through the exponent field — no FP64 arithmetic
// next to the MMAs (FP64 ops were measured to stall the int8 tensor pipe).
// T == I exactly copies X bit for bit; tiny / huge / non-finite rows take exact
// slow paths.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace enkf {

constexpr int I8_N = 128;         // ensemble size handled by this kernel
constexpr int I8_TILE = 32;       // X rows per tile
constexpr int I8_NBUF = 4;        // pipeline depth (raw X stages and digit buffers)
#ifndef I8_CHUNK_ROWS
#define I8_CHUNK_ROWS 16
#endif
constexpr int I8_CHUNK = I8_CHUNK_ROWS;  // rows per MMA (N of the instruction)
// TMEM: 192 columns of T digits + accumulators: two 16-row chunk buffers, or one
// 32-row buffer (N = 32 halves the MMA count; the epilogue drains before reuse)
constexpr int I8_ABUF = I8_CHUNK == 16 ? 2 : 1;
constexpr int I8_ND = 6;          // byte digits per value
#ifndef I8_TBAL
#define I8_TBAL 0   // balanced (zero-mean) digits for T: the p+q > I8_LMAX truncation is then unbiased
#endif
#ifndef I8_LMAX_DEF
#define I8_LMAX_DEF 8
#endif
constexpr int I8_LMAX = I8_LMAX_DEF;  // keep digit pairs with p + q <= I8_LMAX (8; 7 measured in DESIGN §5)
constexpr int I8_NLEV = I8_LMAX - 1;  // levels 2..8
#ifndef I8_SW
#define I8_SW 4
#endif
#ifndef I8_EW
#define I8_EW 8
#endif
constexpr int I8_SLICE_WARPS = I8_SW;
constexpr int I8_EPI_WARPS = I8_EW;   // I8_EW/4 per TMEM lane quadrant, each a slice of a chunk's rows
constexpr int I8_EPI_GROUPS = I8_EPI_WARPS / 4;
constexpr int I8_RPT = I8_CHUNK / I8_EPI_GROUPS;  // chunk rows per epilogue thread
static_assert(I8_RPT == 4 || I8_RPT == 8, "epilogue rows per thread");
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
  return 1024 /*align slack*/ + I8_NBUF * ((size_t)I8_XBUF_BYTES + (size_t)I8_STAGE_BYTES) +
         I8_NBUF * I8_TILE * sizeof(double) + 2 * I8_NBUF * I8_SLICE_WARPS * sizeof(int) + 512;
}

// K order of the digit planes: word w of a plane row holds k = 2w, 2w+1, 64+2w,
// 65+2w (bytes 0..3).  Any permutation of k applied to both operands leaves the
// products unchanged; this one lets a slicer lane fetch its 4 values with two
// contiguous 512-byte LDS.128 rows (no bank conflicts).
__host__ __device__ __forceinline__ int i8_kperm(int w, int b) { return (b < 2 ? 2 * w + b : 64 + 2 * w + b - 2); }

#ifndef I8_WARP_ARRIVE
#define I8_WARP_ARRIVE 0
#endif
__device__ __forceinline__ void i8_wait_a(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      " @!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity), "r"(0x100000u)
      : "memory");
}
__device__ __forceinline__ void i8_arrive_a(uint32_t addr) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(addr) : "memory");
}
// one arrival per warp (barrier counts are in warps) or per thread
__device__ __forceinline__ void i8_arrive(uint64_t* bar) {
#if I8_WARP_ARRIVE
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(bar);
#else
  mbar_arrive(bar);
#endif
}
constexpr int I8_ARRIVE_UNIT = I8_WARP_ARRIVE ? 1 : 32;

// d 2^k for rows whose exponent shift leaves the exponent-field fast path
// (|x| near the fp64 range limits): exact scaling, or NaN for non-finite rows.
__device__ __noinline__ double i8_scale_slow(double d, int k) {
  if (k == INT_MIN) return __longlong_as_double(0x7ff8000000000000ll);
  if (d == 0.0) return 0.0;
  if (k > 2000) return d * INFINITY;
  if (k < -2200) return d * 0.0;
  const int k1 = k / 2;
  return d * ldexp(1.0, k1) * ldexp(1.0, k - k1);
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
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t (&v)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(taddr));
}
template <int R>
__device__ __forceinline__ void tmem_ldr(uint32_t taddr, uint32_t (&v)[R]) {
  if constexpr (R == 8) tmem_ld8(taddr, v); else tmem_ld4(taddr, v);
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
// Profiling-only trace (CTA 0): [tile][event] globaltimer stamps, events:
// 0 TMA issued, 1 stage landed (slicer view), 2 slicing done, 3 MMA issue start,
// 4 MMA issue end, 5 epilogue first chunk ready, 6 epilogue done.
constexpr int I8_TRACE_TILES = 256;
__device__ unsigned long long g_i8_trace[I8_TRACE_TILES][16];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#ifdef I8_TRACE_ON  // profiling builds only (tools/probe/i8_trace.py builds the "trace" variant)
#define I8_TRACE(it, ev) \
  do { if ((dbg & 8) && blockIdx.x == 0 && (it) < I8_TRACE_TILES) g_i8_trace[(it)][(ev)] = gtime(); } while (0)
#else
#define I8_TRACE(it, ev) do { } while (0)
#endif

__global__ void __launch_bounds__(I8_THREADS, 1)
anomaly_i8_kernel(const double* __restrict__ X, const double* __restrict__ T,
                  double* __restrict__ XA, int64_t n_rows, int dbg_arg, uint32_t uz /* = 0 */) {
  // dbg (profiling builds only, -DI8_DBG_BUILD; the product build compiles every dbg
  // branch out): bit0 skip MMAs, bit1 skip slicing, bit2 skip the epilogue,
  // bit4 drain TMEM but skip the recombination, bit5 stores into an L2-resident window.
#ifdef I8_DBG_BUILD
  const int dbg = dbg_arg;
#else
  constexpr int dbg = 0;
  (void)dbg_arg;
#endif
  // Measured with these (tools/probe/i8_trace.py): FP64 arithmetic (DFMA/DADD/DMUL)
  // issued by other warps slows the int8 MMAs roughly in proportion to its count,
  // integer ops and int->fp64 conversions do not.
  extern __shared__ __align__(1024) unsigned char i8sm_raw[];
  // realign by a byte offset (not an integer round trip) so the compiler keeps
  // the shared address space and emits LDS/STS, not generic LD/ST
  unsigned char* i8sm = i8sm_raw + ((1024u - (smem_u32(i8sm_raw) & 1023u)) & 1023u);
  unsigned char* xdig = i8sm;                                                  // [NBUF][6][32][128 B]
  double* stage = reinterpret_cast<double*>(xdig + I8_NBUF * I8_XBUF_BYTES);  // [NBUF][32][128]
  // per-row exponent shift k [2*NBUF][32] (X^A = S' 2^k; INT_MIN for non-finite rows),
  // a ring twice the stage depth so the slicers never overwrite a tile the epilogue reads
  int* rinfo = reinterpret_cast<int*>(stage + I8_NBUF * I8_TILE * I8_N);
  // [2*NBUF][slicer warp]: 1 if one of that warp's 8 rows needs the slow scaling path
  int* rflag = rinfo + 2 * I8_NBUF * I8_TILE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(rflag + 2 * I8_NBUF * I8_SLICE_WARPS);
  uint64_t* sfull = bars;                  // [NBUF] TMA -> slicers/epilogue      (count 1 + tx)
  uint64_t* sempty = bars + I8_NBUF;       // [NBUF] slicers -> producer              (count slicer warps)
  uint64_t* xfull = bars + 2 * I8_NBUF;    // [NBUF] slicers -> MMA               (count slicer threads)
  uint64_t* xempty = bars + 3 * I8_NBUF;   // [NBUF] MMA commit -> slicers        (count 1)
  uint64_t* afull = bars + 4 * I8_NBUF;    // [2] MMA commit -> epilogue          (count 1)
  uint64_t* aempty = bars + 4 * I8_NBUF + 2;  // [2] epilogue -> MMA              (count epi threads)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4 * I8_NBUF + 4);
  unsigned long long* cmax_s = reinterpret_cast<unsigned long long*>(bars + 4 * I8_NBUF + 5);  // max |T| bits
  int* nonid_s = reinterpret_cast<int*>(bars + 4 * I8_NBUF + 6);  // T != I
  // [2*NBUF] slicers -> epilogue: row exponents of a tile are in rinfo (count slicer
  // threads).  Its own ring (depth 8 > the at most 5 tiles the slicers run ahead of
  // the epilogue) keeps the parity waits unambiguous.
  uint64_t* rfull = bars + 4 * I8_NBUF + 8;
  const uint32_t sfull_a = smem_u32(sfull), sempty_a = smem_u32(sempty), xfull_a = smem_u32(xfull);
  const uint32_t xempty_a = smem_u32(xempty), afull_a = smem_u32(afull), aempty_a = smem_u32(aempty);
  const uint32_t rfull_a = smem_u32(rfull);

  // Epilogue warps sit at warp ids 4..4+EW-1 (a warp may only touch the TMEM lane
  // quadrant warp_id % 4); slicers 0..3, then the MMA issuer and the producer.
  // (Giving the MMA issuer an SMSP without a slicer was measured 20% slower.)
  constexpr int EPI0 = 4;
  static_assert(I8_SLICE_WARPS == 4, "role layout assumes 4 slicer warps");
  constexpr int MMAW = EPI0 + I8_EPI_WARPS;
  constexpr int TMAW = MMAW + 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int sw = warp < 4 ? warp : -1;  // slicer index
  const int64_t ntiles = (n_rows + I8_TILE - 1) / I8_TILE;
  const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

  if (tid == 0) {
    for (int i = 0; i < I8_NBUF; ++i) {
      mbar_init(&sfull[i], 1);
      mbar_init(&sempty[i], I8_ARRIVE_UNIT * I8_SLICE_WARPS);
      mbar_init(&xfull[i], I8_ARRIVE_UNIT * I8_SLICE_WARPS);
      mbar_init(&xempty[i], 1);
    }
    for (int i = 0; i < 2 * I8_NBUF; ++i) mbar_init(&rfull[i], I8_ARRIVE_UNIT * I8_SLICE_WARPS);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&afull[i], 1);
      mbar_init(&aempty[i], I8_ARRIVE_UNIT * I8_EPI_WARPS);
    }
    fence_mbar_init();
    *cmax_s = 0ull;
    *nonid_s = 0;
  }
  __syncthreads();
  {
    // One power-of-two scale 2^fT for all of T (max|T| < 2^fT): the epilogue's
    // per-output work then needs a per-row exponent only.  T == I exactly (zero
    // spread) is detected so X^A = X comes out bit-exact.
    unsigned long long lm = 0ull;
    int nonid = 0;
    for (int e = tid; e < I8_N * I8_N; e += I8_THREADS) {
      const double tv = T[e];
      const unsigned long long b = (unsigned long long)__double_as_longlong(tv) & 0x7fffffffffffffffull;
      lm = b > lm ? b : lm;
      nonid |= tv != ((e >> 7) == (e & 127) ? 1.0 : 0.0);
    }
    atomicMax(cmax_s, lm);
    if (nonid) atomicOr(nonid_s, 1);
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
  const int fT = exp_above(*cmax_s);  // max|T| < 2^fT
  if (*nonid_s == 0) {
    // T == I: X^A = X exactly (the reference's zero-spread identity, test_enkf.py:208-213)
    const int64_t ntiles_all = (n_rows + I8_TILE - 1) / I8_TILE;
    for (int64_t tile = blockIdx.x; tile < ntiles_all; tile += gridDim.x) {
      const int64_t g0 = tile * I8_TILE;
      const int64_t rows = n_rows - g0 < I8_TILE ? n_rows - g0 : I8_TILE;
      const double2* src = reinterpret_cast<const double2*>(X + g0 * I8_N);
      double2* dst = reinterpret_cast<double2*>(XA + g0 * I8_N);
      for (int64_t e = tid; e < rows * (I8_N / 2); e += I8_THREADS) dst[e] = src[e];
    }
  } else if (warp == TMAW) {
    // ---- producer: one bulk copy per tile (the tile's rows are contiguous) -----
    if (lane == 0) {
      for (int64_t it = 0; it < my_tiles; ++it) {
        const int buf = (int)(it % I8_NBUF);
        const int64_t tile = blockIdx.x + it * gridDim.x;
        if (it >= I8_NBUF) i8_wait_a(sempty_a + 8u * (uint32_t)(buf), (uint32_t)(((it / I8_NBUF) - 1) & 1));
        fence_proxy_async();
        const int64_t g0 = tile * I8_TILE;
        const int rows = (int)(n_rows - g0 < I8_TILE ? n_rows - g0 : I8_TILE);
        const uint32_t bytes = (uint32_t)rows * I8_N * 8u;
        mbar_arrive_expect_tx(&sfull[buf], bytes);
        I8_TRACE(it, 0);
        double* dst = stage + buf * I8_TILE * I8_N;
        const double* src = X + g0 * I8_N;
        for (uint32_t off = 0; off < bytes; off += 16384u) {
          const uint32_t len = bytes - off < 16384u ? bytes - off : 16384u;
          bulk_g2s(reinterpret_cast<unsigned char*>(dst) + off, reinterpret_cast<const unsigned char*>(src) + off,
                   len, &sfull[buf]);
        }
      }
    }
  } else if (warp >= EPI0 && warp < EPI0 + I8_EPI_WARPS) {
    // ---- epilogue warps: thread = output column j = TMEM lane ------------------
    const int quad = warp & 3;            // TMEM lane quadrant this warp may access
    const int half = (warp - EPI0) >> 2;  // which I8_RPT rows of each 16-row chunk
    const int j = 32 * quad + lane;
    // T^T digit planes into TMEM (A operand), one scale 2^(47-fT) for all of T
    // (T = I + (I - 11'/N) A / sqrt(N-1) from the levels kernel)
    auto cval = [&](int k) { return T[k * I8_N + j]; };
    if (half == 0) {
      const double cscale = pow2(I8_TBAL ? 46 - fT : 47 - fT);
#pragma unroll 1
      for (int p = 0; p < I8_ND; ++p) {
#pragma unroll 1
        for (int w = 0; w < 32; ++w) {
          uint32_t word = 0;
#pragma unroll
          for (int b = 0; b < 4; ++b) {
#if I8_TBAL
            // balanced digits of T (bytes of W + 0x808080808080, each ^ 0x80; |W| <= 2^46)
            const long long v = round_scaled(cval(i8_kperm(w, b)), cscale) + 0x808080808080ll;
            word |= (byte_of(v, 5 - p) ^ 0x80u) << (8 * b);
#else
            const long long v = round_scaled(cval(i8_kperm(w, b)), cscale);
            word |= byte_of(v, 5 - p) << (8 * b);
#endif
          }
          tmem_st1(tmem + ((uint32_t)(32 * quad) << 16) + (uint32_t)(32 * p + w), word);
        }
      }
      tmem_st_wait();
    }
    tc_fence_before();
    asm volatile("bar.sync 1, %0;\n" ::"n"(32 * (I8_EPI_WARPS + 1)) : "memory");  // C planes in TMEM before the first MMA
    int chunk_ctr = 0;
    for (int64_t it = 0; it < my_tiles; ++it) {
      const int64_t tile = blockIdx.x + it * gridDim.x;
      i8_wait_a(rfull_a + 8u * (uint32_t)(it % (2 * I8_NBUF)), (uint32_t)((it / (2 * I8_NBUF)) & 1));  // the tile's row exponents
      const int* rk = rinfo + (int)(it % (2 * I8_NBUF)) * I8_TILE;
      for (int c = 0; c < I8_TILE / I8_CHUNK; ++c, ++chunk_ctr) {
        const int ab = chunk_ctr % I8_ABUF;
        const int r0 = c * I8_CHUNK + I8_RPT * half;  // first tile row of this thread's I8_RPT
        const int64_t g0 = tile * I8_TILE + r0;
        i8_wait_a(afull_a + 8u * (uint32_t)(ab), (uint32_t)((chunk_ctr / I8_ABUF) & 1));
        tc_fence_after();
        if (c == 0 && warp == EPI0 && lane == 0) I8_TRACE(it, 5);
        if (warp == EPI0 && lane == 0) I8_TRACE(it, 12 + c);
        if (dbg & 4) {
          tc_fence_before();
          i8_arrive_a(aempty_a + 8u * (uint32_t)(ab));
          continue;
        }
        const uint32_t tbase = tmem + ((uint32_t)(32 * quad) << 16) +
                               (uint32_t)(I8_ACC0 + ab * I8_ACCBUF + I8_RPT * half);
        uint32_t v[I8_NLEV][I8_RPT];
#pragma unroll
        for (int l = 0; l < I8_NLEV; ++l) tmem_ldr<I8_RPT>(tbase + (uint32_t)(l * I8_CHUNK), v[l]);
        tmem_ld_wait();
        tc_fence_before();
        i8_arrive_a(aempty_a + 8u * (uint32_t)(ab));  // accumulators copied out: the MMA may reuse them
        if (dbg & 16) {          // profiling: drain TMEM but skip the recombination and stores
          if (v[0][0] == 0x7fffffffu) XA[0] = 0.0;
          continue;
        }
        // profiling (dbg 32): stores cycle through a 1 MiB window (L2-resident, no DRAM writes)
        double* orow = XA + ((dbg & 32) ? (g0 & 1023) : g0) * I8_N + j;
        const int nvalid = (int)(n_rows - g0 < I8_RPT ? n_rows - g0 : I8_RPT);
        // X T = 2^(e+fT-94) sum_l acc_l 256^(12-l).  On B200 FP64 arithmetic
        // (DFMA/DMUL/DADD) shares hardware with the tensor cores: every FP64 op here
        // stalls the concurrent int8 MMAs (measured, tools/probe/i8_trace.py; integer
        // ops and int->fp64 conversions do not).  So the 7 levels are combined in
        // INTEGER arithmetic into
        //   S' = acc2 2^36 + acc3 2^28 + acc4 2^20 + acc5 2^12 + acc6 2^4 + (acc7 >> 4) + (acc8 >> 12)
        // (|S'| < 2^63; S' is S / 2^12 up to 2 units, ~2^-57 of max|X||T|, far below
        // the digit truncation), converted once (I2F.S64, one rounding) and scaled by
        // 2^k, k = e + fT - 50, with an integer add to the exponent field.
        int kr[I8_RPT];
#pragma unroll
        for (int r = 0; r < I8_RPT; r += 4) {
          const int4 k4 = *reinterpret_cast<const int4*>(rk + r0 + r);
          kr[r] = k4.x; kr[r + 1] = k4.y; kr[r + 2] = k4.z; kr[r + 3] = k4.w;
        }
        // rows near the fp64 range limits or non-finite (warp-uniform, rare); the
        // slicer warp that formed these 8 rows flagged them
        static_assert(I8_TILE / I8_SLICE_WARPS == 8 && 8 % I8_RPT == 0, "epilogue rows within one slicer row group");
        const bool slow = rflag[(int)(it % (2 * I8_NBUF)) * I8_SLICE_WARPS + (r0 >> 3)] != 0;
        // Instruction count matters here: the epilogue is ~45 % of the kernel's issued
        // instructions, and under the board's power cap (SM clock ~1.3 GHz) issue slots
        // bound the tile time.  sext(small) + d2 2^36 is formed directly as a register
        // pair (high word (small >> 31) + 16 d2), then three mad.wide add d5 2^12,
        // d4 2^20, d3 2^28: 8 integer instructions per output before the conversion.
        auto sprime = [&](int r) {
          const int d2 = (int)v[0][r], d3 = (int)v[1][r], d4 = (int)v[2][r], d5 = (int)v[3][r];
          const int d6 = (int)v[4][r], d7 = (int)v[5][r];
          int small = d6 * 16 + (d7 >> 4);  // |.| < 2^31
          if constexpr (I8_NLEV > 6) small += (int)v[I8_NLEV > 6 ? 6 : 0][r] >> 12;
          const int hi0 = (small >> 31) + d2 * 16;
          long long sp = __double_as_longlong(__hiloint2double(hi0, small));  // register pair, no instruction
          sp = (long long)d5 * 4096 + sp;
          sp = (long long)d4 * 1048576 + sp;
          sp = (long long)d3 * 268435456 + sp;
          return (double)sp;
        };
        // scale by 2^k through the exponent field; an exact zero stays zero
        auto scaled = [&](int r) {
          const double dd = sprime(r);
          int hi = __double2hiint(dd);
          asm("{\n.reg .pred p;\nsetp.ne.s32 p, %0, 0;\n@p mad.lo.s32 %0, %1, 1048576, %0;\n}" : "+r"(hi) : "r"(kr[r]));
          return __hiloint2double(hi, __double2loint(dd));
        };
        if (!slow && nvalid == I8_RPT) {
#pragma unroll
          for (int r = 0; r < I8_RPT; ++r) orow[r * I8_N] = scaled(r);
        } else if (!slow) {
#pragma unroll
          for (int r = 0; r < I8_RPT; ++r)
            if (r < nvalid) orow[r * I8_N] = scaled(r);
        } else {
#pragma unroll
          for (int r = 0; r < I8_RPT; ++r)
            if (r < nvalid) orow[r * I8_N] = i8_scale_slow(sprime(r), kr[r]);
        }
        if (warp == EPI0 && lane == 0) I8_TRACE(it, 14 + c);
      }
      if (warp == EPI0 && lane == 0) I8_TRACE(it, 6);
    }
  } else if (warp == MMAW) {
    // ---- MMA issuer ---------------------------------------------------------------
    asm volatile("bar.sync 1, %0;\n" ::"n"(32 * (I8_EPI_WARPS + 1)) : "memory");
    tc_fence_after();
    const uint32_t xbase = smem_u32(xdig);
    int chunk_ctr = 0;
    for (int64_t it = 0; it < my_tiles; ++it) {
      const int buf = (int)(it % I8_NBUF);
      i8_wait_a(xfull_a + 8u * (uint32_t)(buf), (uint32_t)((it / I8_NBUF) & 1));
      tc_fence_after();
      if (lane == 0) I8_TRACE(it, 3);
      for (int c = 0; c < I8_TILE / I8_CHUNK; ++c, ++chunk_ctr) {
        const int ab = chunk_ctr % I8_ABUF;
        if (chunk_ctr >= I8_ABUF)
          i8_wait_a(aempty_a + 8u * (uint32_t)(ab), (uint32_t)(((chunk_ctr / I8_ABUF) - 1) & 1));
        tc_fence_after();
        if (lane == 0) I8_TRACE(it, 8 + 2 * c);
        if (!(dbg & 1)) {
          // uz is a kernel parameter equal to 0: deriving every operand from it
          // keeps the addresses in uniform registers (UIADD3 from the constant
          // bank) instead of materialising 50+ immediates through vector registers.
          const uint32_t dacc = uz + (uint32_t)(I8_ACC0 + ab * I8_ACCBUF);
          const uint64_t desc0 = umma_desc_sw128(xbase + (uint32_t)(buf * I8_XBUF_BYTES + c * I8_CHUNK * 128));
          // k-step outermost: consecutive MMAs hit different level accumulators,
          // and each k-step needs only 6 A addresses, 6 B descriptors, 7 D addresses
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
            for (int p = 1; p <= I8_ND; ++p) {
#pragma unroll
              for (int q = 1; q <= I8_ND; ++q) {
                if (p + q > I8_LMAX) continue;
                const int l = p + q;
                // the first pair of level l (at k-step 0) overwrites the accumulator
                const bool first = ks == 0 && ((p == 1) || (l > I8_ND + 1 && p == l - I8_ND));
                // A = C digits (q: all signed when balanced), B = X digits (p: top one signed)
                const uint32_t idesc = uz + idesc_i8(I8_TBAL ? true : q == 1, p == 1);
                const uint64_t bdesc = desc0 + (uint64_t)(((p - 1) * I8_PLANE_BYTES + 32 * ks) >> 4);
                const uint32_t atm = uz + (uint32_t)(32 * (q - 1) + 8 * ks);
                umma_i8_ts(dacc + (uint32_t)((l - 2) * I8_CHUNK), atm, bdesc, idesc, first ? 0u : 1u);
              }
            }
          }
        }
        umma_commit_elect(&afull[ab]);
        if (lane == 0) I8_TRACE(it, 9 + 2 * c);
        __syncwarp();
      }
      umma_commit_elect(&xempty[buf]);
      if (lane == 0) I8_TRACE(it, 4);
      __syncwarp();
    }
  } else {
    // ---- slicer warps: rows 16w .. 16w+15 of each tile, from the smem stage ----
    // k = e + fT - 50 with e = bc - 1022 (T scale 2^(47-fT)); one more with balanced T digits
    const int kbias = fT - (I8_TBAL ? 1071 : 1072);
    for (int64_t it = 0; it < my_tiles; ++it) {
      const int buf = (int)(it % I8_NBUF);
      i8_wait_a(sfull_a + 8u * (uint32_t)(buf), (uint32_t)((it / I8_NBUF) & 1));
      if (sw == 0 && lane == 0) I8_TRACE(it, 1);
      if (it >= I8_NBUF) i8_wait_a(xempty_a + 8u * (uint32_t)(buf), (uint32_t)(((it / I8_NBUF) - 1) & 1));
      if (sw == 0 && lane == 0) I8_TRACE(it, 7);
      bool wslow = false;
      unsigned char* planes = xdig + buf * I8_XBUF_BYTES;
      const double* xs = stage + buf * I8_TILE * I8_N;
      if (!(dbg & 2)) {
        // rows in flight (independent load -> max -> split chains); fewer when the
        // 16-epilogue-warp layout caps registers near 88 per thread
        constexpr int RG_MAX = I8_THREADS > 512 ? 4 : 8;
        constexpr int RG = (I8_TILE / I8_SLICE_WARPS) < RG_MAX ? (I8_TILE / I8_SLICE_WARPS) : RG_MAX;
#pragma unroll 1
        for (int rb = 0; rb < I8_TILE / I8_SLICE_WARPS; rb += RG) {
          double xv[RG][4];
          uint32_t m[RG];
#pragma unroll
          for (int u = 0; u < RG; ++u) {
            const int r = (I8_TILE / I8_SLICE_WARPS) * sw + rb + u;
            // k = 2l, 2l+1 and 64+2l, 65+2l (i8_kperm): two conflict-free 512 B rows
            const double2 a0 = *reinterpret_cast<const double2*>(xs + r * I8_N + 2 * lane);
            const double2 a1 = *reinterpret_cast<const double2*>(xs + r * I8_N + 64 + 2 * lane);
            xv[u][0] = a0.x; xv[u][1] = a0.y; xv[u][2] = a1.x; xv[u][3] = a1.y;
          }
#pragma unroll
          for (int u = 0; u < RG; ++u) {
            // max exponent of the row from the high words of |x| (exact for the exponent)
            m[u] = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) m[u] = max(m[u], (uint32_t)__double2hiint(xv[u][b]) & 0x7fffffffu);
          }
#pragma unroll
          for (int u = 0; u < RG; ++u) m[u] = __reduce_max_sync(0xffffffffu, m[u]);  // one REDUX per row
          // Tiny rows (max|x| < 2^-977, including subnormals) would need a scale above
          // the fp64 range: rescale them exactly by 2^600 first (warp-uniform, rare), and
          // take the 600 back out of their exponent shift k.
          int tsh[RG];
          bool anytiny = false;
#pragma unroll
          for (int u = 0; u < RG; ++u) {
            tsh[u] = 0;
            anytiny |= (m[u] != 0u) & ((m[u] >> 20) < 46u);
          }
          if (anytiny) {
#pragma unroll
            for (int u = 0; u < RG; ++u) {
              if ((m[u] != 0u) & ((m[u] >> 20) < 46u)) {
                uint32_t mm = 0;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                  xv[u][b] *= 0x1p600;
                  mm = max(mm, (uint32_t)__double2hiint(xv[u][b]) & 0x7fffffffu);
                }
                m[u] = __reduce_max_sync(0xffffffffu, mm);
                tsh[u] = 600;
              }
            }
          }
#pragma unroll
          for (int u = 0; u < RG; ++u) {
            const int r = (I8_TILE / I8_SLICE_WARPS) * sw + rb + u;
            const int bexp = (int)(m[u] >> 20);  // biased exponent of max|x|
            // Branch-free (so the RG rows interleave): with the biased exponent
            // clamped to bc, scale = 2^(47-e) and rs = 2^(e-30), e = bc - 1022.
            //  * zero row: any finite scale (the digits are 0 and X^A = X exactly);
            //  * tiny rows were rescaled by 2^600 above (bexp >= 46 now);
            //  * non-finite row: the digits are don't-care and rs = NaN makes the
            //    row NaN, what x T gives in fp64.
            const bool finite_row = bexp != 0x7ff;
            const int bc = (m[u] == 0) ? 1023 : max(bexp, 46);
            const double scale = __longlong_as_double((long long)(2092 - bc) << 52);
            const double rs = finite_row ? __longlong_as_double((long long)(bc - 29) << 52)
                                         : __longlong_as_double(0x7ff8000000000000ll);
            // round(x 2^(47-e)) as a 48-bit integer: the low word of fma(x, s, 1.5 2^52)
            // is the low word of the integer, the high word is offset by 0x43380000
            uint32_t vlo[4], vhi[4];
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              const double t = fma(xv[u][b], scale, 6755399441055744.0);
              vlo[b] = (uint32_t)__double2loint(t);
              vhi[b] = (uint32_t)__double2hiint(t) - 0x43380000u;
            }
            // K-major, 128B-swizzled row r: 16-byte chunk (lane/4) ^ (r%8), word lane%4
            const uint32_t off = (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + (((lane >> 2) ^ (r & 7)) << 4) +
                                            ((lane & 3) << 2));
            // digit plane p = byte 5-p of the 48-bit values, packed 4 per word.
            // Two planes per 4 PRMT: A = [v0.bi, v1.bi, v0.bj, v1.bj],
            // B = [v2.bi, v3.bi, v2.bj, v3.bj] -> plane i = (A,B)[0,1,4,5], j = [2,3,6,7]
            auto two_planes = [&](uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3, uint32_t bi, uint32_t bj,
                                  uint32_t& wi, uint32_t& wj) {
              const uint32_t sel = bi | ((bi + 4u) << 4) | (bj << 8) | ((bj + 4u) << 12);
              const uint32_t A = __byte_perm(x0, x1, sel);
              const uint32_t B = __byte_perm(x2, x3, sel);
              wi = __byte_perm(A, B, 0x5410);
              wj = __byte_perm(A, B, 0x7632);
            };
            uint32_t w[I8_ND];
            two_planes(vhi[0], vhi[1], vhi[2], vhi[3], 1u, 0u, w[0], w[1]);  // bytes 5, 4
            two_planes(vlo[0], vlo[1], vlo[2], vlo[3], 3u, 2u, w[2], w[3]);  // bytes 3, 2
            two_planes(vlo[0], vlo[1], vlo[2], vlo[3], 1u, 0u, w[4], w[5]);  // bytes 1, 0
#pragma unroll
            for (int p = 0; p < I8_ND; ++p) *reinterpret_cast<uint32_t*>(planes + p * I8_PLANE_BYTES + off) = w[p];
            const int kv = finite_row ? bc + kbias - tsh[u] : INT_MIN;
            wslow |= (kv < -1022) | (kv > 961);  // outside the exponent-field fast path
            if (lane == 0) rinfo[(int)(it % (2 * I8_NBUF)) * I8_TILE + r] = kv;
          }
        }
      }
      if (lane == 0) rflag[(int)(it % (2 * I8_NBUF)) * I8_SLICE_WARPS + sw] = wslow;
      fence_proxy_async();
      if (sw == 0 && lane == 0) I8_TRACE(it, 2);
      i8_arrive_a(xfull_a + 8u * (uint32_t)(buf));
      i8_arrive_a(rfull_a + 8u * (uint32_t)(it % (2 * I8_NBUF)));
      i8_arrive_a(sempty_a + 8u * (uint32_t)(buf));
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
