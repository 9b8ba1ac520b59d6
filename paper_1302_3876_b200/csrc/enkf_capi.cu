// enkf_capi.cu — the C ABI (include/enkf_b200.h) over the sm_100a kernels.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <type_traits>
#include <cmath>
#include <cstdio>
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <new>
#include <thread>
#include <vector>

#include "../../include/enkf_b200.h"
#include "enkf_kernels.cuh"
#include "anomaly_i8.cuh"
#include "localized.cuh"
#include "l96.cuh"
#include "gram_i8.cuh"
#include "host_stream.cuh"
#include "tiny.cuh"
#include "nccl_comm.cuh"
#include "levels_cluster.cuh"

using namespace enkf;

struct enkf_plan {
  int64_t n_state = 0, n_obs = 0;
  int n = 0;
  int device = 0;
  int num_sms = 0;
  int splits = 1;
  int64_t rows_per_split = 0;
  bool use_ws = true;          // warp-specialised TMA kernels (even N, aligned rows)
  bool use_128 = true;         // N == 128 specialisation of the Gram pass
  bool anomaly_i8 = true;      // tensor-core (int8 digit) anomaly update, N == 128
  int i8_dbg = 0;              // profiling-only role skips (ENKF_I8_DBG)
  bool levels_blocked = true;  // blocked (LB levels per barrier) Sherman-Morrison recursion
  bool levels_cluster = true;  // ... on a 4-CTA cluster (ENKF_LEVELS=single: one CTA; =level: level by level)
  bool host_streamed = true;   // pipelined host path for pinned X / XA (ENKF_HOST_STREAM=0 disables)
  size_t host_chunk_bytes = (size_t)256 << 20;
  bool host_trace = false;      // ENKF_HOST_TRACE=1: phase times of the streamed host path on stderr
  bool gram_i8 = true;         // tensor-core (int8 digit) Gram, N == 128 analysis mode (ENKF_GRAM=fp64: DMMA)
  int g8_groups = 0;           // groups of 4 CTAs over the observation rows
  double* g8_sr = nullptr;                // [n_obs] sqrt(1/r) of the call's observation rows
  double* g8_ls_partial = nullptr;        // [groups][4][256][128] (level-split form)
  int* g8_ls_progress = nullptr;          // [groups][4] blocks issued per CTA (level-split pacing)
  bool loc_dmma = true;                   // localized update on FP64 DMMA (ENKF_LOCALIZED=fma: CUDA-core form)
  bool tiny = true;                       // desk-scale problems: the whole step in one CTA (ENKF_TINY=0: off)
  char* small_h = nullptr;                // host path for small problems: page-locked staging block
  char* small_d = nullptr;                // and its device twin
  bool g8_events = false;                 // measurement: events around the slice and MMA passes
  cudaEvent_t g8_ev[3] = {nullptr, nullptr, nullptr};
  unsigned char* g8_planes = nullptr;     // [ceil(n_obs/32)][48 KiB] digit-plane operand images (two-kernel form)
  unsigned long long* g8_meta = nullptr;  // [256] sampled column maxima, then the overflow flag
  int ws_blocks = 1, ws_ctas_per_block = 1;
  int64_t ws_rows_per_cta = 0;
  int g128_cpb_vv = 1, g128_cpb_vd = 1;     // gram128: CTAs for the V'V / V'D blocks
  int64_t g128_rows_vv = 0, g128_rows_vd = 0;
  double* partial = nullptr;  // [splits][n][2n]
  double* gram = nullptr;     // [n][2n]
  double* A = nullptr;        // [n][n]
  double* T = nullptr;        // [n][n]
  double* den = nullptr;      // [n]
  DevStatus* dstatus = nullptr;
  DevStatus* hstatus = nullptr;  // pinned
  // host-path staging (lazily allocated)
  double* hx = nullptr;
  double* hy = nullptr;
  double* hr = nullptr;
  int64_t* hidx = nullptr;
  cudaStream_t hstream = nullptr;
  // streamed host path (pinned X and XA): compact observed rows, copy streams,
  // one event per X chunk
  double* hxo = nullptr;
  cudaStream_t hs_in = nullptr, hs_out = nullptr;
  cudaEvent_t ev_obs = nullptr, ev_anom = nullptr;
  std::vector<cudaEvent_t> chunk_ev;
  // pinned staging rings for pageable host buffers (ring: inbound / any; oring: X^A outbound)
  char* oring[2] = {nullptr, nullptr};
  cudaEvent_t oring_ev[2] = {nullptr, nullptr};
  size_t pageable_stream_min = (size_t)1 << 30;  // X bytes from which pageable calls stream (ENKF_HOST_STREAM_MIN_MB)
  char* ring[2] = {nullptr, nullptr};
  cudaEvent_t ring_ev[2] = {nullptr, nullptr};
  bool ring_busy[2] = {false, false};  // an async DMA may still touch the slot
  int ring_next = 0;
  size_t ring_bytes = 0;
  size_t ring_bytes_cfg = (size_t)256 << 20;  // slot size (ENKF_HOST_RING_MB; small values for tests)
  // localized-analysis workspace (lazily allocated): V, D, Z [n_obs][n]
  double* locV = nullptr;
  double* locD = nullptr;
  double* locZ = nullptr;
  // Lorenz-96 forecast workspace for rings too long for shared memory: 3 x [n_state][n]
  double* l96ws = nullptr;
  DevStatus* cyc_status = nullptr;  // per-cycle status of enkf_cycle_l96_f64
  int cyc_cap = 0;
  // multi-GPU: the NCCL communicator of this shard (caller-owned) and the last NCCL error
  ncclComm_t comm = nullptr;
  int comm_ranks = 1, comm_rank = 0;
  int nccl_rc = 0;
  // measurement: events at the stage boundaries of the analysis step
  bool stage_events = false;
  static constexpr int ST_SETS = 64;  // stage-event sets: one per step, a ring (the last 64 steps are kept)
  cudaEvent_t st_evs[ST_SETS][5] = {};
  cudaEvent_t* st_ev = st_evs[0];     // the set the current step records into
  long st_steps = 0;                  // steps recorded since the events were switched on
};

namespace {

const char* kVersion = "enkf_b200 0.1.0 sm_100a";
constexpr size_t kSmallHostBytes = (size_t)1 << 20;  // small-problem host path: all inputs <= 1 MiB

// NVTX range for the host-side phases (visible in Nsight Systems; header-only, no
// library dependency, no cost without a profiler attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

void set_status(enkf_status* st, int code, const char* fmt, ...) {
  if (!st) return;
  st->code = code;
  st->level = 0;
  st->denominator = 0.0;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(st->message, sizeof(st->message), fmt, ap);
  va_end(ap);
}

int cuda_fail(enkf_status* st, cudaError_t e, const char* where) {
  set_status(st, ENKF_CUDA_ERROR, "%s: %s", where, cudaGetErrorString(e));
  return ENKF_CUDA_ERROR;
}

#define CUDA_TRY(expr, st)                                  \
  do {                                                      \
    cudaError_t _e = (expr);                                \
    if (_e != cudaSuccess) return cuda_fail(st, _e, #expr); \
  } while (0)

inline bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

template <bool ANALYSIS, bool VEC16>
cudaError_t launch_gram_t(const enkf_plan* p, const double* X, const double* Y,
                          const int64_t* idx, const double* r, cudaStream_t s) {
  const int n = p->n;
  const int ld = padded_ld(n);
  dim3 grid((2 * n + G_BN - 1) / G_BN, (n + G_BM - 1) / G_BM, p->splits);
  const size_t smem = (size_t)(2 * G_STAGES * G_RT * ld + 2 * G_STAGES * G_RT) * sizeof(double);
  auto kern = gram_kernel<ANALYSIS, VEC16>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, G_THREADS, smem, s>>>(X, Y, idx, r, p->n_state, p->n_obs, n, ld, p->rows_per_split,
                                      p->partial, p->dstatus);
  return cudaGetLastError();
}

template <bool ANALYSIS>
cudaError_t launch_gram_ws_t(const enkf_plan* p, const double* X, const double* Y,
                             const int64_t* idx, const double* r, cudaStream_t s) {
  const int n = p->n;
  if (n == W_TILE && p->use_128) {
    const int ld = padded_ld(W_TILE);
    const size_t smem = gram128_smem_bytes(ld);
    auto kern = gram128_kernel<ANALYSIS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<p->g128_cpb_vv + p->g128_cpb_vd, 32 * (G128_MMA_WARPS + 4), smem, s>>>(
        X, Y, idx, r, p->n_state, p->n_obs, ld, p->g128_cpb_vv, p->g128_rows_vv, p->g128_rows_vd,
        p->partial, p->dstatus, nullptr);
    return cudaGetLastError();
  }
  const int ld = padded_ld(W_TILE);  // operand tiles are 128 wide whatever n is
  const size_t smem = gram_ws_smem_bytes(ld);
  auto kern = gram_ws_kernel<ANALYSIS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<p->ws_blocks * p->ws_ctas_per_block, W_THREADS, smem, s>>>(
      X, Y, idx, r, p->n_state, p->n_obs, n, ld, p->ws_ctas_per_block, p->ws_rows_per_cta, p->partial,
      p->dstatus);
  return cudaGetLastError();
}

bool use_ws(const enkf_plan* p, const void* a, const void* b) {
  return p->use_ws && (p->n % 2 == 0) && aligned16(a) && aligned16(b);
}

cudaError_t launch_gram_i8(enkf_plan* p, const double* X, const double* Y, const int64_t* idx,
                           const double* r, double* gram, cudaStream_t s);

cudaError_t launch_gram(enkf_plan* p, bool analysis, const double* X, const double* Y,
                        const int64_t* idx, const double* r, double* gram, cudaStream_t s) {
  const int n = p->n;
  if (p->n_obs == 0) return cudaMemsetAsync(gram, 0, sizeof(double) * n * 2 * n, s);
  if (analysis && n == G8_N && p->gram_i8 && p->use_128 && use_ws(p, X, Y))
    return launch_gram_i8(p, X, Y, idx, r, gram, s);
  if (use_ws(p, X, Y)) {
    cudaError_t e = analysis ? launch_gram_ws_t<true>(p, X, Y, idx, r, s)
                             : launch_gram_ws_t<false>(p, X, Y, idx, r, s);
    if (e != cudaSuccess) return e;
    const double svv = analysis ? 1.0 / (double)(n - 1) : 1.0;
    const double svd = analysis ? 1.0 / std::sqrt((double)(n - 1)) : 1.0;
    const int64_t count = (int64_t)n * 2 * n;
    if (n == W_TILE && p->use_128)
      gram128_reduce<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(p->partial, p->g128_cpb_vv,
                                                                     p->g128_cpb_vd, svv, svd, gram, nullptr);
    else
      gram_ws_reduce<<<(unsigned)((count + 31) / 32), 32 * GWR_SPLIT, 0, s>>>(p->partial, n, p->ws_ctas_per_block,
                                                                            svv, svd, gram);
    return cudaGetLastError();
  }
  const bool vec = (n % 2 == 0) && aligned16(X) && aligned16(Y);
  cudaError_t e;
  if (analysis) e = vec ? launch_gram_t<true, true>(p, X, Y, idx, r, s) : launch_gram_t<true, false>(p, X, Y, idx, r, s);
  else e = vec ? launch_gram_t<false, true>(p, X, Y, idx, r, s) : launch_gram_t<false, false>(p, X, Y, idx, r, s);
  if (e != cudaSuccess) return e;
  const double svv = analysis ? 1.0 / (double)(n - 1) : 1.0;
  const double svd = analysis ? 1.0 / std::sqrt((double)(n - 1)) : 1.0;
  const int64_t count = (int64_t)n * 2 * n;
  gram_reduce<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(p->partial, p->splits, n, svv, svd, gram);
  return cudaGetLastError();
}

// Workspace of the int8 Gram for the plan's shape (allocated by enkf_plan_create
// when the int8 Gram is the plan's analysis Gram, so the compute calls allocate
// nothing and a CUDA-graph capture needs no warm-up call).
cudaError_t ensure_gram_i8_workspace(enkf_plan* p) {
  cudaError_t e = cudaSuccess;
  const int64_t n_blocks = (p->n_obs + G8_KB - 1) / G8_KB;
  if (!p->g8_meta && (e = cudaMalloc(&p->g8_meta, sizeof(unsigned long long) * (2 * G8_N + 2))) != cudaSuccess)
    return e;
  if (!p->g8_planes && n_blocks > 0 &&
      (e = cudaMalloc(&p->g8_planes, (size_t)n_blocks * G8_BLOCK_BYTES)) != cudaSuccess)
    return e;
  if (!p->g8_sr && p->n_obs > 0 && (e = cudaMalloc(&p->g8_sr, sizeof(double) * (size_t)p->n_obs)) != cudaSuccess)
    return e;
  if (!p->g8_ls_partial &&
      (e = cudaMalloc(&p->g8_ls_partial, sizeof(double) * (size_t)p->g8_groups * 4 * 2 * G8_N * G8_N)) != cudaSuccess)
    return e;
  if (!p->g8_ls_progress &&
      (e = cudaMalloc(&p->g8_ls_progress, sizeof(int) * 4 * p->g8_groups)) != cudaSuccess)
    return e;
  return cudaSuccess;
}

// int8 tensor-core Gram (gram_i8.cuh): sampled column scales, the slice pass
// (operand images in HBM), the MMA pass, the reduce, and the FP64 gram128 pass
// gated on the overflow flag.
cudaError_t launch_gram_i8(enkf_plan* p, const double* X, const double* Y, const int64_t* idx,
                           const double* r, double* gram, cudaStream_t s) {
  const int n = p->n;
  cudaError_t e = cudaSuccess;
  const int64_t n_blocks = (p->n_obs + G8_KB - 1) / G8_KB;
  if ((e = ensure_gram_i8_workspace(p)) != cudaSuccess) return e;
  int* overflow = reinterpret_cast<int*>(p->g8_meta + 2 * G8_N);
  if ((e = cudaMemsetAsync(p->g8_meta, 0, sizeof(unsigned long long) * (2 * G8_N + 2), s)) != cudaSuccess) return e;
  gram_i8_scales_kernel<<<p->num_sms * 2, 256, 0, s>>>(X, Y, idx, r, p->n_state, p->n_obs, p->g8_meta);
  const int64_t bpg = (n_blocks + p->g8_groups - 1) / p->g8_groups;
  if (p->g8_events) {
    for (cudaEvent_t& ev : p->g8_ev)
      if (!ev && (e = cudaEventCreate(&ev)) != cudaSuccess) return e;
    cudaEventRecord(p->g8_ev[0], s);
  }
  const size_t smem = gram_i8_slice_smem_bytes();
  if ((e = cudaFuncSetAttribute(gram_i8_slice_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
      cudaSuccess)
    return e;
  // 2 CTAs per SM are resident (120 registers x 256 threads): one full wave, no tail
  const int64_t grid = std::min<int64_t>(n_blocks, (int64_t)p->num_sms * G8_SLICE_CTAS_PER_SM);
  gram_i8_sqrt_rho_kernel<<<(unsigned)std::min<int64_t>((p->n_obs + 255) / 256, (int64_t)p->num_sms * 8), 256, 0, s>>>(
      r, p->n_obs, p->g8_sr, p->dstatus);
  gram_i8_slice_kernel<<<(unsigned)grid, G8_SLICE_THREADS, smem, s>>>(X, Y, idx, p->g8_sr, p->g8_meta, p->n_state,
                                                                       p->n_obs, n_blocks, p->g8_planes, overflow,
                                                                       p->dstatus);
  if (p->g8_events) cudaEventRecord(p->g8_ev[1], s);
  const size_t lsmem = gram_i8_ls_smem_bytes();
  if ((e = cudaFuncSetAttribute(gram_i8_mma_ls_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsmem)) !=
      cudaSuccess)
    return e;
  if ((e = cudaMemsetAsync(p->g8_ls_progress, 0, sizeof(int) * 4 * p->g8_groups, s)) != cudaSuccess) return e;
  gram_i8_mma_ls_kernel<<<4 * p->g8_groups, G8LS_THREADS, lsmem, s>>>(p->g8_planes, p->g8_meta, n_blocks, bpg,
                                                                      p->g8_ls_partial, overflow, p->g8_ls_progress);
  if (p->g8_events) cudaEventRecord(p->g8_ev[2], s);
  const double svv = 1.0 / (double)(n - 1), svd = 1.0 / std::sqrt((double)(n - 1));
  gram_i8_ls_reduce<<<(2 * G8_N * G8_N + 255) / 256, 256, 0, s>>>(p->g8_ls_partial, p->g8_groups, svv, svd, overflow,
                                                                  gram);
  // FP64 fallback, a no-op unless an element fell outside the sampled scales
  {
    const int ld = padded_ld(W_TILE);
    const size_t gsmem = gram128_smem_bytes(ld);
    auto kern = gram128_kernel<true>;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsmem)) != cudaSuccess)
      return e;
    kern<<<p->g128_cpb_vv + p->g128_cpb_vd, 32 * (G128_MMA_WARPS + 4), gsmem, s>>>(X, Y, idx, r, p->n_state, p->n_obs, ld, p->g128_cpb_vv,
                                                                   p->g128_rows_vv, p->g128_rows_vd, p->partial,
                                                                   p->dstatus, overflow);
    gram128_reduce<<<(2 * G8_N * G8_N + 255) / 256, 256, 0, s>>>(p->partial, p->g128_cpb_vv, p->g128_cpb_vd, svv,
                                                                 svd, gram, overflow);
  }
  return cudaGetLastError();
}

// The analysis step's Gram over ALL observation rows into p->gram: the local pass,
// then (a communicator attached) one in-place ncclAllReduce of [Gram | input-check
// flags] on the compute stream and the reduced flags folded back into the status,
// so every rank runs the levels on the same Gram and reports the same outcome.
cudaError_t launch_gram_global(enkf_plan* p, const double* X, const double* Y, const int64_t* idx,
                               const double* r, cudaStream_t s) {
  cudaError_t e = launch_gram(p, true, X, Y, idx, r, p->gram, s);
  if (e != cudaSuccess || !p->comm) return e;
  const size_t count = (size_t)2 * p->n * p->n + COMM_FLAG_SLOTS;
  double* tail = p->gram + (size_t)2 * p->n * p->n;
  comm_pack_flags<<<1, 32, 0, s>>>(p->dstatus, tail);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (p->stage_events) cudaEventRecord(p->st_ev[1], s);
  const ncclResult_t rc = nccl_api().all_reduce(p->gram, p->gram, count, ncclFloat64, ncclSum, p->comm, s);
  if (rc != ncclSuccess) {
    p->nccl_rc = (int)rc;
    return cudaErrorUnknown;
  }
  if (p->stage_events) cudaEventRecord(p->st_ev[2], s);
  comm_unpack_flags<<<1, 32, 0, s>>>(tail, p->dstatus);
  return cudaGetLastError();
}

// Desk-scale analysis in one CTA (tiny.cuh); flags into p->dstatus.
cudaError_t launch_tiny(const enkf_plan* p, const double* X, const double* Y, const int64_t* idx, const double* r,
                        double* XA, cudaStream_t s) {
  const size_t smem = (size_t)tiny_smem_doubles(p->n_obs, p->n) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(analysis_tiny_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  analysis_tiny_kernel<<<1, TINY_THREADS, smem, s>>>(X, Y, idx, r, XA, p->n_state, p->n_obs, p->n,
                                                     std::sqrt((double)(p->n - 1)), p->dstatus);
  return cudaGetLastError();
}

cudaError_t launch_levels(const enkf_plan* p, const double* gram, double* A, double* T,
                          double* den, double cscale, cudaStream_t s) {
  if (p->levels_cluster && p->n >= 2 && p->n <= 128) {
    // the blocked recursion on a cluster of LC_CTAS CTAs (levels_cluster.cuh)
    const size_t smem = (size_t)levels_cluster_smem_doubles(p->n) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(ism_levels_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(LC_CTAS);
    cfg.blockDim = dim3(LC_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = LC_CTAS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, ism_levels_cluster_kernel, gram, p->n, cscale, A, T, den, p->dstatus);
    if (e == cudaSuccess) return e;
    // a context that cannot place a 4-CTA cluster (SM-limited partitions, MPS):
    // the one-CTA kernel computes the same bits
    cudaGetLastError();
  }
  if (p->levels_blocked) {
    const size_t smem = (size_t)levels_blk_smem_doubles(p->n) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(ism_levels_blocked_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    ism_levels_blocked_kernel<<<1, LV_THREADS, smem, s>>>(gram, p->n, cscale, A, T, den, p->dstatus);
    return cudaGetLastError();
  }
  const size_t smem = (size_t)levels_smem_doubles(p->n) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(ism_levels_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  ism_levels_kernel<<<1, 1024, smem, s>>>(gram, p->n, cscale, A, T, den, p->dstatus);
  return cudaGetLastError();
}

template <int NP, int MODE, bool VEC16>
cudaError_t launch_rowgemm_t(const enkf_plan* p, const double* P, const double* Q, const double* C,
                             const double* r, double* out, int64_t n_rows, cudaStream_t s) {
  const int n = p->n;
  const int ld = padded_ld(NP);  // the k loop reads NP >= n columns
  const size_t smem = (size_t)R_STAGES * R_ROWS * ld * sizeof(double);
  auto kern = rowgemm_kernel<NP, MODE, VEC16>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t ntiles = (n_rows + R_ROWS - 1) / R_ROWS;
  int grid = (int)(ntiles < p->num_sms ? ntiles : p->num_sms);
  if (grid < 1) return cudaSuccess;
  kern<<<grid, R_THREADS, smem, s>>>(P, Q, C, r, out, n_rows, n, ld);
  return cudaGetLastError();
}

template <int NP, int MODE>
cudaError_t launch_rowgemm_ws_t(const enkf_plan* p, const double* P, const double* Q, const double* C,
                                const double* r, double* out, int64_t n_rows, cudaStream_t s) {
  const int n = p->n;
  const int ld = padded_ld(NP);  // the k loop reads NP >= n columns
  const size_t smem = (size_t)R_STAGES * R_ROWS * ld * sizeof(double) + 2 * R_STAGES * sizeof(uint64_t);
  auto kern = rowgemm_ws_kernel<NP, MODE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t ntiles = (n_rows + R_ROWS - 1) / R_ROWS;
  int grid = (int)(ntiles < p->num_sms ? ntiles : p->num_sms);
  if (grid < 1) return cudaSuccess;
  kern<<<grid, R_THREADS, smem, s>>>(P, Q, C, r, out, n_rows, n, ld);
  return cudaGetLastError();
}

cudaError_t launch_anomaly_i8(const enkf_plan* p, const double* X, const double* T, double* XA,
                              int64_t n_rows, cudaStream_t s) {
  const size_t smem = anomaly_i8_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(anomaly_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t ntiles = (n_rows + I8_TILE - 1) / I8_TILE;
  const int grid = (int)(ntiles < p->num_sms ? ntiles : p->num_sms);
  if (grid < 1) return cudaSuccess;
  anomaly_i8_kernel<<<grid, I8_THREADS, smem, s>>>(X, T, XA, n_rows, p->i8_dbg, 0u);
  return cudaGetLastError();
}

template <int MODE>
cudaError_t launch_rowgemm(const enkf_plan* p, const double* P, const double* Q, const double* C,
                           const double* r, double* out, int64_t n_rows, cudaStream_t s) {
  const int n = p->n;
  if (MODE == 0 && p->anomaly_i8 && n == I8_N && aligned16(P) && aligned16(out))
    return launch_anomaly_i8(p, P, Q, out, n_rows, s);
  if (use_ws(p, P, out) && (C == nullptr || aligned16(C))) {
#define ENKF_RW(NPV) \
    if (n <= NPV) return launch_rowgemm_ws_t<NPV, MODE>(p, P, Q, C, r, out, n_rows, s);
    ENKF_RW(8) ENKF_RW(16) ENKF_RW(32) ENKF_RW(48) ENKF_RW(64) ENKF_RW(96) ENKF_RW(128)
#undef ENKF_RW
  }
  const bool vec = (n % 2 == 0) && aligned16(P) && aligned16(out) && (C == nullptr || aligned16(C));
#define ENKF_RG(NPV)                                                                   \
  if (n <= NPV) return vec ? launch_rowgemm_t<NPV, MODE, true>(p, P, Q, C, r, out, n_rows, s) \
                           : launch_rowgemm_t<NPV, MODE, false>(p, P, Q, C, r, out, n_rows, s);
  ENKF_RG(8) ENKF_RG(16) ENKF_RG(32) ENKF_RG(48) ENKF_RG(64) ENKF_RG(96) ENKF_RG(128)
#undef ENKF_RG
  return cudaErrorInvalidValue;
}

// ---- host <-> device copies for the host-buffer entry point -----------------
// Pinned (page-locked or registered) host buffers are DMA'd directly.  Pageable
// buffers go through a 2 x 256 MiB pinned ring: the host side is copied by a
// pool of threads (first-touch page faults of fresh numpy arrays are the real
// cost of pageable transfers and parallelise), the DMA of one ring slot
// overlaps the host copy of the other.
bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void parallel_memcpy(void* dst, const void* src, size_t bytes) {
  const size_t min_chunk = (size_t)8 << 20;
  unsigned nt = std::thread::hardware_concurrency();
  if (nt == 0) nt = 1;
  if (nt > 16) nt = 16;
  size_t want = (bytes + min_chunk - 1) / min_chunk;
  if (want < nt) nt = (unsigned)(want ? want : 1);
  if (nt <= 1) {
    memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> th;
  const size_t per = (bytes + nt - 1) / nt;
  for (unsigned t = 0; t < nt; ++t) {
    const size_t lo = t * per;
    if (lo >= bytes) break;
    const size_t len = (lo + per > bytes) ? bytes - lo : per;
    th.emplace_back([=] { memcpy((char*)dst + lo, (const char*)src + lo, len); });
  }
  for (auto& t : th) t.join();
}

cudaError_t ensure_ring(enkf_plan* p) {
  if (p->ring[0]) return cudaSuccess;
  p->ring_bytes = p->ring_bytes_cfg;
  for (int i = 0; i < 2; ++i) {
    cudaError_t e = cudaMallocHost(&p->ring[i], p->ring_bytes);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ring_ev[i], cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// Take the next ring slot, waiting until its previous DMA (of any direction,
// from this or an earlier call) has completed.
cudaError_t take_slot(enkf_plan* p, int* slot) {
  *slot = p->ring_next;
  p->ring_next ^= 1;
  if (p->ring_busy[*slot]) {
    cudaError_t e = cudaEventSynchronize(p->ring_ev[*slot]);
    if (e != cudaSuccess) return e;
    p->ring_busy[*slot] = false;
  }
  return cudaSuccess;
}

cudaError_t copy_h2d(enkf_plan* p, void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return cudaSuccess;
  if (is_pinned(src)) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
  cudaError_t e = ensure_ring(p);
  if (e != cudaSuccess) return e;
  for (size_t off = 0; off < bytes;) {
    const size_t len = bytes - off < p->ring_bytes ? bytes - off : p->ring_bytes;
    int slot;
    if ((e = take_slot(p, &slot)) != cudaSuccess) return e;
    parallel_memcpy(p->ring[slot], (const char*)src + off, len);
    if ((e = cudaMemcpyAsync((char*)dst + off, p->ring[slot], len, cudaMemcpyHostToDevice, s)) != cudaSuccess) return e;
    if ((e = cudaEventRecord(p->ring_ev[slot], s)) != cudaSuccess) return e;
    p->ring_busy[slot] = true;
    off += len;
  }
  return cudaSuccess;
}

cudaError_t copy_d2h(enkf_plan* p, void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return cudaSuccess;
  if (is_pinned(dst)) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s);
  cudaError_t e = ensure_ring(p);
  if (e != cudaSuccess) return e;
  const size_t nchunks = (bytes + p->ring_bytes - 1) / p->ring_bytes;
  int slot_of[2] = {0, 0};
  auto launch = [&](size_t k) -> cudaError_t {
    const size_t off = k * p->ring_bytes;
    const size_t len = bytes - off < p->ring_bytes ? bytes - off : p->ring_bytes;
    int slot;
    cudaError_t err = take_slot(p, &slot);
    if (err != cudaSuccess) return err;
    slot_of[k & 1] = slot;
    if ((err = cudaMemcpyAsync(p->ring[slot], (const char*)src + off, len, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return err;
    if ((err = cudaEventRecord(p->ring_ev[slot], s)) != cudaSuccess) return err;
    p->ring_busy[slot] = true;
    return cudaSuccess;
  };
  // keep up to two chunks in flight; drain in order
  for (size_t k = 0; k < nchunks && k < 2; ++k)
    if ((e = launch(k)) != cudaSuccess) return e;
  for (size_t k = 0; k < nchunks; ++k) {
    const int slot = slot_of[k & 1];
    const size_t off = k * p->ring_bytes;
    const size_t len = bytes - off < p->ring_bytes ? bytes - off : p->ring_bytes;
    if ((e = cudaEventSynchronize(p->ring_ev[slot])) != cudaSuccess) return e;
    p->ring_busy[slot] = false;
    parallel_memcpy((char*)dst + off, p->ring[slot], len);
    if (k + 2 < nchunks && (e = launch(k + 2)) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// Rows idx[0..nrows) of the row-major [*][row_bytes] host array src, gathered into
// dst by a pool of threads (the observed rows of a pageable X).
void parallel_gather_rows(char* dst, const char* src, const int64_t* idx, int64_t nrows, size_t row_bytes) {
  unsigned nt = std::thread::hardware_concurrency();
  if (nt == 0) nt = 1;
  if (nt > 16) nt = 16;
  if ((int64_t)nt > nrows / 1024) nt = (unsigned)(nrows / 1024 > 0 ? nrows / 1024 : 1);
  auto run = [=](int64_t lo, int64_t hi) {
    for (int64_t k = lo; k < hi; ++k) memcpy(dst + (size_t)k * row_bytes, src + (size_t)idx[k] * row_bytes, row_bytes);
  };
  if (nt <= 1) {
    run(0, nrows);
    return;
  }
  std::vector<std::thread> th;
  const int64_t per = (nrows + nt - 1) / nt;
  for (unsigned t = 0; t < nt; ++t) {
    const int64_t lo = t * per, hi = lo + per < nrows ? lo + per : nrows;
    if (lo >= hi) break;
    th.emplace_back(run, lo, hi);
  }
  for (auto& t : th) t.join();
}

int translate_status(const enkf_plan* p, enkf_status* st) {
  const DevStatus& d = *p->hstatus;
  if (d.flags & FLAG_DIVERGED) {  // the forecast precedes the analysis of its cycle
    const unsigned long long key = ~(unsigned long long)d.bad_index;
    const int member = (int)(key & 0xffffffffu);
    set_status(st, ENKF_DIVERGED, "state became non-finite (ensemble member %d, step %d)", member,
               (int)(key >> 32));
    if (st) st->level = member;
    return ENKF_DIVERGED;
  }
  if (d.flags & (FLAG_IDX_RANGE)) {
    set_status(st, ENKF_INDEX_RANGE, "observation index out of range for state size %lld",
               (long long)p->n_state);
    return ENKF_INDEX_RANGE;
  }
  if (d.flags & FLAG_IDX_ORDER) {
    set_status(st, ENKF_INVALID_ARGUMENT, "indices must be strictly increasing");
    return ENKF_INVALID_ARGUMENT;
  }
  if (d.flags & FLAG_R_NONPOS) {
    set_status(st, ENKF_INVALID_ARGUMENT, "observation variances must be positive");
    return ENKF_INVALID_ARGUMENT;
  }
  if (d.flags & FLAG_NONFINITE) {
    set_status(st, ENKF_INVALID_ARGUMENT, "inputs contain non-finite entries");
    return ENKF_INVALID_ARGUMENT;
  }
  if (d.flags & FLAG_SINGULAR) {
    set_status(st, ENKF_SINGULAR_UPDATE, "rank-one update %d is numerically singular (1 + v'u = %.3e)",
               d.level, d.den);
    if (st) {
      st->level = d.level;
      st->denominator = d.den;
    }
    return ENKF_SINGULAR_UPDATE;
  }
  set_status(st, ENKF_OK, "ok");
  return ENKF_OK;
}

// Every plan entry point runs on the plan's device and leaves the caller's
// current device as it found it (torch and other callers keep theirs).
struct DeviceGuard {
  int prev = -1;
  DeviceGuard() {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      prev = -1;
      cudaGetLastError();
    }
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

int check_plan(const enkf_plan* p, enkf_status* st) {
  if (!p) {
    set_status(st, ENKF_INVALID_ARGUMENT, "null plan");
    return ENKF_INVALID_ARGUMENT;
  }
  if (cudaSetDevice(p->device) != cudaSuccess) {
    set_status(st, ENKF_CUDA_ERROR, "cudaSetDevice(%d) failed", p->device);
    return ENKF_CUDA_ERROR;
  }
  return ENKF_OK;
}

}  // namespace

extern "C" {

const char* enkf_version(void) { return kVersion; }

int32_t enkf_max_ens(void) { return 128; }

int32_t enkf_set_device(int32_t device) {
  return cudaSetDevice(device) == cudaSuccess ? ENKF_OK : ENKF_CUDA_ERROR;
}

int32_t enkf_get_device(int32_t* device) {
  int d = 0;
  if (!device || cudaGetDevice(&d) != cudaSuccess) return ENKF_CUDA_ERROR;
  *device = d;
  return ENKF_OK;
}

int32_t enkf_plan_options_default(enkf_plan_options* o) {
  if (!o) return ENKF_INVALID_ARGUMENT;
  memset(o, 0, sizeof(*o));
  o->struct_size = (int32_t)sizeof(*o);
  o->gram_kernel = ENKF_GRAM_INT8;
  o->anomaly_kernel = ENKF_ANOMALY_INT8;
  o->levels_kernel = ENKF_LEVELS_CLUSTER;
  o->localized_dmma = 1;
  o->tiny_kernel = 1;
  o->host_stream = 1;
  o->host_trace = 0;
  o->host_chunk_bytes = (int64_t)256 << 20;
  o->host_ring_bytes = (int64_t)256 << 20;
  o->host_stream_min_bytes = (int64_t)1 << 30;
  // process-wide overrides (A/B measurements without recompiling the caller)
  if (const char* env = getenv("ENKF_GRAM")) o->gram_kernel = strcmp(env, "fp64") == 0 ? ENKF_GRAM_FP64 : ENKF_GRAM_INT8;
  if (const char* env = getenv("ENKF_ANOMALY"))
    o->anomaly_kernel = strcmp(env, "fp64") == 0 ? ENKF_ANOMALY_FP64 : ENKF_ANOMALY_INT8;
  if (const char* env = getenv("ENKF_LEVELS"))
    o->levels_kernel = strcmp(env, "level") == 0    ? ENKF_LEVELS_PER_LEVEL
                       : strcmp(env, "single") == 0 ? ENKF_LEVELS_SINGLE_CTA
                                                    : ENKF_LEVELS_CLUSTER;
  if (const char* env = getenv("ENKF_LOCALIZED")) o->localized_dmma = strcmp(env, "fma") != 0;
  if (const char* env = getenv("ENKF_TINY")) o->tiny_kernel = env[0] != '0';
  if (const char* env = getenv("ENKF_HOST_STREAM")) o->host_stream = env[0] != '0';
  if (const char* env = getenv("ENKF_HOST_TRACE")) o->host_trace = env[0] == '1';
  if (const char* env = getenv("ENKF_HOST_CHUNK_MB")) o->host_chunk_bytes = (int64_t)atol(env) << 20;
  if (const char* env = getenv("ENKF_HOST_STREAM_MIN_MB")) o->host_stream_min_bytes = (int64_t)atol(env) << 20;
  if (const char* env = getenv("ENKF_HOST_RING_MB")) {
    const int64_t mb = atol(env);
    o->host_ring_bytes = (mb > 0 ? mb : 1) << 20;
  }
  return ENKF_OK;
}

int32_t enkf_plan_create(int64_t n_state, int64_t n_obs, int64_t n_ens, enkf_plan** out,
                         enkf_status* st) {
  return enkf_plan_create_ex(n_state, n_obs, n_ens, nullptr, out, st);
}

int32_t enkf_plan_create_ex(int64_t n_state, int64_t n_obs, int64_t n_ens, const enkf_plan_options* options,
                            enkf_plan** out, enkf_status* st) {
  enkf_plan_options opt;
  enkf_plan_options_default(&opt);
  if (options) {
    if (options->struct_size != (int32_t)sizeof(enkf_plan_options) || options->gram_kernel < 0 ||
        options->gram_kernel > ENKF_GRAM_FP64 || options->anomaly_kernel < 0 ||
        options->anomaly_kernel > ENKF_ANOMALY_FP64 || options->levels_kernel < 0 ||
        options->levels_kernel > ENKF_LEVELS_PER_LEVEL || options->host_chunk_bytes < 0 ||
        options->host_ring_bytes <= 0 || options->host_stream_min_bytes < 0) {
      set_status(st, ENKF_INVALID_ARGUMENT, "invalid enkf_plan_options (start from enkf_plan_options_default)");
      if (out) *out = nullptr;
      return ENKF_INVALID_ARGUMENT;
    }
    opt = *options;
  }
  if (!out) {
    set_status(st, ENKF_INVALID_ARGUMENT, "null plan pointer");
    return ENKF_INVALID_ARGUMENT;
  }
  *out = nullptr;
  if (n_ens < 1 || n_obs < 0 || n_state < 0) {
    set_status(st, ENKF_INVALID_ARGUMENT, "invalid sizes (n_state=%lld n_obs=%lld n_ens=%lld)",
               (long long)n_state, (long long)n_obs, (long long)n_ens);
    return ENKF_INVALID_ARGUMENT;
  }
  if (n_ens > enkf_max_ens()) {
    set_status(st, ENKF_NOT_SUPPORTED, "n_ens=%lld exceeds the supported maximum %d",
               (long long)n_ens, enkf_max_ens());
    return ENKF_NOT_SUPPORTED;
  }
  enkf_plan* p = new (std::nothrow) enkf_plan();
  if (!p) {
    set_status(st, ENKF_CUDA_ERROR, "host allocation failed");
    return ENKF_CUDA_ERROR;
  }
  p->n_state = n_state;
  p->n_obs = n_obs;
  p->n = (int)n_ens;
  cudaError_t e = cudaGetDevice(&p->device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, p->device);
  if (e != cudaSuccess) {
    delete p;
    return cuda_fail(st, e, "device query");
  }
  const int n = p->n;
  const int blocks = ((2 * n + G_BN - 1) / G_BN) * ((n + G_BM - 1) / G_BM);
  int splits = (2 * p->num_sms) / blocks;
  if (splits < 1) splits = 1;
  const int64_t max_splits = (n_obs + G_RT - 1) / G_RT;
  if (splits > max_splits) splits = (int)(max_splits > 0 ? max_splits : 1);
  int64_t rps = (n_obs + splits - 1) / splits;
  rps = (rps + G_RT - 1) / G_RT * G_RT;
  if (rps < G_RT) rps = G_RT;
  splits = (int)((n_obs + rps - 1) / rps);
  if (splits < 1) splits = 1;
  p->splits = splits;
  p->rows_per_split = rps;

  // warp-specialised Gram: 128 x 128 blocks, one CTA per SM
  p->ws_blocks = (2 * n + W_TILE - 1) / W_TILE;
  int cpb = p->num_sms / p->ws_blocks;
  if (cpb < 1) cpb = 1;
  const int64_t max_cpb = (n_obs + W_RT - 1) / W_RT;
  if (cpb > max_cpb) cpb = (int)(max_cpb > 0 ? max_cpb : 1);
  int64_t rpc = (n_obs + cpb - 1) / cpb;
  rpc = (rpc + W_RT - 1) / W_RT * W_RT;
  if (rpc < W_RT) rpc = W_RT;
  cpb = (int)((n_obs + rpc - 1) / rpc);
  if (cpb < 1) cpb = 1;
  p->ws_ctas_per_block = cpb;
  p->ws_rows_per_cta = rpc;
  if (const char* env = getenv("ENKF_DISABLE_WS")) p->use_ws = (env[0] == '0');
  if (const char* env = getenv("ENKF_DISABLE_G128")) p->use_128 = (env[0] == '0');
#ifdef I8_DBG_BUILD  // profiling variants only (tools/build_variant.py NAME -DI8_DBG_BUILD)
  if (const char* env = getenv("ENKF_I8_DBG")) p->i8_dbg = atoi(env);
#endif
  p->gram_i8 = opt.gram_kernel == ENKF_GRAM_INT8;
  p->anomaly_i8 = opt.anomaly_kernel == ENKF_ANOMALY_INT8;
  p->levels_blocked = opt.levels_kernel != ENKF_LEVELS_PER_LEVEL;
  p->levels_cluster = opt.levels_kernel == ENKF_LEVELS_CLUSTER;
  p->loc_dmma = opt.localized_dmma != 0;
  p->tiny = opt.tiny_kernel != 0;
  p->host_streamed = opt.host_stream != 0;
  p->host_trace = opt.host_trace != 0;
  p->host_chunk_bytes = (size_t)opt.host_chunk_bytes;
  p->pageable_stream_min = (size_t)opt.host_stream_min_bytes;
  p->ring_bytes_cfg = (size_t)opt.host_ring_bytes;
  p->g8_groups = p->num_sms / 4 > 0 ? p->num_sms / 4 : 1;

  // gram128 split: the V'V CTAs do 3/4 of the DMMA work of the V'D CTAs (and
  // lighter transforms), so they get fewer CTAs with more rows each.
  {
    double frac = 0.43;
    if (const char* env = getenv("ENKF_VV_FRAC")) frac = atof(env);
    int vv = (int)(p->num_sms * frac + 0.5);
    if (vv < 1) vv = 1;
    if (vv > p->num_sms - 1) vv = p->num_sms - 1;
    int vd = p->num_sms - vv;
    auto rows_for = [&](int ctas) {
      int64_t rr = (n_obs + ctas - 1) / ctas;
      rr = (rr + W_RT - 1) / W_RT * W_RT;
      return rr < W_RT ? (int64_t)W_RT : rr;
    };
    p->g128_rows_vv = rows_for(vv);
    p->g128_rows_vd = rows_for(vd);
    p->g128_cpb_vv = (int)((n_obs + p->g128_rows_vv - 1) / p->g128_rows_vv);
    p->g128_cpb_vd = (int)((n_obs + p->g128_rows_vd - 1) / p->g128_rows_vd);
    if (p->g128_cpb_vv < 1) p->g128_cpb_vv = 1;
    if (p->g128_cpb_vd < 1) p->g128_cpb_vd = 1;
  }
  const size_t nn = (size_t)n * n;
  size_t partial_elems = (size_t)splits * 2 * nn;
  size_t ws_elems = (size_t)p->ws_blocks * cpb * W_TILE * W_TILE;
  const size_t g128_elems = (size_t)(p->g128_cpb_vv + p->g128_cpb_vd) * W_TILE * W_TILE;
  if (g128_elems > ws_elems) ws_elems = g128_elems;
  if (ws_elems > partial_elems) partial_elems = ws_elems;
  e = cudaMalloc(&p->partial, sizeof(double) * partial_elems);
  if (e == cudaSuccess) e = cudaMalloc(&p->gram, sizeof(double) * (2 * nn + COMM_FLAG_SLOTS));
  if (e == cudaSuccess) e = cudaMalloc(&p->A, sizeof(double) * nn);
  if (e == cudaSuccess) e = cudaMalloc(&p->T, sizeof(double) * nn);
  if (e == cudaSuccess) e = cudaMalloc(&p->den, sizeof(double) * n);
  if (e == cudaSuccess) e = cudaMalloc(&p->dstatus, sizeof(DevStatus));
  if (e == cudaSuccess) e = cudaMallocHost(&p->hstatus, sizeof(DevStatus));
  if (e != cudaSuccess) {
    enkf_plan_destroy(p);
    return cuda_fail(st, e, "workspace allocation");
  }
  memset(p->hstatus, 0, sizeof(DevStatus));
  if (n == G8_N && p->gram_i8 && p->use_128 && n_obs > 0 && !(p->tiny && tiny_eligible(n_state, n_obs, n))) {
    e = ensure_gram_i8_workspace(p);
    if (e != cudaSuccess) {
      enkf_plan_destroy(p);
      return cuda_fail(st, e, "int8 Gram workspace allocation");
    }
  }
  *out = p;
  set_status(st, ENKF_OK, "ok");
  return ENKF_OK;
}

void enkf_plan_destroy(enkf_plan* p) {
  if (!p) return;
  DeviceGuard device_guard;
  cudaSetDevice(p->device);
  cudaFree(p->partial);
  cudaFree(p->gram);
  cudaFree(p->A);
  cudaFree(p->T);
  cudaFree(p->den);
  cudaFree(p->dstatus);
  if (p->hstatus) cudaFreeHost(p->hstatus);
  cudaFree(p->hx);
  cudaFree(p->hy);
  cudaFree(p->hr);
  cudaFree(p->hidx);
  if (p->hstream) cudaStreamDestroy(p->hstream);
  cudaFree(p->hxo);
  if (p->small_h) cudaFreeHost(p->small_h);
  cudaFree(p->small_d);
  if (p->hs_in) cudaStreamDestroy(p->hs_in);
  if (p->hs_out) cudaStreamDestroy(p->hs_out);
  if (p->ev_obs) cudaEventDestroy(p->ev_obs);
  if (p->ev_anom) cudaEventDestroy(p->ev_anom);
  for (cudaEvent_t ev : p->chunk_ev) cudaEventDestroy(ev);
  cudaFree(p->locV);
  cudaFree(p->locD);
  cudaFree(p->locZ);
  cudaFree(p->l96ws);
  cudaFree(p->g8_planes);
  for (cudaEvent_t ev : p->g8_ev)
    if (ev) cudaEventDestroy(ev);
  cudaFree(p->g8_meta);
  cudaFree(p->g8_sr);
  cudaFree(p->g8_ls_partial);
  cudaFree(p->g8_ls_progress);
  cudaFree(p->cyc_status);
  for (auto& set : p->st_evs)
    for (cudaEvent_t ev : set)
      if (ev) cudaEventDestroy(ev);
  for (int i = 0; i < 2; ++i) {
    if (p->ring[i]) cudaFreeHost(p->ring[i]);
    if (p->ring_ev[i]) cudaEventDestroy(p->ring_ev[i]);
    if (p->oring[i]) cudaFreeHost(p->oring[i]);
    if (p->oring_ev[i]) cudaEventDestroy(p->oring_ev[i]);
  }
  delete p;
}

int32_t enkf_ism_gram_f64(enkf_plan* p, const double* X, const double* Y, const int64_t* idx,
                          const double* r, double* gram, void* stream) {
  DeviceGuard device_guard;
  if (check_plan(p, nullptr)) return ENKF_INVALID_ARGUMENT;
  if (p->n < 2) return ENKF_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = launch_gram(p, true, X, Y, idx, r, gram, s);
  return e == cudaSuccess ? ENKF_OK : ENKF_CUDA_ERROR;
}

int32_t enkf_ism_levels_f64(enkf_plan* p, const double* gram, double* A, double* T, double* den,
                            void* stream) {
  DeviceGuard device_guard;
  if (check_plan(p, nullptr)) return ENKF_INVALID_ARGUMENT;
  const double cscale = p->n > 1 ? 1.0 / std::sqrt((double)(p->n - 1)) : 0.0;
  cudaError_t e = launch_levels(p, gram, A, T, den, cscale, (cudaStream_t)stream);
  return e == cudaSuccess ? ENKF_OK : ENKF_CUDA_ERROR;
}

int32_t enkf_anomaly_update_f64(enkf_plan* p, const double* X, const double* T, double* XA,
                                int64_t n_rows, void* stream) {
  DeviceGuard device_guard;
  if (check_plan(p, nullptr)) return ENKF_INVALID_ARGUMENT;
  cudaError_t e = launch_rowgemm<0>(p, X, T, nullptr, nullptr, XA, n_rows, (cudaStream_t)stream);
  return e == cudaSuccess ? ENKF_OK : ENKF_CUDA_ERROR;
}

int32_t enkf_analysis_async_f64(enkf_plan* p, const double* X, const double* Y, const int64_t* idx,
                                const double* r, double* XA, void* stream) {
  NvtxRange nvtx("enkf_analysis");
  DeviceGuard device_guard;
  if (check_plan(p, nullptr)) return ENKF_INVALID_ARGUMENT;
  if (p->n < 2) return ENKF_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(p->dstatus, 0, sizeof(DevStatus), s);
  if (e == cudaSuccess && !p->comm && p->tiny && tiny_eligible(p->n_state, p->n_obs, p->n)) {
    e = launch_tiny(p, X, Y, idx, r, XA, s);
    return e == cudaSuccess ? ENKF_OK : ENKF_CUDA_ERROR;
  }
  if (p->stage_events) {
    p->st_ev = p->st_evs[p->st_steps % enkf_plan::ST_SETS];
    ++p->st_steps;
    for (int i = 0; i < 5; ++i)
      if (!p->st_ev[i] && cudaEventCreate(&p->st_ev[i]) != cudaSuccess) return ENKF_CUDA_ERROR;
    cudaEventRecord(p->st_ev[0], s);
  }
  if (e == cudaSuccess) e = launch_gram_global(p, X, Y, idx, r, s);
  if (p->stage_events && !p->comm) {  // no exchange: gram | allreduce boundaries coincide
    cudaEventRecord(p->st_ev[1], s);
    cudaEventRecord(p->st_ev[2], s);
  }
  const double cscale = 1.0 / std::sqrt((double)(p->n - 1));
  if (e == cudaSuccess) e = launch_levels(p, p->gram, p->A, p->T, p->den, cscale, s);
  if (p->stage_events) cudaEventRecord(p->st_ev[3], s);
  if (e == cudaSuccess) e = launch_rowgemm<0>(p, X, p->T, nullptr, nullptr, XA, p->n_state, s);
  if (p->stage_events) cudaEventRecord(p->st_ev[4], s);
  if (e == cudaErrorUnknown && p->nccl_rc) return ENKF_CUDA_ERROR;
  return e == cudaSuccess ? ENKF_OK : ENKF_CUDA_ERROR;
}

int32_t enkf_plan_sync_status(enkf_plan* p, void* stream, enkf_status* st) {
  DeviceGuard device_guard;
  if (check_plan(p, st)) return ENKF_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaMemcpyAsync(p->hstatus, p->dstatus, sizeof(DevStatus), cudaMemcpyDeviceToHost, s), st);
  CUDA_TRY(cudaStreamSynchronize(s), st);
  return translate_status(p, st);
}

int32_t enkf_plan_reset_status(enkf_plan* p, void* stream) {
  DeviceGuard device_guard;
  if (check_plan(p, nullptr)) return ENKF_INVALID_ARGUMENT;
  return cudaMemsetAsync(p->dstatus, 0, sizeof(DevStatus), (cudaStream_t)stream) == cudaSuccess
             ? ENKF_OK : ENKF_CUDA_ERROR;
}

int32_t enkf_analysis_f64(enkf_plan* p, const double* X, const double* Y, const int64_t* idx,
                          const double* r, double* XA, void* stream, enkf_status* st) {
  DeviceGuard device_guard;
  if (check_plan(p, st)) return ENKF_INVALID_ARGUMENT;
  if (p->n < 2) {
    set_status(st, ENKF_INVALID_ARGUMENT, "analysis needs at least 2 ensemble members");
    return ENKF_INVALID_ARGUMENT;
  }
  int rc = enkf_analysis_async_f64(p, X, Y, idx, r, XA, stream);
  if (rc != ENKF_OK) {
    if (p->nccl_rc) {
      set_status(st, ENKF_CUDA_ERROR, "ncclAllReduce of the Gram failed: %s",
                 nccl_api().error_string((ncclResult_t)p->nccl_rc));
      p->nccl_rc = 0;
      return ENKF_CUDA_ERROR;
    }
    CUDA_TRY(cudaGetLastError(), st);
    set_status(st, rc, "launch failed");
    return rc;
  }
  return enkf_plan_sync_status(p, stream, st);
}

namespace {
// Device address of a page-locked, mapped host buffer (cudaHostAlloc'd memory,
// torch pin_memory, or cudaHostRegister'ed with mapping), or null.
const void* mapped_device_ptr(const void* h) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

// Host-buffer analysis with page-locked X and XA (enkf.py:167-192 on host
// arrays).  Only the observed rows and Y are needed before T exists, so:
//   1. r, idx, Y by DMA; X[idx] gathered by SM loads over PCIe (gather_rows_kernel)
//   2. Gram pass on the compact rows (identity H), levels -> T
//   3. X by DMA in chunks on a second stream (starts right after step 1's
//      traffic, overlapping the Gram), the anomaly update of each chunk as it
//      lands, X^A chunks out by DMA on a third stream: the two PCIe directions
//      run concurrently.
// The status is read after step 2 (a failed step returns before any X^A is
// copied, after the in-flight X DMA has drained).
int analysis_host_streamed(enkf_plan* p, const double* X_h, const double* Xmap, const double* Y_h,
                           const int64_t* idx_h, const double* r_h, double* XA_h, enkf_status* st) {
  const size_t n = (size_t)p->n;
  const size_t row_bytes = n * sizeof(double);
  cudaStream_t s = p->hstream;
  if (!p->hxo) {
    CUDA_TRY(cudaMalloc(&p->hxo, row_bytes * (size_t)p->n_obs + 16), st);
    CUDA_TRY(cudaStreamCreateWithFlags(&p->hs_in, cudaStreamNonBlocking), st);
    CUDA_TRY(cudaStreamCreateWithFlags(&p->hs_out, cudaStreamNonBlocking), st);
    CUDA_TRY(cudaEventCreateWithFlags(&p->ev_obs, cudaEventDisableTiming), st);
    CUDA_TRY(cudaEventCreateWithFlags(&p->ev_anom, cudaEventDisableTiming), st);
  }
  // On any early return below, wait for the copies already queued: the caller's
  // buffers must not be touched by DMA or kernels after the call returns.
  struct Drain {
    cudaStream_t a, b, c;
    ~Drain() {
      cudaStreamSynchronize(a);
      cudaStreamSynchronize(b);
      cudaStreamSynchronize(c);
    }
  } drain{s, p->hs_in, p->hs_out};
  int64_t chunk_rows = (int64_t)(p->host_chunk_bytes / row_bytes);
  if (chunk_rows < 1024) chunk_rows = 1024;
  const int64_t nchunks = (p->n_state + chunk_rows - 1) / chunk_rows;
  while ((int64_t)p->chunk_ev.size() < nchunks) {
    cudaEvent_t ev;
    CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), st);
    p->chunk_ev.push_back(ev);
  }
  cudaEvent_t tr[7] = {};
  if (p->host_trace)
    for (auto& ev : tr) cudaEventCreate(&ev);
  auto mark = [&](int i, cudaStream_t ms) {
    if (p->host_trace) cudaEventRecord(tr[i], ms);
  };
  // 1. observation side
  NvtxRange nvtx1("host_streamed: observation side + Gram + levels");
  mark(0, s);
  CUDA_TRY(cudaMemsetAsync(p->dstatus, 0, sizeof(DevStatus), s), st);
  CUDA_TRY(copy_h2d(p, p->hr, r_h, sizeof(double) * (size_t)p->n_obs, s), st);
  CUDA_TRY(copy_h2d(p, p->hidx, idx_h, sizeof(int64_t) * (size_t)p->n_obs, s), st);
  CUDA_TRY(copy_h2d(p, p->hy, Y_h, row_bytes * (size_t)p->n_obs, s), st);
  mark(1, s);
  {
    const int grid = p->num_sms * 8;
    const bool vec = (n % 2 == 0) && aligned16(Xmap) && aligned16(p->hxo);
    if (vec)
      gather_rows_kernel<true><<<grid, GATHER_THREADS, 0, s>>>(Xmap, p->hidx, p->hxo, p->n_obs, p->n_state,
                                                               (int)n, p->dstatus);
    else
      gather_rows_kernel<false><<<grid, GATHER_THREADS, 0, s>>>(Xmap, p->hidx, p->hxo, p->n_obs, p->n_state,
                                                                (int)n, p->dstatus);
    CUDA_TRY(cudaGetLastError(), st);
  }
  mark(2, s);  // X[idx] gathered
  CUDA_TRY(cudaEventRecord(p->ev_obs, s), st);
  // 3a. the X stream starts once the observation traffic is through
  CUDA_TRY(cudaStreamWaitEvent(p->hs_in, p->ev_obs, 0), st);
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t r0 = c * chunk_rows;
    const int64_t rows = std::min<int64_t>(chunk_rows, p->n_state - r0);
    CUDA_TRY(cudaMemcpyAsync(p->hx + (size_t)r0 * n, X_h + (size_t)r0 * n, (size_t)rows * row_bytes,
                             cudaMemcpyHostToDevice, p->hs_in), st);
    CUDA_TRY(cudaEventRecord(p->chunk_ev[c], p->hs_in), st);
  }
  // 2. Gram on the compact observed rows, levels
  {
    CUDA_TRY(launch_gram_global(p, p->hxo, p->hy, nullptr, p->hr, s), st);
    const double cscale = 1.0 / std::sqrt((double)(p->n - 1));
    CUDA_TRY(launch_levels(p, p->gram, p->A, p->T, p->den, cscale, s), st);
  }
  mark(3, s);  // T ready
  {
    int rc = enkf_plan_sync_status(p, s, st);
    if (rc != ENKF_OK) return rc;  // (Drain waits for the X copies in flight)
  }
  // 3b. anomaly update chunk by chunk (in place), X^A out
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t r0 = c * chunk_rows;
    const int64_t rows = std::min<int64_t>(chunk_rows, p->n_state - r0);
    double* dx = p->hx + (size_t)r0 * n;
    CUDA_TRY(cudaStreamWaitEvent(s, p->chunk_ev[c], 0), st);
    CUDA_TRY(launch_rowgemm<0>(p, dx, p->T, nullptr, nullptr, dx, rows, s), st);
    CUDA_TRY(cudaEventRecord(p->ev_anom, s), st);
    CUDA_TRY(cudaStreamWaitEvent(p->hs_out, p->ev_anom, 0), st);
    CUDA_TRY(cudaMemcpyAsync(XA_h + (size_t)r0 * n, dx, (size_t)rows * row_bytes, cudaMemcpyDeviceToHost,
                             p->hs_out), st);
  }
  mark(4, p->hs_in);   // all of X in
  mark(5, s);          // last anomaly chunk
  mark(6, p->hs_out);  // all of X^A out
  CUDA_TRY(cudaStreamSynchronize(p->hs_out), st);
  CUDA_TRY(cudaStreamSynchronize(s), st);
  if (p->host_trace) {
    cudaStreamSynchronize(p->hs_in);
    float t[7] = {};
    for (int i = 1; i < 7; ++i) cudaEventElapsedTime(&t[i], tr[0], tr[i]);
    const double ob = (double)(row_bytes * (size_t)p->n_obs);
    fprintf(stderr,
            "[enkf host] Y in %.1f ms (%.1f GB/s)  gather %.1f ms (%.1f GB/s)  T ready %.1f  X in %.1f  "
            "anomaly done %.1f  XA out %.1f ms\n",
            t[1], ob / (t[1] * 1e6), t[2] - t[1], ob / ((t[2] - t[1]) * 1e6), t[3], t[4], t[5], t[6]);
    for (auto& ev : tr) cudaEventDestroy(ev);
  }
  return ENKF_OK;
}
// Host-buffer analysis with the caller's ordinary (pageable) X and X^A: the same
// schedule as analysis_host_streamed through pinned staging rings.  The observed rows
// X[idx] are gathered on the host (thread pool) into the inbound ring and copied in
// first; the Gram and the levels run on them; then X streams in chunk by chunk (host
// copy into an inbound ring slot, DMA), each chunk's anomaly update runs as it lands,
// and its X^A returns through the outbound ring while the next chunk comes in — the
// two PCIe directions and the host copies overlap.  Bound by host-memory copy
// bandwidth (both directions pass through the rings).
int analysis_host_pageable_streamed(enkf_plan* p, const double* X_h, const double* Y_h, const int64_t* idx_h,
                                    const double* r_h, double* XA_h, enkf_status* st) {
  const size_t n = (size_t)p->n;
  const size_t row_bytes = n * sizeof(double);
  cudaStream_t s = p->hstream;
  if (!p->hxo) {
    CUDA_TRY(cudaMalloc(&p->hxo, row_bytes * (size_t)p->n_obs + 16), st);
    CUDA_TRY(cudaStreamCreateWithFlags(&p->hs_in, cudaStreamNonBlocking), st);
    CUDA_TRY(cudaStreamCreateWithFlags(&p->hs_out, cudaStreamNonBlocking), st);
    CUDA_TRY(cudaEventCreateWithFlags(&p->ev_obs, cudaEventDisableTiming), st);
    CUDA_TRY(cudaEventCreateWithFlags(&p->ev_anom, cudaEventDisableTiming), st);
  }
  CUDA_TRY(ensure_ring(p), st);
  for (int i = 0; i < 2; ++i)
    if (!p->oring[i]) {
      CUDA_TRY(cudaMallocHost(&p->oring[i], p->ring_bytes), st);
      CUDA_TRY(cudaEventCreateWithFlags(&p->oring_ev[i], cudaEventDisableTiming), st);
    }
  struct Drain {
    cudaStream_t a, b, c;
    ~Drain() {
      cudaStreamSynchronize(a);
      cudaStreamSynchronize(b);
      cudaStreamSynchronize(c);
    }
  } drain{s, p->hs_in, p->hs_out};
  // host-side phase clock (ENKF_HOST_TRACE=1)
  const auto t_start = std::chrono::steady_clock::now();
  auto ms_since = [&] {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
  };
  double t_obs = 0, t_T = 0, t_loop = 0, t_memcpy_in = 0, t_wait_slot = 0;
  // 1. r, idx, Y (ring), the observed rows gathered on the host (ring)
  CUDA_TRY(cudaMemsetAsync(p->dstatus, 0, sizeof(DevStatus), s), st);
  CUDA_TRY(copy_h2d(p, p->hr, r_h, sizeof(double) * (size_t)p->n_obs, s), st);
  CUDA_TRY(copy_h2d(p, p->hidx, idx_h, sizeof(int64_t) * (size_t)p->n_obs, s), st);
  CUDA_TRY(copy_h2d(p, p->hy, Y_h, row_bytes * (size_t)p->n_obs, s), st);
  {
    // index checks the gather relies on (the device re-checks order and range)
    const int64_t ring_rows = (int64_t)(p->ring_bytes / row_bytes);
    for (int64_t k0 = 0; k0 < p->n_obs; k0 += ring_rows) {
      const int64_t rows = std::min<int64_t>(ring_rows, p->n_obs - k0);
      for (int64_t k = k0; k < k0 + rows; ++k) {
        if (idx_h[k] < 0 || idx_h[k] >= p->n_state) {
          set_status(st, ENKF_INDEX_RANGE, "observation index out of range for state size %lld",
                     (long long)p->n_state);
          return ENKF_INDEX_RANGE;
        }
        if (k > 0 && idx_h[k] <= idx_h[k - 1]) {
          set_status(st, ENKF_INVALID_ARGUMENT, "indices must be strictly increasing");
          return ENKF_INVALID_ARGUMENT;
        }
      }
      int slot;
      CUDA_TRY(take_slot(p, &slot), st);
      parallel_gather_rows(p->ring[slot], (const char*)X_h, idx_h + k0, rows, row_bytes);
      CUDA_TRY(cudaMemcpyAsync((char*)p->hxo + (size_t)k0 * row_bytes, p->ring[slot], (size_t)rows * row_bytes,
                               cudaMemcpyHostToDevice, s), st);
      CUDA_TRY(cudaEventRecord(p->ring_ev[slot], s), st);
      p->ring_busy[slot] = true;
    }
  }
  t_obs = ms_since();
  // 2. Gram on the compact observed rows, levels; the status before any X traffic
  CUDA_TRY(launch_gram_global(p, p->hxo, p->hy, nullptr, p->hr, s), st);
  CUDA_TRY(launch_levels(p, p->gram, p->A, p->T, p->den, 1.0 / std::sqrt((double)(p->n - 1)), s), st);
  {
    int rc = enkf_plan_sync_status(p, s, st);
    if (rc != ENKF_OK) return rc;
  }
  t_T = ms_since();
  // 3. X in (inbound ring, hs_in), anomaly per chunk in place (s), X^A out (outbound ring, hs_out)
  const int64_t chunk_rows = (int64_t)(p->ring_bytes / row_bytes);
  const int64_t nchunks = (p->n_state + chunk_rows - 1) / chunk_rows;
  while ((int64_t)p->chunk_ev.size() < nchunks) {
    cudaEvent_t ev;
    CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), st);
    p->chunk_ev.push_back(ev);
  }
  auto drain_out = [&](int64_t c) -> cudaError_t {
    const int64_t r0 = c * chunk_rows, rows = std::min<int64_t>(chunk_rows, p->n_state - r0);
    cudaError_t e = cudaEventSynchronize(p->oring_ev[c & 1]);
    if (e != cudaSuccess) return e;
    parallel_memcpy((char*)XA_h + (size_t)r0 * row_bytes, p->oring[c & 1], (size_t)rows * row_bytes);
    return cudaSuccess;
  };
  // (a page-locked X or X^A - e.g. the Python layer's page-locked result arrays - is
  // DMA'd directly instead of through its ring)
  const bool x_pinned = is_pinned(X_h), xa_pinned = is_pinned(XA_h);
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t r0 = c * chunk_rows, rows = std::min<int64_t>(chunk_rows, p->n_state - r0);
    const size_t bytes = (size_t)rows * row_bytes;
    double* dx = p->hx + (size_t)r0 * n;
    if (x_pinned) {
      CUDA_TRY(cudaMemcpyAsync(dx, (const char*)X_h + (size_t)r0 * row_bytes, bytes, cudaMemcpyHostToDevice,
                               p->hs_in), st);
    } else {
      int slot;
      const double t0 = ms_since();
      CUDA_TRY(take_slot(p, &slot), st);
      const double t1 = ms_since();
      parallel_memcpy(p->ring[slot], (const char*)X_h + (size_t)r0 * row_bytes, bytes);
      t_wait_slot += t1 - t0;
      t_memcpy_in += ms_since() - t1;
      CUDA_TRY(cudaMemcpyAsync(dx, p->ring[slot], bytes, cudaMemcpyHostToDevice, p->hs_in), st);
      CUDA_TRY(cudaEventRecord(p->ring_ev[slot], p->hs_in), st);
      p->ring_busy[slot] = true;
    }
    CUDA_TRY(cudaEventRecord(p->chunk_ev[c], p->hs_in), st);
    CUDA_TRY(cudaStreamWaitEvent(s, p->chunk_ev[c], 0), st);
    CUDA_TRY(launch_rowgemm<0>(p, dx, p->T, nullptr, nullptr, dx, rows, s), st);
    CUDA_TRY(cudaEventRecord(p->ev_anom, s), st);
    CUDA_TRY(cudaStreamWaitEvent(p->hs_out, p->ev_anom, 0), st);
    if (xa_pinned) {
      CUDA_TRY(cudaMemcpyAsync((char*)XA_h + (size_t)r0 * row_bytes, dx, bytes, cudaMemcpyDeviceToHost, p->hs_out),
               st);
    } else {
      // the outbound slot of chunk c was drained by the host when chunk c - 1 was queued
      CUDA_TRY(cudaMemcpyAsync(p->oring[c & 1], dx, bytes, cudaMemcpyDeviceToHost, p->hs_out), st);
      CUDA_TRY(cudaEventRecord(p->oring_ev[c & 1], p->hs_out), st);
      if (c >= 1) CUDA_TRY(drain_out(c - 1), st);
    }
  }
  if (!xa_pinned && nchunks >= 1) CUDA_TRY(drain_out(nchunks - 1), st);
  t_loop = ms_since();
  CUDA_TRY(cudaStreamSynchronize(p->hs_out), st);
  if (p->host_trace)
    fprintf(stderr,
            "[enkf host pageable] obs side queued %.1f ms, T ready %.1f ms, X loop queued %.1f ms (slot waits %.1f, "
            "host copies in %.1f), X^A out done %.1f ms\n",
            t_obs, t_T, t_loop, t_wait_slot, t_memcpy_in, ms_since());
  CUDA_TRY(cudaStreamSynchronize(s), st);
  return ENKF_OK;
}
}  // namespace

int32_t enkf_analysis_host_f64(enkf_plan* p, const double* X_h, const double* Y_h,
                               const int64_t* idx_h, const double* r_h, double* XA_h,
                               enkf_status* st) {
  NvtxRange nvtx("enkf_analysis_host");
  DeviceGuard device_guard;
  if (check_plan(p, st)) return ENKF_INVALID_ARGUMENT;
  if (p->n < 2) {
    set_status(st, ENKF_INVALID_ARGUMENT, "analysis needs at least 2 ensemble members");
    return ENKF_INVALID_ARGUMENT;
  }
  const size_t n = (size_t)p->n;
  if (!p->hstream) CUDA_TRY(cudaStreamCreateWithFlags(&p->hstream, cudaStreamNonBlocking), st);
  if (!p->hx) {
    CUDA_TRY(cudaMalloc(&p->hx, sizeof(double) * (size_t)p->n_state * n + 16), st);
    CUDA_TRY(cudaMalloc(&p->hy, sizeof(double) * (size_t)p->n_obs * n + 16), st);
    CUDA_TRY(cudaMalloc(&p->hr, sizeof(double) * (size_t)p->n_obs + 16), st);
    CUDA_TRY(cudaMalloc(&p->hidx, sizeof(int64_t) * (size_t)p->n_obs + 16), st);
  }
  cudaStream_t s = p->hstream;
  {
    // Small problems: every input packed into one page-locked staging block, one
    // copy in, the step (in place), X^A and the status out, one synchronisation.
    const size_t xb = sizeof(double) * (size_t)p->n_state * n, yb = sizeof(double) * (size_t)p->n_obs * n;
    const size_t rb = sizeof(double) * (size_t)p->n_obs, ib = idx_h ? sizeof(int64_t) * (size_t)p->n_obs : 0;
    auto al = [](size_t v) { return (v + 255) & ~(size_t)255; };
    const size_t total = al(xb) + al(yb) + al(rb) + al(ib);
    if (total <= kSmallHostBytes) {
      if (!p->small_h) {
        CUDA_TRY(cudaMallocHost(&p->small_h, kSmallHostBytes), st);
        CUDA_TRY(cudaMalloc(&p->small_d, kSmallHostBytes), st);
      }
      char* h = p->small_h;
      char* d = p->small_d;
      memcpy(h, X_h, xb);
      memcpy(h + al(xb), Y_h, yb);
      memcpy(h + al(xb) + al(yb), r_h, rb);
      if (ib) memcpy(h + al(xb) + al(yb) + al(rb), idx_h, ib);
      CUDA_TRY(cudaMemcpyAsync(d, h, total, cudaMemcpyHostToDevice, s), st);
      double* dx = reinterpret_cast<double*>(d);
      const double* dy = reinterpret_cast<const double*>(d + al(xb));
      const double* dr = reinterpret_cast<const double*>(d + al(xb) + al(yb));
      const int64_t* di = ib ? reinterpret_cast<const int64_t*>(d + al(xb) + al(yb) + al(rb)) : nullptr;
      int rc = enkf_analysis_async_f64(p, dx, dy, di, dr, dx, s);  // in place
      if (rc != ENKF_OK) {
        cudaStreamSynchronize(s);
        CUDA_TRY(cudaGetLastError(), st);
        set_status(st, rc, "launch failed");
        return rc;
      }
      CUDA_TRY(cudaMemcpyAsync(h, dx, xb, cudaMemcpyDeviceToHost, s), st);
      CUDA_TRY(cudaMemcpyAsync(p->hstatus, p->dstatus, sizeof(DevStatus), cudaMemcpyDeviceToHost, s), st);
      CUDA_TRY(cudaStreamSynchronize(s), st);
      const int rc2 = translate_status(p, st);
      if (rc2 == ENKF_OK) memcpy(XA_h, h, xb);
      return rc2;
    }
  }
  if (idx_h && p->n_obs > 0 && p->host_streamed) {
    const void* Xmap = mapped_device_ptr(X_h);
    if (Xmap && is_pinned(XA_h))
      return analysis_host_streamed(p, X_h, (const double*)Xmap, Y_h, idx_h, r_h, XA_h, st);
    if (sizeof(double) * (size_t)p->n_state * n >= p->pageable_stream_min)
      return analysis_host_pageable_streamed(p, X_h, Y_h, idx_h, r_h, XA_h, st);
  }
  struct Drain {
    cudaStream_t a;
    ~Drain() { cudaStreamSynchronize(a); }
  } drain{s};  // no queued copy outlives the call, on any return path
  CUDA_TRY(copy_h2d(p, p->hx, X_h, sizeof(double) * (size_t)p->n_state * n, s), st);
  CUDA_TRY(copy_h2d(p, p->hy, Y_h, sizeof(double) * (size_t)p->n_obs * n, s), st);
  CUDA_TRY(copy_h2d(p, p->hr, r_h, sizeof(double) * (size_t)p->n_obs, s), st);
  const int64_t* didx = nullptr;
  if (idx_h) {
    CUDA_TRY(copy_h2d(p, p->hidx, idx_h, sizeof(int64_t) * (size_t)p->n_obs, s), st);
    didx = p->hidx;
  }
  // In place: XA overwrites the device copy of X.
  int rc = enkf_analysis_async_f64(p, p->hx, p->hy, didx, p->hr, p->hx, s);
  if (rc != ENKF_OK) {
    CUDA_TRY(cudaGetLastError(), st);
    set_status(st, rc, "launch failed");
    return rc;
  }
  // Read the status before the (long) copy-out so a failed step raises
  // without paying for it.
  int rc2 = enkf_plan_sync_status(p, s, st);
  if (rc2 != ENKF_OK) return rc2;
  CUDA_TRY(copy_d2h(p, XA_h, p->hx, sizeof(double) * (size_t)p->n_state * n, s), st);
  CUDA_TRY(cudaStreamSynchronize(s), st);
  return ENKF_OK;
}

int32_t enkf_ism_solve_f64(enkf_plan* p, const double* r, const double* V, const double* D,
                           double* Z, double* A, void* stream, enkf_status* st) {
  NvtxRange nvtx("enkf_ism_solve");
  DeviceGuard device_guard;
  if (check_plan(p, st)) return ENKF_INVALID_ARGUMENT;
  if (p->comm) {
    set_status(st, ENKF_NOT_SUPPORTED, "solve_sherman on a sharded plan (communicator attached) is not provided");
    return ENKF_NOT_SUPPORTED;
  }
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaMemsetAsync(p->dstatus, 0, sizeof(DevStatus), s), st);
  CUDA_TRY(launch_gram(p, false, V, D, nullptr, r, p->gram, s), st);
  double* Aout = A ? A : p->A;
  CUDA_TRY(launch_levels(p, p->gram, Aout, nullptr, p->den, 0.0, s), st);
  CUDA_TRY(launch_rowgemm<1>(p, V, Aout, D, r, Z, p->n_obs, s), st);
  return enkf_plan_sync_status(p, s, st);
}

int32_t enkf_member_deviations_f64(const double* X, double* S, int64_t n_rows, int64_t n_ens,
                                   void* stream) {
  if (n_ens < 2) return ENKF_INVALID_ARGUMENT;
  if (n_rows == 0) return ENKF_OK;
  const double root = std::sqrt((double)n_ens - 1.0);
  const int64_t threads = n_rows * 32;
  deviations_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(X, S, n_rows, (int)n_ens, root);
  return cudaGetLastError() == cudaSuccess ? ENKF_OK : ENKF_CUDA_ERROR;
}

int32_t enkf_innovations_f64(const double* X, const double* Y, const int64_t* idx, double* D,
                             int64_t n_obs, int64_t n_ens, void* stream) {
  if (n_ens < 1) return ENKF_INVALID_ARGUMENT;
  if (n_obs == 0) return ENKF_OK;
  const int64_t threads = n_obs * 32;
  innovations_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, (cudaStream_t)stream>>>(X, Y, idx, D, n_obs, (int)n_ens);
  return cudaGetLastError() == cudaSuccess ? ENKF_OK : ENKF_CUDA_ERROR;
}

namespace {
// Shared body of the two localized entry points (enkf.py:187-199).
// The launches of one localized analysis (enkf.py:187-199) on stream s, flags into
// p->dstatus: V, D rows; Gram -> levels -> Z; X + (Delta o (S V')) Z.  XA may alias X
// (each CTA of the update kernel reads and writes only its own state rows).
cudaError_t launch_localized(enkf_plan* p, const double* X, const double* Y, const int64_t* idx, const double* r,
                             const double* delta, double scale, int mode, double* XA, cudaStream_t s) {
  const int n = p->n;
  const size_t obs_elems = (size_t)p->n_obs * (size_t)n;
  cudaError_t e = cudaSuccess;
  if (!p->locV && obs_elems) {
    if ((e = cudaMalloc(&p->locV, sizeof(double) * obs_elems)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&p->locD, sizeof(double) * obs_elems)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&p->locZ, sizeof(double) * obs_elems)) != cudaSuccess) return e;
  }
  const double root = std::sqrt((double)n - 1.0);
  if (p->n_obs > 0) {
    const int64_t threads = p->n_obs * 32;
    obs_rows_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(X, Y, idx, p->locV, p->locD, p->n_obs,
                                                                      p->n_state, n, root, p->dstatus);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = launch_gram(p, false, p->locV, p->locD, nullptr, r, p->gram, s)) != cudaSuccess) return e;
    if ((e = launch_levels(p, p->gram, p->A, nullptr, p->den, 0.0, s)) != cudaSuccess) return e;
    if ((e = launch_rowgemm<1>(p, p->locV, p->A, p->locD, r, p->locZ, p->n_obs, s)) != cudaSuccess) return e;
  }
  if (p->n_state > 0 && p->loc_dmma) {
    auto run = [&](auto np_tag) -> cudaError_t {
      constexpr int NPV = decltype(np_tag)::value;
      const size_t smem = localized_dmma_smem_bytes(NPV);
      const unsigned grid = (unsigned)((p->n_state + LD_TI - 1) / LD_TI);
      cudaError_t err;
      if (mode == 0) {
        if ((err = cudaFuncSetAttribute(localized_update_dmma_kernel<NPV, 0>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
          return err;
        localized_update_dmma_kernel<NPV, 0><<<grid, LD_THREADS, smem, s>>>(X, p->locV, p->locZ, delta, idx, scale,
                                                                          XA, p->n_state, p->n_obs, n, root);
      } else {
        if ((err = cudaFuncSetAttribute(localized_update_dmma_kernel<NPV, 1>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
          return err;
        localized_update_dmma_kernel<NPV, 1><<<grid, LD_THREADS, smem, s>>>(X, p->locV, p->locZ, nullptr, idx,
                                                                          scale, XA, p->n_state, p->n_obs, n, root);
      }
      return cudaGetLastError();
    };
    if (n <= 8) return run(std::integral_constant<int, 8>{});
    if (n <= 16) return run(std::integral_constant<int, 16>{});
    if (n <= 32) return run(std::integral_constant<int, 32>{});
    if (n <= 64) return run(std::integral_constant<int, 64>{});
    if (n <= 96) return run(std::integral_constant<int, 96>{});
    return run(std::integral_constant<int, 128>{});
  }
  if (p->n_state > 0) {
    const size_t smem = localized_smem_bytes(n);
    const unsigned grid = (unsigned)((p->n_state + LOC_TI - 1) / LOC_TI);
    if (mode == 0) {
      if ((e = cudaFuncSetAttribute(localized_update_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem)) != cudaSuccess)
        return e;
      localized_update_kernel<0><<<grid, LOC_THREADS, smem, s>>>(X, p->locV, p->locZ, delta, idx, scale, XA,
                                                                p->n_state, p->n_obs, n, root);
    } else {
      if ((e = cudaFuncSetAttribute(localized_update_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem)) != cudaSuccess)
        return e;
      localized_update_kernel<1><<<grid, LOC_THREADS, smem, s>>>(X, p->locV, p->locZ, nullptr, idx, scale, XA,
                                                                p->n_state, p->n_obs, n, root);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

int localized_common(enkf_plan* p, const double* X, const double* Y, const int64_t* idx, const double* r,
                     const double* delta, double scale, int mode, double* XA, void* stream, enkf_status* st) {
  DeviceGuard device_guard;
  if (check_plan(p, st)) return ENKF_INVALID_ARGUMENT;
  if (p->comm) {
    set_status(st, ENKF_NOT_SUPPORTED, "not provided on a sharded plan (communicator attached)");
    return ENKF_NOT_SUPPORTED;
  }
  if (p->n < 2) {
    set_status(st, ENKF_INVALID_ARGUMENT, "analysis needs at least 2 ensemble members");
    return ENKF_INVALID_ARGUMENT;
  }
  if (mode == 1 && !(scale > 0.0)) {
    set_status(st, ENKF_INVALID_ARGUMENT, "influence scale must be positive");
    return ENKF_INVALID_ARGUMENT;
  }
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaMemsetAsync(p->dstatus, 0, sizeof(DevStatus), s), st);
  CUDA_TRY(launch_localized(p, X, Y, idx, r, delta, scale, mode, XA, s), st);
  return enkf_plan_sync_status(p, stream, st);
}
}  // namespace

int32_t enkf_analysis_localized_f64(enkf_plan* p, const double* X, const double* Y, const int64_t* idx,
                                    const double* r, const double* delta, double* XA, void* stream,
                                    enkf_status* st) {
  if (p && p->n_state > 0 && p->n_obs > 0 && !delta) {
    set_status(st, ENKF_INVALID_ARGUMENT, "null influence matrix");
    return ENKF_INVALID_ARGUMENT;
  }
  return localized_common(p, X, Y, idx, r, delta, 0.0, 0, XA, stream, st);
}

int32_t enkf_analysis_localized_cyclic_f64(enkf_plan* p, const double* X, const double* Y,
                                           const int64_t* idx, const double* r, double scale, double* XA,
                                           void* stream, enkf_status* st) {
  return localized_common(p, X, Y, idx, r, nullptr, scale, 1, XA, stream, st);
}

namespace {
// n_steps RK4 steps of the plan's ensemble, X -> Xout (may alias), on stream s.
cudaError_t launch_l96(enkf_plan* p, const double* X, double* Xout, double dt, double forcing, int n_steps,
                       cudaStream_t s) {
  const int64_t ns = p->n_state;
  const int n = p->n;
  const double half_dt = 0.5 * dt, dt6 = dt / 6.0;  // the reference's scalar factors
  if (ns == 0 || n == 0) return cudaSuccess;
  if (n_steps == 0) {
    return X == Xout ? cudaSuccess
                     : cudaMemcpyAsync(Xout, X, sizeof(double) * (size_t)ns * n, cudaMemcpyDeviceToDevice, s);
  }
  // register path: as few members per CTA as one wave of CTAs allows (the stages are
  // barrier-latency-bound, so the points per thread set the time), rings <= 8192 points
  if (ns <= 8 * L96R_THREADS && ns * (int64_t)n < (1ll << 31)) {
    int mbr = (n + p->num_sms - 1) / p->num_sms;
    if ((int64_t)mbr * ns > 8 * L96R_THREADS) mbr = (int)(8 * L96R_THREADS / ns);
    const int len = (int)ns * mbr;
    const int pt = (len + L96R_THREADS - 1) / L96R_THREADS;
    const size_t smem = 24 * (size_t)len;
    const int grid = (n + mbr - 1) / mbr;
    auto go = [&](auto kern) -> cudaError_t {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      kern<<<grid, L96R_THREADS, smem, s>>>(X, Xout, (int)ns, n, mbr, half_dt, dt, dt6, forcing, n_steps, p->dstatus);
      return cudaGetLastError();
    };
    if (pt <= 1) return go(l96_rk4_reg_kernel<1>);
    if (pt <= 2) return go(l96_rk4_reg_kernel<2>);
    if (pt <= 4) return go(l96_rk4_reg_kernel<4>);
    return go(l96_rk4_reg_kernel<8>);
  }
  int mb = (int)std::min<int64_t>((int64_t)(L96_SMEM_MAX / (32 * (size_t)ns)), (int64_t)n);
  if (mb >= 1) {
    const size_t smem = 32 * (size_t)ns * mb;
    cudaError_t e = cudaFuncSetAttribute(l96_rk4_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    l96_rk4_smem_kernel<<<(n + mb - 1) / mb, L96_THREADS, smem, s>>>(X, Xout, ns, n, mb, half_dt, dt, dt6,
                                                                      forcing, n_steps, p->dstatus);
    return cudaGetLastError();
  }
  if (!p->l96ws) {
    cudaError_t e = cudaMalloc(&p->l96ws, 3 * sizeof(double) * (size_t)ns * n);
    if (e != cudaSuccess) return e;
  }
  double* sa = p->l96ws;
  double* sb = sa + (size_t)ns * n;
  double* acc = sb + (size_t)ns * n;
  if (X != Xout) {
    cudaError_t e = cudaMemcpyAsync(Xout, X, sizeof(double) * (size_t)ns * n, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
  }
  const int grid = std::max(1, std::min(p->num_sms * 8, (int)((ns * n + 255) / 256)));
  for (int step = 0; step < n_steps; ++step) {
    l96_stage_kernel<<<grid, 256, 0, s>>>(Xout, Xout, acc, sa, ns, n, 0, half_dt, dt, dt6, forcing, step, p->dstatus);
    l96_stage_kernel<<<grid, 256, 0, s>>>(Xout, sa, acc, sb, ns, n, 1, half_dt, dt, dt6, forcing, step, p->dstatus);
    l96_stage_kernel<<<grid, 256, 0, s>>>(Xout, sb, acc, sa, ns, n, 2, half_dt, dt, dt6, forcing, step, p->dstatus);
    l96_stage_kernel<<<grid, 256, 0, s>>>(Xout, sa, acc, Xout, ns, n, 3, half_dt, dt, dt6, forcing, step, p->dstatus);
  }
  return cudaGetLastError();
}

int check_l96(const enkf_plan* p, double dt, int n_steps, enkf_status* st) {
  if (p->n_state < 4) {
    set_status(st, ENKF_INVALID_ARGUMENT, "state must have at least 4 components");
    return ENKF_INVALID_ARGUMENT;
  }
  if (!(dt > 0.0)) {
    set_status(st, ENKF_INVALID_ARGUMENT, "dt must be positive");
    return ENKF_INVALID_ARGUMENT;
  }
  if (n_steps < 0) {
    set_status(st, ENKF_INVALID_ARGUMENT, "negative step count");
    return ENKF_INVALID_ARGUMENT;
  }
  return ENKF_OK;
}
}  // namespace

int32_t enkf_forecast_l96_f64(enkf_plan* p, const double* X, double* Xout, double dt, double forcing,
                              int32_t n_steps, void* stream, enkf_status* st) {
  DeviceGuard device_guard;
  if (check_plan(p, st)) return ENKF_INVALID_ARGUMENT;
  if (int rc = check_l96(p, dt, n_steps, st)) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaMemsetAsync(p->dstatus, 0, sizeof(DevStatus), s), st);
  CUDA_TRY(launch_l96(p, X, Xout, dt, forcing, n_steps, s), st);
  return enkf_plan_sync_status(p, stream, st);
}

int32_t enkf_inflate_f64(const double* X, double* Xout, int64_t n_rows, int64_t n_ens, double alpha,
                         void* stream) {
  if (!(alpha >= 1.0) || n_ens < 1 || n_rows < 0) return ENKF_INVALID_ARGUMENT;
  if (n_rows == 0) return ENKF_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (alpha == 1.0) {  // the reference returns x itself
    if (X == Xout) return ENKF_OK;
    return cudaMemcpyAsync(Xout, X, sizeof(double) * (size_t)n_rows * n_ens, cudaMemcpyDeviceToDevice, s) == cudaSuccess
               ? ENKF_OK : ENKF_CUDA_ERROR;
  }
  inflate_kernel<<<(unsigned)((n_rows * 32 + 255) / 256), 256, 0, s>>>(X, Xout, n_rows, (int)n_ens, alpha);
  return cudaGetLastError() == cudaSuccess ? ENKF_OK : ENKF_CUDA_ERROR;
}

namespace {
// forecast -> (inflation) -> analysis cycles; loc_scale > 0: the analysis is localized
// with the cyclic influence matrix of that scale (evaluated in-kernel)
int cycle_l96(enkf_plan* p, double* X, const double* Ys, const int64_t* idx, const double* r, int32_t n_cycles,
              int32_t steps_per_cycle, double dt, double forcing, double inflation, double loc_scale,
              double* mean_f, double* mean_a, void* stream, enkf_status* st, int32_t* failed_cycle) {
  if (failed_cycle) *failed_cycle = -1;
  DeviceGuard device_guard;
  if (check_plan(p, st)) return ENKF_INVALID_ARGUMENT;
  if (p->comm) {
    set_status(st, ENKF_NOT_SUPPORTED, "not provided on a sharded plan (communicator attached)");
    return ENKF_NOT_SUPPORTED;
  }
  if (p->n < 2) {
    set_status(st, ENKF_INVALID_ARGUMENT, "analysis needs at least 2 ensemble members");
    return ENKF_INVALID_ARGUMENT;
  }
  if (int rc = check_l96(p, dt, steps_per_cycle, st)) return rc;
  if (!(inflation >= 1.0)) {
    set_status(st, ENKF_INVALID_ARGUMENT, "inflation factor must be >= 1, got %g", inflation);
    return ENKF_INVALID_ARGUMENT;
  }
  if (n_cycles < 0) {
    set_status(st, ENKF_INVALID_ARGUMENT, "negative cycle count");
    return ENKF_INVALID_ARGUMENT;
  }
  if (n_cycles == 0) {
    set_status(st, ENKF_OK, "ok");
    return ENKF_OK;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (p->cyc_cap < n_cycles) {
    cudaFree(p->cyc_status);
    p->cyc_status = nullptr;
    p->cyc_cap = 0;
    CUDA_TRY(cudaMalloc(&p->cyc_status, sizeof(DevStatus) * (size_t)n_cycles), st);
    p->cyc_cap = n_cycles;
  }
  CUDA_TRY(cudaMemsetAsync(p->cyc_status, 0, sizeof(DevStatus) * (size_t)n_cycles, s), st);
  DevStatus* saved = p->dstatus;
  const double cscale = 1.0 / std::sqrt((double)(p->n - 1));
  const size_t yelems = (size_t)p->n_obs * p->n;
  const unsigned mean_grid = (unsigned)((p->n_state * 32 + 255) / 256);
  cudaError_t e = cudaSuccess;
  for (int c = 0; c < n_cycles && e == cudaSuccess; ++c) {
    p->dstatus = p->cyc_status + c;  // every kernel of cycle c flags into its own status
    e = launch_l96(p, X, X, dt, forcing, steps_per_cycle, s);
    if (e == cudaSuccess && mean_f) {
      row_mean_kernel<<<mean_grid, 256, 0, s>>>(X, mean_f + (size_t)c * p->n_state, p->n_state, p->n);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess && inflation > 1.0) {  // experiment.py:466-467, after the forecast error
      inflate_kernel<<<mean_grid, 256, 0, s>>>(X, X, p->n_state, p->n, inflation);
      e = cudaGetLastError();
    }
    if (loc_scale > 0.0) {  // experiment.py:470-473 with localization=influence_matrix_cyclic(...)
      if (e == cudaSuccess) e = launch_localized(p, X, Ys + (size_t)c * yelems, idx, r, nullptr, loc_scale, 1, X, s);
    } else if (p->tiny && tiny_eligible(p->n_state, p->n_obs, p->n)) {
      if (e == cudaSuccess) e = launch_tiny(p, X, Ys + (size_t)c * yelems, idx, r, X, s);
    } else {
      if (e == cudaSuccess) e = launch_gram(p, true, X, Ys + (size_t)c * yelems, idx, r, p->gram, s);
      if (e == cudaSuccess) e = launch_levels(p, p->gram, p->A, p->T, p->den, cscale, s);
      if (e == cudaSuccess) e = launch_rowgemm<0>(p, X, p->T, nullptr, nullptr, X, p->n_state, s);
    }
    if (e == cudaSuccess && mean_a) {
      row_mean_kernel<<<mean_grid, 256, 0, s>>>(X, mean_a + (size_t)c * p->n_state, p->n_state, p->n);
      e = cudaGetLastError();
    }
  }
  p->dstatus = saved;
  if (e != cudaSuccess) return cuda_fail(st, e, "enkf_cycle_l96_f64 launch");
  std::vector<DevStatus> hs((size_t)n_cycles);
  CUDA_TRY(cudaMemcpyAsync(hs.data(), p->cyc_status, sizeof(DevStatus) * (size_t)n_cycles, cudaMemcpyDeviceToHost,
                           s), st);
  CUDA_TRY(cudaStreamSynchronize(s), st);
  for (int c = 0; c < n_cycles; ++c) {
    if (hs[(size_t)c].flags == 0) continue;
    *p->hstatus = hs[(size_t)c];
    if (failed_cycle) *failed_cycle = c;
    return translate_status(p, st);
  }
  set_status(st, ENKF_OK, "ok");
  return ENKF_OK;
}
}  // namespace

int32_t enkf_cycle_l96_f64(enkf_plan* p, double* X, const double* Ys, const int64_t* idx, const double* r,
                           int32_t n_cycles, int32_t steps_per_cycle, double dt, double forcing, double inflation,
                           double* mean_f, double* mean_a, void* stream, enkf_status* st,
                           int32_t* failed_cycle) {
  return cycle_l96(p, X, Ys, idx, r, n_cycles, steps_per_cycle, dt, forcing, inflation, 0.0, mean_f, mean_a,
                   stream, st, failed_cycle);
}

int32_t enkf_cycle_l96_localized_f64(enkf_plan* p, double* X, const double* Ys, const int64_t* idx,
                                     const double* r, int32_t n_cycles, int32_t steps_per_cycle, double dt,
                                     double forcing, double inflation, double loc_scale, double* mean_f,
                                     double* mean_a, void* stream, enkf_status* st, int32_t* failed_cycle) {
  if (!(loc_scale > 0.0)) {
    if (failed_cycle) *failed_cycle = -1;
    set_status(st, ENKF_INVALID_ARGUMENT, "influence scale must be positive");
    return ENKF_INVALID_ARGUMENT;
  }
  return cycle_l96(p, X, Ys, idx, r, n_cycles, steps_per_cycle, dt, forcing, inflation, loc_scale, mean_f, mean_a,
                   stream, st, failed_cycle);
}

// Profiling-only: per-block phase clocks of the blocked levels kernel (-DLV_TRACE_ON)
__attribute__((visibility("default"))) int32_t enkf_debug_lv_trace(long long* out) {
  return cudaMemcpyFromSymbol(out, enkf::g_lv_trace, sizeof(enkf::g_lv_trace)) == cudaSuccess ? 0 : 5;
}
// Profiling-only (not part of include/enkf_b200.h): CTA-0 event trace of the
// int8 anomaly kernel, filled when ENKF_I8_DBG has bit 3 set.
__attribute__((visibility("default"))) int32_t enkf_debug_i8_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, enkf::g_i8_trace, sizeof(enkf::g_i8_trace)) == cudaSuccess ? 0 : 5;
}

// ---- multi-GPU: NCCL communicator (nccl_comm.cuh) ----
int32_t enkf_comm_unique_id(unsigned char* id, enkf_status* st) {
  const NcclApi& api = nccl_api();
  if (!api.ok) {
    set_status(st, ENKF_NOT_SUPPORTED, "%s", api.why);
    return ENKF_NOT_SUPPORTED;
  }
  if (!id) {
    set_status(st, ENKF_INVALID_ARGUMENT, "null id buffer");
    return ENKF_INVALID_ARGUMENT;
  }
  ncclUniqueId u;
  const ncclResult_t rc = api.get_unique_id(&u);
  if (rc != ncclSuccess) {
    set_status(st, ENKF_CUDA_ERROR, "ncclGetUniqueId: %s", api.error_string(rc));
    return ENKF_CUDA_ERROR;
  }
  memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  set_status(st, ENKF_OK, "ok");
  return ENKF_OK;
}

int32_t enkf_comm_init(const unsigned char* id, int32_t nranks, int32_t rank, int32_t device, void** comm,
                       enkf_status* st) {
  const NcclApi& api = nccl_api();
  if (!api.ok) {
    set_status(st, ENKF_NOT_SUPPORTED, "%s", api.why);
    return ENKF_NOT_SUPPORTED;
  }
  if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks) {
    set_status(st, ENKF_INVALID_ARGUMENT, "invalid communicator arguments (nranks=%d rank=%d)", nranks, rank);
    return ENKF_INVALID_ARGUMENT;
  }
  DeviceGuard device_guard;
  if (cudaSetDevice(device) != cudaSuccess) {
    set_status(st, ENKF_CUDA_ERROR, "cudaSetDevice(%d) failed", device);
    return ENKF_CUDA_ERROR;
  }
  ncclUniqueId u;
  memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
  ncclComm_t c = nullptr;
  const ncclResult_t rc = api.comm_init_rank(&c, nranks, u, rank);
  if (rc != ncclSuccess) {
    set_status(st, ENKF_CUDA_ERROR, "ncclCommInitRank(nranks=%d, rank=%d): %s", nranks, rank, api.error_string(rc));
    return ENKF_CUDA_ERROR;
  }
  *comm = c;
  set_status(st, ENKF_OK, "ok");
  return ENKF_OK;
}

int32_t enkf_comm_destroy(void* comm) {
  if (!comm) return ENKF_OK;
  const NcclApi& api = nccl_api();
  if (!api.ok) return ENKF_NOT_SUPPORTED;
  return api.comm_destroy((ncclComm_t)comm) == ncclSuccess ? ENKF_OK : ENKF_CUDA_ERROR;
}

int32_t enkf_plan_set_comm(enkf_plan* p, void* comm, enkf_status* st) {
  DeviceGuard device_guard;
  if (check_plan(p, st)) return ENKF_INVALID_ARGUMENT;
  if (!comm) {
    p->comm = nullptr;
    p->comm_ranks = 1;
    p->comm_rank = 0;
    set_status(st, ENKF_OK, "ok");
    return ENKF_OK;
  }
  const NcclApi& api = nccl_api();
  if (!api.ok) {
    set_status(st, ENKF_NOT_SUPPORTED, "%s", api.why);
    return ENKF_NOT_SUPPORTED;
  }
  int ranks = 0, rank = 0;
  if (api.comm_count((ncclComm_t)comm, &ranks) != ncclSuccess ||
      api.comm_user_rank((ncclComm_t)comm, &rank) != ncclSuccess) {
    set_status(st, ENKF_INVALID_ARGUMENT, "not a valid ncclComm_t");
    return ENKF_INVALID_ARGUMENT;
  }
  if (p->n < 2) {
    set_status(st, ENKF_INVALID_ARGUMENT, "analysis needs at least 2 ensemble members");
    return ENKF_INVALID_ARGUMENT;
  }
  p->comm = (ncclComm_t)comm;
  p->comm_ranks = ranks;
  p->comm_rank = rank;
  set_status(st, ENKF_OK, "ok");
  return ENKF_OK;
}

// Measurement-only (not part of include/enkf_b200.h): CUDA events at the stage
// boundaries of enkf_analysis_async_f64 (gram | allreduce | levels | anomaly).
__attribute__((visibility("default"))) int32_t enkf_debug_set_stage_events(enkf_plan* p, int32_t on) {
  if (!p) return ENKF_INVALID_ARGUMENT;
  if (on && !p->stage_events) p->st_steps = 0;  // a new measurement window
  p->stage_events = on != 0;
  return ENKF_OK;
}
// ms of the last step's gram, allreduce, levels and anomaly stages (caller synchronised)
__attribute__((visibility("default"))) int32_t enkf_debug_stage_times(enkf_plan* p, float* out4) {
  if (!p || !p->st_ev[4]) return ENKF_INVALID_ARGUMENT;
  for (int i = 0; i < 4; ++i)
    if (cudaEventElapsedTime(&out4[i], p->st_ev[i], p->st_ev[i + 1]) != cudaSuccess) return ENKF_CUDA_ERROR;
  return ENKF_OK;
}
// mean ms of the four stages over the steps recorded since the events were switched on
// (at most the last 64; caller synchronised); *n_steps = how many were averaged
__attribute__((visibility("default"))) int32_t enkf_debug_stage_times_mean(enkf_plan* p, float* out4, int32_t* n_steps) {
  if (!p || p->st_steps <= 0) return ENKF_INVALID_ARGUMENT;
  const long n = p->st_steps < enkf_plan::ST_SETS ? p->st_steps : (long)enkf_plan::ST_SETS;
  double acc[4] = {0, 0, 0, 0};
  for (long k = 0; k < n; ++k) {
    cudaEvent_t* ev = p->st_evs[(p->st_steps - 1 - k) % enkf_plan::ST_SETS];
    for (int i = 0; i < 4; ++i) {
      float ms = 0.f;
      if (!ev[i] || !ev[i + 1] || cudaEventElapsedTime(&ms, ev[i], ev[i + 1]) != cudaSuccess) return ENKF_CUDA_ERROR;
      acc[i] += ms;
    }
  }
  for (int i = 0; i < 4; ++i) out4[i] = (float)(acc[i] / (double)n);
  if (n_steps) *n_steps = (int32_t)n;
  return ENKF_OK;
}

// Measurement-only (not part of include/enkf_b200.h): CUDA events around the
// int8 Gram's slice pass and MMA pass (two-kernel form) of this plan.
__attribute__((visibility("default"))) int32_t enkf_debug_set_gram_events(enkf_plan* p, int32_t on) {
  if (!p) return ENKF_INVALID_ARGUMENT;
  p->g8_events = on != 0;
  return ENKF_OK;
}
// ms of the last slice and MMA passes (the caller has synchronised)
__attribute__((visibility("default"))) int32_t enkf_debug_gram_times(enkf_plan* p, float* out2) {
  if (!p || !p->g8_ev[2]) return ENKF_INVALID_ARGUMENT;
  if (cudaEventElapsedTime(&out2[0], p->g8_ev[0], p->g8_ev[1]) != cudaSuccess) return ENKF_CUDA_ERROR;
  if (cudaEventElapsedTime(&out2[1], p->g8_ev[1], p->g8_ev[2]) != cudaSuccess) return ENKF_CUDA_ERROR;
  return ENKF_OK;
}

}  // extern "C"
