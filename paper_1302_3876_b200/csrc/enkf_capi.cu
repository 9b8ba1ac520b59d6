// enkf_capi.cu — the C ABI (include/enkf_b200.h) over the sm_100a kernels.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdarg>
#include <cstring>
#include <new>

#include "../../include/enkf_b200.h"
#include "enkf_kernels.cuh"

using namespace enkf;

struct enkf_plan {
  int64_t n_state = 0, n_obs = 0;
  int n = 0;
  int device = 0;
  int num_sms = 0;
  int splits = 1;
  int64_t rows_per_split = 0;
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
};

namespace {

const char* kVersion = "enkf_b200 0.1.0 sm_100a";

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

cudaError_t launch_gram(const enkf_plan* p, bool analysis, const double* X, const double* Y,
                        const int64_t* idx, const double* r, double* gram, cudaStream_t s) {
  const int n = p->n;
  if (p->n_obs == 0) return cudaMemsetAsync(gram, 0, sizeof(double) * n * 2 * n, s);
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

cudaError_t launch_levels(const enkf_plan* p, const double* gram, double* A, double* T,
                          double* den, double cscale, cudaStream_t s) {
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
  const int ld = padded_ld(n);
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

template <int MODE>
cudaError_t launch_rowgemm(const enkf_plan* p, const double* P, const double* Q, const double* C,
                           const double* r, double* out, int64_t n_rows, cudaStream_t s) {
  const int n = p->n;
  const bool vec = (n % 2 == 0) && aligned16(P) && aligned16(out) && (C == nullptr || aligned16(C));
#define ENKF_RG(NPV)                                                                   \
  if (n <= NPV) return vec ? launch_rowgemm_t<NPV, MODE, true>(p, P, Q, C, r, out, n_rows, s) \
                           : launch_rowgemm_t<NPV, MODE, false>(p, P, Q, C, r, out, n_rows, s);
  ENKF_RG(8) ENKF_RG(16) ENKF_RG(32) ENKF_RG(48) ENKF_RG(64) ENKF_RG(96) ENKF_RG(128)
#undef ENKF_RG
  return cudaErrorInvalidValue;
}

int translate_status(const enkf_plan* p, enkf_status* st) {
  const DevStatus& d = *p->hstatus;
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

int32_t enkf_plan_create(int64_t n_state, int64_t n_obs, int64_t n_ens, enkf_plan** out,
                         enkf_status* st) {
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

  const size_t nn = (size_t)n * n;
  e = cudaMalloc(&p->partial, sizeof(double) * (size_t)splits * 2 * nn);
  if (e == cudaSuccess) e = cudaMalloc(&p->gram, sizeof(double) * 2 * nn);
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
  *out = p;
  set_status(st, ENKF_OK, "ok");
  return ENKF_OK;
}

void enkf_plan_destroy(enkf_plan* p) {
  if (!p) return;
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
  delete p;
}

int32_t enkf_ism_gram_f64(enkf_plan* p, const double* X, const double* Y, const int64_t* idx,
                          const double* r, double* gram, void* stream) {
  if (check_plan(p, nullptr)) return ENKF_INVALID_ARGUMENT;
  if (p->n < 2) return ENKF_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = launch_gram(p, true, X, Y, idx, r, gram, s);
  return e == cudaSuccess ? ENKF_OK : ENKF_CUDA_ERROR;
}

int32_t enkf_ism_levels_f64(enkf_plan* p, const double* gram, double* A, double* T, double* den,
                            void* stream) {
  if (check_plan(p, nullptr)) return ENKF_INVALID_ARGUMENT;
  const double cscale = p->n > 1 ? 1.0 / std::sqrt((double)(p->n - 1)) : 0.0;
  cudaError_t e = launch_levels(p, gram, A, T, den, cscale, (cudaStream_t)stream);
  return e == cudaSuccess ? ENKF_OK : ENKF_CUDA_ERROR;
}

int32_t enkf_anomaly_update_f64(enkf_plan* p, const double* X, const double* T, double* XA,
                                int64_t n_rows, void* stream) {
  if (check_plan(p, nullptr)) return ENKF_INVALID_ARGUMENT;
  cudaError_t e = launch_rowgemm<0>(p, X, T, nullptr, nullptr, XA, n_rows, (cudaStream_t)stream);
  return e == cudaSuccess ? ENKF_OK : ENKF_CUDA_ERROR;
}

int32_t enkf_analysis_async_f64(enkf_plan* p, const double* X, const double* Y, const int64_t* idx,
                                const double* r, double* XA, void* stream) {
  if (check_plan(p, nullptr)) return ENKF_INVALID_ARGUMENT;
  if (p->n < 2) return ENKF_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(p->dstatus, 0, sizeof(DevStatus), s);
  if (e == cudaSuccess) e = launch_gram(p, true, X, Y, idx, r, p->gram, s);
  const double cscale = 1.0 / std::sqrt((double)(p->n - 1));
  if (e == cudaSuccess) e = launch_levels(p, p->gram, p->A, p->T, p->den, cscale, s);
  if (e == cudaSuccess) e = launch_rowgemm<0>(p, X, p->T, nullptr, nullptr, XA, p->n_state, s);
  return e == cudaSuccess ? ENKF_OK : ENKF_CUDA_ERROR;
}

int32_t enkf_plan_sync_status(enkf_plan* p, void* stream, enkf_status* st) {
  if (check_plan(p, st)) return ENKF_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaMemcpyAsync(p->hstatus, p->dstatus, sizeof(DevStatus), cudaMemcpyDeviceToHost, s), st);
  CUDA_TRY(cudaStreamSynchronize(s), st);
  return translate_status(p, st);
}

int32_t enkf_plan_reset_status(enkf_plan* p, void* stream) {
  if (check_plan(p, nullptr)) return ENKF_INVALID_ARGUMENT;
  return cudaMemsetAsync(p->dstatus, 0, sizeof(DevStatus), (cudaStream_t)stream) == cudaSuccess
             ? ENKF_OK : ENKF_CUDA_ERROR;
}

int32_t enkf_analysis_f64(enkf_plan* p, const double* X, const double* Y, const int64_t* idx,
                          const double* r, double* XA, void* stream, enkf_status* st) {
  if (check_plan(p, st)) return ENKF_INVALID_ARGUMENT;
  if (p->n < 2) {
    set_status(st, ENKF_INVALID_ARGUMENT, "analysis needs at least 2 ensemble members");
    return ENKF_INVALID_ARGUMENT;
  }
  int rc = enkf_analysis_async_f64(p, X, Y, idx, r, XA, stream);
  if (rc != ENKF_OK) {
    CUDA_TRY(cudaGetLastError(), st);
    set_status(st, rc, "launch failed");
    return rc;
  }
  return enkf_plan_sync_status(p, stream, st);
}

int32_t enkf_analysis_host_f64(enkf_plan* p, const double* X_h, const double* Y_h,
                               const int64_t* idx_h, const double* r_h, double* XA_h,
                               enkf_status* st) {
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
  CUDA_TRY(cudaMemcpyAsync(p->hx, X_h, sizeof(double) * (size_t)p->n_state * n, cudaMemcpyHostToDevice, s), st);
  CUDA_TRY(cudaMemcpyAsync(p->hy, Y_h, sizeof(double) * (size_t)p->n_obs * n, cudaMemcpyHostToDevice, s), st);
  CUDA_TRY(cudaMemcpyAsync(p->hr, r_h, sizeof(double) * (size_t)p->n_obs, cudaMemcpyHostToDevice, s), st);
  const int64_t* didx = nullptr;
  if (idx_h) {
    CUDA_TRY(cudaMemcpyAsync(p->hidx, idx_h, sizeof(int64_t) * (size_t)p->n_obs, cudaMemcpyHostToDevice, s), st);
    didx = p->hidx;
  }
  // In place: XA overwrites the device copy of X.
  int rc = enkf_analysis_async_f64(p, p->hx, p->hy, didx, p->hr, p->hx, s);
  if (rc != ENKF_OK) {
    CUDA_TRY(cudaGetLastError(), st);
    set_status(st, rc, "launch failed");
    return rc;
  }
  CUDA_TRY(cudaMemcpyAsync(XA_h, p->hx, sizeof(double) * (size_t)p->n_state * n, cudaMemcpyDeviceToHost, s), st);
  return enkf_plan_sync_status(p, s, st);
}

int32_t enkf_ism_solve_f64(enkf_plan* p, const double* r, const double* V, const double* D,
                           double* Z, double* A, void* stream, enkf_status* st) {
  if (check_plan(p, st)) return ENKF_INVALID_ARGUMENT;
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

}  // extern "C"
