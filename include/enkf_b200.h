/*
 * enkf_b200.h — C ABI of the B200-native EnKF analysis step
 * (iterative Sherman-Morrison, arXiv 1302.3876).
 *
 * Plain pointers and sizes only; no torch types.  Every entry point names the
 * reference interface it replaces (files under /root/reference/pkg/src/enkfkit,
 * read-only, not shipped):
 *
 *   enkf_analysis_f64       enkf.py:167-192   analysis_step(x, obs, h, r, "sherman")
 *                                              (unlocalized branch, workers ignored)
 *   enkf_analysis_host_f64  same, host buffers (copies in/out inside the call)
 *   enkf_ism_solve_f64      sherman.py:253-286 solve_sherman(r, v, d) -> SolverResult.z
 *   enkf_ism_gram_f64       sherman.py:149-205 level 0 + the per-level dots v_k'u (K4/K5/K8),
 *                           fused into one Gram pass; the multi-GPU split point
 *   enkf_ism_levels_f64     sherman.py:164-187 the N Sherman-Morrison levels (den_k, singular
 *                           guard, composition), run on the reduced N x 2N Gram
 *   enkf_anomaly_update_f64 enkf.py:192        x + s @ A  (A = v' z), as X @ T
 *   enkf_member_deviations_f64 enkf.py:82-92   member_deviations
 *   enkf_innovations_f64    enkf.py:114-120    innovations (Y - H X)
 *   enkf_analysis_localized_f64        enkf.py:193-199  analysis_step(..., localization=delta)
 *   enkf_analysis_localized_cyclic_f64 enkf.py:193-199 with delta = influence_matrix_cyclic
 *                           (enkf.py:138-164) evaluated on the fly (matrix-free)
 *   enkf_forecast_l96_f64   models/lorenz96.py:31-78  Lorenz96.advance (RK4 steps), bit-exact
 *   enkf_cycle_l96_f64      experiment.py:457-479     forecast -> (inflation) -> analysis cycles, device-resident
 *   enkf_cycle_l96_localized_f64 experiment.py:457-479 the same with the localized (cyclic taper) analysis
 *   enkf_inflate_f64        enkf.py:123-135           inflate (covariance inflation about the row mean)
 *
 * Layouts (all fp64 row-major, the reference's C-order arrays):
 *   X, XA : [n_state][n_ens]      Y, D, V, Z : [n_obs][n_ens]
 *   idx   : int64 [n_obs], strictly increasing, or NULL for the identity H
 *   r     : [n_obs] observation-error variances (> 0)
 *   gram  : [n_ens][2 n_ens]      A, T : [n_ens][n_ens]
 * Device pointers unless the name says _host.  Stream = cudaStream_t as void*.
 *
 * Status codes map 1:1 onto the reference's exceptions (errors.py, enkf.py):
 *   ENKF_OK                 -> (return value)
 *   ENKF_INVALID_ARGUMENT   -> ValueError        (sherman.py:85-108, enkf.py:185-186)
 *   ENKF_INDEX_RANGE        -> IndexError        (enkf.py:54-58)
 *   ENKF_SINGULAR_UPDATE    -> SingularUpdateError(level, denominator) (sherman.py:171-174)
 *   ENKF_NOT_SUPPORTED      -> NotImplementedError (shape outside the kernels' range)
 *   ENKF_CUDA_ERROR         -> RuntimeError
 *   ENKF_DIVERGED           -> DivergenceError(member) (models/lorenz96.py:52-58; status.level
 *                              = the first non-finite ensemble column)
 */
#ifndef ENKF_B200_H
#define ENKF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum enkf_code {
  ENKF_OK = 0,
  ENKF_INVALID_ARGUMENT = 1,
  ENKF_INDEX_RANGE = 2,
  ENKF_SINGULAR_UPDATE = 3,
  ENKF_NOT_SUPPORTED = 4,
  ENKF_CUDA_ERROR = 5,
  ENKF_DIVERGED = 6
};

typedef struct enkf_status {
  int32_t code;        /* enum enkf_code */
  int32_t level;       /* 1-based Sherman-Morrison level for ENKF_SINGULAR_UPDATE */
  double denominator;  /* 1 + v_k' u_k at that level */
  char message[256];
} enkf_status;

typedef struct enkf_plan enkf_plan;

/* Library identification: "enkf_b200 <version> sm_100a". */
const char* enkf_version(void);
/* Largest ensemble size the kernels accept (the N x 2N Gram recursion runs in
 * one CTA's shared memory). */
int32_t enkf_max_ens(void);

/* Select the CUDA device for subsequent plan creation / helper calls on this
 * host thread (the library links its own CUDA runtime; callers that manage
 * devices elsewhere, e.g. torch, pass their device index here). */
int32_t enkf_set_device(int32_t device);
/* The calling thread's current CUDA device (so a caller can restore it after
 * enkf_set_device; every plan entry point already restores it on return). */
int32_t enkf_get_device(int32_t* device);

/* Plan: owns the device workspace (Gram partials, the int8 Gram's operand
 * images, Gram, A, T, status) for one (n_state, n_obs, n_ens) shape on the
 * current device, all allocated here: the device-buffer analysis calls
 * (enkf_analysis_f64 / _async_f64 and the staged form) allocate nothing, so they
 * can be captured into a CUDA graph without a warm-up call.  Entries that need
 * workspace only some callers use allocate it on their first call and keep it
 * with the plan: the host-buffer entry (device copies of X, Y, r, idx), the
 * localized analysis (V, D, Z) and the Lorenz-96 forecast / cycle entries.
 * Every entry point runs on the plan's device and restores the caller's current
 * device before returning.  Thread-safe per plan (one call at a time). */
int32_t enkf_plan_create(int64_t n_state, int64_t n_obs, int64_t n_ens,
                         enkf_plan** plan, enkf_status* status);

/* Kernel and host-path choices of a plan (the reference has no counterpart: its
 * module constants GROUP_LEVELS / SINGULAR_TOL are fixed, sherman.py:51, 146).
 * enkf_plan_options_default() fills the product defaults, then applies the
 * process-wide ENKF_* environment overrides;
 * enkf_plan_create(...) == enkf_plan_create_ex(..., NULL, ...) uses exactly that.
 * Every choice computes the same analysis within the parity tolerance; they exist
 * for A/B measurement and for callers that require IEEE FP64 arithmetic. */
enum enkf_gram_kernel { ENKF_GRAM_INT8 = 0 /* exact int8-digit tcgen05 (N = 128) */, ENKF_GRAM_FP64 = 1 /* DMMA */ };
enum enkf_anomaly_kernel { ENKF_ANOMALY_INT8 = 0, ENKF_ANOMALY_FP64 = 1 };
enum enkf_levels_kernel { ENKF_LEVELS_CLUSTER = 0, ENKF_LEVELS_SINGLE_CTA = 1, ENKF_LEVELS_PER_LEVEL = 2 };
typedef struct enkf_plan_options {
  int32_t struct_size;        /* sizeof(enkf_plan_options): set by enkf_plan_options_default */
  int32_t gram_kernel;        /* enum enkf_gram_kernel */
  int32_t anomaly_kernel;     /* enum enkf_anomaly_kernel */
  int32_t levels_kernel;      /* enum enkf_levels_kernel */
  int32_t localized_dmma;     /* 1: DMMA localized update (default), 0: CUDA-core form */
  int32_t tiny_kernel;        /* 1: single-CTA step for desk-scale shapes (default), 0: multi-kernel */
  int32_t host_stream;        /* 1: streamed host entry (default), 0: copy in / step / copy out */
  int32_t host_trace;         /* 1: phase times of the host entry on stderr */
  int64_t host_chunk_bytes;   /* X / XA chunk of the streamed host entry (default 256 MiB; 0 = the smallest chunk) */
  int64_t host_ring_bytes;    /* pinned staging-ring slot for pageable buffers (default 256 MiB) */
  int64_t host_stream_min_bytes; /* pageable X from this size streams through the rings (default 1 GiB) */
} enkf_plan_options;
int32_t enkf_plan_options_default(enkf_plan_options* options);
int32_t enkf_plan_create_ex(int64_t n_state, int64_t n_obs, int64_t n_ens,
                            const enkf_plan_options* options /* NULL = defaults */,
                            enkf_plan** plan, enkf_status* status);
void enkf_plan_destroy(enkf_plan* plan);

/* Full analysis step on device buffers (single GPU or one shard whose obs rows
 * are all local).  XA may equal X (in-place update).  Synchronous: returns
 * after the stream is drained and the status is read. */
int32_t enkf_analysis_f64(enkf_plan* plan, const double* X, const double* Y,
                          const int64_t* idx, const double* r, double* XA,
                          void* stream, enkf_status* status);

/* Same, without the final synchronisation: the status stays on the device
 * until enkf_plan_sync_status().  Graph-capturable. */
int32_t enkf_analysis_async_f64(enkf_plan* plan, const double* X, const double* Y,
                                const int64_t* idx, const double* r, double* XA,
                                void* stream);
int32_t enkf_plan_sync_status(enkf_plan* plan, void* stream, enkf_status* status);
/* Clear the device status word (start of a staged step). */
int32_t enkf_plan_reset_status(enkf_plan* plan, void* stream);

/* Full analysis step on HOST buffers: copies X, Y, idx, r in, runs the step,
 * copies XA out; returns after every copy has completed.  With page-locked X and
 * XA (and idx given) the call streams: X[idx] gathered over PCIe, the Gram pass,
 * then X chunks in and XA chunks out concurrently.  Pageable buffers go through
 * a pinned staging ring. */
int32_t enkf_analysis_host_f64(enkf_plan* plan, const double* X_h, const double* Y_h,
                               const int64_t* idx_h, const double* r_h, double* XA_h,
                               enkf_status* status);

/* Localized analysis (enkf.py:193-199): XA = X + (delta o (S V')) Z, Z from the
 * ISM solve of (r, V, D).  delta: device fp64 [n_state][n_obs] (row-major, the
 * reference's (nstate, nobs) influence matrix).  S V' is never materialised.
 * Same status semantics as enkf_analysis_f64; synchronous. */
int32_t enkf_analysis_localized_f64(enkf_plan* plan, const double* X, const double* Y,
                                    const int64_t* idx, const double* r, const double* delta,
                                    double* XA, void* stream, enkf_status* status);
/* Matrix-free variant: delta_ij = exp(-d(i, p_j) / scale), d the cyclic distance
 * min(|i - p_j|, n_state - |i - p_j|), p_j = idx[j] (or j when idx is NULL), as
 * influence_matrix_cyclic (enkf.py:138-164).  scale <= 0 -> INVALID_ARGUMENT. */
int32_t enkf_analysis_localized_cyclic_f64(enkf_plan* plan, const double* X, const double* Y,
                                           const int64_t* idx, const double* r, double scale,
                                           double* XA, void* stream, enkf_status* status);

/* Lorenz-96 ensemble forecast (models/lorenz96.py:31-78, enkf.py:202-212):
 * n_steps RK4 steps of size dt with forcing F on the plan's [n_state][n_ens]
 * ensemble, every member independently; X and Xout may alias.  Same
 * operation order as the reference (no FMA contraction): bit-identical.
 * A non-finite state returns ENKF_DIVERGED with status.level = first bad member. */
int32_t enkf_forecast_l96_f64(enkf_plan* plan, const double* X, double* Xout, double dt, double forcing,
                              int32_t n_steps, void* stream, enkf_status* status);
/* Device-resident cycled assimilation (the experiment.py:457-479 loop with the
 * lorenz96 model and pre-staged perturbed observations):
 *   for c in [0, n_cycles): X <- forecast(X, steps_per_cycle); X <- analysis(X, Ys[c], idx, r)
 * X is updated in place.  Ys: [n_cycles][n_obs][n_ens].  mean_f / mean_a
 * (optional, [n_cycles][n_state]) receive the forecast / analysis ensemble
 * means.  inflation > 1 inflates the forecast (after mean_f) as experiment.py:466-467.  No host round trip between cycles; the first failing cycle (0-based)
 * is returned in *failed_cycle (-1 if none) with its error in status. */
int32_t enkf_cycle_l96_f64(enkf_plan* plan, double* X, const double* Ys, const int64_t* idx, const double* r,
                           int32_t n_cycles, int32_t steps_per_cycle, double dt, double forcing, double inflation,
                           double* mean_f, double* mean_a, void* stream, enkf_status* status,
                           int32_t* failed_cycle);
/* The same loop with the localized analysis (experiment.py:470-473 with
 * localization = influence_matrix_cyclic(n_state, h, loc_scale), enkf.py:138-164,
 * 193-199), the taper evaluated in-kernel — the lorenz-small preset's loop.
 * loc_scale <= 0 -> INVALID_ARGUMENT. */
int32_t enkf_cycle_l96_localized_f64(enkf_plan* plan, double* X, const double* Ys, const int64_t* idx,
                                     const double* r, int32_t n_cycles, int32_t steps_per_cycle, double dt,
                                     double forcing, double inflation, double loc_scale, double* mean_f,
                                     double* mean_a, void* stream, enkf_status* status, int32_t* failed_cycle);
/* Covariance inflation (enkf.py:123-135): Xout = mean + alpha (X - mean) per row of the
 * [n_rows][n_ens] ensemble (X may alias Xout); alpha < 1 -> INVALID_ARGUMENT, alpha == 1 copies. */
int32_t enkf_inflate_f64(const double* X, double* Xout, int64_t n_rows, int64_t n_ens, double alpha,
                         void* stream);

/* --- staged form (multi-GPU: partial Gram -> allreduce by the caller -> levels) --- */

/* Level 0 + Gram over this plan's obs rows: gram = [V'R^-1 V | V'R^-1 D]
 * (n_ens x 2 n_ens), V = H S, D = Y - H X, S = (X - mean)/sqrt(N-1).
 * Input checks (non-finite, r <= 0, idx order/range) are flagged on the device. */
int32_t enkf_ism_gram_f64(enkf_plan* plan, const double* X, const double* Y,
                          const int64_t* idx, const double* r, double* gram,
                          void* stream);
/* The N Sherman-Morrison levels on a (globally reduced) Gram.  Writes
 * A = V'Z (n_ens x n_ens), the anomaly transform T = I + (I - 11'/N) A/sqrt(N-1),
 * and den[k] = 1 + v_k'u_k (n_ens) when den != NULL. */
int32_t enkf_ism_levels_f64(enkf_plan* plan, const double* gram, double* A, double* T,
                            double* den, void* stream);
/* XA[rows] = X[rows] @ T  ==  X + S (V'Z).  XA may equal X. */
int32_t enkf_anomaly_update_f64(enkf_plan* plan, const double* X, const double* T,
                                double* XA, int64_t n_rows, void* stream);

/* --- multi-GPU: one process per GPU, state rows sharded ---
 *
 * Rank g owns the contiguous state rows [lo_g, hi_g) and the observation rows whose
 * (sorted) index falls in that range; its plan is created for the LOCAL sizes and
 * its idx is relative to lo_g.  With a communicator attached to the plan,
 * enkf_analysis_f64 / _async_f64 / _host_f64 run one shard of the step: the local
 * level-0 Gram, ONE ncclAllReduce (sum, fp64, on the call's stream) of the N x 2N
 * Gram with the shard's input-check flags appended, the N levels on the identical
 * global Gram (every rank, no broadcast), the anomaly update of the local rows.
 * Every rank returns the same status (an input error on one rank raises on all),
 * with no extra collective or host synchronisation; the async form stays
 * graph-capturable.  Replaces the reference's thread-blocked column sweep
 * (sherman.py:162, 189-203, solve_sherman_blocked) as the parallel scheme.
 * NCCL is loaded at run time (libnccl.so.2); ENKF_NOT_SUPPORTED if it is absent.
 * The localized, cycled and solve_sherman entries return ENKF_NOT_SUPPORTED on a
 * plan with a communicator. */

/* ncclGetUniqueId on rank 0: 128 bytes to hand to every rank (e.g. broadcast over
 * torch.distributed). */
int32_t enkf_comm_unique_id(unsigned char* id /* [128] */, enkf_status* status);
/* ncclCommInitRank for `rank` of `nranks` on CUDA device `device`; *comm receives
 * the ncclComm_t (caller-owned: enkf_comm_destroy). */
int32_t enkf_comm_init(const unsigned char* id /* [128] */, int32_t nranks, int32_t rank, int32_t device,
                       void** comm, enkf_status* status);
int32_t enkf_comm_destroy(void* comm);
/* Attach an ncclComm_t (from enkf_comm_init or the caller's own NCCL) to a plan;
 * NULL detaches.  The communicator must outlive the plan's use of it. */
int32_t enkf_plan_set_comm(enkf_plan* plan, void* comm, enkf_status* status);

/* --- solve_sherman parity (sherman.py:253-286): Z = (R + V V')^-1 D --- */
int32_t enkf_ism_solve_f64(enkf_plan* plan, const double* r, const double* V,
                           const double* D, double* Z, double* A, void* stream,
                           enkf_status* status);

/* --- row-local helpers of the path --- */
int32_t enkf_member_deviations_f64(const double* X, double* S, int64_t n_rows,
                                   int64_t n_ens, void* stream);
int32_t enkf_innovations_f64(const double* X, const double* Y, const int64_t* idx,
                             double* D, int64_t n_obs, int64_t n_ens, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ENKF_B200_H */
