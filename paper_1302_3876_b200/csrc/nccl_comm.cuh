// nccl_comm.cuh — the multi-GPU exchange of the analysis step in the
// native layer: ONE ncclAllReduce per step, on the compute stream, of the N x 2N
// level-0 Gram with the shard's input-check flags appended, so every rank runs the
// N Sherman-Morrison levels on the identical global Gram and agrees on the outcome
// (a bad input on one rank raises the same error on all ranks) without a second
// collective or a host synchronisation.  Graph-capturable (NCCL collectives are).
//
// NCCL is loaded at run time (dlopen of libnccl.so.2, resolved with dlsym): a
// single-GPU user never loads it, and inside a torch process the library shares
// the libnccl torch already loaded (same soname) instead of pinning another build.
// nccl.h supplies the types only.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "enkf_kernels.cuh"

namespace enkf {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*comm_count)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*comm_user_rank)(const ncclComm_t, int*) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
  char why[256] = {0};
};

inline const NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      snprintf(api.why, sizeof(api.why), "libnccl.so.2 not loadable: %s", dlerror());
      return;
    }
#define ENKF_NCCL_SYM(field, name)                                                  \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));                \
  if (!api.field) {                                                                 \
    snprintf(api.why, sizeof(api.why), "libnccl.so.2 lacks %s", name);              \
    return;                                                                         \
  }
    ENKF_NCCL_SYM(get_unique_id, "ncclGetUniqueId")
    ENKF_NCCL_SYM(comm_init_rank, "ncclCommInitRank")
    ENKF_NCCL_SYM(all_reduce, "ncclAllReduce")
    ENKF_NCCL_SYM(comm_destroy, "ncclCommDestroy")
    ENKF_NCCL_SYM(comm_count, "ncclCommCount")
    ENKF_NCCL_SYM(comm_user_rank, "ncclCommUserRank")
    ENKF_NCCL_SYM(error_string, "ncclGetErrorString")
#undef ENKF_NCCL_SYM
    api.ok = true;
  });
  return api;
}

// Input-check flags that travel with the Gram (one fp64 slot per bit: the sum over
// ranks is > 0 iff some rank raised the bit).
constexpr int COMM_FLAG_SLOTS = 8;
constexpr int COMM_FLAG_MASK = FLAG_NONFINITE | FLAG_R_NONPOS | FLAG_IDX_ORDER | FLAG_IDX_RANGE;

__global__ void comm_pack_flags(const DevStatus* __restrict__ st, double* __restrict__ tail) {
  const int b = threadIdx.x;
  if (b < COMM_FLAG_SLOTS) tail[b] = ((st->flags & COMM_FLAG_MASK) >> b) & 1 ? 1.0 : 0.0;
}

__global__ void comm_unpack_flags(const double* __restrict__ tail, DevStatus* __restrict__ st) {
  if (threadIdx.x != 0) return;
  int f = 0;
  for (int b = 0; b < COMM_FLAG_SLOTS; ++b)
    if (tail[b] > 0.5) f |= 1 << b;
  st->flags |= f & COMM_FLAG_MASK;
}

}  // namespace enkf
