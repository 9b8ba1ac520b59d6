// tcgen05.mma kind::i8 throughput vs N and A source (TMEM vs SMEM).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1302_3876_b200/csrc/enkf_kernels.cuh"
#include "../../paper_1302_3876_b200/csrc/anomaly_i8.cuh"
using namespace enkf;

__device__ __forceinline__ uint32_t idesc_n(int n) {
  uint32_t d = 0;
  d |= 2u << 4; d |= 1u << 7; d |= 1u << 10;
  d |= (uint32_t)(n >> 3) << 17; d |= (uint32_t)(128 >> 4) << 24;
  return d;
}
__device__ __forceinline__ void umma_i8_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
               "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
               :: "r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc) : "memory");
}

template <bool A_TMEM>
__global__ void __launch_bounds__(128, 1) probe(int n, int iters, int nacc, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = (uint64_t*)(base + 64 * 1024);
  uint32_t* slot = (uint32_t*)(bar + 2);
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0x01010101u;
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" :: "r"(smem_u32(slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  fence_proxy_async();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = *slot;
  unsigned long long t0 = clock64();
  if (threadIdx.x < 32) {
    const uint64_t adesc = umma_desc_sw128(smem_u32(base));
    const uint64_t bdesc = umma_desc_sw128(smem_u32(base + 32768));
    const uint32_t idesc = idesc_n(n);
    for (int it = 0; it < iters; ++it) {
      const uint32_t d = tmem + 256 + (uint32_t)((it % nacc) * 0);  // accumulators at col 256
      if (A_TMEM) umma_i8_ts(tmem + 256 + (uint32_t)(it % nacc) * (uint32_t)n / 2 * 0 + 0, tmem + 0, bdesc, idesc, 1u);
      else umma_i8_ss(d, adesc, bdesc, idesc, 1u);
    }
    umma_commit_elect(bar);
    mbar_wait(bar, 0);
  }
  tc_fence_before(); __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (threadIdx.x < 32) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" :: "r"(tmem) : "memory");
  }
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 148 * 8);
  unsigned long long h[148];
  const int iters = 4096;
  printf("{");
  for (int a_tmem = 0; a_tmem < 2; ++a_tmem) {
    for (int n : {16, 32, 64, 128, 256}) {
      size_t smem = 64 * 1024 + 2048;
      auto k = a_tmem ? probe<true> : probe<false>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k<<<148, 128, smem>>>(n, iters, 1, d);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k<<<148, 128, smem>>>(n, iters, 1, d);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      cudaError_t err = cudaGetLastError();
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double ops = 2.0 * 128 * n * 32 * iters * 148;
      printf("\"%s_n%d\": {\"cyc_per_mma\": %.1f, \"tops\": %.1f, \"err\": \"%s\"}, ", a_tmem ? "ts" : "ss", n,
             (double)h[0] / iters, ops / ms / 1e9, cudaGetErrorString(err));
    }
  }
  printf("\"done\": 1}\n");
  return 0;
}
