// Rate of the int8 Gram's MMA issue pattern (gram_i8.cuh) in isolation: per "block",
// optionally 6 tcgen05.cp (A planes smem -> TMEM) then 26 TS MMAs (M=128, N=64, K=32)
// into 7 rotating level accumulators, with the B operand in SWIZZLE_32B (the Gram's
// layout) or SWIZZLE_128B descriptors.  Prints cycles per MMA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1302_3876_b200/csrc/enkf_kernels.cuh"
#include "../../paper_1302_3876_b200/csrc/anomaly_i8.cuh"
#include "../../paper_1302_3876_b200/csrc/gram_i8.cuh"
using namespace enkf;

__global__ void __launch_bounds__(128, 1) probe(int blocks, int use_cp, int sw128, int nacc, int qouter,
                                                unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = (uint64_t*)(base + 96 * 1024);
  uint32_t* slot = (uint32_t*)(bar + 2);
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0x01010101u;
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
    const uint32_t abuf = smem_u32(base), bbuf = smem_u32(base + 32768);
    const uint32_t idesc = idesc_g8();
    for (int k = 0; k < blocks; ++k) {
      if (use_cp) {
#pragma unroll
        for (int p = 0; p < 6; ++p)
          asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                       "@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n}\n" ::"r"(tmem + 448u + 8u * p),
                       "l"(umma_desc_sw32(abuf + p * 4096u)) : "memory");
      }
      int cnt = 0;
#pragma unroll
      for (int o = 1; o <= 6; ++o)
#pragma unroll
        for (int i = 1; i <= 6; ++i) {
          const int p = qouter ? i : o, q = qouter ? o : i;
          if (p + q > 8) continue;
          const int l = (p + q - 2) % nacc;
          const uint64_t bd = sw128 ? umma_desc_sw128(bbuf + (uint32_t)(q - 1) * 8192u)
                                    : umma_desc_sw32(bbuf + (uint32_t)(q - 1) * 2048u);
          umma_i8_ts(tmem + (uint32_t)(l * 64), tmem + 448u + 8u * (p - 1), bd, idesc, 1u);
          ++cnt;
        }
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
  const int blocks = 2000;
  printf("{");
  for (int use_cp = 0; use_cp < 2; ++use_cp)
    for (int sw128 = 0; sw128 < 1; ++sw128)
      for (int qouter = 0; qouter < 2; ++qouter)
      for (int nacc : {7}) {
        size_t smem = 96 * 1024 + 2048;
        cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        probe<<<148, 128, smem>>>(blocks, use_cp, sw128, nacc, qouter, d);
        cudaDeviceSynchronize();
        probe<<<148, 128, smem>>>(blocks, use_cp, sw128, nacc, qouter, d);
        cudaError_t err = cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("\"cp%d_sw%s_acc%d_qouter%d\": {\"cyc_per_mma\": %.1f, \"err\": \"%s\"}, ", use_cp, sw128 ? "128" : "32", nacc, qouter,
               (double)h[0] / (blocks * 26.0), cudaGetErrorString(err));
      }
  printf("\"done\": 1}\n");
  return 0;
}
