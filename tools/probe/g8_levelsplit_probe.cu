// Costing the level-split form of the int8 Gram MMA pass: cycles per
// tcgen05.mma kind::i8 (M = 128, K = 32, A from TMEM, B SWIZZLE_32B K-major) at
// N = 64 / 128 / 256, with and without the six tcgen05.cp of the A planes per
// block, and with 26 (column split, today) or 7 (level split) MMAs per block.
// use_cp = 2: A from shared memory (SS mode, no tcgen05.cp).
// One CTA per SM, MMAs on resident data (issue pattern only, no streaming).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1302_3876_b200/csrc/enkf_kernels.cuh"
#include "../../paper_1302_3876_b200/csrc/anomaly_i8.cuh"
#include "../../paper_1302_3876_b200/csrc/gram_i8.cuh"
using namespace enkf;

__device__ __forceinline__ uint32_t idesc_n(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

template <int nN, int nacc, int nmma, int use_cp>
__global__ void __launch_bounds__(128, 1) probe(int blocks, unsigned long long* out) {
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
    const uint32_t idesc = idesc_n(nN);
    const uint32_t plane_b = (uint32_t)nN * 32u;  // B plane bytes: N rows x 32 B
    for (int k = 0; k < blocks; ++k) {
      if (use_cp == 1) {
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
          if (o + i > 8 || cnt >= nmma) continue;
          const int l = (o + i - 2) % nacc;
          const uint64_t bd = umma_desc_sw32(bbuf + (uint32_t)(i - 1) * plane_b);
          if (use_cp == 2)
            umma_i8_ss(tmem + (uint32_t)(l * nN), umma_desc_sw32(abuf + (uint32_t)(o - 1) * 4096u), bd, idesc, 1u);
          else
            umma_i8_ts(tmem + (uint32_t)(l * nN), tmem + 448u + 8u * (o - 1), bd, idesc, 1u);
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

template <int nN, int nacc, int nmma, int use_cp>
void run1(int blocks, unsigned long long* d) {
  unsigned long long h[148];
  {
    size_t smem = 96 * 1024 + 2048;
    cudaFuncSetAttribute(probe<nN, nacc, nmma, use_cp>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe<nN, nacc, nmma, use_cp><<<148, 128, smem>>>(blocks, d);
    cudaDeviceSynchronize();
    probe<nN, nacc, nmma, use_cp><<<148, 128, smem>>>(blocks, d);
    cudaError_t err = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    const double cyc_block = (double)h[0] / blocks;
    const double floor_block = nmma * 32.0 * nN / 64.0;  // int8 math floor, 8K MAC/cycle/SM
    printf("\"N%d_acc%d_mma%d_cp%d\": {\"cyc_per_mma\": %.1f, \"cyc_per_block\": %.0f, \"math_floor_per_block\": %.0f, \"err\": \"%s\"}, ",
           nN, nacc, nmma, use_cp, cyc_block / nmma, cyc_block, floor_block, cudaGetErrorString(err));
  }
}

template <int nN, int nacc, int nmma>
void run(int blocks, unsigned long long* d) {
  run1<nN, nacc, nmma, 0>(blocks, d);
  run1<nN, nacc, nmma, 1>(blocks, d);
  run1<nN, nacc, nmma, 2>(blocks, d);
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 148 * 8);
  const int blocks = 2000;
  printf("{");
  run<64, 7, 26>(blocks, d);
  run<64, 7, 7>(blocks, d);
  run<128, 3, 26>(blocks, d);
  run<128, 3, 7>(blocks, d);
  run<256, 1, 26>(blocks, d);
  run<256, 1, 7>(blocks, d);
  run<256, 2, 26>(blocks, d);  // two level accumulators of 256 columns (SS mode: no A staging)
  printf("\"done\": 1}\n");
  return 0;
}
