// FP64 pipe probe for B200 (sm_100a): DFMA vs DMMA (mma.sync f64) issue
// throughput, plus a streaming fp64 copy. Used once to choose the kernel
// shapes of the sweep and the anomaly GEMM; results go to profiles/.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("{\"error\": \"%s line %d\"}\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_loop(double* out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double m = 0.999999, c = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], m, c);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dmma_m8n8k4(double* out, int iters) {
  double c[8][2];
  for (int i = 0; i < 8; ++i) { c[i][0] = 0; c[i][1] = 0; }
  double a = threadIdx.x * 1e-3, b = 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dmma_m16n8k4(double* out, int iters) {
  double c[4][4];
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  double a0 = threadIdx.x * 1e-3, a1 = 2e-3, b = 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dmma_m16n8k16(double* out, int iters) {
  double c[4][4];
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1e-3 * i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) s += c[i][j];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void copy_f64(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

template <typename K>
float time_kernel(K kern, int blocks, int threads, double* out, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, iters);
  cudaEventRecord(e0);
  for (int r = 0; r < 3; ++r) kern<<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / 3;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, 1 << 20));
  const int iters = 20000;
  printf("{\"sms\": %d, \"name\": \"%s\"", sms, p.name);
  for (int occ : {1, 2, 4}) {
    int blocks = sms * occ, threads = 256;
    float ms = time_kernel(dfma_loop, blocks, threads, out, iters);
    double fl = 2.0 * 8 * iters * (double)blocks * threads;
    printf(", \"dfma_occ%d_tflops\": %.2f", occ, fl / ms / 1e9);
    ms = time_kernel(dmma_m8n8k4, blocks, threads, out, iters / 4);
    fl = 2.0 * 8 * 8 * 4 * 8 * (iters / 4) * (double)blocks * (threads / 32);
    printf(", \"dmma_m8n8k4_occ%d_tflops\": %.2f", occ, fl / ms / 1e9);
    ms = time_kernel(dmma_m16n8k4, blocks, threads, out, iters / 4);
    fl = 2.0 * 16 * 8 * 4 * 4 * (iters / 4) * (double)blocks * (threads / 32);
    printf(", \"dmma_m16n8k4_occ%d_tflops\": %.2f", occ, fl / ms / 1e9);
    ms = time_kernel(dmma_m16n8k16, blocks, threads, out, iters / 16);
    fl = 2.0 * 16 * 8 * 16 * 4 * (iters / 16) * (double)blocks * (threads / 32);
    printf(", \"dmma_m16n8k16_occ%d_tflops\": %.2f", occ, fl / ms / 1e9);
  }
  size_t n = (size_t)1 << 30;  // 1 Gi doubles = 8 GiB per buffer
  double2 *a, *b;
  CK(cudaMalloc(&a, n * 8)); CK(cudaMalloc(&b, n * 8));
  cudaMemset(a, 0, n * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 6; ++r) {
    cudaEventRecord(e0);
    copy_f64<<<sms * 8, 512>>>(a, b, n / 2);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  printf(", \"copy_f64_gbs\": %.1f", 2.0 * n * 8 / best / 1e6);
  CK(cudaGetLastError());
  printf("}\n");
  return 0;
}
