// Measured FP32 (FFMA) and SFU (MUFU.EX2) lane throughput per SM per clock on
// this B200: the denominators of the FP32/SFU issue roofline.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_ffma(float* out, int iters) {
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const float m = 0.9999f, c = 1e-4f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      a0 = fmaf(a0, m, c); a1 = fmaf(a1, m, c); a2 = fmaf(a2, m, c); a3 = fmaf(a3, m, c);
      a4 = fmaf(a4, m, c); a5 = fmaf(a5, m, c); a6 = fmaf(a6, m, c); a7 = fmaf(a7, m, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void k_ex2(float* out, int iters) {
  float x0 = -threadIdx.x * 1e-3f, x1 = x0 - 1, x2 = x0 - 2, x3 = x0 - 3, acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    float e0, e1, e2, e3;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(x0));
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(x1));
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e2) : "f"(x2));
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e3) : "f"(x3));
    acc += (e0 + e1) + (e2 + e3);
    x0 -= 1e-6f; x1 -= 1e-6f; x2 -= 1e-6f; x3 -= 1e-6f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* d; cudaMalloc(&d, sms * 8 * 1024 * sizeof(float));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int blocks = sms * 8, threads = 256, iters = 20000;
  float ms;
  for (int rep = 0; rep < 3; ++rep) { cudaEventRecord(a); k_ffma<<<blocks, threads>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b); }
  cudaEventElapsedTime(&ms, a, b);
  double ffma = double(blocks) * threads * iters * 64;
  printf("{\"sms\": %d, \"ffma_lane_ops_per_s\": %.4e, \"ffma_ms\": %.3f", sms, ffma / (ms * 1e-3), ms);
  for (int rep = 0; rep < 3; ++rep) { cudaEventRecord(a); k_ex2<<<blocks, threads>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b); }
  cudaEventElapsedTime(&ms, a, b);
  double ex2 = double(blocks) * threads * iters * 4;
  printf(", \"ex2_lane_ops_per_s\": %.4e, \"ex2_ms\": %.3f}\n", ex2 / (ms * 1e-3), ms);
  return 0;
}
