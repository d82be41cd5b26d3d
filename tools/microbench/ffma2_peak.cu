// FFMA2 (packed f32x2 FMA, sm_100a) vs FFMA: flop and issue throughput per SM per clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t pk(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float lo(uint64_t v) { float a, b; asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); return a + b; }
__global__ void k2(float* out, int iters) {
  uint64_t a[8];
  for (int j = 0; j < 8; ++j) a[j] = pk(threadIdx.x * 1e-3f + j, j * 0.5f);
  const uint64_t m = pk(0.9999f, 0.9998f), c = pk(1e-4f, 2e-4f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[j]) : "l"(m), "l"(c));
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += lo(a[j]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k1(float* out, int iters) {
  float a[8];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3f + j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[j]) : "f"(0.9999f), "f"(1e-4f));
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* d; cudaMalloc(&d, sms * 8 * 256 * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int blocks = sms * 8, iters = 4000; float ms;
  for (int r = 0; r < 3; ++r) { cudaEventRecord(a); k1<<<blocks, 256>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b); }
  cudaEventElapsedTime(&ms, a, b);
  double inst = double(blocks) * 256 * iters * 64;
  printf("FFMA : %.3f ms, %.1f fma-lanes/clk/SM, %.2f warp-inst/clk/SM @1.965GHz\n", ms, inst / (ms * 1e-3) / sms / 1.965e9, inst / 32 / (ms * 1e-3) / sms / 1.965e9);
  for (int r = 0; r < 3; ++r) { cudaEventRecord(a); k2<<<blocks, 256>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b); }
  cudaEventElapsedTime(&ms, a, b);
  printf("FFMA2: %.3f ms, %.1f fma-lanes/clk/SM, %.2f warp-inst/clk/SM @1.965GHz\n", ms, 2 * inst / (ms * 1e-3) / sms / 1.965e9, inst / 32 / (ms * 1e-3) / sms / 1.965e9);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
