#include <cstdio>
#include <cuda_runtime.h>
// Microbenchmark: shared-memory float atomicAdd throughput vs LDS/FADD/STS, random vs row patterns
__global__ void k_atom(float* out, int iters, int mode) {
  __shared__ float acc[80*129];
  for (int i = threadIdx.x; i < 80*129; i += blockDim.x) acc[i] = 0.f;
  __syncthreads();
  unsigned s = threadIdx.x * 2654435761u + blockIdx.x;
  int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
    s = s * 1664525u + 1013904223u;
    int addr;
    if (mode == 0) addr = (s >> 8) % (80*129);          // random
    else addr = ((s >> 8) % 76) * 129 + lane;          // one row per warp, consecutive
    atomicAdd(&acc[addr], 1.0f);
  }
  __syncthreads();
  float t = 0; for (int i = threadIdx.x; i < 80*129; i += blockDim.x) t += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k_rmw(float* out, int iters, int mode) {
  __shared__ float acc[80*129];
  for (int i = threadIdx.x; i < 80*129; i += blockDim.x) acc[i] = 0.f;
  __syncthreads();
  unsigned s = threadIdx.x * 2654435761u + blockIdx.x;
  int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
    s = s * 1664525u + 1013904223u;
    int addr;
    if (mode == 0) addr = (s >> 8) % (80*129);
    else addr = ((s >> 8) % 76) * 129 + lane;
    acc[addr] += 1.0f;
  }
  __syncthreads();
  float t = 0; for (int i = threadIdx.x; i < 80*129; i += blockDim.x) t += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void k_ex2(float* out, int iters) {
  float x = threadIdx.x * 1e-3f, a = 0.f;
  for (int it = 0; it < iters; ++it) { float e; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x)); a += e; x = x * 0.999f - 1e-4f; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a;
}
int main() {
  float* d; cudaMalloc(&d, 148*8*256*4*4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters = 4096; int blocks = 148*2; int threads = 512;
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a); k_atom<<<blocks, threads>>>(d, iters, mode); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double ops = double(blocks) * threads * iters;
      if (rep) printf("atomics mode %d: %.3f ms, %.1f Gop/s, %.2f lane-ops/clk/SM @1.9GHz\n", mode, ms, ops/ms/1e6, ops/(ms*1e-3)/148/1.9e9);
      cudaEventRecord(a); k_rmw<<<blocks, threads>>>(d, iters, mode); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("lds+fadd+sts mode %d: %.3f ms, %.1f Gop/s, %.2f lane-ops/clk/SM\n", mode, ms, ops/ms/1e6, ops/(ms*1e-3)/148/1.9e9);
    }
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a); k_ex2<<<blocks*4, 256>>>(d, iters*4); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = double(blocks*4) * 256 * iters*4;
    if (rep) printf("ex2: %.3f ms, %.2f lane-ops/clk/SM @1.9GHz\n", ms, ops/(ms*1e-3)/148/1.9e9);
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0); printf("clock attr %d kHz\n", clk);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
