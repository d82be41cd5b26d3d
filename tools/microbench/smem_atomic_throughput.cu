// Throughput of shared-memory accumulation forms on B200 (random addresses in a
// 64 KB buffer, 4 independent updates in flight per thread, 512 threads/CTA).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int W = 8192;  // words (32 KB)
template <int MODE>
__global__ void __launch_bounds__(512) k(float* out, int iters) {
  __shared__ float acc[W];
  for (int i = threadIdx.x; i < W; i += blockDim.x) acc[i] = 0.f;
  __syncthreads();
  unsigned s0 = threadIdx.x * 2654435761u + blockIdx.x * 97u, s1 = s0 ^ 0x9e3779b9u, s2 = s0 * 3u + 7u, s3 = s0 ^ 0x7f4a7c15u;
  for (int it = 0; it < iters; ++it) {
    s0 = s0 * 1664525u + 1013904223u; s1 = s1 * 1664525u + 1013904223u;
    s2 = s2 * 1664525u + 1013904223u; s3 = s3 * 1664525u + 1013904223u;
    unsigned a0 = s0 >> 19, a1 = s1 >> 19, a2 = s2 >> 19, a3 = s3 >> 19;  // 13 bits
    if (MODE == 0) { acc[a0] += 1.f; acc[a1] += 1.f; acc[a2] += 1.f; acc[a3] += 1.f; }
    if (MODE == 1) { atomicAdd(&acc[a0], 1.f); atomicAdd(&acc[a1], 1.f); atomicAdd(&acc[a2], 1.f); atomicAdd(&acc[a3], 1.f); }
    if (MODE == 2) { int* ia = (int*)acc; atomicAdd(&ia[a0], (int)(s0 & 7)); atomicAdd(&ia[a1], (int)(s1 & 7)); atomicAdd(&ia[a2], (int)(s2 & 7)); atomicAdd(&ia[a3], (int)(s3 & 7)); }
    if (MODE == 4) {  // conflict-free: lane l hits bank l, random row
      int* ia = (int*)acc; const unsigned l = threadIdx.x & 31;
      atomicAdd(&ia[(a0 & ~31u) | l], 1); atomicAdd(&ia[(a1 & ~31u) | l], 1); atomicAdd(&ia[(a2 & ~31u) | l], 1); atomicAdd(&ia[(a3 & ~31u) | l], 1); }
    if (MODE == 5) {  // 2-way: lane pairs share a bank (different rows)
      int* ia = (int*)acc; const unsigned l = threadIdx.x & 31;
      atomicAdd(&ia[(a0 & ~31u) | (l >> 1)], 1); atomicAdd(&ia[(a1 & ~31u) | (l >> 1)], 1); atomicAdd(&ia[(a2 & ~31u) | (l >> 1)], 1); atomicAdd(&ia[(a3 & ~31u) | (l >> 1)], 1); }
    if (MODE == 6) {  // 8 lanes per row segment of 8 consecutive words (4 random segments per warp)
      int* ia = (int*)acc; const unsigned l = threadIdx.x & 31;
      unsigned b0 = __shfl_sync(0xffffffffu, a0, l & 24), b1 = __shfl_sync(0xffffffffu, a1, l & 24), b2 = __shfl_sync(0xffffffffu, a2, l & 24), b3 = __shfl_sync(0xffffffffu, a3, l & 24);
      atomicAdd(&ia[(b0 + (l & 7)) & (W - 1)], 1); atomicAdd(&ia[(b1 + (l & 7)) & (W - 1)], 1); atomicAdd(&ia[(b2 + (l & 7)) & (W - 1)], 1); atomicAdd(&ia[(b3 + (l & 7)) & (W - 1)], 1); }
    if (MODE == 7) {  // random, but only 16 lanes active
      int* ia = (int*)acc;
      if (threadIdx.x & 16) { atomicAdd(&ia[a0], 1); atomicAdd(&ia[a1], 1); atomicAdd(&ia[a2], 1); atomicAdd(&ia[a3], 1); } }
    if (MODE == 3) { unsigned long long* la = (unsigned long long*)acc; atomicAdd(&la[a0 >> 1], 1ull); atomicAdd(&la[a1 >> 1], 1ull); atomicAdd(&la[a2 >> 1], 1ull); atomicAdd(&la[a3 >> 1], 1ull); }
  }
  __syncthreads();
  float t = 0; for (int i = threadIdx.x; i < W; i += blockDim.x) t += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int MODE> void run(float* d, int sms, const char* name) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int blocks = sms * 3, iters = 2000; float ms = 0;
  for (int r = 0; r < 3; ++r) { cudaEventRecord(a); k<MODE><<<blocks, 512>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b); }
  cudaEventElapsedTime(&ms, a, b);
  double ops = double(blocks) * 512 * iters * 4;
  printf("%-28s %8.3f ms  %6.2f lane-updates/clk/SM @1.965GHz\n", name, ms, ops / (ms * 1e-3) / sms / 1.965e9);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* d; cudaMalloc(&d, sms * 3 * 512 * 4);
  run<0>(d, sms, "LDS+FADD+STS (racy)");
  run<1>(d, sms, "atomicAdd f32 smem (CAS)");
  run<2>(d, sms, "atomicAdd i32 smem");
  run<3>(d, sms, "atomicAdd u64 smem");
  run<4>(d, sms, "atomicAdd i32 conflict-free");
  run<5>(d, sms, "atomicAdd i32 2-way");
  run<6>(d, sms, "atomicAdd i32 4x8-run segs");
  run<7>(d, sms, "atomicAdd i32 16 lanes rnd");
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
