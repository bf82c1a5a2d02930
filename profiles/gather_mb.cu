// Microbenchmark: DRAM bytes per isolated random 4-byte gather on B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_gather(const float* __restrict__ X, const uint64_t* __restrict__ idx, int n, float* out, int mode) {
  float acc = 0.f;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float* p = X + idx[i];
    float v;
    if (mode == 0) v = __ldg(p);
    else if (mode == 1) v = __ldcg(p);
    else { asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p)); }
    acc += v;
  }
  if (acc == 12345.f) out[0] = acc;
}
__global__ void k_pairs(const float* __restrict__ X, const uint64_t* __restrict__ idx, int n, float* out) {
  // each random sector read as 8 consecutive floats by 8 lanes (full 32B sector)
  float acc = 0.f;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n * 8; i += gridDim.x * blockDim.x) {
    acc += __ldcg(X + (idx[i >> 3] & ~7ull) + (i & 7));
  }
  if (acc == 12345.f) out[0] = acc;
}
int main() {
  const size_t N = 4ull << 30;  // 4G floats = 16 GB
  float* X; cudaMalloc(&X, N * 4); cudaMemset(X, 0, N * 4);
  const int n = 64 << 20;
  uint64_t* idx; cudaMalloc(&idx, n * 8);
  uint64_t* h = (uint64_t*)malloc(n * 8);
  uint64_t s = 88172645463325252ull;
  for (int i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = s % N; }
  cudaMemcpy(idx, h, n * 8, cudaMemcpyHostToDevice);
  float* out; cudaMalloc(&out, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (mode < 3) k_gather<<<148 * 16, 256>>>(X, idx, n, out, mode);
      else k_pairs<<<148 * 16, 256>>>(X, idx, n, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("mode %d: %.3f ms  %.2f Ggathers/s  sector-model %.1f GB/s\n", mode, ms, n / ms / 1e6, n * 32.0 / ms / 1e6);
    }
  }
  return 0;
}
