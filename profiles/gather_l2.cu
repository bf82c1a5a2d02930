// Random 4-byte gathers hitting an L2-resident window vs. DRAM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_gather(const float* __restrict__ X, const uint32_t* __restrict__ idx, int n, uint64_t mask, float* out) {
  float acc = 0.f;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) acc += __ldcg(X + (idx[i] & mask));
  if (acc == 12345.f) out[0] = acc;
}
// 8 independent gathers per thread per iteration
__global__ void k_gather8(const float* __restrict__ X, const uint32_t* __restrict__ idx, int n, uint64_t mask, float* out) {
  float acc = 0.f;
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += 8 * stride) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) { int j = i + u * stride; v[u] = j < n ? __ldcg(X + (idx[j] & mask)) : 0.f; }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u];
  }
  if (acc == 12345.f) out[0] = acc;
}
int main() {
  const size_t N = 4ull << 30;
  float* X; cudaMalloc(&X, N * 4); cudaMemset(X, 0, N * 4);
  const int n = 256 << 20;
  uint32_t* idx; cudaMalloc(&idx, size_t(n) * 4);
  uint32_t* h = (uint32_t*)malloc(size_t(n) * 4);
  uint64_t s = 88172645463325252ull;
  for (int i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = uint32_t(s); }
  cudaMemcpy(idx, h, size_t(n) * 4, cudaMemcpyHostToDevice);
  float* out; cudaMalloc(&out, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int kern = 0; kern < 2; ++kern)
  for (uint64_t win_mb : {4ull, 16ull, 32ull, 64ull, 96ull, 4096ull, 16384ull}) {
    const uint64_t mask = (win_mb << 20) / 4 - 1;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (kern == 0) k_gather<<<148 * 16, 256>>>(X, idx, n, mask, out);
      else k_gather8<<<148 * 16, 256>>>(X, idx, n, mask, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("kern %d window %6llu MB: %.3f ms  %.1f Ggathers/s\n", kern, (unsigned long long)win_mb, ms, n / ms / 1e6);
    }
  }
  return 0;
}
