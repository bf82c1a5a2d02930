// Microbenchmark: DRAM bytes moved per 4-byte read for strided (partition-like: one float per
// 384-byte sample block) and random-sector (boundary-pick-like) access, per load flavour.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int F>
__device__ __forceinline__ float ld(const float* p) {
  float v;
  if constexpr (F == 0) v = __ldg(p);
  else if constexpr (F == 1) asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
  else if constexpr (F == 2) asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  else if constexpr (F == 3) asm volatile("ld.global.nc.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(p));
  else asm volatile("ld.global.nc.L2::256B.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

template <int F>
__global__ void k_strided(const float* __restrict__ V, uint64_t n, uint32_t stride, float* out) {
  float acc = 0.f;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
    acc += ld<F>(V + i * stride);
  if (acc == 12345.f) out[0] = acc;
}

template <int F>
__global__ void k_random(const float* __restrict__ V, uint64_t n_words, uint64_t n, float* out) {
  float acc = 0.f;
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t h = (i + 1) * 0x9E3779B97F4A7C15ull;
    h ^= h >> 29;
    acc += ld<F>(V + (h % n_words));
  }
  if (acc == 12345.f) out[0] = acc;
}

int main() {
  const uint64_t words = uint64_t(6) << 30;  // 24 GB
  float* V;
  float* out;
  if (cudaMalloc(&V, words * 4) != cudaSuccess) return 1;
  cudaMalloc(&out, 4);
  cudaMemset(V, 0, words * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const uint64_t ns = words / 96;  // one float per 384 B
  const uint64_t nr = uint64_t(256) << 20;
  auto run = [&](auto kern, const char* name, auto... args) {
    kern<<<148 * 16, 256>>>(V, args..., out);
    cudaEventRecord(a);
    kern<<<148 * 16, 256>>>(V, args..., out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-22s %8.3f ms (%s)\n", name, ms, cudaGetErrorString(cudaGetLastError()));
  };
  run(k_strided<0>, "strided ldg", ns, 96u);
  run(k_strided<1>, "strided cg", ns, 96u);
  run(k_strided<2>, "strided nc no_alloc", ns, 96u);
  run(k_strided<3>, "strided L2::64B", ns, 96u);
  run(k_strided<4>, "strided L2::256B", ns, 96u);
  run(k_random<0>, "random ldg", words, nr);
  run(k_random<1>, "random cg", words, nr);
  run(k_random<3>, "random L2::64B", words, nr);
  return 0;
}
