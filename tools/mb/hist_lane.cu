// Microbenchmark: histogram binning with lane = projection row (transposed, bank-private search
// trees and counters) vs the current lane = sample layout (k_hist_count: 8 rows per CTA).
// V sample-major, pitch 96 (R = 96 rows), random boundaries per row.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

constexpr int BP = 256, LT = 8, RP = 96, CH = 8192;

// current layout: CTA = 8 rows x CH samples, lane = sample, shared search trees [8][256]
__global__ void __launch_bounds__(256) k_cur(const float* __restrict__ V, const uint8_t* __restrict__ lab,
                                             const float* __restrict__ bnd, uint32_t* out) {
  extern __shared__ __align__(16) unsigned char smx[];
  uint32_t* cnt_s = reinterpret_cast<uint32_t*>(smx);  // [8][256][2]
  float* bnd_s = reinterpret_cast<float*>(cnt_s + 8 * BP * 2);
  uint8_t* lab_s = reinterpret_cast<uint8_t*>(bnd_s + 8 * BP);
  const uint64_t s0 = uint64_t(blockIdx.x) * CH;
  const int g0 = blockIdx.y * 8;
  for (int i = threadIdx.x; i < 8 * BP; i += 256) bnd_s[i] = bnd[(g0 + i / BP) * BP + i % BP];
  for (int i = threadIdx.x; i < 8 * BP * 2; i += 256) cnt_s[i] = 0;
  for (int i = threadIdx.x; i < CH; i += 256) lab_s[i] = lab[s0 + i];
  __syncthreads();
  float root[8];
#pragma unroll
  for (int g = 0; g < 8; ++g) root[g] = bnd_s[g * BP + 1];
  for (uint32_t j = threadIdx.x; j < CH; j += 256) {
    const float4* src = reinterpret_cast<const float4*>(V + (s0 + j) * RP + g0);
    const float4 a = __ldg(src), b = __ldg(src + 1);
    const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    const uint32_t y = lab_s[j];
    int t[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) t[g] = 2 + (root[g] <= v[g] ? 1 : 0);
#pragma unroll
    for (int l = 1; l < LT; ++l) {
#pragma unroll
      for (int g = 0; g < 8; ++g) t[g] = 2 * t[g] + (bnd_s[g * BP + t[g]] <= v[g] ? 1 : 0);
    }
#pragma unroll
    for (int g = 0; g < 8; ++g) atomicAdd(&cnt_s[(g * BP + (t[g] - BP)) * 2 + y], 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(out, cnt_s[5]);
}

// lane = row: CTA = 32 rows x CH samples; warp w takes samples w*U.., U per lane in flight.
// tree[t][32] and cnt[bin][32] (u16 class 0 | u16 class 1): lane s only ever touches bank s.
template <int U>
__global__ void __launch_bounds__(256) k_lane(const float* __restrict__ V, const uint8_t* __restrict__ lab,
                                              const float* __restrict__ bnd, uint32_t* out) {
  extern __shared__ __align__(16) unsigned char smx[];
  float* tree = reinterpret_cast<float*>(smx);                 // [256][32]
  uint32_t* cnt = reinterpret_cast<uint32_t*>(tree + BP * 32);  // [256][32]
  uint8_t* lab_s = reinterpret_cast<uint8_t*>(cnt + BP * 32);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t s0 = uint64_t(blockIdx.x) * CH;
  const int g0 = blockIdx.y * 32;
  for (int i = threadIdx.x; i < BP * 32; i += 256) {
    const int t = i >> 5, s = i & 31;
    tree[i] = bnd[(g0 + s) * BP + t];
    cnt[i] = 0;
  }
  for (int i = threadIdx.x; i < CH; i += 256) lab_s[i] = lab[s0 + i];
  __syncthreads();
  const float root = tree[32 + lane];
  const float* Vl = V + s0 * RP + g0 + lane;
  for (int j0 = w * U; j0 < CH; j0 += 8 * U) {
    float v[U];
    uint32_t inc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u] = __ldg(Vl + uint64_t(j0 + u) * RP);
      inc[u] = lab_s[j0 + u] ? 0x10000u : 1u;
    }
    int t[U];
#pragma unroll
    for (int u = 0; u < U; ++u) t[u] = 2 + (root <= v[u] ? 1 : 0);
#pragma unroll
    for (int l = 1; l < LT; ++l) {
#pragma unroll
      for (int u = 0; u < U; ++u) t[u] = 2 * t[u] + (tree[t[u] * 32 + lane] <= v[u] ? 1 : 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) atomicAdd(&cnt[(t[u] - BP) * 32 + lane], inc[u]);
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(out, cnt[5]);
}

int main() {
  const int nblk = 1024;
  const size_t n = size_t(nblk) * CH;
  std::vector<float> hV(n * RP);
  std::mt19937 rng(1);
  std::normal_distribution<float> nd;
  for (auto& x : hV) x = nd(rng);
  std::vector<uint8_t> hl(n);
  for (auto& x : hl) x = rng() & 1;
  std::vector<float> hb(RP * BP);
  for (int g = 0; g < RP; ++g) {
    std::vector<float> s(255);
    for (auto& x : s) x = nd(rng);
    std::sort(s.begin(), s.end());
    hb[g * BP] = __builtin_nanf("");
    for (int t = 1; t < BP; ++t) {
      int l = 31 - __builtin_clz(t);
      int sidx = ((2 * (t - (1 << l)) + 1) << (LT - 1 - l)) - 1;
      hb[g * BP + t] = s[sidx];
    }
  }
  float *V, *B;
  uint8_t* L;
  uint32_t* out;
  cudaMalloc(&V, n * RP * 4);
  cudaMalloc(&B, hb.size() * 4);
  cudaMalloc(&L, n);
  cudaMalloc(&out, 4);
  cudaMemcpy(V, hV.data(), n * RP * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(L, hl.data(), n, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto kern, const char* name, dim3 grid, size_t smem) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    for (int w = 0; w < 2; ++w) kern<<<grid, 256, smem>>>(V, L, B, out);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int w = 0; w < reps; ++w) kern<<<grid, 256, smem>>>(V, L, B, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    const double vals = double(n) * RP;
    printf("%-24s %8.3f ms  %.2f Gval/s  %.0f GB/s V  (%s)\n", name, ms, vals / ms / 1e6, vals * 4 / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  };
  run(k_cur, "lane=sample (current)", dim3(nblk, RP / 8), 8 * BP * 2 * 4 + 8 * BP * 4 + CH);
  const size_t ls = BP * 32 * 4 * 2 + CH;
  run(k_lane<1>, "lane=row U=1", dim3(nblk, RP / 32), ls);
  run(k_lane<2>, "lane=row U=2", dim3(nblk, RP / 32), ls);
  run(k_lane<4>, "lane=row U=4", dim3(nblk, RP / 32), ls);
  run(k_lane<8>, "lane=row U=8", dim3(nblk, RP / 32), ls);
  return 0;
}
