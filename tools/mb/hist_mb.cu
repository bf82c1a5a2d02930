// Microbenchmark: histogram binning building blocks on B200 (search vs shared atomics).
// Layout mimics k_hist_count: V sample-major with pitch Rp=96, CTA = 8 rows x chunk of samples.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

constexpr int BP = 256, LT = 8, RP = 96, CH = 8192;

template <int MODE>  // 0 search+atomic(k=2 words), 1 search only, 2 search+packed atomic, 3 atomic only (bin from value bits)
__global__ void __launch_bounds__(256) k_hist(const float* __restrict__ V, const uint8_t* __restrict__ lab,
                                              const float* __restrict__ bnd, uint32_t* out) {
  __shared__ float bnd_s[8 * BP];
  __shared__ uint32_t cnt_s[8 * BP * 2];
  __shared__ uint8_t lab_s[CH];
  const uint64_t s0 = uint64_t(blockIdx.x) * CH;
  for (int i = threadIdx.x; i < 8 * BP; i += 256) bnd_s[i] = bnd[i];
  for (int i = threadIdx.x; i < 8 * BP * 2; i += 256) cnt_s[i] = 0;
  for (int i = threadIdx.x; i < CH; i += 256) lab_s[i] = lab[s0 + i];
  __syncthreads();
  float root[8];
#pragma unroll
  for (int g = 0; g < 8; ++g) root[g] = bnd_s[g * BP + 1];
  uint32_t acc = 0;
  for (uint32_t j = threadIdx.x; j < CH; j += 256) {
    const float4* src = reinterpret_cast<const float4*>(V + (s0 + j) * RP);
    const float4 a = __ldg(src), b = __ldg(src + 1);
    const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    const uint32_t y = lab_s[j];
    int t[8];
    if (MODE == 3) {
#pragma unroll
      for (int g = 0; g < 8; ++g) t[g] = BP + ((__float_as_uint(v[g]) >> 7) & 255);
    } else {
#pragma unroll
      for (int g = 0; g < 8; ++g) t[g] = 2 + (root[g] <= v[g] ? 1 : 0);
#pragma unroll
      for (int l = 1; l < LT; ++l) {
#pragma unroll
        for (int g = 0; g < 8; ++g) t[g] = 2 * t[g] + (bnd_s[g * BP + t[g]] <= v[g] ? 1 : 0);
      }
    }
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      if (MODE == 0 || MODE == 3) atomicAdd(&cnt_s[(g * BP + (t[g] - BP)) * 2 + y], 1u);
      else if (MODE == 2) atomicAdd(&cnt_s[g * BP + (t[g] - BP)], 1u << (16 * y));
      else acc += t[g];
    }
  }
  __syncthreads();
  uint32_t s = acc;
  for (int i = threadIdx.x; i < 8 * BP * 2; i += 256) s += cnt_s[i];
  atomicAdd(out, s);
}

int main() {
  const int nblk = 2048;
  const size_t n = size_t(nblk) * CH;
  std::vector<float> hV(n * 8);
  std::mt19937 rng(1);
  std::normal_distribution<float> nd;
  for (size_t i = 0; i < n; ++i)
    for (int r = 0; r < 8; ++r) hV[i * 8 + r] = nd(rng);
  std::vector<uint8_t> hl(n);
  for (auto& x : hl) x = rng() & 1;
  // Eytzinger trees of 255 sorted boundaries per row (NaN pad at index 0)
  std::vector<float> hb(8 * BP);
  for (int g = 0; g < 8; ++g) {
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
  cudaMemcpy2D(V, RP * 4, hV.data(), 32, 32, n, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(L, hl.data(), n, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto kern, const char* name) {
    for (int w = 0; w < 2; ++w) kern<<<nblk, 256>>>(V, L, B, out);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int w = 0; w < reps; ++w) kern<<<nblk, 256>>>(V, L, B, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    const double vals = double(n) * 8;
    printf("%-28s %8.3f ms  %6.3f ns/val  %.2f Gval/s  (%s)\n", name, ms, ms * 1e6 / vals, vals / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  };
  run(k_hist<0>, "search+atomic[bin][y]");
  run(k_hist<1>, "search only");
  run(k_hist<2>, "search+packed atomic");
  run(k_hist<3>, "atomic only");
  return 0;
}
