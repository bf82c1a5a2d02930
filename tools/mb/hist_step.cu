// Microbenchmark: the lane = row search step of k_hist_count_lr (split.cu) in three instruction
// forms, same shared-memory layout (word t of row s at tree + 128 t + 4 s), same counts checked.
//   A  production: FSETP + SEL + IADD3/IMAD per level (3 ALU-pipe instructions)
//   B  FSET (float 0/1) + FFMA into a 2^23-magic float whose bits carry the offset + IMAD
//   C  FSET + IMAD + IMAD.HI (hi(bits(1.0f) * 517) = 128)
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

constexpr int BP = 256, LT = 8, RP = 96, CH = 8192, U = 8;

template <int VAR>
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
  const uint32_t lane_base = uint32_t(__cvta_generic_to_shared(tree)) + 4u * uint32_t(lane);
  const uint32_t k0 = 0u - lane_base, k1 = 128u - lane_base;
  const uint32_t cnt_off = uint32_t(__cvta_generic_to_shared(cnt)) - uint32_t(__cvta_generic_to_shared(tree)) - BP * 128u;
  constexpr uint32_t BU = 0x4B000000u + (1u << 20);
  const float M = __uint_as_float(BU - lane_base);
  for (int j0 = w * U; j0 < CH; j0 += 8 * U) {
    float v[U];
    uint32_t inc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u] = __ldg(Vl + uint64_t(j0 + u) * RP);
      inc[u] = lab_s[j0 + u] ? 0x10000u : 1u;
    }
    uint32_t a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = lane_base + (root <= v[u] ? 3u * 128u : 2u * 128u);
    if constexpr (VAR == 0) {
#pragma unroll
      for (int l = 1; l < LT; ++l) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          float b;
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(b) : "r"(a[u]));
          a[u] = 2u * a[u] + (b <= v[u] ? k1 : k0);
        }
      }
    } else if constexpr (VAR == 1) {
      uint32_t D = 0;  // a = true address + D (D uniform)
#pragma unroll
      for (int l = 1; l < LT; ++l) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          float b, s;
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(b) : "r"(a[u] - D));
          asm("set.le.f32.f32 %0, %1, %2;" : "=f"(s) : "f"(b), "f"(v[u]));
          a[u] = 2u * a[u] + __float_as_uint(__fmaf_rn(s, 128.f, M));
        }
        D = 2u * D + BU;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) a[u] -= D;
    } else {
#pragma unroll
      for (int l = 1; l < LT; ++l) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          float b, s;
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(b) : "r"(a[u]));
          asm("set.le.f32.f32 %0, %1, %2;" : "=f"(s) : "f"(b), "f"(v[u]));
          a[u] = __umulhi(__float_as_uint(s), 517u) + (2u * a[u] + k0);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a[u] + cnt_off), "r"(inc[u]) : "memory");
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < BP * 32; i += 256) atomicAdd(out + (i & 255), cnt[i]);
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
  cudaMalloc(&out, 4 * 256);
  cudaMemcpy(V, hV.data(), n * RP * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(L, hl.data(), n, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<uint32_t> ref;
  auto run = [&](auto kern, const char* name) {
    const dim3 grid(nblk, RP / 32);
    const size_t smem = BP * 32 * 4 * 2 + CH;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaMemset(out, 0, 1024);
    kern<<<grid, 256, smem>>>(V, L, B, out);
    std::vector<uint32_t> h(256);
    cudaMemcpy(h.data(), out, 1024, cudaMemcpyDeviceToHost);
    if (ref.empty()) ref = h;
    const bool same = h == ref;
    cudaEventRecord(e0);
    const int reps = 5;
    for (int w = 0; w < reps; ++w) kern<<<grid, 256, smem>>>(V, L, B, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    const double vals = double(n) * RP;
    printf("%-12s %8.3f ms  %.2f Gval/s  counts %s (%s)\n", name, ms, vals / ms / 1e6, same ? "same" : "DIFFER",
           cudaGetErrorString(cudaGetLastError()));
  };
  run(k_lane<0>, "A sel");
  run(k_lane<1>, "B ffma");
  run(k_lane<2>, "C imad.hi");
  return 0;
}
