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

// Per-warp private histograms (8 rows x 256 bins, u32 = c0 | c1 << 16), no atomics: the lanes that
// share a bin in one step elect a leader (ballot-derived key match, MODE 5; match.any, MODE 6)
// that adds the group's counts with a plain read-modify-write.
template <int MODE>
__global__ void __launch_bounds__(256) k_hist_leader(const float* __restrict__ V, const uint8_t* __restrict__ lab,
                                                     const float* __restrict__ bnd, uint32_t* out) {
  extern __shared__ __align__(16) unsigned char smx[];
  uint32_t (*cnt_s)[8 * 256] = reinterpret_cast<uint32_t (*)[8 * 256]>(smx);  // [warp][row][bin]
  float* bnd_s = reinterpret_cast<float*>(smx + 8 * 8 * 256 * 4);
  uint8_t* lab_s = reinterpret_cast<uint8_t*>(bnd_s + 8 * BP);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t s0 = uint64_t(blockIdx.x) * CH;
  for (int i = threadIdx.x; i < 8 * BP; i += 256) bnd_s[i] = bnd[i];
  for (int i = threadIdx.x; i < 8 * 8 * 256; i += 256) (&cnt_s[0][0])[i] = 0;
  for (int i = threadIdx.x; i < CH; i += 256) lab_s[i] = lab[s0 + i];
  __syncthreads();
  float root[8];
#pragma unroll
  for (int g = 0; g < 8; ++g) root[g] = bnd_s[g * BP + 1];
  uint32_t* mc = cnt_s[w];
  for (uint32_t j = threadIdx.x; j < CH; j += 256) {
    const float4* src = reinterpret_cast<const float4*>(V + (s0 + j) * RP);
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
    const unsigned yb = __ballot_sync(0xffffffffu, y != 0);
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const uint32_t bin = uint32_t(t[g] - BP);
      unsigned same;
      if (MODE == 5) {
        same = 0xffffffffu;
#pragma unroll
        for (int bit = 0; bit < 8; ++bit) {
          const unsigned bb = __ballot_sync(0xffffffffu, (bin >> bit) & 1u);
          same &= ((bin >> bit) & 1u) ? bb : ~bb;
        }
      } else {
        same = __match_any_sync(0xffffffffu, bin);
      }
      const uint32_t c1 = __popc(same & yb), c0 = __popc(same) - c1;
      if ((__ffs(same) - 1) == lane) {
        uint32_t* c = mc + g * 256 + bin;
        *c += c0 | (c1 << 16);
      }
    }
  }
  __syncthreads();
  uint32_t s = 0;
  for (int i = threadIdx.x; i < 8 * 8 * 256; i += 256) s += (&cnt_s[0][0])[i];
  atomicAdd(out, s);
}

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

// warp = row; lane-private u8 counters (class 0 low byte, class 1 high byte of a u16 per
// (bin, lane)); V tile staged through smem with a 9-float pitch; chunk <= 255 * 32 samples.
constexpr int TS = 1024;
constexpr int UU = 8;  // samples per staged tile
__global__ void __launch_bounds__(256) k_hist_priv(const float* __restrict__ V, const uint8_t* __restrict__ lab,
                                                   const float* __restrict__ bnd, uint32_t* out, int chunk) {
  extern __shared__ __align__(16) unsigned char sm[];
  uint16_t* pc = reinterpret_cast<uint16_t*>(sm);                  // [8 warps][256 bins][32 lanes]
  float* bnd_s = reinterpret_cast<float*>(sm + 8 * 256 * 32 * 2);   // [8][256]
  float* tv = bnd_s + 8 * BP;                                       // [TS][9]
  uint8_t* lab_s = reinterpret_cast<uint8_t*>(tv + TS * 9);         // [TS]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t s0 = uint64_t(blockIdx.x) * chunk;
  for (int i = threadIdx.x; i < 8 * BP; i += 256) bnd_s[i] = bnd[i];
  for (int i = threadIdx.x; i < 8 * 256 * 32 / 2; i += 256) reinterpret_cast<uint32_t*>(pc)[i] = 0;
  uint16_t* my = pc + w * 256 * 32 + lane;
  const float* tr = bnd_s + w * BP;
  const float root = tr[1];
  for (int t0 = 0; t0 < chunk; t0 += TS) {
    __syncthreads();
    const int ts = min(TS, chunk - t0);
    for (int j = threadIdx.x; j < ts; j += 256) {
      const float4* src = reinterpret_cast<const float4*>(V + (s0 + t0 + j) * RP);
      const float4 a = __ldg(src), b = __ldg(src + 1);
      float* d = tv + j * 9;
      d[0] = a.x; d[1] = a.y; d[2] = a.z; d[3] = a.w; d[4] = b.x; d[5] = b.y; d[6] = b.z; d[7] = b.w;
      lab_s[j] = lab[s0 + t0 + j];
    }
    __syncthreads();
    for (int j0 = 0; j0 < ts; j0 += 32 * UU) {
      float v[UU];
      uint32_t y[UU];
      int t[UU];
#pragma unroll
      for (int u = 0; u < UU; ++u) {
        const int j = j0 + u * 32 + lane;
        v[u] = j < ts ? tv[j * 9 + w] : __int_as_float(0x7fc00000);
        y[u] = j < ts ? lab_s[j] : 2u;
        t[u] = 2 + (root <= v[u] ? 1 : 0);
      }
#pragma unroll
      for (int l = 1; l < LT; ++l) {
#pragma unroll
        for (int u = 0; u < UU; ++u) t[u] = 2 * t[u] + (tr[t[u]] <= v[u] ? 1 : 0);
      }
#pragma unroll
      for (int u = 0; u < UU; ++u) {
        if (y[u] < 2) {
          uint16_t* c = my + (t[u] - BP) * 32;
          *c = uint16_t(*c + (1u << (8 * y[u])));
        }
      }
    }
  }
  __syncthreads();
  // reduce: lane L sums bins 8L..8L+7 over the 32 lane columns of this warp's row
  uint32_t s = 0;
  for (int b = lane * 8; b < lane * 8 + 8; ++b) {
    const uint4* row = reinterpret_cast<const uint4*>(pc + w * 256 * 32 + b * 32);
    uint32_t c0 = 0, c1 = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 x = row[(q + lane) & 3];
      const uint32_t ws[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        c0 += (ws[i] & 0xff) + ((ws[i] >> 16) & 0xff);
        c1 += ((ws[i] >> 8) & 0xff) + (ws[i] >> 24);
      }
    }
    s += c0 * 3 + c1;
  }
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
  auto run = [&](auto kern, const char* name, size_t smem = 0) {
    if (smem) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    for (int w = 0; w < 2; ++w) kern<<<nblk, 256, smem>>>(V, L, B, out);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int w = 0; w < reps; ++w) kern<<<nblk, 256, smem>>>(V, L, B, out);
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
  const size_t lsm = 8 * 8 * 256 * 4 + 8 * BP * 4 + CH;
  run(k_hist_leader<5>, "leader ballot-match RMW", lsm);
  run(k_hist_leader<6>, "leader match.any RMW", lsm);
  {
    const int chunk = 8160;
    const int nb2 = int(n / chunk);
    const size_t smem = 8 * 256 * 32 * 2 + 8 * BP * 4 + TS * 9 * 4 + TS;
    cudaFuncSetAttribute(k_hist_priv, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    for (int w = 0; w < 2; ++w) k_hist_priv<<<nb2, 256, smem>>>(V, L, B, out, chunk);
    cudaEventRecord(e0);
    for (int w = 0; w < 5; ++w) k_hist_priv<<<nb2, 256, smem>>>(V, L, B, out, chunk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    const double vals = double(nb2) * chunk * 8;
    printf("%-28s %8.3f ms  %.2f Gval/s  (%s)\n", "private u8 counters", ms, vals / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
