// Device-side helpers off the split-finding path: synthetic data, a standalone projection kernel
// (apply_projection parity) and batch prediction (reference predict, forest.hpp:88-121).
#include <cuda_runtime.h>

#include <algorithm>

#include "common.hpp"
#include "dev_util.cuh"
#include "kernels.hpp"
#include "mt64.cuh"

namespace sofg {
namespace dev {

// Counter-based normal draw (splitmix64 hash -> two uniforms -> Box-Muller, double precision).
__device__ __forceinline__ double hashed_normal(uint64_t seed, uint64_t i, uint64_t f) {
  const uint64_t h1 = split_mix64(seed ^ split_mix64(i * 0x9E3779B97F4A7C15ull + f));
  const uint64_t h2 = split_mix64(h1 ^ 0xD1B54A32D192ED03ull);
  const double u1 = (double(h1 >> 11) + 0.5) * 0x1p-53;
  const double u2 = double(h2 >> 11) * 0x1p-53;
  return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

// Trunk-style synthetic table (the reference's generate_trunk, dataset.hpp:306-329, draws one
// serial mt19937_64 stream; this is the same model — x_f = s_{c,f} * mu_f + N(0,1),
// mu_f = 1/sqrt(f+1), class = i % k — from a counter-based generator so 16 GB fills in ms.
// s_{c,f} = -1 iff bit (f mod ceil(log2 k)) of c is set; for k = 2 that is the trunk sign.
__global__ void k_generate_trunk(float* __restrict__ X, uint64_t ld, uint8_t* __restrict__ lab,
                                 uint64_t n, uint64_t f0, int k, int kbits, uint64_t seed) {
  const uint64_t f = f0 + blockIdx.y;
  const double mu = 1.0 / sqrt(double(f + 1));
  const int bit = kbits > 0 ? int(f % uint64_t(kbits)) : 0;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const int c = int(i % uint64_t(k));
    const double s = ((c >> bit) & 1) ? -1.0 : 1.0;
    X[f * ld + i] = float(s * mu + hashed_normal(seed, i, f));
    if (f == 0) lab[i] = uint8_t(c);
  }
}

__global__ void k_apply_projection(const float* __restrict__ X, uint64_t ld,
                                   const uint32_t* __restrict__ terms, int nt,
                                   const uint32_t* __restrict__ active, uint64_t n,
                                   float* __restrict__ out) {
  for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
       j += uint64_t(gridDim.x) * blockDim.x)
    out[j] = project_sample(X, ld, terms, nt, active[j]);
}

// One thread per (row, tree): walks the tree, adds a vote. rows are row-major [n_rows][d].
__global__ void k_predict(const float* __restrict__ rows, uint64_t n_rows, uint64_t d,
                          const int64_t* __restrict__ tree_off, int n_trees,
                          const int32_t* __restrict__ left, const int32_t* __restrict__ right,
                          const int32_t* __restrict__ pred, const float* __restrict__ thr,
                          const int64_t* __restrict__ term_off, const uint32_t* __restrict__ terms,
                          int k, uint32_t* __restrict__ votes) {
  const uint64_t gid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid >= n_rows * uint64_t(n_trees)) return;
  const uint64_t i = gid / uint64_t(n_trees);
  const int t = int(gid % uint64_t(n_trees));
  const float* x = rows + i * d;
  const int64_t base = tree_off[t];
  int64_t nd = base;
  while (left[nd] >= 0) {
    double acc = 0.0;
    for (int64_t q = term_off[nd]; q < term_off[nd + 1]; ++q) {
      const uint32_t tm = terms[q];
      const double v = (tm & 1u) ? -double(x[tm >> 1]) : double(x[tm >> 1]);
      acc = (q == term_off[nd]) ? v : __dadd_rn(acc, v);
    }
    nd = base + ((__double2float_rn(acc) <= thr[nd]) ? left[nd] : right[nd]);
  }
  atomicAdd(&votes[i * uint64_t(k) + uint64_t(pred[nd])], 1u);
}

// Root segments of a tree batch: labels gathered from the resident label column, and per-tree
// class counts (tree b owns [off[b], off[b+1]) of the level buffer).
__global__ void __launch_bounds__(256) k_root_labels(const uint32_t* __restrict__ idx,
                                                     const uint64_t* __restrict__ off,
                                                     const uint8_t* __restrict__ labels,
                                                     uint8_t* __restrict__ lab_out, int k,
                                                     uint32_t* __restrict__ counts) {
  __shared__ uint32_t s_cnt[kMaxClassesWide];
  const uint32_t b = blockIdx.y;
  for (int c = threadIdx.x; c < k; c += blockDim.x) s_cnt[c] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t p1 = off[b + 1];
  for (uint64_t p0 = off[b] + uint64_t(blockIdx.x) * blockDim.x; p0 < p1; p0 += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t p = p0 + threadIdx.x;
    int y = -1;
    if (p < p1) {
      y = labels[idx[p]];
      lab_out[p] = uint8_t(y);
    }
    const unsigned same = __match_any_sync(0xffffffffu, y);  // one shared atomic per distinct label
    if (y >= 0 && (__ffs(same) - 1) == lane) atomicAdd(&s_cnt[y], uint32_t(__popc(same)));
  }
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x)
    if (s_cnt[c]) atomicAdd(&counts[size_t(b) * k + c], s_cnt[c]);
}


// One CTA per tree: thread t takes words [t * per, (t + 1) * per), counts their bits, a block scan
// gives its first rank, then it writes the ids of its set bits in order.
__global__ void __launch_bounds__(1024) k_bits_to_ids(const uint32_t* __restrict__ bits, uint64_t W,
                                                     const uint64_t* __restrict__ off, uint32_t* __restrict__ ids) {
  __shared__ uint32_t s_warp[32];
  const uint32_t b = blockIdx.x;
  const uint32_t* bw = bits + uint64_t(b) * W;
  const uint64_t per = (W + blockDim.x - 1) / blockDim.x;
  const uint64_t w0 = uint64_t(threadIdx.x) * per, w1 = min(W, w0 + per);
  uint32_t c = 0;
  for (uint64_t i = w0; i < w1; ++i) c += __popc(bw[i]);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t wt;
  const uint32_t ex = warp_excl_scan_u32(c, lane, &wt);
  if (lane == 0) s_warp[w] = wt;
  __syncthreads();
  uint32_t pos = ex;
  for (int i = 0; i < w; ++i) pos += s_warp[i];
  uint32_t* out = ids + off[b];
  for (uint64_t i = w0; i < w1; ++i) {
    uint32_t x = bw[i];
    while (x) {
      const int t = __ffs(x) - 1;
      x &= x - 1;
      out[pos++] = uint32_t(i * 32 + uint64_t(t));
    }
  }
}
}  // namespace dev

cudaError_t launch_root_labels(const uint32_t* idx, const uint64_t* off, uint32_t B,
                               uint64_t max_per_tree, const uint8_t* labels, uint8_t* lab_out,
                               int k, uint32_t* counts, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(uint32_t) * size_t(k) * B, st);
  if (e != cudaSuccess || B == 0) return e;
  const unsigned gx = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((max_per_tree + 255) / 256, 256)));
  dev::k_root_labels<<<dim3(gx, B), 256, 0, st>>>(idx, off, labels, lab_out, k, counts);
  return cudaGetLastError();
}

cudaError_t launch_generate_trunk(float* X, uint64_t ld, uint8_t* labels, uint64_t n, uint64_t d,
                                  int k, uint64_t seed, cudaStream_t st) {
  int kbits = 0;
  while ((1 << kbits) < k) ++kbits;
  const unsigned gx = unsigned(std::min<uint64_t>((n + 255) / 256, 4096));
  if (k < 1) return cudaErrorInvalidValue;
  for (uint64_t f0 = 0; f0 < d; f0 += 65535) {
    const unsigned gy = unsigned(std::min<uint64_t>(65535, d - f0));
    dev::k_generate_trunk<<<dim3(gx, gy), 256, 0, st>>>(X, ld, labels, n, f0, k, kbits, seed);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_apply_projection(const float* X, uint64_t ld, const uint32_t* terms, int nt,
                                    const uint32_t* active, uint64_t n, float* out,
                                    cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const unsigned g = unsigned(std::min<uint64_t>((n + 255) / 256, 65535));
  dev::k_apply_projection<<<g, 256, 0, st>>>(X, ld, terms, nt, active, n, out);
  return cudaGetLastError();
}

cudaError_t launch_predict(const float* rows, uint64_t n_rows, uint64_t d, const int64_t* tree_off,
                           int n_trees, const int32_t* left, const int32_t* right,
                           const int32_t* pred, const float* thr, const int64_t* term_off,
                           const uint32_t* terms, int k, uint32_t* votes, cudaStream_t st) {
  const uint64_t work = n_rows * uint64_t(n_trees);
  if (work == 0) return cudaSuccess;
  dev::k_predict<<<unsigned((work + 255) / 256), 256, 0, st>>>(
      rows, n_rows, d, tree_off, n_trees, left, right, pred, thr, term_off, terms, k, votes);
  return cudaGetLastError();
}

cudaError_t launch_bits_to_ids(const uint32_t* bits, uint64_t W, uint32_t B, const uint64_t* off, uint32_t* ids,
                               cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  dev::k_bits_to_ids<<<B, 1024, 0, st>>>(bits, W, off, ids);
  return cudaGetLastError();
}

}  // namespace sofg
