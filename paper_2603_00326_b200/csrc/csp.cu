// Column-sweep gather: the projection stage of a wave, scheduled for L2 reuse.
//
// Every term of every node's projection matrix gathers one column of the table over the node's
// sample ids (reference apply_projection, projection.hpp:86-108). With a batch of trees each
// column is gathered by dozens of nodes per level, but a scattered 4-byte load that misses L2
// pulls a whole 128-byte line from HBM. So the wave's (node, term, chunk) work items are
// counting-sorted by feature and gathered in feature order: all gathers of a column run back to
// back while its lines are L2-resident. The raw values land in G (per node: z x n floats, term q
// of the node at G[gbase + q*n + j], coalesced writes); the split kernels combine a row's terms
// from G in ascending feature order with double accumulation, exactly as the reference does.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.hpp"
#include "dev_util.cuh"
#include "kernels.hpp"

namespace sofg {
namespace dev {

constexpr int kChunkShift = 10;  // 1024 samples per gather item
constexpr int kChunk = 1 << kChunkShift;

__device__ __forceinline__ uint32_t n_chunks(uint32_t n) { return (n + kChunk - 1) >> kChunkShift; }

// Per-feature item counts (block-local histogram in shared memory, merged with one atomic per
// non-empty bin).
__global__ void __launch_bounds__(256) k_items_count(const NodeIn* __restrict__ nodes, int n_nodes,
                                                     const uint32_t* __restrict__ terms, uint32_t d,
                                                     uint32_t* __restrict__ cnt) {
  extern __shared__ uint32_t loc[];
  for (uint32_t f = threadIdx.x; f < d; f += blockDim.x) loc[f] = 0;
  __syncthreads();
  for (int node = blockIdx.x; node < n_nodes; node += gridDim.x) {
    const NodeIn nd = nodes[node];
    const uint32_t nch = n_chunks(nd.n);
    for (uint32_t q = threadIdx.x; q < nd.z; q += blockDim.x)
      atomicAdd(&loc[terms[nd.term_off + q] >> 1], nch);
  }
  __syncthreads();
  for (uint32_t f = threadIdx.x; f < d; f += blockDim.x)
    if (loc[f]) atomicAdd(&cnt[f], loc[f]);
}

// Exclusive scan of the feature counts into cursors (one block of 1024 threads).
__global__ void __launch_bounds__(1024) k_items_scan(uint32_t* __restrict__ cnt, uint32_t d) {
  __shared__ uint32_t s_warp[32];
  __shared__ uint32_t s_carry;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < d; base += blockDim.x) {
    const uint32_t f = base + threadIdx.x;
    const uint32_t v = f < d ? cnt[f] : 0;
    uint32_t wt, bt = 0;
    const uint32_t ex = warp_excl_scan_u32(v, lane, &wt);
    if (lane == 0) s_warp[w] = wt;
    __syncthreads();
    if (w == 0) s_warp[lane] = warp_excl_scan_u32(s_warp[lane], lane, &bt);
    __syncthreads();
    const uint32_t carry = s_carry;
    if (f < d) cnt[f] = carry + s_warp[w] + ex;
    __syncthreads();
    if (threadIdx.x == 0) s_carry = carry + bt;
    __syncthreads();
  }
}

// Scatter items (node, q, chunk) into feature order. Same block decomposition as the count.
__global__ void __launch_bounds__(256) k_items_scatter(const NodeIn* __restrict__ nodes,
                                                       int n_nodes,
                                                       const uint32_t* __restrict__ terms,
                                                       uint32_t d, uint32_t* __restrict__ cursor,
                                                       uint64_t* __restrict__ items) {
  extern __shared__ uint32_t sm[];
  uint32_t* loc = sm;       // [d] local counts, then local ranks
  uint32_t* base = sm + d;  // [d] block base inside each feature
  for (uint32_t f = threadIdx.x; f < d; f += blockDim.x) loc[f] = 0;
  __syncthreads();
  for (int node = blockIdx.x; node < n_nodes; node += gridDim.x) {
    const NodeIn nd = nodes[node];
    const uint32_t nch = n_chunks(nd.n);
    for (uint32_t q = threadIdx.x; q < nd.z; q += blockDim.x)
      atomicAdd(&loc[terms[nd.term_off + q] >> 1], nch);
  }
  __syncthreads();
  for (uint32_t f = threadIdx.x; f < d; f += blockDim.x) {
    base[f] = loc[f] ? atomicAdd(&cursor[f], loc[f]) : 0u;
    loc[f] = 0;
  }
  __syncthreads();
  for (int node = blockIdx.x; node < n_nodes; node += gridDim.x) {
    const NodeIn nd = nodes[node];
    const uint32_t nch = n_chunks(nd.n);
    for (uint32_t q = threadIdx.x; q < nd.z; q += blockDim.x) {
      const uint32_t f = terms[nd.term_off + q] >> 1;
      const uint32_t r = atomicAdd(&loc[f], nch);
      for (uint32_t c = 0; c < nch; ++c)
        items[base[f] + r + c] = (uint64_t(node) << 32) | (uint64_t(q) << 16) | uint64_t(c);
    }
  }
}

// One warp per item: G[gbase(node) + q*n + j] = X[f][idx[begin + j]] for the item's chunk.
__global__ void __launch_bounds__(256) k_csp_gather(const NodeIn* __restrict__ nodes,
                                                    const uint64_t* __restrict__ gbase,
                                                    const uint32_t* __restrict__ terms,
                                                    const uint64_t* __restrict__ items,
                                                    uint64_t n_items,
                                                    const uint32_t* __restrict__ idx,
                                                    const float* __restrict__ X, uint64_t ld,
                                                    float* __restrict__ G) {
  const uint64_t it = uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (it >= n_items) return;
  const int lane = threadIdx.x & 31;
  const uint64_t item = items[it];
  const uint32_t node = uint32_t(item >> 32);
  const uint32_t q = uint32_t(item >> 16) & 0xffffu;
  const uint32_t c = uint32_t(item) & 0xffffu;
  const NodeIn nd = nodes[node];
  const uint32_t f = terms[nd.term_off + q] >> 1;
  const float* col = X + uint64_t(f) * ld;
  const uint32_t* seg = idx + nd.begin;
  float* out = G + gbase[node] + uint64_t(q) * nd.n;
  const uint32_t j0 = c << kChunkShift;
  const uint32_t j1 = min(nd.n, j0 + uint32_t(kChunk));
  for (uint32_t j = j0 + lane; j < j1; j += 256) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t jj = j + uint32_t(u * 32);
      v[u] = jj < j1 ? __ldcg(col + seg[jj]) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t jj = j + uint32_t(u * 32);
      if (jj < j1) out[jj] = v[u];
    }
  }
}

}  // namespace dev

uint64_t csp_items(uint32_t n, uint32_t z) {
  return uint64_t(z) * ((uint64_t(n) + dev::kChunk - 1) >> dev::kChunkShift);
}

cudaError_t launch_csp(const NodeIn* nodes, int n_nodes, const uint64_t* gbase,
                       const uint32_t* terms, uint32_t d, uint64_t n_items, uint32_t* cnt,
                       uint64_t* items, const uint32_t* idx, const float* X, uint64_t ld, float* G,
                       cudaStream_t st) {
  if (n_nodes == 0 || n_items == 0) return cudaSuccess;
  if (n_items >= (1ull << 32)) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * d, st);
  if (e != cudaSuccess) return e;
  const int blocks = std::min(n_nodes, 148 * 4);
  const size_t smem1 = sizeof(uint32_t) * d, smem2 = 2 * sizeof(uint32_t) * d;
  if (smem2 > 48 * 1024) {
    cudaFuncSetAttribute(dev::k_items_count, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem1));
    cudaFuncSetAttribute(dev::k_items_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem2));
  }
  dev::k_items_count<<<blocks, 256, smem1, st>>>(nodes, n_nodes, terms, d, cnt);
  dev::k_items_scan<<<1, 1024, 0, st>>>(cnt, d);
  dev::k_items_scatter<<<blocks, 256, smem2, st>>>(nodes, n_nodes, terms, d, cnt, items);
  const uint64_t grid = (n_items + 7) / 8;
  dev::k_csp_gather<<<unsigned(grid), 256, 0, st>>>(nodes, gbase, terms, items, n_items, idx, X, ld, G);
  return cudaGetLastError();
}

}  // namespace sofg
