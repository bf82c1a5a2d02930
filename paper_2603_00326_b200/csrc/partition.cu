// Stable two-way partition of every split node's segment (reference forest.hpp:197-212:
// values <= threshold stay left in order, the rest follow in order).
//
//  k_part_flags_w    per 1024-element tile (one warp): read the winning row's projected value,
//                    flag v <= thr, store the flag bits, count lefts per tile and per class.
//  k_part_scan       per node: exclusive scan of tile left-counts; fills n_left, the stream
//                    position after the attempt and the winning row's terms in NodeRes.
//  k_part_scatter_w  per tile (one warp): rank inside the tile from the flag bits, scatter sample
//                    ids and labels into the next level's buffers.
#include <cuda_runtime.h>

#include "common.hpp"
#include "dev_util.cuh"
#include "kernels.hpp"

#ifndef SOFG_PART_TPC
#define SOFG_PART_TPC 8  // partition tiles (warps) per CTA
#endif

namespace sofg {
namespace dev {

// One warp per node: scan its tiles (tiles of a node are contiguous, first = tile_first[node]).
__global__ void k_part_scan(const NodeIn* __restrict__ nodes, int n_nodes, uint32_t R,
                            const uint32_t* __restrict__ tile_first,
                            const uint32_t* __restrict__ terms, const uint32_t* __restrict__ row_ptr,
                            const uint32_t* __restrict__ pos_proj,
                            const uint32_t* __restrict__ pos_split, uint32_t* __restrict__ tile_left,
                            NodeRes* __restrict__ res) {
  const int lane = threadIdx.x & 31;
  const int node = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (node >= n_nodes) return;
  const NodeIn nd = nodes[node];
  NodeRes& o = res[node];
  if (lane == 0) o.pos_after = (nd.flags & kNodeHist) ? pos_split[node] : pos_proj[node];
  const int row = o.row;
  if (row < 0) return;
  const uint32_t t0 = tile_first[node], t1 = tile_first[node + 1];
  uint32_t carry = 0;
  for (uint32_t base = t0; base < t1; base += 32) {
    const uint32_t t = base + lane;
    const uint32_t c = t < t1 ? tile_left[t] : 0;
    uint32_t tot;
    const uint32_t ex = warp_excl_scan_u32(c, lane, &tot);
    if (t < t1) tile_left[t] = carry + ex;  // becomes the tile's left offset
    carry += tot;
  }
  const uint32_t* rp = row_ptr + size_t(node) * (R + 1);
  const uint32_t nt = rp[row + 1] - rp[row];
  const uint32_t* rt = terms + nd.term_off + rp[row];
  if (lane == 0) {
    o.n_left = carry;
    o.n_terms = nt;
  }
  for (uint32_t q = lane; q < nt && q < uint32_t(kWinTermsMax); q += 32) o.terms[q] = rt[q];
}

// Flags and scatter, one warp per partition tile (flag word l / 32 of the tile's 32 words covers
// elements [32 word, 32 word + 32)). A CTA takes 8 tiles, so the many small nodes of deep levels
// do not each occupy a 256-thread CTA for a few dozen elements.
__global__ void __launch_bounds__(32 * SOFG_PART_TPC) k_part_flags_w(
    const NodeIn* __restrict__ nodes, const Tile* __restrict__ tiles, int n_tiles, uint32_t R, int k,
    const uint8_t* __restrict__ lab, const uint64_t* __restrict__ gbase, const float* __restrict__ G,
    NodeRes* __restrict__ res, uint32_t* __restrict__ flags, uint32_t* __restrict__ tile_left,
    uint32_t* __restrict__ class_left) {
  const int lane = threadIdx.x & 31;
  const int ti = int(blockIdx.x) * int(blockDim.x >> 5) + int(threadIdx.x >> 5);
  if (ti >= n_tiles) return;
  const Tile tl = tiles[ti];
  const int row = res[tl.node].row;
  if (row < 0) return;
  const NodeIn nd = nodes[tl.node];
  const float thr = res[tl.node].threshold;
  const uint32_t Rp = vpitch(R);
  const float* Vn = G + gbase[tl.node] + row + uint64_t(tl.start) * Rp;
  const uint8_t* ln = lab + nd.begin + tl.start;
  uint32_t my_left = 0;
  uint32_t cls[kMaxClasses];
#pragma unroll
  for (int c = 0; c < kMaxClasses; ++c) cls[c] = 0;
  const int words = int((tl.len + 31) / 32);
#pragma unroll 4
  for (int wd = 0; wd < words; ++wd) {
    const uint32_t l = uint32_t(wd * 32 + lane);
    bool f = false;
    uint32_t y = 0;
    if (l < tl.len) {
      f = ldg_l2_64(Vn + uint64_t(l) * Rp) <= thr;
      y = ln[l];
    }
    const unsigned m = __ballot_sync(0xffffffffu, f);
    if (lane == 0) flags[size_t(ti) * 32 + wd] = m;
    if (k > kMaxClasses) {  // more than kMaxClasses classes: one atomic per distinct label of the step
      const unsigned same = __match_any_sync(0xffffffffu, f ? int(y) : -1);
      if (f && (__ffs(same) - 1) == lane) atomicAdd(&class_left[size_t(tl.node) * k + y], uint32_t(__popc(same)));
      my_left += f ? 1u : 0u;
    } else if (f) {
      ++my_left;
#pragma unroll
      for (int c = 0; c < kMaxClasses; ++c) cls[c] += (c == int(y));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) my_left += __shfl_xor_sync(0xffffffffu, my_left, o);
  if (lane == 0) tile_left[ti] = my_left;
#pragma unroll
  for (int c = 0; c < kMaxClasses; ++c) {
    if (c >= k || k > kMaxClasses) break;
    uint32_t x = cls[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0 && x) atomicAdd(&class_left[size_t(tl.node) * k + c], x);
  }
}

__global__ void __launch_bounds__(32 * SOFG_PART_TPC) k_part_scatter_w(
    const NodeIn* __restrict__ nodes, const Tile* __restrict__ tiles, int n_tiles,
    const NodeRes* __restrict__ res, const uint32_t* __restrict__ flags,
    const uint32_t* __restrict__ tile_off, const uint32_t* __restrict__ idx_in,
    const uint8_t* __restrict__ lab_in, uint32_t* __restrict__ idx_out,
    uint8_t* __restrict__ lab_out, uint32_t* __restrict__ inv, uint32_t B) {
  const int lane = threadIdx.x & 31;
  const int ti = int(blockIdx.x) * int(blockDim.x >> 5) + int(threadIdx.x >> 5);
  if (ti >= n_tiles) return;
  const Tile tl = tiles[ti];
  if (res[tl.node].row < 0) return;
  const NodeIn nd = nodes[tl.node];
  const uint32_t n_left = res[tl.node].n_left;
  const uint32_t* fw = flags + size_t(ti) * 32;
  const int words = int((tl.len + 31) / 32);
  const uint32_t mw = lane < words ? fw[lane] : 0u;
  uint32_t tot;
  const uint32_t wpre = warp_excl_scan_u32(__popc(mw), lane, &tot);
  const uint32_t off = tile_off[ti];
#pragma unroll 4
  for (int wd = 0; wd < words; ++wd) {
    const uint32_t l = uint32_t(wd * 32 + lane);
    const uint32_t m = __shfl_sync(0xffffffffu, mw, wd);
    const uint32_t pre = __shfl_sync(0xffffffffu, wpre, wd);
    if (l >= tl.len) continue;
    const uint32_t lrank = pre + __popc(m & ((1u << lane) - 1u));
    const uint32_t p = tl.start + l;             // position inside the node
    const uint32_t L = off + lrank;              // left elements before p
    const bool left = (m >> lane) & 1u;
    const uint32_t dst = left ? L : n_left + (p - L);
    const uint32_t src = nd.begin + p;
    const uint32_t smp = idx_in[src];
    idx_out[nd.begin + dst] = smp;
    lab_out[nd.begin + dst] = lab_in[src];
    if (inv) inv[uint64_t(smp) * B + nd.tree] = nd.begin + dst;  // sweep.cu inverse map
  }
}

// Roofline accounting: number of distinct 32-byte sectors {idx >> 3} in each node's (sorted)
// sample-id set. Every projection term gathers one column over that set, so the node's gather
// traffic in the sector model is 32 * sectors * z.
__global__ void __launch_bounds__(256) k_sector_count(const NodeIn* __restrict__ nodes,
                                                      const Tile* __restrict__ tiles,
                                                      const uint32_t* __restrict__ idx,
                                                      NodeRes* __restrict__ res) {
  const Tile tl = tiles[blockIdx.x];
  const NodeIn nd = nodes[tl.node];
  uint32_t c = 0;
  for (uint32_t l = threadIdx.x; l < tl.len; l += blockDim.x) {
    const uint32_t p = tl.start + l;
    const uint32_t s = idx[nd.begin + p] >> 3;
    c += (p == 0 || (idx[nd.begin + p - 1] >> 3) != s) ? 1u : 0u;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(&res[tl.node].sectors, c);
}

// Winning-row terms of nodes whose row is longer than NodeRes carries inline (dense projection
// matrices): one warp per listed node copies its row into a compact buffer for one D2H copy.
__global__ void k_win_terms(const NodeIn* __restrict__ nodes, const NodeRes* __restrict__ res,
                            const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ terms,
                            uint32_t R, const uint32_t* __restrict__ list, int n_list,
                            const uint32_t* __restrict__ off, uint32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int li = int(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (li >= n_list) return;
  const uint32_t node = list[li];
  const int row = res[node].row;
  const uint32_t* rp = row_ptr + size_t(node) * (R + 1);
  const uint32_t q0 = rp[row], q1 = rp[row + 1];
  const uint32_t* src = terms + nodes[node].term_off + q0;
  for (uint32_t q = uint32_t(lane); q < q1 - q0; q += 32) out[off[li] + q] = src[q];
}

}  // namespace dev

cudaError_t launch_win_terms(const NodeIn* nodes, const NodeRes* res, const uint32_t* row_ptr,
                             const uint32_t* terms, uint32_t R, const uint32_t* list, int n_list,
                             const uint32_t* off, uint32_t* out, cudaStream_t st) {
  if (n_list == 0) return cudaSuccess;
  dev::k_win_terms<<<(n_list + 3) / 4, 128, 0, st>>>(nodes, res, row_ptr, terms, R, list, n_list, off,
                                                     out);
  return cudaGetLastError();
}

cudaError_t launch_sector_count(const NodeIn* nodes, const Tile* tiles, int n_tiles,
                                const uint32_t* idx, NodeRes* res, cudaStream_t st) {
  if (n_tiles == 0) return cudaSuccess;
  dev::k_sector_count<<<n_tiles, 256, 0, st>>>(nodes, tiles, idx, res);
  return cudaGetLastError();
}

cudaError_t launch_partition(const NodeIn* nodes, int n_nodes, const Tile* tiles, int n_tiles,
                             const uint32_t* tile_first, uint32_t R, int k, const uint32_t* terms,
                             const uint32_t* row_ptr, const uint32_t* pos_proj,
                             const uint32_t* pos_split, const uint32_t* idx_in,
                             const uint8_t* lab_in, uint32_t* idx_out, uint8_t* lab_out,
                             const uint64_t* gbase, const float* G, NodeRes* res, uint32_t* flags,
                             uint32_t* tile_left, uint32_t* inv, uint32_t B, uint32_t* class_left,
                             cudaStream_t st) {
  if (n_nodes == 0) return cudaSuccess;
  if (n_tiles > 0)
    dev::k_part_flags_w<<<(n_tiles + SOFG_PART_TPC - 1) / SOFG_PART_TPC, 32 * SOFG_PART_TPC, 0, st>>>(nodes, tiles, n_tiles, R, k, lab_in, gbase, G, res,
                                                           flags, tile_left, class_left);
  dev::k_part_scan<<<(n_nodes + 3) / 4, 128, 0, st>>>(nodes, n_nodes, R, tile_first, terms,
                                                      row_ptr, pos_proj, pos_split, tile_left, res);
  if (n_tiles > 0)
    dev::k_part_scatter_w<<<(n_tiles + SOFG_PART_TPC - 1) / SOFG_PART_TPC, 32 * SOFG_PART_TPC, 0, st>>>(nodes, tiles, n_tiles, res, flags, tile_left, idx_in,
                                                             lab_in, idx_out, lab_out, inv, B);
  return cudaGetLastError();
}

}  // namespace sofg
