// Exact splitter for large nodes (n > kExactSmemMax): ExactOnly mode, or a breakeven above the
// shared-memory splitter's range (reference best_split_exact, split.hpp:142-194, for every
// non-empty row, split.hpp:306-312).
//
//  1. k_big_keys      per (node, row) segment: the reference's packed sort key
//                     order_key(v) << 32 | label for every sample, from the wave's V block;
//  2. k_seg_radix     one CTA per segment, least-significant-digit radix sort in global memory:
//                     four stable passes (the label byte, then the 32-bit value key in 11 + 11 +
//                     10 bits); each pass counts its digits, then scatters the segment tile by
//                     tile, ranking keys of equal digit in input order (warp match + per-warp
//                     digit offsets in shared memory);
//  3. k_big_scan_wide one CTA per segment (wide.cuh): class counts at every gap between distinct
//                     values, impurity in the reference's FP64 order, minimum X, then the first
//                     position whose gain equals the best (first maximum);
//  4. k_big_select    best row per node (strict '>', lowest row wins, split.hpp:259-263).
#include <cuda_runtime.h>

#include <vector>

#include "common.hpp"
#include "dev_util.cuh"
#include "kernels.hpp"
#include "wide.cuh"

namespace sofg {
namespace dev {

struct BigSeg {
  uint32_t node;  // wave node index
  uint32_t row;
  uint64_t off;   // first key of the segment
};

__global__ void __launch_bounds__(256) k_big_keys(const NodeIn* __restrict__ nodes,
                                                  const BigSeg* __restrict__ segs,
                                                  uint32_t R, const uint8_t* __restrict__ lab,
                                                  const uint64_t* __restrict__ vbase,
                                                  const float* __restrict__ V,
                                                  uint64_t* __restrict__ keys,
                                                  uint64_t* __restrict__ seg_begin,
                                                  uint64_t* __restrict__ seg_end) {
  const BigSeg sg = segs[blockIdx.x];
  const NodeIn nd = nodes[sg.node];
  const uint32_t Rp = vpitch(R);
  const float* Vn = V + vbase[sg.node] + sg.row;
  if (threadIdx.x == 0) {
    seg_begin[blockIdx.x] = sg.off;
    seg_end[blockIdx.x] = sg.off + nd.n;
  }
  for (uint32_t j = threadIdx.x; j < nd.n; j += blockDim.x)
    keys[sg.off + j] = (uint64_t(order_key(__ldg(Vn + uint64_t(j) * Rp))) << 32) |
                       uint64_t(lab[nd.begin + j]);
}

// ------------------------------------------------------------------------------------------
// Segmented LSD radix sort, one CTA per segment: keys [beg, end) of `src` sorted into `dst`
// (ascending 64-bit keys; only bits 0-7 (label) and 32-63 (value key) can be non-zero).
constexpr int kRadixThreads = 256;
constexpr int kRadixMaxDigit = 2048;  // 11-bit digits

__device__ __forceinline__ uint32_t radix_digit(uint64_t key, int pass) {
  switch (pass) {
    case 0: return uint32_t(key) & 0xffu;                     // label
    case 1: return uint32_t(key >> 32) & 0x7ffu;              // value key bits 0-10
    case 2: return uint32_t(key >> 43) & 0x7ffu;              // bits 11-21
    default: return uint32_t(key >> 54) & 0x3ffu;             // bits 22-31
  }
}

__global__ void __launch_bounds__(kRadixThreads) k_seg_radix(const uint64_t* __restrict__ seg_begin,
                                                             const uint64_t* __restrict__ seg_end,
                                                             uint64_t* __restrict__ a, uint64_t* __restrict__ b) {
  __shared__ uint32_t s_base[kRadixMaxDigit];  // next output position of each digit
  extern __shared__ uint32_t s_wc[];           // [8 warps][D]: the current tile's digit counts per warp
  const uint64_t beg = seg_begin[blockIdx.x];
  const uint32_t n = uint32_t(seg_end[blockIdx.x] - beg);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int NW = kRadixThreads / 32;
  for (int i = threadIdx.x; i < NW * kRadixMaxDigit; i += kRadixThreads) s_wc[i] = 0;
  for (int pass = 0; pass < 4; ++pass) {  // a -> b -> a -> b -> a
    const uint32_t D = pass == 0 ? 256u : pass == 3 ? 1024u : 2048u;
    const uint64_t* src = (pass & 1) ? b : a;
    uint64_t* dst = (pass & 1) ? a : b;
    // 1. digit counts, then their exclusive prefix (warp 0)
    for (uint32_t d = threadIdx.x; d < D; d += kRadixThreads) s_base[d] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += kRadixThreads) {
      const uint32_t d = radix_digit(src[beg + i], pass);
      const unsigned peers = __match_any_sync(__activemask(), d);
      if ((__ffs(peers) - 1) == lane) atomicAdd(&s_base[d], uint32_t(__popc(peers)));
    }
    __syncthreads();
    if (w == 0) {
      uint32_t carry = 0;
      for (uint32_t c0 = 0; c0 < D; c0 += 32) {
        const uint32_t x = s_base[c0 + lane];
        uint32_t tot;
        const uint32_t ex = warp_excl_scan_u32(x, lane, &tot);
        s_base[c0 + lane] = carry + ex;
        carry += tot;
      }
    }
    __syncthreads();
    // 2. stable scatter: tiles of 256 keys, thread t holding key t of the tile; a key's place among
    //    the tile's keys of its digit = (keys of that digit in earlier warps) + (earlier lanes)
    for (uint32_t t0 = 0; t0 < n; t0 += kRadixThreads) {
      const uint32_t i = t0 + threadIdx.x;
      const bool in = i < n;
      const uint64_t key = in ? src[beg + i] : 0ull;
      const uint32_t d = in ? radix_digit(key, pass) : 0xffffffffu;
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      const uint32_t cnt = uint32_t(__popc(peers));
      const bool leader = in && (__ffs(peers) - 1) == lane;
      if (leader) s_wc[w * D + d] = cnt;
      __syncthreads();
      uint32_t before = 0, after = 0;
      if (in) {
        for (int ww = 0; ww < w; ++ww) before += s_wc[ww * D + d];
        for (int ww = w + 1; ww < NW; ++ww) after += s_wc[ww * D + d];
        dst[beg + s_base[d] + before + uint32_t(__popc(peers & ((1u << lane) - 1u)))] = key;
      }
      __syncthreads();
      if (leader) {
        if (after == 0) s_base[d] += before + cnt;  // the tile's last warp of digit d advances it
        s_wc[w * D + d] = 0;
      }
      __syncthreads();
    }
  }
}

// The scan: one CTA per segment, class counts in shared memory (wide.cuh), any class count.
__global__ void __launch_bounds__(kWideThreads) k_big_scan_wide(const NodeIn* __restrict__ nodes,
                                                                const BigSeg* __restrict__ segs, uint32_t R, int k,
                                                                const uint32_t* __restrict__ row_ptr,
                                                                const uint64_t* __restrict__ keys,
                                                                const double* __restrict__ xl,
                                                                RowRes* __restrict__ rowres) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const BigSeg sg = segs[blockIdx.x];
  const NodeIn nd = nodes[sg.node];
  const uint32_t* rp = row_ptr + size_t(sg.node) * (R + 1);
  if (rp[sg.row + 1] == rp[sg.row]) {  // empty rows are skipped in exact mode (split.hpp:308)
    if (threadIdx.x == 0) rowres[blockIdx.x] = RowRes{};
    return;
  }
  const WideShared s = wide_carve(smem_raw, k);
  const uint64_t* kk = keys + sg.off;
  const RowRes rr = wide_exact_scan([&](uint32_t p) { return __ldg(kk + p); }, nd.n, k, nd.parent, xl, s.base,
                                    s.run, s.tot, nullptr, s.red, s.ured);
  if (threadIdx.x == 0) rowres[blockIdx.x] = rr;
}

// Best row of each big node: rows arrive in increasing order per node (segments are node-major).
__global__ void k_big_select(const BigSeg* __restrict__ segs, int n_nodes, uint32_t R,
                             const RowRes* __restrict__ rowres, NodeRes* __restrict__ res) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_nodes) return;
  int best = -1;
  double g = 0.0;
  float thr = 0.f;
  uint32_t nl = 0;
  for (uint32_t r = 0; r < R; ++r) {
    const RowRes rr = rowres[size_t(i) * R + r];
    if (rr.valid && (best < 0 || rr.gain > g)) {
      best = int(r);
      g = rr.gain;
      thr = rr.threshold;
      nl = rr.n_left;
    }
  }
  NodeRes& o = res[segs[size_t(i) * R].node];
  o.row = best;
  o.gain = g;
  o.threshold = thr;
  o.n_left_search = nl;
}

}  // namespace dev

// Nodes `list[0..n)` (all exact, n_i > kExactSmemMax). Processes them in chunks that bound the
// key buffers; allocations are stream-ordered.
cudaError_t launch_exact_big(const NodeIn* nodes, const NodeIn* h_nodes, const uint32_t* h_list,
                             int n, uint32_t R, int k, const uint32_t* row_ptr, const uint8_t* lab,
                             const uint64_t* vbase, const float* V, const double* xl, NodeRes* res,
                             Scratch& scratch, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const uint64_t kMaxKeys = 256ull << 20;  // 2 GB of keys (x2 for the sort's double buffer)
  int i0 = 0;
  while (i0 < n) {
    // chunk of nodes
    uint64_t keys = 0;
    int i1 = i0;
    while (i1 < n && (i1 == i0 || keys + uint64_t(h_nodes[h_list[i1]].n) * R <= kMaxKeys)) {
      keys += uint64_t(h_nodes[h_list[i1]].n) * R;
      ++i1;
    }
    const int nn = i1 - i0;
    const int nseg = nn * int(R);
    std::vector<dev::BigSeg> segs(static_cast<size_t>(nseg));
    uint64_t off = 0;
    for (int i = 0; i < nn; ++i) {
      const uint32_t node = h_list[i0 + i];
      for (uint32_t r = 0; r < R; ++r) {
        segs[size_t(i) * R + r] = dev::BigSeg{node, r, off};
        off += h_nodes[node].n;
      }
    }
    // scratch kept across calls (grow-only, owned by the caller's WaveRunner)
    auto ar_get = [&](int i, size_t bytes) { return scratch.get(Scratch::kBigFirst + i, bytes, st); };
    dev::BigSeg* d_segs = static_cast<dev::BigSeg*>(ar_get(0, sizeof(dev::BigSeg) * nseg));
    uint64_t* d_k0 = static_cast<uint64_t*>(ar_get(1, 8 * keys));
    uint64_t* d_k1 = static_cast<uint64_t*>(ar_get(2, 8 * keys));
    uint64_t* d_b = static_cast<uint64_t*>(ar_get(3, 8 * size_t(nseg)));
    uint64_t* d_e = static_cast<uint64_t*>(ar_get(4, 8 * size_t(nseg)));
    RowRes* d_rr = static_cast<RowRes*>(ar_get(5, sizeof(RowRes) * nseg));
    if (!d_segs || !d_k0 || !d_k1 || !d_b || !d_e || !d_rr) return cudaErrorMemoryAllocation;
    cudaError_t e = cudaMemcpyAsync(d_segs, segs.data(), sizeof(dev::BigSeg) * nseg, cudaMemcpyHostToDevice, st);
    if (e) return e;
    dev::k_big_keys<<<nseg, 256, 0, st>>>(nodes, d_segs, R, lab, vbase, V, d_k0, d_b, d_e);
    constexpr size_t kRadixSmem = sizeof(uint32_t) * 8 * dev::kRadixMaxDigit;  // 64 KB per-warp digit counts
    e = cudaFuncSetAttribute(dev::k_seg_radix, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kRadixSmem));
    if (e) return e;
    dev::k_seg_radix<<<nseg, dev::kRadixThreads, kRadixSmem, st>>>(d_b, d_e, d_k0, d_k1);
    // sorted keys are back in d_k0 (four passes)
    dev::k_big_scan_wide<<<nseg, dev::kWideThreads, dev::wide_carve_bytes(k), st>>>(nodes, d_segs, R, k, row_ptr, d_k0,
                                                                                   xl, d_rr);
    dev::k_big_select<<<(nn + 127) / 128, 128, 0, st>>>(d_segs, nn, R, d_rr, res);
    e = cudaGetLastError();
    if (e) return e;
    i0 = i1;
  }
  return cudaSuccess;
}

}  // namespace sofg
