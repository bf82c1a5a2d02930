// Exact splitter for large nodes (n > kExactSmemMax): ExactOnly mode, or a breakeven above the
// shared-memory splitter's range (reference best_split_exact, split.hpp:142-194, for every
// non-empty row, split.hpp:306-312).
//
//  1. k_big_keys    per (node, row) segment: the reference's packed sort key
//                   order_key(v) << 32 | label for every sample, from the wave's V block;
//  2. cub::DeviceSegmentedRadixSort sorts every segment (device-wide, all segments at once);
//  3. k_big_scan    one CTA per segment: block scans of the class counts over the sorted keys,
//                   impurity at every gap between distinct values in the reference's FP64 order,
//                   minimum X, then the first position whose gain equals the best (first maximum);
//  4. k_big_select  best row per node (strict '>', lowest row wins, split.hpp:259-263).
#include <cuda_runtime.h>

#include <vector>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>

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

constexpr int kBigThreads = 256;

// One CTA per segment; the segment's sorted keys are walked in tiles of kBigThreads.
template <int KC>
__global__ void __launch_bounds__(kBigThreads) k_big_scan(const NodeIn* __restrict__ nodes,
                                                          const BigSeg* __restrict__ segs,
                                                          uint32_t R, int k,
                                                          const uint32_t* __restrict__ row_ptr,
                                                          const uint64_t* __restrict__ keys,
                                                          const double* __restrict__ xl,
                                                          RowRes* __restrict__ rowres) {
  using Scan = cub::BlockScan<uint32_t, kBigThreads>;
  using RedD = cub::BlockReduce<double, kBigThreads>;
  using RedU = cub::BlockReduce<uint32_t, kBigThreads>;
  __shared__ union {
    typename Scan::TempStorage scan;
    typename RedD::TempStorage redd;
    typename RedU::TempStorage redu;
  } tmp;
  __shared__ uint32_t s_carry[KC];
  __shared__ double s_xmin;
  __shared__ uint32_t s_first;
  const BigSeg sg = segs[blockIdx.x];
  const NodeIn nd = nodes[sg.node];
  const uint32_t n = nd.n;
  const uint64_t* K = keys + sg.off;
  RowRes out{};
  const uint32_t* rp = row_ptr + size_t(sg.node) * (R + 1);
  if (rp[sg.row + 1] == rp[sg.row]) {  // empty rows are skipped in exact mode (split.hpp:308)
    if (threadIdx.x == 0) rowres[blockIdx.x] = out;
    return;
  }
  // class totals
  uint32_t tot[KC];
  {
    uint32_t c[KC];
#pragma unroll
    for (int cc = 0; cc < KC; ++cc) c[cc] = 0;
    for (uint32_t j = threadIdx.x; j < n; j += kBigThreads) {
      const int y = int(K[j] & 0xffu);
#pragma unroll
      for (int cc = 0; cc < KC; ++cc) c[cc] += (cc == y);
    }
#pragma unroll
    for (int cc = 0; cc < KC; ++cc) {
      const uint32_t t = RedU(tmp.redu).Sum(c[cc]);
      if (threadIdx.x == 0) s_carry[cc] = t;
      __syncthreads();
      tot[cc] = s_carry[cc];
      __syncthreads();
    }
  }
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  const double dn = double(n);
  // Walk the sorted keys; visit(p, X, a, b) for every candidate gap after position p.
  auto walk = [&](auto&& visit) {
    if (threadIdx.x < KC) s_carry[threadIdx.x] = 0;
    __syncthreads();
    for (uint32_t base = 0; base < n; base += kBigThreads) {
      const uint32_t p = base + threadIdx.x;
      const uint64_t key = p < n ? K[p] : ~0ull;
      const int y = int(key & 0xffu);
      uint32_t left[KC];
#pragma unroll
      for (int cc = 0; cc < KC; ++cc) {
        uint32_t agg;
        Scan(tmp.scan).InclusiveSum(p < n && cc == y ? 1u : 0u, left[cc], agg);
        __syncthreads();
        left[cc] += s_carry[cc];
        __syncthreads();
        if (threadIdx.x == kBigThreads - 1) s_carry[cc] = left[cc];
      }
      __syncthreads();
      if (p + 1 < n) {
        const float a = order_key_inv(uint32_t(key >> 32));
        const float b = order_key_inv(uint32_t(K[p + 1] >> 32));
        if (a < b) {
          const uint32_t nl = p + 1;
          const double X = impurity_sum<KC>(xl, left, tot, k, nl, n - nl);
          visit(p, X, a, b);
        }
      }
    }
  };
  double xmin = inf;
  walk([&](uint32_t, double X, float, float) { xmin = fmin(xmin, X); });
  const double bx = RedD(tmp.redd).Reduce(xmin, [](double x, double y) { return fmin(x, y); });
  if (threadIdx.x == 0) s_xmin = bx;
  __syncthreads();
  xmin = s_xmin;
  const double g = gain_from_x(nd.parent, xmin, dn);
  if (!(xmin < inf) || !(g > 0.0)) {
    if (threadIdx.x == 0) rowres[blockIdx.x] = out;
    return;
  }
  const double win = x_window(nd.parent, xmin, dn);
  uint32_t first = 0xffffffffu;
  walk([&](uint32_t p, double X, float, float) {
    if (first == 0xffffffffu && X <= win && (X == xmin || gain_from_x(nd.parent, X, dn) == g)) first = p;
  });
  const uint32_t bf = RedU(tmp.redu).Reduce(first, [](uint32_t x, uint32_t y) { return min(x, y); });
  if (threadIdx.x == 0) {
    const float a = order_key_inv(uint32_t(K[bf] >> 32));
    const float b = order_key_inv(uint32_t(K[bf + 1] >> 32));
    out.valid = 1;
    out.gain = g;
    out.threshold = midpoint_down(a, b);
    out.n_left = bf + 1;
    rowres[blockIdx.x] = out;
  }
}

// More than kMaxClasses classes: one CTA per segment, class counts in shared memory (wide.cuh).
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
    size_t tb = 0;
    e = cub::DeviceSegmentedRadixSort::SortKeys(nullptr, tb, d_k0, d_k1, int64_t(keys), nseg, d_b, d_e, 0, 64, st);
    void* d_tmp = e ? nullptr : ar_get(6, tb ? tb : 1);
    if (!e && !d_tmp) e = cudaErrorMemoryAllocation;
    if (!e) e = cub::DeviceSegmentedRadixSort::SortKeys(d_tmp, tb, d_k0, d_k1, int64_t(keys), nseg, d_b, d_e, 0, 64, st);
    if (e) return e;
    if (k == 2)
      dev::k_big_scan<2><<<nseg, dev::kBigThreads, 0, st>>>(nodes, d_segs, R, k, row_ptr, d_k1, xl, d_rr);
    else if (k <= kMaxClasses)
      dev::k_big_scan<kMaxClasses><<<nseg, dev::kBigThreads, 0, st>>>(nodes, d_segs, R, k, row_ptr, d_k1, xl, d_rr);
    else
      dev::k_big_scan_wide<<<nseg, dev::kWideThreads, dev::wide_carve_bytes(k), st>>>(nodes, d_segs, R, k, row_ptr,
                                                                                     d_k1, xl, d_rr);
    dev::k_big_select<<<(nn + 127) / 128, 128, 0, st>>>(d_segs, nn, R, d_rr, res);
    e = cudaGetLastError();
    if (e) return e;
    i0 = i1;
  }
  return cudaSuccess;
}

}  // namespace sofg
