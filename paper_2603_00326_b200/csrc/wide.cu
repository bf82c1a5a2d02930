// Split search for more than kMaxClasses (8) classes, up to kMaxClassesWide (64): the reference
// puts no bound on class_count (dataset.hpp:36-44); its impurity at a candidate split is a sum
// over all k classes in class order (split.hpp:66-76), so a candidate costs O(k) here as there.
// The class counts do not fit the register-resident kernels (exact.cu, split.cu), so these keep
// them in shared memory and evaluate 32 candidates per warp step, one per lane:
//
//  k_hist_wide   histogram splitter (build_histogram + best_split_histogram, histogram.hpp:180-206,
//                split.hpp:84-120): one CTA per (node, row, chunk of <= 65535 samples); bins by
//                upper_bound over the row's boundaries in shared memory, u16 counters packed in
//                pairs; multi-chunk nodes merge in global counters and the chunk that completes
//                the row scans.
//  k_exact_wide  exact splitter (best_split_exact, split.hpp:142-194) for nodes of <= 2048
//                samples: one CTA per (node, row); the packed keys order_key(v) << 32 | label are
//                bitonic-sorted in shared memory, then scanned.
//  (exact_big.cu's k_big_scan_wide scans the device-sorted segments of nodes above 2048.)
// Each writes one RowRes per (node, row); the node's best row is picked by k_hist_select
// (split.hpp:259-263: strict '>', lowest row wins).
#include <cuda_runtime.h>

#include "common.hpp"
#include "dev_util.cuh"
#include "kernels.hpp"
#include "wide.cuh"

namespace sofg {
namespace dev {

// ------------------------------------------------------------------------------------------
// Exact, nodes of <= kExactSmemMax samples: one CTA per (listed node, row).
__global__ void __launch_bounds__(kWideThreads) k_exact_wide(
    const NodeIn* __restrict__ nodes, const uint32_t* __restrict__ list, uint32_t R, int k,
    const uint32_t* __restrict__ row_ptr, const uint8_t* __restrict__ lab,
    const uint64_t* __restrict__ gbase, const float* __restrict__ G, const double* __restrict__ xl,
    RowRes* __restrict__ rowres) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t li = blockIdx.x / R, r = blockIdx.x % R;
  const uint32_t node = list[li];
  const NodeIn nd = nodes[node];
  const uint32_t* rp = row_ptr + size_t(node) * (R + 1);
  RowRes* out = rowres + size_t(li) * R + r;
  if (rp[r + 1] == rp[r] || nd.n < 2) {  // empty rows are skipped in exact mode (split.hpp:308)
    if (threadIdx.x == 0) *out = RowRes{};
    return;
  }
  WideShared s = wide_carve(smem_raw, k);
  const uint32_t n = nd.n;
  uint32_t P = 1;
  while (P < n) P <<= 1;
  uint64_t* keys = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(s.rest) + 15) & ~uintptr_t(15));
  double* xs = reinterpret_cast<double*>(keys + P);
  const uint32_t Rp = vpitch(R);
  const float* Vn = G + gbase[node] + r;
  for (uint32_t j = threadIdx.x; j < P; j += kWideThreads)
    keys[j] = j < n ? (uint64_t(order_key(__ldg(Vn + uint64_t(j) * Rp))) << 32) | uint64_t(lab[nd.begin + j])
                    : ~0ull;
  __syncthreads();
  for (uint32_t sz = 2; sz <= P; sz <<= 1)  // bitonic sort, ascending
    for (uint32_t st = sz >> 1; st > 0; st >>= 1) {
      for (uint32_t i = threadIdx.x; i < P; i += kWideThreads) {
        const uint32_t j = i ^ st;
        if (j > i) {
          const uint64_t a = keys[i], b = keys[j];
          const bool up = (i & sz) == 0;
          if ((a > b) == up) {
            keys[i] = b;
            keys[j] = a;
          }
        }
      }
      __syncthreads();
    }
  const RowRes rr = wide_exact_scan([&](uint32_t p) { return keys[p]; }, n, k, nd.parent, xl, s.base, s.run, s.tot,
                                    xs, s.red, s.ured);
  if (threadIdx.x == 0) *out = rr;
}

// ------------------------------------------------------------------------------------------
// Histogram: one CTA per WideWork item (node, row, chunk). Counters: u16 pairs [nb + 1][k].
__global__ void __launch_bounds__(kWideThreads) k_hist_wide(
    const NodeIn* __restrict__ nodes, const uint32_t* __restrict__ node_hist_slot, const HistWork* __restrict__ work,
    const uint32_t* __restrict__ multi_slot, uint32_t R, uint32_t bins, int k, int two_level,
    const uint8_t* __restrict__ lab, const uint64_t* __restrict__ gbase, const float* __restrict__ G,
    const float* __restrict__ bnd_g, const uint32_t* __restrict__ nb_g, const double* __restrict__ xl,
    uint32_t* __restrict__ gcnt, uint32_t* __restrict__ done, RowRes* __restrict__ rowres) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_last;
  const HistWork wk = work[blockIdx.x];
  const uint32_t r = wk.row0;
  const NodeIn nd = nodes[wk.node];
  const uint32_t h = node_hist_slot[wk.node];
  const uint32_t nb = nb_g[size_t(h) * R + r];
  const float* bnd = bnd_g + (size_t(h) * R + r) * (bins - 1);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* sb = reinterpret_cast<float*>(smem_raw);                      // [bins] boundaries
  uint32_t* cnt = reinterpret_cast<uint32_t*>(sb + ((bins + 3) & ~3u));  // u16 pairs
  const uint32_t nbin = nb + 1, words = (nbin * uint32_t(k) + 1) / 2;
  for (uint32_t i = threadIdx.x; i < nb; i += kWideThreads) sb[i] = __ldg(bnd + i);
  for (uint32_t i = threadIdx.x; i < words; i += kWideThreads) cnt[i] = 0;
  __syncthreads();
  // NaN: bin 0 under the two-level table (63 / 255 boundaries with two_level_binning), bin nb
  // under the scalar upper_bound lookup (histogram.hpp:72-75,118-131)
  const uint32_t nan_bin = (two_level && (nb == 63 || nb == 255)) ? 0u : nb;
  const uint32_t Rp = vpitch(R);
  const float* Vn = G + gbase[wk.node] + uint64_t(wk.start) * Rp + r;
  const uint8_t* ln = lab + nd.begin + wk.start;
  for (uint32_t j = threadIdx.x; j < wk.len; j += kWideThreads) {
    const float v = __ldg(Vn + uint64_t(j) * Rp);
    uint32_t lo = 0, hi = nb;  // upper_bound: first boundary > v
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (v < sb[mid]) hi = mid; else lo = mid + 1;
    }
    const uint32_t bin = v != v ? nan_bin : lo;
    const uint32_t idx = bin * uint32_t(k) + ln[j];
    atomicAdd(&cnt[idx >> 1], 1u << (16 * (idx & 1u)));
  }
  __syncthreads();
  const uint32_t* src = nullptr;  // counts as u32 [nbin][k]: the chunk's (in shared memory) or merged
  uint32_t* merged = nullptr;
  if (wk.n_chunks > 1) {
    const uint32_t ms = multi_slot[wk.node];
    uint32_t* g = gcnt + (size_t(ms) * R + r) * size_t(bins) * size_t(k);
    for (uint32_t i = threadIdx.x; i < nbin * uint32_t(k); i += kWideThreads) {
      const uint32_t x = (cnt[i >> 1] >> (16 * (i & 1u))) & 0xffffu;
      if (x) atomicAdd(g + i, x);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&done[size_t(ms) * R + r], 1u) == wk.n_chunks - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    merged = g;
    src = g;
  }
  if (w != 0) return;
  auto count_at = [&](uint32_t b, int c) -> uint32_t {
    const uint32_t i = b * uint32_t(k) + uint32_t(c);
    return src ? __ldcg(merged + i) : (cnt[i >> 1] >> (16 * (i & 1u))) & 0xffffu;
  };
  // class totals over every bin (split.hpp:95-101); the running left counts live in tot_run
  uint32_t* s_tot = reinterpret_cast<uint32_t*>(cnt + words);  // [k]
  uint32_t* s_run = s_tot + k;                                   // [k]
  double* s_x = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(s_run + k) + 7) & ~uintptr_t(7));  // [nb]
  uint32_t n = 0;
  for (int c = 0; c < k; ++c) {
    uint32_t t = 0;
    for (uint32_t b = lane; b < nbin; b += 32) t += count_at(b, c);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) {
      s_tot[c] = t;
      s_run[c] = 0;
    }
    n += t;
  }
  __syncwarp();
  RowRes res{};
  if (nb == 0 || n < 2) {  // split.hpp:101
    if (lane == 0) rowres[size_t(h) * R + r] = res;
    return;
  }
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  const double dn = double(n);
  double xmin = inf;
  for (uint32_t q = 0; q < nb; q += 32) {
    const uint32_t b = q + uint32_t(lane);
    const bool in = b < nb;
    double sl = 0.0, sr = 0.0;
    uint32_t nl = 0;
    for (int c = 0; c < k; ++c) {
      uint32_t x = in ? count_at(b, c) : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {  // inclusive scan over the chunk's candidates
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      const uint32_t base = s_run[c];
      const uint32_t l = base + x;
      nl += l;
      sl = __dadd_rn(sl, __ldg(xl + l));
      sr = __dadd_rn(sr, __ldg(xl + (s_tot[c] - l)));
      __syncwarp();
      if (lane == 31) s_run[c] = l;
      __syncwarp();
    }
    const uint32_t nr = n - nl;
    double X = inf;
    if (in && nl != 0 && nr != 0) {
      X = __dsub_rn(__dadd_rn(__dsub_rn(__ldg(xl + nl), sl), __ldg(xl + nr)), sr);
      xmin = fmin(xmin, X);
    }
    if (in) s_x[b] = X;
    // s_x also keeps nl for the winner: recomputed below from the counts
  }
  xmin = warp_min_f64(xmin);
  __syncwarp();
  if (xmin < inf) {
    const double g = gain_from_x(nd.parent, xmin, dn);
    if (g > 0.0) {
      const double win = x_window(nd.parent, xmin, dn);
      uint32_t first = 0xffffffffu;
      for (uint32_t b = lane; b < nb; b += 32) {
        const double X = s_x[b];
        if (X < inf && X <= win && gain_from_x(nd.parent, X, dn) == g) {
          first = b;
          break;
        }
      }
      const uint32_t fb = warp_min_u32(first);
      uint32_t nl = 0;  // left count at the winning boundary: bins [0, fb]
      for (uint32_t b = lane; b <= fb; b += 32)
        for (int c = 0; c < k; ++c) nl += count_at(b, c);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nl += __shfl_xor_sync(0xffffffffu, nl, o);
      res.valid = 1;
      res.gain = g;
      res.threshold = sb[fb];
      res.n_left = nl;
    }
  }
  if (lane == 0) rowres[size_t(h) * R + r] = res;
}

}  // namespace dev

// ---------------------------------------------------------------------------- launchers
size_t exact_wide_smem(uint32_t nmax, int k) {
  uint32_t P = 1;
  while (P < nmax) P <<= 1;
  return dev::wide_carve_bytes(k) + 16 + size_t(P) * 16;
}

cudaError_t launch_exact_wide(const NodeIn* nodes, const uint32_t* list, int n_list, uint32_t nmax, uint32_t R,
                              int k, const uint32_t* row_ptr, const uint8_t* lab, const uint64_t* gbase,
                              const float* G, const double* xl, RowRes* rowres, cudaStream_t st) {
  if (n_list == 0) return cudaSuccess;
  const size_t smem = exact_wide_smem(nmax, k);
  if (smem > size_t(kSmemOptin)) return cudaErrorInvalidValue;
  cudaFuncSetAttribute(dev::k_exact_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptin);
  dev::k_exact_wide<<<unsigned(n_list) * R, dev::kWideThreads, smem, st>>>(nodes, list, R, k, row_ptr, lab, gbase,
                                                                           G, xl, rowres);
  return cudaGetLastError();
}

size_t hist_wide_smem(uint32_t bins, int k) {
  return size_t((bins + 3) & ~3u) * 4 + (size_t(bins) * k + 1) / 2 * 4 + size_t(2 * k) * 4 + 8 + size_t(bins) * 8;
}

cudaError_t launch_hist_wide(const NodeIn* nodes, const uint32_t* node_hist_slot, const HistWork* work, int n_work,
                             const uint32_t* multi_slot, uint32_t R, uint32_t bins, int k, int two_level,
                             const uint8_t* lab, const uint64_t* gbase, const float* G, const float* bnd,
                             const uint32_t* nb, const double* xl, uint32_t* gcnt, uint32_t* done, RowRes* rowres,
                             cudaStream_t st) {
  if (n_work == 0) return cudaSuccess;
  const size_t smem = hist_wide_smem(bins, k);
  if (smem > size_t(kSmemOptin)) return cudaErrorInvalidValue;
  cudaFuncSetAttribute(dev::k_hist_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptin);
  dev::k_hist_wide<<<n_work, dev::kWideThreads, smem, st>>>(nodes, node_hist_slot, work, multi_slot, R, bins, k,
                                                            two_level, lab, gbase, G, bnd, nb, xl, gcnt, done,
                                                            rowres);
  return cudaGetLastError();
}

}  // namespace sofg
