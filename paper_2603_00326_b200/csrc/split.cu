// Split search for one wave of nodes.
//
//  k_hist_count   histogram splitter (reference build_histogram + best_split_histogram,
//                 histogram.hpp:180-206, split.hpp:84-120). One CTA = 8 rows (one warp each) x
//                 one chunk of the node's samples. Each lane reads a sample's 8 projected rows
//                 (one 32-byte sector of V), bins each by an upper_bound over that row's
//                 boundaries (implicit search tree in shared memory) and counts with shared
//                 atomics. Single-chunk nodes scan in place; multi-chunk nodes merge into global
//                 counters and the last CTA of the (node, row group) scans.
//  k_hist_select  best row of a histogram node (split.hpp:259-263: strict '>', lowest row wins).
//  k_exact        exact splitter (split.hpp:142-194) for nodes of <= kExactSmemMax samples:
//                 per row, gather, sort (order_key(v) << 32 | label), scan, min impurity.
#include <cuda_runtime.h>

#include "common.hpp"
#include "dev_util.cuh"
#include "kernels.hpp"

namespace sofg {
namespace dev {

// Count-vector scan of one histogram row, warp-cooperative. cnt is bin-major [nbins][k] in
// shared memory, nb boundaries in bnd. Returns the reference's best candidate for this row.
template <int KC, class Get>
__device__ RowRes hist_row_scan_g(const Get& cnt_at, const float* bnd, uint32_t nb, int k,
                                  int bpad, double parent, const double* __restrict__ xl,
                                  int lane) {
  RowRes res;
  res.valid = 0;
  res.gain = 0.0;
  res.threshold = 0.f;
  res.n_left = 0;
  res._pad = 0;
  const int E = bpad / 32;
  const int b0 = lane * E;
  uint32_t loc[KC], pre[KC], tot[KC];
#pragma unroll
  for (int c = 0; c < KC; ++c) loc[c] = 0;
  for (int e = 0; e < E; ++e) {
    const int b = b0 + e;
    if (b <= int(nb)) {
#pragma unroll
      for (int c = 0; c < KC; ++c)
        if (c < k) loc[c] += cnt_at(b, c);
    }
  }
  uint32_t n = 0;
#pragma unroll
  for (int c = 0; c < KC; ++c) {
    if (c < k) {
      pre[c] = warp_excl_scan_u32(loc[c], lane, &tot[c]);
      n += tot[c];
    } else {
      pre[c] = 0;
      tot[c] = 0;
    }
  }
  if (n < 2) return res;  // split.hpp:101
  const double dn = double(n);

  // pass 1: min impurity over candidate boundaries b < nb
  double xmin = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  {
    uint32_t left[KC];
#pragma unroll
    for (int c = 0; c < KC; ++c) left[c] = pre[c];
    for (int e = 0; e < E; ++e) {
      const int b = b0 + e;
      if (b >= int(nb)) break;
      uint32_t nl = 0;
#pragma unroll
      for (int c = 0; c < KC; ++c)
        if (c < k) {
          left[c] += cnt_at(b, c);
          nl += left[c];
        }
      const uint32_t nr = n - nl;
      if (nl == 0 || nr == 0) continue;
      const double X = impurity_sum<KC>(xl, left, tot, k, nl, nr);
      xmin = fmin(xmin, X);
    }
  }
  xmin = warp_min_f64(xmin);
  if (!(xmin < __longlong_as_double(0x7ff0000000000000ll))) return res;
  const double gbest = gain_from_x(parent, xmin, dn);
  if (!(gbest > 0.0)) return res;
  const double win = x_window(parent, xmin, dn);
  // pass 2: first boundary whose gain equals gbest
  uint32_t first = 0xffffffffu, first_nl = 0;
  {
    uint32_t left[KC];
#pragma unroll
    for (int c = 0; c < KC; ++c) left[c] = pre[c];
    for (int e = 0; e < E; ++e) {
      const int b = b0 + e;
      if (b >= int(nb)) break;
      uint32_t nl = 0;
#pragma unroll
      for (int c = 0; c < KC; ++c)
        if (c < k) {
          left[c] += cnt_at(b, c);
          nl += left[c];
        }
      const uint32_t nr = n - nl;
      if (nl == 0 || nr == 0) continue;
      const double X = impurity_sum<KC>(xl, left, tot, k, nl, nr);
      if (X <= win && gain_from_x(parent, X, dn) == gbest) {
        first = uint32_t(b);
        first_nl = nl;
        break;
      }
    }
  }
  const uint32_t fb = warp_min_u32(first);
  const uint32_t src = __ffs(__ballot_sync(0xffffffffu, first == fb)) - 1;
  const uint32_t nl = __shfl_sync(0xffffffffu, first_nl, src);
  res.valid = 1;
  res.gain = gbest;
  res.threshold = __ldg(bnd + fb);  // sorted boundaries (global)
  res.n_left = nl;
  return res;
}

// Two-class form of hist_row_scan_g for E = bpad / 32 candidates per lane (compile time): every
// candidate's six table values are loaded before any is used (no data-dependent exits in the load
// phase) and the impurity sums stay in registers for the first-maximum pass. Same operations in
// the same order as impurity_sum<2> / gain_from_x, so the result is identical.
template <int E, class Get>
__device__ RowRes hist_row_scan2(const Get& cnt_at, const float* bnd, uint32_t nb, double parent,
                                 const double* __restrict__ xl, int lane) {
  RowRes res;
  res.valid = 0;
  res.gain = 0.0;
  res.threshold = 0.f;
  res.n_left = 0;
  res._pad = 0;
  const int b0 = lane * E;
  uint32_t c0[E], c1[E], s0 = 0, s1 = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const bool in = b0 + e <= int(nb);
    c0[e] = in ? cnt_at(b0 + e, 0) : 0u;
    c1[e] = in ? cnt_at(b0 + e, 1) : 0u;
    s0 += c0[e];
    s1 += c1[e];
  }
  uint32_t t0, t1;
  const uint32_t p0 = warp_excl_scan_u32(s0, lane, &t0), p1 = warp_excl_scan_u32(s1, lane, &t1);
  const uint32_t n = t0 + t1;
  if (n < 2) return res;  // split.hpp:101
  const double dn = double(n);
  double X[E];
  bool ok[E];
  uint32_t nlv[E];
  {
    uint32_t l0 = p0, l1 = p1;
    uint32_t i0[E], i1[E], inl[E], inr[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      l0 += c0[e];
      l1 += c1[e];
      const uint32_t nl = l0 + l1, nr = n - nl;
      ok[e] = b0 + e < int(nb) && nl != 0 && nr != 0;
      nlv[e] = nl;
      i0[e] = ok[e] ? l0 : 0u;
      i1[e] = ok[e] ? l1 : 0u;
      inl[e] = ok[e] ? nl : 0u;
      inr[e] = ok[e] ? nr : 0u;
    }
    double a0[E], a1[E], r0[E], r1[E], fl[E], fr[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      a0[e] = __ldg(xl + i0[e]);
      a1[e] = __ldg(xl + i1[e]);
      r0[e] = __ldg(xl + (ok[e] ? t0 - i0[e] : 0u));
      r1[e] = __ldg(xl + (ok[e] ? t1 - i1[e] : 0u));
      fl[e] = __ldg(xl + inl[e]);
      fr[e] = __ldg(xl + inr[e]);
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const double sl = __dadd_rn(a0[e], a1[e]), sr = __dadd_rn(r0[e], r1[e]);
      X[e] = __dsub_rn(__dadd_rn(__dsub_rn(fl[e], sl), fr[e]), sr);
    }
  }
  double xmin = __longlong_as_double(0x7ff0000000000000ll);  // +inf
#pragma unroll
  for (int e = 0; e < E; ++e)
    if (ok[e]) xmin = fmin(xmin, X[e]);
  xmin = warp_min_f64(xmin);
  if (!(xmin < __longlong_as_double(0x7ff0000000000000ll))) return res;
  const double gbest = gain_from_x(parent, xmin, dn);
  if (!(gbest > 0.0)) return res;
  const double win = x_window(parent, xmin, dn);
  uint32_t first = 0xffffffffu, first_nl = 0;
#pragma unroll
  for (int e = E - 1; e >= 0; --e)  // the lowest qualifying candidate of this lane wins
    if (ok[e] && X[e] <= win && gain_from_x(parent, X[e], dn) == gbest) {
      first = uint32_t(b0 + e);
      first_nl = nlv[e];
    }
  const uint32_t fb = warp_min_u32(first);
  const uint32_t src = __ffs(__ballot_sync(0xffffffffu, first == fb)) - 1;
  res.valid = 1;
  res.gain = gbest;
  res.threshold = __ldg(bnd + fb);  // sorted boundaries (global)
  res.n_left = __shfl_sync(0xffffffffu, first_nl, src);
  return res;
}

// Bin-major counts [nbins][k] of one row in shared memory.
template <int KC>
__device__ RowRes hist_row_scan(const uint32_t* cnt, const float* bnd, uint32_t nb, int k,
                                int bpad, double parent, const double* __restrict__ xl,
                                int lane) {
  return hist_row_scan_g<KC>([&](int b, int c) { return cnt[b * k + c]; }, bnd, nb, k, bpad, parent, xl, lane);
}

// ------------------------------------------------------------------------------------------
// LT > 0: compile-time search depth (bpad == 1 << LT); the 8 rows' searches interleave.
template <int KC, int LT>
__global__ void __launch_bounds__(256) k_hist_count(
    const NodeIn* __restrict__ nodes, const uint32_t* __restrict__ node_hist_slot,
    const HistWork* __restrict__ work, const uint32_t* __restrict__ multi_slot,
    uint32_t R, uint32_t bins, int bpad, int k, int chunk_cap, int two_level,
    const uint32_t* __restrict__ terms, const uint32_t* __restrict__ row_ptr,
    const uint8_t* __restrict__ lab, const uint64_t* __restrict__ gbase,
    const float* __restrict__ G, const float* __restrict__ bnd_g,
    const uint32_t* __restrict__ nb_g, const double* __restrict__ xl,
    uint32_t* __restrict__ gcnt, uint32_t* __restrict__ done, RowRes* __restrict__ rowres) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const HistWork wk = work[blockIdx.x];
  const NodeIn nd = nodes[wk.node];
  const uint32_t h = node_hist_slot[wk.node];
  // smem layout
  uint32_t* cnt_s = reinterpret_cast<uint32_t*>(smem_raw);                  // [8][bpad][k]
  float* bnd_s = reinterpret_cast<float*>(cnt_s + size_t(8) * bpad * k);      // [8][bpad]
  uint8_t* lab_s = reinterpret_cast<uint8_t*>(bnd_s + size_t(8) * bpad);     // [chunk_cap]
  __shared__ int s_last;
  __shared__ int s_nan_leaf[8];  // search-tree leaf of NaN values per row (see below)

  const uint32_t r = wk.row0 + uint32_t(w);  // the row this warp scans at the end
  const bool row_ok = r < R;
  const uint32_t nb = row_ok ? nb_g[size_t(h) * R + r] : 0;
  uint32_t* my_cnt = cnt_s + size_t(w) * bpad * k;
  const float pad = __int_as_float(0x7fc00000);  // NaN
  const float* gb = bnd_g + (size_t(h) * R + (row_ok ? r : 0)) * (bins - 1);
  // Boundaries of the 8 rows as implicit search trees (Eytzinger order: node t >= 1 holds the
  // sorted boundary ((2(t - 2^l) + 1) << (L-1-l)) - 1 at level l), padded with NaN (pad <= v is false for
  // every v, so v = +inf lands in bin nb as in the reference; NaN values land in bin 0,
  // the reference's two-level lookup result, histogram.hpp:117-131). A search
  // step at level l touches one of 2^l consecutive words, so the 32 lanes' probes spread over
  // the banks instead of piling onto one (sorted-order probes are power-of-two strided).
  int L = 0;
  while ((1 << L) < bpad) ++L;
  for (int i = threadIdx.x; i < 8 * bpad; i += blockDim.x) {
    const int g = i / bpad, t = i % bpad;
    float v = pad;
    const uint32_t rg = wk.row0 + uint32_t(g);
    if (t > 0 && rg < R) {
      const int l = 31 - __clz(t);
      const int sidx = ((2 * (t - (1 << l)) + 1) << (L - 1 - l)) - 1;
      const uint32_t nbg = nb_g[size_t(h) * R + rg];
      if (uint32_t(sidx) < nbg) v = bnd_g[(size_t(h) * R + rg) * (bins - 1) + sidx];
    }
    bnd_s[i] = v;
  }
  for (int i = threadIdx.x; i < 8 * bpad * k; i += blockDim.x) cnt_s[i] = 0;
  // NaN values: bin 0 under the reference's two-level table (used for 63 or 255 boundaries when
  // two_level_binning is set: every `boundary <= NaN` is false), bin nb under its scalar
  // std::upper_bound lookup (histogram.hpp:72-75,118-131; split.hpp:281-283).
  if (threadIdx.x < 8) {
    const uint32_t rg = wk.row0 + threadIdx.x;
    const uint32_t nbr = rg < R ? nb_g[size_t(h) * R + rg] : 0u;
    const bool scalar = !(two_level && (nbr == 63 || nbr == 255));
    s_nan_leaf[threadIdx.x] = bpad + (scalar ? int(nbr) : 0);
  }
  // stage the chunk's labels
  const uint8_t* lseg = lab + nd.begin + wk.start;
  for (uint32_t j = threadIdx.x; j < wk.len; j += blockDim.x) lab_s[j] = lseg[j];
  __syncthreads();

  {
    // Each lane takes one sample at a time and bins its 8 rows (one aligned 32-byte load).
    const uint32_t Rp = vpitch(R);
    const float* Vn = G + gbase[wk.node] + wk.row0;  // rows row0.. of the node's V block
    uint32_t live = 0;  // rows of this group with boundaries
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const uint32_t rg = wk.row0 + uint32_t(g);
      if (rg < R && nb_g[size_t(h) * R + rg] > 0) live |= 1u << g;
    }
    float root[8];  // each row's tree root (the median boundary): level 0 without a load
#pragma unroll
    for (int g = 0; g < 8; ++g) root[g] = bnd_s[g * bpad + 1];
    for (uint32_t j = uint32_t(threadIdx.x); j < wk.len; j += blockDim.x) {
      const float4* src = reinterpret_cast<const float4*>(Vn + uint64_t(wk.start + j) * Rp);
      const float4 a = __ldg(src), b = __ldg(src + 1);
      const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      const uint32_t y = lab_s[j];
      if constexpr (LT > 0) {
        // all 8 searches advance one level per step: 8 independent shared loads in flight
        constexpr int BP = 1 << LT;
        int t[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) t[g] = 2 + (root[g] <= v[g] ? 1 : 0);  // level 0 from registers
#pragma unroll
        for (int l = 1; l < LT; ++l) {
#pragma unroll
          for (int g = 0; g < 8; ++g) t[g] = 2 * t[g] + (bnd_s[g * BP + t[g]] <= v[g] ? 1 : 0);
        }
        bool nan = false;
#pragma unroll
        for (int g = 0; g < 8; ++g) nan |= v[g] != v[g];
        if (nan) {
#pragma unroll
          for (int g = 0; g < 8; ++g)
            if (v[g] != v[g]) t[g] = s_nan_leaf[g];
        }
#pragma unroll
        for (int g = 0; g < 8; ++g)
          if (live & (1u << g))  // uniform
            atomicAdd(&cnt_s[(size_t(g) * BP + size_t(t[g] - BP)) * k + y], 1u);
      } else {
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          if (!(live & (1u << g))) continue;  // uniform
          const float* tr = bnd_s + g * bpad;
          int t = 1;
          for (int l = 0; l < L; ++l) t = 2 * t + (tr[t] <= v[g] ? 1 : 0);
          if (v[g] != v[g]) t = s_nan_leaf[g];
          atomicAdd(&cnt_s[(size_t(g) * bpad + size_t(t - bpad)) * k + y], 1u);
        }
      }
    }
  }
  __syncthreads();

  if (wk.n_chunks == 1) {
    if (nb > 0) {
      const RowRes rr = hist_row_scan<KC>(my_cnt, gb, nb, k, bpad, nd.parent, xl, lane);
      if (lane == 0) rowres[size_t(h) * R + r] = rr;
    } else if (row_ok && lane == 0) {
      RowRes z{};
      rowres[size_t(h) * R + r] = z;
    }
    return;
  }
  // multi-chunk: merge into global counters, last CTA scans
  const uint32_t ms = multi_slot[wk.node];
  if (nb > 0) {
    uint32_t* g = gcnt + (size_t(ms) * R + r) * size_t(bpad) * k;
    for (int i = lane; i < int(nb + 1) * k; i += 32) {
      const uint32_t c = my_cnt[i];
      if (c) atomicAdd(g + i, c);
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(&done[size_t(ms) * ((R + 7) / 8) + wk.row0 / 8], 1u);
    s_last = prev == wk.n_chunks - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (nb > 0) {
    const uint32_t* g = gcnt + (size_t(ms) * R + r) * size_t(bpad) * k;
    for (int i = lane; i < int(nb + 1) * k; i += 32) my_cnt[i] = __ldcg(g + i);
    __syncwarp();
    const RowRes rr = hist_row_scan<KC>(my_cnt, gb, nb, k, bpad, nd.parent, xl, lane);
    if (lane == 0) rowres[size_t(h) * R + r] = rr;
  } else if (row_ok && lane == 0) {
    RowRes z{};
    rowres[size_t(h) * R + r] = z;
  }
}

// ------------------------------------------------------------------------------------------
// Histogram counting, lane = row (two classes, <= 256 bins). One CTA = 32 consecutive rows
// (row0 = 32 g) x one chunk of a node's samples; lane s of every warp owns row row0 + s. Each row's
// search tree lives in shared memory transposed — word t of row s at [t * 32 + s] — and so do its
// counters (u16 class 0 | u16 class 1 per bin; chunk <= 65535), so lane s only ever touches bank
// s: the search and the count atomics have no bank conflicts and no same-address collisions (the
// lane = sample layout of k_hist_count spends 57 % of its shared wavefronts on conflict replays:
// profiles/r01_ncu_hist_count.txt). Warp w takes samples w U + 8 U i with U = 8 searches in flight
// per lane; a warp's V load of one sample is 32 consecutive rows. The counters are then transposed
// 32 x 32 tile by tile (conflict-free both ways) into skewed row-major rows and each warp scans 4
// rows; multi-chunk nodes merge into the global counters first and the chunk that completes a
// (node, row group) scans.
#ifndef SOFG_LR_FFMA
#define SOFG_LR_FFMA 1  // FSET + FFMA + IMAD search step (177 -> 170 ms per step; 0: FSETP + SEL + IADD3)
#endif
#ifndef SOFG_LRU
#define SOFG_LRU 8
#endif
constexpr int kLrU = SOFG_LRU;  // searches in flight per lane (divides 32: a step's labels sit in one word)
template <int LT>
struct LrLayout {
  static constexpr int BP = 1 << LT;
  static constexpr int E = BP / 32;            // bins per lane in hist_row_scan_g
  static constexpr int PITCH = BP + 32 + 1;    // skewed row: bin b at b + b / E (lane-contiguous bins hit distinct banks)
  static constexpr int AREA = BP * 32 > 32 * PITCH ? BP * 32 : 32 * PITCH;  // words: trees, then rows
  __device__ static int at(int s, int b) { return s * PITCH + b + b / E; }
};

template <int LT>
__global__ void __launch_bounds__(256) k_hist_count_lr(
    const NodeIn* __restrict__ nodes, const uint32_t* __restrict__ node_hist_slot,
    const HistWork* __restrict__ work, const uint32_t* __restrict__ multi_slot, uint32_t R, uint32_t bins,
    int two_level, const uint8_t* __restrict__ lab, const uint64_t* __restrict__ gbase,
    const float* __restrict__ G, const float* __restrict__ bnd_g, const uint32_t* __restrict__ nb_g,
    const double* __restrict__ xl, uint32_t* __restrict__ gcnt, uint32_t* __restrict__ done,
    RowRes* __restrict__ rowres) {
  using Lay = LrLayout<LT>;
  constexpr int BP = Lay::BP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* tree = reinterpret_cast<float*>(smem_raw);                       // [BP][32], then rows
  uint32_t* cnt = reinterpret_cast<uint32_t*>(smem_raw) + Lay::AREA;       // [BP][32] packed
  uint32_t* lbits = cnt + BP * 32;                                         // [chunk / 32] label bits
  __shared__ int s_last;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const HistWork wk = work[blockIdx.x];
  const NodeIn nd = nodes[wk.node];
  const uint32_t h = node_hist_slot[wk.node];
  const uint32_t r = wk.row0 + uint32_t(lane);  // this lane's row
  const uint32_t nb = r < R ? nb_g[size_t(h) * R + r] : 0u;
  // Eytzinger trees of the 32 rows (as k_hist_count), NaN pads: pad <= v is false for every v.
  // Warp w moves sorted boundaries [32 w, 32 w + 32) of all 32 rows: coalesced row reads, a
  // 32 x 32 transpose through XOR-swizzled staging (conflict-free), then lane l writes row l's
  // words (bank l). Sorted index q sits at Eytzinger node t: i = q + 1, z = ctz(i),
  // t = 2^(LT-1-z) + (i >> (z + 1)).
  const float pad = __int_as_float(0x7fc00000);
  {
    uint32_t* stage = cnt + w * 1024;  // the counters are zeroed afterwards
    const float* brow = bnd_g + size_t(h) * R * (bins - 1);
    for (int m = w; m < BP / 32; m += 8) {
      float v[32];  // all 32 rows' loads in flight before the first store
      const uint32_t q = uint32_t(32 * m + lane);
#pragma unroll
      for (int i = 0; i < 32; ++i) {  // row i of the group, boundaries 32 m + lane (nb 0 past R)
        const uint32_t nbi = __shfl_sync(0xffffffffu, nb, i);
        v[i] = q < nbi ? __ldg(brow + (wk.row0 + uint32_t(i)) * (bins - 1) + q) : pad;
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) stage[i * 32 + (lane ^ i)] = __float_as_uint(v[i]);
      __syncwarp();
      for (int i = 0; i < 32; ++i) {  // boundary 32 m + i of row `lane`
        const uint32_t q1 = uint32_t(32 * m + i + 1);
        if (q1 < uint32_t(BP)) {
          const int z = __ffs(int(q1)) - 1;
          const int t = (1 << (LT - 1 - z)) + int(q1 >> (z + 1));
          tree[t * 32 + lane] = __uint_as_float(stage[lane * 32 + (i ^ lane)]);
        }
      }
      __syncwarp();
    }
    tree[lane] = pad;  // node 0 (unused)
  }
  __syncthreads();
  for (int i = threadIdx.x; i < BP * 32; i += blockDim.x) cnt[i] = 0;
  const uint8_t* lseg = lab + nd.begin + wk.start;
  for (uint32_t j0 = uint32_t(threadIdx.x) & ~31u; j0 < wk.len; j0 += blockDim.x) {
    const uint32_t j = j0 + uint32_t(lane);
    const unsigned b = __ballot_sync(0xffffffffu, j < wk.len && lseg[j] != 0);
    if (lane == 0) lbits[j0 >> 5] = b;
  }
  // NaN: bin 0 under the two-level table (63 / 255 boundaries with two_level_binning), bin nb
  // under the scalar upper_bound lookup (histogram.hpp:72-75,118-131; split.hpp:281-283)
  const int nan_leaf = BP + ((two_level && (nb == 63 || nb == 255)) ? 0 : int(nb));
  __syncthreads();

  {
    const uint32_t Rp = vpitch(R);
    const float root = tree[32 + lane];
    const float* Vl = G + gbase[wk.node] + uint64_t(wk.start) * Rp + min(r, Rp - 1);
    const uint32_t len = wk.len;
    // The search walks shared byte addresses A(t) = tree + 128 t + 4 lane: A(2t + p) =
    // 2 A(t) + (p ? 128 : 0) - (tree + 4 lane), one select and one shift-add per level.
    const uint32_t lane_base = uint32_t(__cvta_generic_to_shared(tree)) + 4u * uint32_t(lane);
    const uint32_t k0 = 0u - lane_base, k1 = 128u - lane_base;
#if SOFG_LR_FFMA
    constexpr uint32_t kMagicBits = 0x4B000000u + (1u << 20);  // float 2^23 + 2^20: unit mantissa steps
    const float magic = __uint_as_float(kMagicBits - lane_base);  // bits - lane_base stays in [2^23, 2^24)
#endif
    auto step = [&](const float (&v)[kLrU], const uint32_t (&inc)[kLrU], bool nan_fix) {
      uint32_t a[kLrU];
#pragma unroll
      for (int u = 0; u < kLrU; ++u) a[u] = lane_base + (root <= v[u] ? 3u * 128u : 2u * 128u);
#if SOFG_LR_FFMA
      // One ALU instruction per level instead of three: the comparison as a float 0 / 1 (FSET), the
      // branch offset through the mantissa of 2^23-scaled magic (FFMA), the address update by IMAD.
      // a holds the address plus a uniform, level-dependent offset D (D_{l+1} = 2 D_l + BU).
      {
        uint32_t D = 0;
#pragma unroll
        for (int l = 1; l < LT; ++l) {
#pragma unroll
          for (int u = 0; u < kLrU; ++u) {
            float b, sel;
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(b) : "r"(a[u] - D));
            asm("set.le.f32.f32 %0, %1, %2;" : "=f"(sel) : "f"(b), "f"(v[u]));
            a[u] = 2u * a[u] + __float_as_uint(__fmaf_rn(sel, 128.f, magic));
          }
          D = 2u * D + kMagicBits;
        }
#pragma unroll
        for (int u = 0; u < kLrU; ++u) a[u] -= D;
      }
#else
#pragma unroll
      for (int l = 1; l < LT; ++l) {
#pragma unroll
        for (int u = 0; u < kLrU; ++u) {
          float b;
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(b) : "r"(a[u]));
          a[u] = 2u * a[u] + (b <= v[u] ? k1 : k0);
        }
      }
#endif
      int t[kLrU];
#pragma unroll
      for (int u = 0; u < kLrU; ++u) t[u] = int((a[u] - lane_base) >> 7);
      if (nan_fix) {  // warp-uniform: NaN falls to leaf BP (bin 0) by itself; scalar rows move it
#pragma unroll
        for (int u = 0; u < kLrU; ++u)
          if (v[u] != v[u]) t[u] = nan_leaf;
      }
#pragma unroll
      for (int u = 0; u < kLrU; ++u) atomicAdd(&cnt[(t[u] - BP) * 32 + lane], inc[u]);
    };
    const bool nan_fix = __any_sync(0xffffffffu, nan_leaf != BP);
    // full steps: U consecutive samples per warp, the next step's values loaded while this one
    // searches (software pipeline); j0 is a multiple of U, so a step's labels sit in one word
    uint32_t j0 = uint32_t(w) * kLrU;
    float vn[kLrU];
    if (j0 + kLrU <= len) {
#pragma unroll
      for (int u = 0; u < kLrU; ++u) vn[u] = __ldg(Vl + uint64_t(j0 + u) * Rp);
    }
    for (; j0 + kLrU <= len; j0 += 8 * kLrU) {
      float v[kLrU];
      uint32_t inc[kLrU];
      const uint32_t bits = lbits[j0 >> 5] >> (j0 & 31);
#pragma unroll
      for (int u = 0; u < kLrU; ++u) {
        v[u] = vn[u];
        inc[u] = ((bits >> u) & 1u) ? 0x10000u : 1u;
      }
      const uint32_t jn = j0 + 8 * kLrU;
      if (jn + kLrU <= len) {
#pragma unroll
        for (int u = 0; u < kLrU; ++u) vn[u] = __ldg(Vl + uint64_t(jn + u) * Rp);
      }
      step(v, inc, nan_fix);
    }
    if (j0 < len) {  // this warp's last, partial step
      float v[kLrU];
      uint32_t inc[kLrU];
#pragma unroll
      for (int u = 0; u < kLrU; ++u) {
        const uint32_t j = j0 + uint32_t(u);
        const bool ok = j < len;
        v[u] = ok ? __ldg(Vl + uint64_t(j) * Rp) : 0.f;
        inc[u] = ok ? (((lbits[j >> 5] >> (j & 31)) & 1u) ? 0x10000u : 1u) : 0u;
      }
      step(v, inc, nan_fix);
    }
  }
  __syncthreads();
  // transpose the packed counters into skewed row-major rows (32 x 32 tiles through registers)
  uint32_t* rows = reinterpret_cast<uint32_t*>(smem_raw);
  for (int T = w; T < BP / 32; T += 8) {
    uint32_t x[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = cnt[(T * 32 + i) * 32 + lane];
#pragma unroll
    for (int i = 0; i < 32; ++i) rows[Lay::at(lane, T * 32 + i)] = x[i];
  }
  __syncthreads();

  if (wk.n_chunks == 1) {
    for (int sl = w; sl < 32; sl += 8) {
      const uint32_t rg = wk.row0 + uint32_t(sl);
      if (rg >= R) break;
      const uint32_t nbr = nb_g[size_t(h) * R + rg];
      RowRes rr{};
      if (nbr > 0) {
        const uint32_t* row = rows;
        rr = hist_row_scan2<Lay::E>(
            [&](int b, int c) {
              const uint32_t x = row[Lay::at(sl, b)];
              return c ? x >> 16 : x & 0xffffu;
            },
            bnd_g + (size_t(h) * R + rg) * (bins - 1), nbr, nd.parent, xl, lane);
      }
      if (lane == 0) rowres[size_t(h) * R + rg] = rr;
    }
    return;
  }
  // multi-chunk: merge into the global counters [ms][R][BP][2]; the last chunk of this
  // (node, row group) scans the totals
  const uint32_t ms = multi_slot[wk.node];
  for (int sl = w; sl < 32; sl += 8) {
    const uint32_t rg = wk.row0 + uint32_t(sl);
    if (rg >= R) break;
    uint32_t* g = gcnt + (size_t(ms) * R + rg) * size_t(BP) * 2;
    for (int b = lane; b < BP; b += 32) {
      const uint32_t x = rows[Lay::at(sl, b)];
      if (x & 0xffffu) atomicAdd(g + 2 * b, x & 0xffffu);
      if (x >> 16) atomicAdd(g + 2 * b + 1, x >> 16);
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(&done[size_t(ms) * ((R + 31) / 32) + wk.row0 / 32], 1u);
    s_last = prev == wk.n_chunks - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  uint32_t* mine = reinterpret_cast<uint32_t*>(smem_raw) + size_t(w) * BP * 2;  // [BP][2] per warp
  for (int sl = w; sl < 32; sl += 8) {
    const uint32_t rg = wk.row0 + uint32_t(sl);
    if (rg >= R) break;
    const uint32_t nbr = nb_g[size_t(h) * R + rg];
    RowRes rr{};
    if (nbr > 0) {
      const uint32_t* g = gcnt + (size_t(ms) * R + rg) * size_t(BP) * 2;
      for (int i = lane; i < int(nbr + 1) * 2; i += 32) mine[i] = __ldcg(g + i);
      __syncwarp();
      rr = hist_row_scan2<Lay::E>([&](int b, int c) { return mine[2 * b + c]; },
                                  bnd_g + (size_t(h) * R + rg) * (bins - 1), nbr, nd.parent, xl, lane);
      __syncwarp();
    }
    if (lane == 0) rowres[size_t(h) * R + rg] = rr;
  }
}

// ------------------------------------------------------------------------------------------
__global__ void k_hist_select(const uint32_t* __restrict__ hist_nodes, int n_hist, uint32_t R,
                              const RowRes* __restrict__ rowres, NodeRes* __restrict__ res) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= n_hist) return;
  int best = -1;
  double g = 0.0;
  float thr = 0.f;
  uint32_t nl = 0;
  for (uint32_t r = 0; r < R; ++r) {
    const RowRes rr = rowres[size_t(h) * R + r];
    if (rr.valid && (best < 0 || rr.gain > g)) {
      best = int(r);
      g = rr.gain;
      thr = rr.threshold;
      nl = rr.n_left;
    }
  }
  NodeRes& o = res[hist_nodes[h]];
  o.row = best;
  o.gain = g;
  o.threshold = thr;
  o.n_left_search = nl;
}

}  // namespace dev

// ---------------------------------------------------------------------------- launchers
static int pow2_at_least(int x, int lo) {
  int p = lo;
  while (p < x) p <<= 1;
  return p;
}

size_t hist_count_smem(uint32_t bins, int k, int chunk_cap) {
  const int bpad = pow2_at_least(int(bins), 32);
  return size_t(8) * bpad * k * 4 + size_t(8) * bpad * 4 + size_t(chunk_cap) + 16;
}

cudaError_t launch_hist_count(const NodeIn* nodes, const uint32_t* node_hist_slot,
                              const HistWork* work, int n_work, const uint32_t* multi_slot,
                              uint32_t R, uint32_t bins, int k, int chunk_cap, int two_level,
                              const uint32_t* terms, const uint32_t* row_ptr, const uint8_t* lab,
                              const uint64_t* gbase, const float* G, const float* bnd,
                              const uint32_t* nb, const double* xl, uint32_t* gcnt,
                              uint32_t* done, RowRes* rowres, cudaStream_t st) {
  if (n_work == 0) return cudaSuccess;
  const int bpad = pow2_at_least(int(bins), 32);
  const size_t smem = hist_count_smem(bins, k, chunk_cap);
  // class-count specialised (k = 2 is the trunk workload; generic up to kMaxClasses)
  auto kern = k == 2 ? (bpad == 256   ? dev::k_hist_count<2, 8>
                        : bpad == 128 ? dev::k_hist_count<2, 7>
                        : bpad == 64  ? dev::k_hist_count<2, 6>
                        : bpad == 32  ? dev::k_hist_count<2, 5>
                                      : dev::k_hist_count<2, 0>)
                     : (bpad == 256 ? dev::k_hist_count<kMaxClasses, 8> : dev::k_hist_count<kMaxClasses, 0>);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptin);
  kern<<<n_work, 256, smem, st>>>(nodes, node_hist_slot, work, multi_slot, R, bins, bpad, k,
                                  chunk_cap, two_level, terms, row_ptr, lab, gbase, G, bnd, nb, xl, gcnt,
                                  done, rowres);
  return cudaGetLastError();
}

bool hist_count_lane_rows(uint32_t R, uint32_t bins, int k) {
  // lane = row needs two classes and <= 256 bins; a row group of 32 is worth it when it is
  // mostly full (measured ~2.2x the lane = sample kernel's throughput per value)
  return k == 2 && bins <= 256 && (R + 31) / 32 * 32 < 2 * R;
}

size_t hist_count_lr_smem(uint32_t bins, int chunk_cap) {
  const int bpad = pow2_at_least(int(bins), 32);
  const int pitch = bpad + 33;
  const int area = bpad * 32 > 32 * pitch ? bpad * 32 : 32 * pitch;
  return size_t(area) * 4 + size_t(bpad) * 32 * 4 + size_t((chunk_cap + 31) / 32) * 4 + 16;
}

cudaError_t launch_hist_count_lr(const NodeIn* nodes, const uint32_t* node_hist_slot, const HistWork* work,
                                 int n_work, const uint32_t* multi_slot, uint32_t R, uint32_t bins, int chunk_cap,
                                 int two_level, const uint8_t* lab, const uint64_t* gbase, const float* G,
                                 const float* bnd, const uint32_t* nb, const double* xl, uint32_t* gcnt,
                                 uint32_t* done, RowRes* rowres, cudaStream_t st) {
  if (n_work == 0) return cudaSuccess;
  const int bpad = pow2_at_least(int(bins), 32);
  const size_t smem = hist_count_lr_smem(bins, chunk_cap);
  auto kern = bpad == 256 ? dev::k_hist_count_lr<8>
              : bpad == 128 ? dev::k_hist_count_lr<7>
              : bpad == 64  ? dev::k_hist_count_lr<6>
                            : dev::k_hist_count_lr<5>;
  if (bpad > 256) return cudaErrorInvalidValue;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptin);
  kern<<<n_work, 256, smem, st>>>(nodes, node_hist_slot, work, multi_slot, R, bins, two_level, lab, gbase, G, bnd,
                                  nb, xl, gcnt, done, rowres);
  return cudaGetLastError();
}

cudaError_t launch_hist_select(const uint32_t* hist_nodes, int n_hist, uint32_t R,
                               const RowRes* rowres, NodeRes* res, cudaStream_t st) {
  if (n_hist == 0) return cudaSuccess;
  dev::k_hist_select<<<(n_hist + 127) / 128, 128, 0, st>>>(hist_nodes, n_hist, R, rowres, res);
  return cudaGetLastError();
}

}  // namespace sofg
