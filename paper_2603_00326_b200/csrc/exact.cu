// Exact splitter, register-resident (reference best_split_exact, split.hpp:142-194, driven per
// row by find_node_split, split.hpp:306-312).
//
// Nodes are bucketed by padded size P = 32*E (E keys per lane, blocked layout: lane l holds
// sorted positions [l*E, (l+1)*E)). Per row a warp
//   1. gathers the node's projected values, G rows at a time so G*E loads are in flight,
//   2. builds keys (order_key(v) << 32 | label) — the reference's packed sort key,
//   3. bitonic-sorts them in registers (intra-lane compare-exchange for strides < E, shuffles
//      for strides >= E),
//   4. scans class counts and evaluates the impurity sum at every gap between distinct values,
//   5. resolves the reference's first-maximum position (see dev_util.cuh: impurity_sum).
// E <= 4: one warp per node (four nodes per CTA). E >= 8: four warps per node, rows split
// round-robin, reduced in shared memory (lowest row wins ties, as split.hpp:259-263).
#include <cuda_runtime.h>

#include <cstdlib>

#include "common.hpp"
#include "dev_util.cuh"
#include "kernels.hpp"

#ifndef SOFG_PRUNE_MINB
#define SOFG_PRUNE_MINB 0  // min CTAs per SM of the prune pass (0: no register cap; 9: 120.6 vs 121.7 ms, within noise)
#endif
#ifndef SOFG_TEAM_MINB
#define SOFG_TEAM_MINB 4  // min CTAs per SM of the team splitters (3: 40.2, 4: 37.1 ms per step at <= 512 samples)
#endif
#ifndef SOFG_REG_MINB
// min CTAs per SM of the register splitters, i.e. their register cap (ptxas' own choice at E = 1, 2,
// 4, 8 -> 34.4 / 54.4 / 20.1 / 43.0 ms per step; 6 CTAs: 31.2 / 47.1 / 10.6 / 31.4; 8: 28.6 / 46.3 / 12.3 / 32.9)
#define SOFG_REG_MINB(E) ((E) <= 2 ? 8 : 6)
#endif
// rows in flight per warp of the register splitters for n <= 32 / 64 / 128 (variant builds)
#ifndef SOFG_TEAM512
#define SOFG_TEAM512 2  // warps per node of the radix splitter for 257..512 samples (4: 56.6 vs 40.2 ms per step)
#endif
static_assert(32 * 8 * SOFG_TEAM512 >= 512, "a team holds 256 W positions: 257..512 samples need W >= 2");
#ifndef SOFG_GR32
#define SOFG_GR32 2  // measured: 8 -> 35.9, 4 -> 34.9, 2 -> 31.2, 1 -> 32.0 ms per step
#endif
#ifndef SOFG_GR64
#define SOFG_GR64 2   // 2 -> 49.1, 4 -> 48.5, 8 -> 56.1; under the 8-CTA register cap: 2 -> 44.7, 4 -> 46.4, 8 -> 47.5
#endif
#ifndef SOFG_GR128
#define SOFG_GR128 1  // 2 -> 18.8, 1 -> 17.3
#endif

namespace sofg {
namespace dev {

template <int E>
__device__ __forceinline__ void reg_bitonic_sort(uint64_t (&key)[E], int lane) {
  reg_bitonic_sort_k<E, uint64_t, (E >= 8)>(key, lane);  // compact stages for E >= 8 (i-cache)
}

struct Best {
  double gain;
  float thr;
  uint32_t nl;
  int row;
  double xmin;   // impurity sum of the best row (monotone proxy for its gain)
  double inv_n;  // 1/n (window bound only; every compared gain uses the exact division)
};

// Search one sorted row (keys in blocked layout). Updates `b` when this row's best gain is
// strictly larger (rows are visited in increasing order by the calling warp).
// Pass 1 evaluates every candidate gap in float; only candidates whose float impurity lies within
// 2 eps of the row's float minimum (a superset of every candidate whose exact gain can equal the
// row's best) are evaluated exactly in double, in the reference's operation order.
// Key policies for scan_row.
// Packed keys: order_key(v) << 32 | label (the reference's sort key, split.hpp:173-176).
struct Key64Ops {
  __device__ int cls(uint64_t k) const { return int(k & 0xffu); }
  __device__ bool gap(uint64_t a, uint64_t b) const {
    return order_key_inv(uint32_t(a >> 32)) < order_key_inv(uint32_t(b >> 32));
  }
  __device__ void values(uint64_t a, uint64_t b, int, float* fa, float* fb) const {
    *fa = order_key_inv(uint32_t(a >> 32));
    *fb = order_key_inv(uint32_t(b >> 32));
  }
};
// Folded 32-bit keys for two classes: (order_key(v) & ~1) | label. Valid only when no two
// samples of the row share the upper 31 key bits and no value is +-0 or +-denorm_min (checked by
// the caller): then sorted order equals value order, every neighbouring pair is a gap between
// distinct values, and the winner's exact values are recovered from the original keys.
template <int E>
struct Key32FoldOps {
  const uint32_t (&orig)[E];  // this lane's unsorted order keys
  __device__ int cls(uint32_t k) const { return int(k & 1u); }
  __device__ bool gap(uint32_t, uint32_t) const { return true; }
  __device__ uint32_t recover(uint32_t folded) const {
    uint32_t hit = 0;
    bool found = false;
#pragma unroll
    for (int e = 0; e < E; ++e)
      if ((orig[e] >> 1) == (folded >> 1)) {
        hit = orig[e];
        found = true;
      }
    const unsigned m = __ballot_sync(0xffffffffu, found);
    return __shfl_sync(0xffffffffu, hit, __ffs(m) - 1);
  }
  __device__ void values(uint32_t a, uint32_t b, int, float* fa, float* fb) const {
    *fa = order_key_inv(recover(a));
    *fb = order_key_inv(recover(b));
  }
};

template <int E, int KC, class K, class Ops>
__device__ __forceinline__ void scan_row(const K (&key)[E], const Ops& ops, uint32_t n, int k,
                                         const uint32_t* tot, double parent,
                                         const double* __restrict__ xl,
                                         const float* __restrict__ xlf, int row, int lane,
                                         Best& b) {
  // per-lane class counts
  uint32_t loc[KC], pre[KC];
#pragma unroll
  for (int c = 0; c < KC; ++c) loc[c] = 0;
  const int p0 = lane * E;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if (uint32_t(p0 + e) < n) {
      const int c = ops.cls(key[e]);
#pragma unroll
      for (int cc = 0; cc < KC; ++cc) loc[cc] += (cc == c);
    }
  }
#pragma unroll
  for (int c = 0; c < KC; ++c) {
    uint32_t t;
    pre[c] = warp_excl_scan_u32(loc[c], lane, &t);
  }
  const K next_first = __shfl_down_sync(0xffffffffu, key[0], 1);
  const double dn = double(n);
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  const float inff = __int_as_float(0x7f800000);

  // pass 1: float impurity per candidate gap (a < b between consecutive sorted values)
  float Xf[E];
  float xminf = inff;
  {
    uint32_t left[KC];
#pragma unroll
    for (int c = 0; c < KC; ++c) left[c] = pre[c];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      Xf[e] = inff;
      const uint32_t p = uint32_t(p0 + e);
      if (p + 1 < n) {
        const int c = ops.cls(key[e]);
#pragma unroll
        for (int cc = 0; cc < KC; ++cc) left[cc] += (cc == c);
        const K kb = (e + 1 < E) ? key[(e + 1) % E] : next_first;
        if (ops.gap(key[e], kb)) {
          if constexpr (KC == 2) {
            uint32_t lf[2] = {(p + 1) - left[1], left[1]};
            Xf[e] = impurity_sum_f<2>(xlf, lf, tot, k, p + 1, n - (p + 1));
          } else {
            Xf[e] = impurity_sum_f<KC>(xlf, left, tot, k, p + 1, n - (p + 1));
          }
          xminf = fminf(xminf, Xf[e]);
        }
      }
    }
  }
  xminf = warp_min_f32(xminf);
  if (!(xminf < inff)) return;
  const double eps = prefilter_eps(__ldg(xl + n), k);
  // the row cannot beat the best row so far (its exact minimum exceeds the best's)
  if (b.row >= 0 && double(xminf) - 2.0 * eps > b.xmin) return;
  const double lim = double(xminf) + 3.0 * eps;  // 2 eps + slack for the equal-gain window
  // pass 2: exact impurity of the prefiltered candidates (the pass is repeated below to find the
  // first position; the exact values are not kept, so wide E costs no extra registers)
  auto exact_pass = [&](auto&& visit) {
    uint32_t left[KC];
#pragma unroll
    for (int c = 0; c < KC; ++c) left[c] = pre[c];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t p = uint32_t(p0 + e);
      if (p + 1 < n) {
        const int c = ops.cls(key[e]);
#pragma unroll
        for (int cc = 0; cc < KC; ++cc) left[cc] += (cc == c);
        if (double(Xf[e]) <= lim) {
          const uint32_t nl = p + 1;
          double X;
          if constexpr (KC == 2) {
            const uint32_t l1 = left[1], l0 = nl - l1;
            const double sl = __dadd_rn(__ldg(xl + l0), __ldg(xl + l1));
            const double sr = __dadd_rn(__ldg(xl + tot[0] - l0), __ldg(xl + tot[1] - l1));
            X = __dsub_rn(__dadd_rn(__dsub_rn(__ldg(xl + nl), sl), __ldg(xl + (n - nl))), sr);
          } else {
            X = impurity_sum<KC>(xl, left, tot, k, nl, n - nl);
          }
          visit(e, X);
        }
      }
    }
  };
  constexpr bool kKeep = E < 8;  // small E: keep the exact values; wide E: recompute (registers)
  double Xd[kKeep ? E : 1];
#pragma unroll
  for (int e = 0; e < (kKeep ? E : 1); ++e) Xd[e] = inf;
  double xmin = inf;
  exact_pass([&](int e, double X) {
    xmin = fmin(xmin, X);
    if constexpr (kKeep) Xd[e] = X;
  });
  xmin = warp_min_f64(xmin);
  // gain = parent - X / n is monotone non-increasing in X: a row whose minimum impurity is not
  // below the best row's cannot have a strictly larger gain (split.hpp:260 keeps earlier rows).
  if (b.row >= 0 && !(xmin < b.xmin)) return;
  const double g = gain_from_x(parent, xmin, dn);
  if (!(g > 0.0)) return;
  if (b.row >= 0 && !(g > b.gain)) return;
  const double win = x_window_fast(parent, xmin, dn, b.inv_n);
  uint32_t first = 0xffffffffu;
  int fe = 0;
  auto take = [&](int e, double X) {
    if (first == 0xffffffffu && X <= win && (X == xmin || gain_from_x(parent, X, dn) == g)) {
      first = uint32_t(p0 + e);
      fe = e;
    }
  };
  if constexpr (kKeep) {
#pragma unroll
    for (int e = 0; e < E; ++e) take(e, Xd[e]);
  } else {
    exact_pass(take);
  }
  const uint32_t fp = warp_min_u32(first);
  const int src = __ffs(__ballot_sync(0xffffffffu, first == fp)) - 1;
  // the two keys around the winning gap (positions fp, fp+1)
  K ka = 0, kb = 0;
#pragma unroll
  for (int e = 0; e < E; ++e)
    if (e == fe) {
      ka = key[e];
      kb = (e + 1 < E) ? key[(e + 1) % E] : next_first;
    }
  ka = __shfl_sync(0xffffffffu, ka, src);
  kb = __shfl_sync(0xffffffffu, kb, src);
  b.xmin = xmin;
  b.row = row;
  b.gain = g;
  float fa, fb;
  ops.values(ka, kb, lane, &fa, &fb);
  b.thr = midpoint_down(fa, fb);
  b.nl = fp + 1;
}

// ------------------------------------------------------------------------------------------
// Row bounds for the exact splitter (branch and bound). For each (node, row): 31 pivots (row
// values at fixed positions, sorted) split the row into 32 value buckets; one pass counts each
// bucket's classes. The split "v < pivot" is a real candidate gap, so its exact impurity X is an
// achievable value: xstar[node] = min over rows of those. Every other gap lies inside one bucket,
// whose left class counts (l0, l1) range over a box; X = sum over children of n_c * H(child) is
// concave in (l0, l1), so its minimum over the box is at a corner. rowlb = min(pivot X, bucket
// corner minima) bounds every candidate of the row from below. A row with rowlb > xstar (+ a
// margin far above rounding) cannot contain the node's best split nor tie it (gain = parent - X/n
// is monotone), and the exact kernels skip sorting it.
// ------------------------------------------------------------------------------------------
// Rows whose bound exceeds the limit are skipped. The reference X is the smaller of xstar (an
// achievable candidate of some row) and the best X found so far by this warp / team (also
// achievable); the margin is far above rounding and above x_window, so a skipped row can neither
// beat nor tie the best.
__device__ __forceinline__ bool pruned(const float* rowlb, size_t at, const unsigned long long* xstar,
                                       uint32_t li, const Best& b) {
  double xs = __longlong_as_double((long long)xstar[li]);
  if (b.row >= 0) xs = fmin(xs, b.xmin);
  return double(rowlb[at]) > xs + fabs(xs) * 0x1p-30 + 0x1p-30;
}

template <int KC>
__device__ __forceinline__ double x_at(const double* __restrict__ xl, uint32_t l0, uint32_t l1,
                                       const uint32_t* tot, int k, uint32_t n) {
  uint32_t left[2] = {l0, l1};
  return impurity_sum<2>(xl, left, tot, k, l0 + l1, n - (l0 + l1));
}


// One warp per (node, group of 8 rows): each sample's 8 projected values of the group are one
// 32-byte sector of V (the sample-major pitch is a multiple of 8), read with two vector loads.
// 4 warps per CTA; per warp the sorted pivots and the bucket class counts of its 8 rows live in
// shared memory.
// kPB value buckets per row (32 or 64), kPBE per lane.
template <int kPB, int KC>
__global__ void __launch_bounds__(128, SOFG_PRUNE_MINB) k_exact_prune(
    const NodeIn* __restrict__ nodes, const uint32_t* __restrict__ list, int n_list, uint32_t R,
    const uint32_t* __restrict__ row_ptr, const uint8_t* __restrict__ lab,
    const uint64_t* __restrict__ gbase, const float* __restrict__ G,
    const double* __restrict__ xl, float* __restrict__ rowlb, unsigned long long* __restrict__ xstar,
    int k) {
  constexpr int GR = 8;
  constexpr int kPBE = kPB / 32;
  __shared__ __align__(16) uint32_t s_cnt[4][GR][kPB][KC];
  // pivot i at word i + i/32: positions i and i+32 fall in different banks (a search step's probes
  // are spread over both halves)
  constexpr int kPP = kPB + kPB / 32;
  __shared__ uint32_t s_piv[4][GR][kPP];
  auto pslot = [](uint32_t i) { return i + (i >> 5); };
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t RG = (R + GR - 1) / GR;
  const uint64_t gw = uint64_t(blockIdx.x) * 4 + uint64_t(w);
  if (gw >= uint64_t(n_list) * RG) return;
  const uint32_t li = uint32_t(gw / RG), r0 = uint32_t(gw % RG) * GR;
  const uint32_t node = list[li];
  const NodeIn nd = nodes[node];
  const uint32_t n = nd.n;
  const uint32_t* rp = row_ptr + size_t(node) * (R + 1);
  const uint32_t Rp = vpitch(R);
  const float* Vn = G + gbase[node] + r0;
  // pivots of each row: the values at positions n*(i+1)/kPB, i < kPB - 1, sorted (last: +inf);
  // lane l holds sorted positions l*kPBE .. l*kPBE + kPBE - 1
  {
    float v[kPBE][GR];
#pragma unroll
    for (int e = 0; e < kPBE; ++e) {
      const uint32_t i = uint32_t(lane * kPBE + e);
      const uint32_t pos = uint32_t((uint64_t(n) * (i + 1)) / kPB);
      const float4* src = reinterpret_cast<const float4*>(Vn + uint64_t(i < kPB - 1 ? pos : 0u) * Rp);
      const float4 a = __ldg(src), b = __ldg(src + 1);
      v[e][0] = a.x; v[e][1] = a.y; v[e][2] = a.z; v[e][3] = a.w;
      v[e][4] = b.x; v[e][5] = b.y; v[e][6] = b.z; v[e][7] = b.w;
    }
#pragma unroll
    for (int g = 0; g < GR; ++g) {
      uint32_t k[kPBE];
#pragma unroll
      for (int e = 0; e < kPBE; ++e)
        k[e] = uint32_t(lane * kPBE + e) < uint32_t(kPB - 1) ? order_key(v[e][g]) : 0xFFFFFFFFu;
      reg_bitonic_sort_k<kPBE, uint32_t>(k, lane);
#pragma unroll
      for (int e = 0; e < kPBE; ++e) {
        s_piv[w][g][pslot(lane * kPBE + e)] = k[e];
#pragma unroll
        for (int cc = 0; cc < KC; ++cc) s_cnt[w][g][lane * kPBE + e][cc] = 0;
      }
    }
  }
  __syncwarp();
  uint32_t mid[GR];  // each row's middle pivot: the search's first step without a load
#pragma unroll
  for (int g = 0; g < GR; ++g) mid[g] = s_piv[w][g][pslot(kPB / 2 - 1)];
  for (uint32_t j = uint32_t(lane); j < n; j += 32) {
    const float4* src = reinterpret_cast<const float4*>(Vn + uint64_t(j) * Rp);
    const float4 a = __ldg(src), b = __ldg(src + 1);
    const float v[GR] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    const uint32_t y = min(uint32_t(__ldg(lab + nd.begin + j)), uint32_t(KC - 1));
    uint32_t lo[GR];
#pragma unroll
    for (int g = 0; g < GR; ++g) lo[g] = mid[g] <= order_key(v[g]) ? uint32_t(kPB / 2) : 0u;
#pragma unroll
    for (uint32_t step = kPB / 4; step > 0; step >>= 1) {
#pragma unroll
      for (int g = 0; g < GR; ++g)
        if (s_piv[w][g][pslot(lo[g] + step - 1)] <= order_key(v[g])) lo[g] += step;
    }
#pragma unroll
    for (int g = 0; g < GR; ++g) atomicAdd(&s_cnt[w][g][lo[g]][y], 1u);
  }
  __syncwarp();
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  double xbest = inf;
  // Row g's lane partial bounds go to the row's own (then dead) bucket counters; one transposed
  // reduction over all rows at the end replaces a warp-wide shuffle reduction per row.
  unsigned scored = 0;
#pragma unroll 1
  for (int g = 0; g < GR; ++g) {
    const uint32_t r = r0 + uint32_t(g);
    if (r >= R) break;
    float* out = rowlb + size_t(li) * R + r;
    if (__ldg(rp + r + 1) == __ldg(rp + r)) {  // empty: skipped by the exact kernels anyway
      if (lane == 0) *out = __int_as_float(0x7f800000);
      continue;
    }
    uint32_t cnt[kPBE][KC], sum[KC];
#pragma unroll
    for (int cc = 0; cc < KC; ++cc) sum[cc] = 0;
#pragma unroll
    for (int e = 0; e < kPBE; ++e)
#pragma unroll
      for (int cc = 0; cc < KC; ++cc) {
        cnt[e][cc] = s_cnt[w][g][lane * kPBE + e][cc];
        sum[cc] += cnt[e][cc];
      }
    uint32_t a[KC], tot[KC];
#pragma unroll
    for (int cc = 0; cc < KC; ++cc) a[cc] = warp_excl_scan_u32(sum[cc], lane, &tot[cc]);
    auto xat = [&](const uint32_t (&left)[KC]) {
      uint32_t nl = 0;
#pragma unroll
      for (int cc = 0; cc < KC; ++cc) nl += left[cc];
      return impurity_sum<KC>(xl, left, tot, k, nl, n - nl);
    };
    // X at every bucket's end point (its left counts after the bucket); the pivot candidates are
    // the valid ones among them. A bucket's candidates lie in the box [a, L] of left counts; X is
    // concave there, so its minimum is at a vertex (start and end are the shared end points; the
    // other vertices only matter when at least two classes are present in the bucket).
    double xe[kPBE];
    double xp = inf, lb = inf;
#pragma unroll
    for (int e = 0; e < kPBE; ++e) {
      const uint32_t bk = uint32_t(lane * kPBE + e);
      uint32_t L[KC], nl = 0, classes = 0;
#pragma unroll
      for (int cc = 0; cc < KC; ++cc) {
        L[cc] = a[cc] + cnt[e][cc];
        nl += L[cc];
        classes += cnt[e][cc] > 0 ? 1u : 0u;
      }
      xe[e] = xat(L);
      // pivot candidate: split after bucket bk ("v < pivot_bk"), a real gap when 0 < nl < n —
      // except at a +0 pivot, where -0 values (a smaller key, the same float) sit on the left
      if (bk < uint32_t(kPB - 1) && nl > 0 && nl < n && s_piv[w][g][pslot(bk)] != 0x80000000u)
        xp = fmin(xp, xe[e]);
      if (classes >= 2) {
#pragma unroll 1
        for (uint32_t m = 1; m + 1 < (1u << KC); ++m) {
          uint32_t v[KC];
#pragma unroll
          for (int cc = 0; cc < KC; ++cc) v[cc] = (m >> cc) & 1u ? L[cc] : a[cc];
          lb = fmin(lb, xat(v));
        }
      }
      lb = fmin(lb, xe[e]);
#pragma unroll
      for (int cc = 0; cc < KC; ++cc) a[cc] = L[cc];
    }
    // start point of this lane's first bucket = end point of the previous lane's last one
    double xs0 = __shfl_up_sync(0xffffffffu, xe[kPBE - 1], 1);
    if (lane == 0) {
      uint32_t z[KC];
#pragma unroll
      for (int cc = 0; cc < KC; ++cc) z[cc] = 0;
      xs0 = xat(z);
    }
    lb = fmin(lb, xs0);
    xbest = fmin(xbest, xp);
    __syncwarp();  // every lane has read row g's counters
    reinterpret_cast<double*>(&s_cnt[w][g][0][0])[lane] = fmin(lb, xp);  // 256 bytes: the whole row (kPB = 32, KC = 2) or part of it
    scored |= 1u << g;
  }
  __syncwarp();
  {  // lanes 4g .. 4g + 3 reduce row g's 32 partials: 8 each, then two shuffle steps
    const int g = lane >> 2, part = lane & 3;
    double m = inf;
    if (g < GR && ((scored >> g) & 1u)) {
      const double* pg = reinterpret_cast<const double*>(&s_cnt[w][g][0][0]) + 8 * part;
#pragma unroll
      for (int i = 0; i < 8; ++i) m = fmin(m, pg[i]);
    }
    m = fmin(m, __shfl_xor_sync(0xffffffffu, m, 1));
    m = fmin(m, __shfl_xor_sync(0xffffffffu, m, 2));
    if (part == 0 && g < GR && ((scored >> g) & 1u))
      rowlb[size_t(li) * R + r0 + uint32_t(g)] = __double2float_rd(m);  // rounded down: a conservative bound
  }
  xbest = warp_min_f64(xbest);
  if (lane == 0 && xbest < inf) atomicMin(xstar + li, (unsigned long long)__double_as_longlong(xbest));
}

// E keys per lane, G rows in flight per warp, WPN warps per node, KC class-count registers.
template <int E, int GR, int WPN, int KC>
__global__ void __launch_bounds__(128, SOFG_REG_MINB(E)) k_exact_reg(
    const NodeIn* __restrict__ nodes, const uint32_t* __restrict__ list, int n_list, uint32_t R,
    int k, const uint32_t* __restrict__ terms, const uint32_t* __restrict__ row_ptr,
    const uint8_t* __restrict__ lab, const uint64_t* __restrict__ gbase,
    const float* __restrict__ G, const double* __restrict__ xl, const float* __restrict__ xlf,
    NodeRes* __restrict__ res, const float* __restrict__ rowlb,
    const unsigned long long* __restrict__ xstar) {
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int li = (WPN == 1) ? int(blockIdx.x) * 4 + w : int(blockIdx.x);
  const int wr = (WPN == 1) ? 0 : w;  // rank of this warp within the node
  __shared__ Best s_best[4];
  if (li >= n_list) return;  // only reachable when WPN == 1 (whole warp exits)
  const uint32_t node = list[li];
  const NodeIn nd = nodes[node];
  const uint32_t n = nd.n;

  const float* Gn = G + gbase[node];
  uint32_t cnt[KC];
#pragma unroll
  for (int c = 0; c < KC; ++c) cnt[c] = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t p = uint32_t(lane * E + e);
    if (p < n) {
      const int yy = lab[nd.begin + p];
#pragma unroll
      for (int c = 0; c < KC; ++c) cnt[c] += (c == yy);
    }
  }
  uint32_t tot[KC];
#pragma unroll
  for (int c = 0; c < KC; ++c) {
    uint32_t x = cnt[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    tot[c] = x;
  }

  const uint32_t* rp = row_ptr + size_t(node) * (R + 1);
  const uint32_t Rp = vpitch(R);
  Best best{0.0, 0.f, 0, -1, 0.0, 1.0 / double(n)};

  for (uint32_t r0 = uint32_t(wr * GR); r0 < R; r0 += uint32_t(WPN * GR)) {
    int nt[GR];
#pragma unroll
    for (int g = 0; g < GR; ++g) {
      const uint32_t r = r0 + uint32_t(g);
      nt[g] = r < R ? int(__ldg(rp + r + 1) - __ldg(rp + r)) : 0;
    }
    // Rows r0..r0+GR-1 of this lane's samples: one aligned vector load each (GR divides the
    // 8-row pitch, so the group never crosses a sample's sector).
    float val[GR][E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t j = uint32_t(lane * E + e);
      const float* src = Gn + uint64_t(j < n ? j : 0u) * Rp + r0;
      if constexpr (GR == 8) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(src));
        const float4 b = __ldg(reinterpret_cast<const float4*>(src) + 1);
        val[0][e] = a.x; val[1][e] = a.y; val[2][e] = a.z; val[3][e] = a.w;
        val[4][e] = b.x; val[5][e] = b.y; val[6][e] = b.z; val[7][e] = b.w;
      } else if constexpr (GR == 4) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(src));
        val[0][e] = a.x; val[1][e] = a.y; val[2][e] = a.z; val[3][e] = a.w;
      } else if constexpr (GR == 2) {
        const float2 a = __ldg(reinterpret_cast<const float2*>(src));
        val[0][e] = a.x; val[1][e] = a.y;
      } else {
#pragma unroll
        for (int g = 0; g < GR; ++g) val[g][e] = __ldg(src + g);
      }
    }
    // One copy of the sort/scan code for all GR rows (instruction-cache footprint): the row's
    // values are picked out of the unrolled registers with selects.
#pragma unroll 1
    for (int g = 0; g < GR; ++g) {
      const uint32_t r = r0 + uint32_t(g);
      int ntg = 0;
#pragma unroll
      for (int gg = 0; gg < GR; ++gg)
        if (gg == g) ntg = nt[gg];
      if (r >= R || ntg == 0) continue;  // empty rows are skipped in exact mode (split.hpp:308)
      if (rowlb && pruned(rowlb, size_t(li) * R + r, xstar, uint32_t(li), best)) continue;  // bound
      if constexpr (KC == 2) {
        // fast path: 32-bit folded keys (half the shuffle/compare work of the packed 64-bit key)
        uint32_t ok[E], k32[E];
        bool special = false;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          float v = 0.f;
#pragma unroll
          for (int gg = 0; gg < GR; ++gg)
            if (gg == g) v = val[gg][e];
          if (uint32_t(lane * E + e) < n) {
            ok[e] = order_key(v);
            const uint32_t top = ok[e] >> 1;
            special |= top == 0x3FFFFFFFu || top == 0x40000000u;  // +-0, +-denorm_min
            k32[e] = (ok[e] & ~1u) | uint32_t(__ldg(lab + nd.begin + lane * E + e));
          } else {
            ok[e] = 0xFFFFFFFFu;
            k32[e] = 0xFFFFFFFFu;
          }
        }
        if (!__any_sync(0xffffffffu, special)) {
          reg_bitonic_sort_k<E, uint32_t, (E >= 8)>(k32, lane);
          // collision: neighbours (among the n real samples) with equal upper 31 bits
          bool coll = false;
          const uint32_t nf = __shfl_down_sync(0xffffffffu, k32[0], 1);
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const uint32_t p = uint32_t(lane * E + e);
            const uint32_t nx = (e + 1 < E) ? k32[(e + 1) % E] : nf;
            coll |= p + 1 < n && (k32[e] >> 1) == (nx >> 1);
          }
          if (!__any_sync(0xffffffffu, coll)) {
            scan_row<E, 2>(k32, Key32FoldOps<E>{ok}, n, k, tot, nd.parent, xl, xlf, int(r), lane, best);
            continue;
          }
        }
      }
      uint64_t key[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        float v = 0.f;
#pragma unroll
        for (int gg = 0; gg < GR; ++gg)
          if (gg == g) v = val[gg][e];
        if (uint32_t(lane * E + e) < n) {
          key[e] = (uint64_t(order_key(v)) << 32) | uint64_t(__ldg(lab + nd.begin + lane * E + e));
        } else {
          key[e] = ~0ull;
        }
      }
      reg_bitonic_sort<E>(key, lane);
      scan_row<E, KC>(key, Key64Ops{}, n, k, tot, nd.parent, xl, xlf, int(r), lane, best);
    }
  }

  if (WPN == 1) {
    if (lane == 0) {
      NodeRes& o = res[node];
      o.row = best.row;
      o.gain = best.gain;
      o.threshold = best.thr;
      o.n_left_search = best.nl;
    }
    return;
  }
  if (lane == 0) s_best[w] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    Best bb{0.0, 0.f, 0, -1, 0.0, 0.0};
    for (int i = 0; i < WPN; ++i) {
      const Best& c = s_best[i];
      if (c.row < 0) continue;
      if (bb.row < 0 || c.gain > bb.gain || (c.gain == bb.gain && c.row < bb.row)) bb = c;
    }
    NodeRes& o = res[node];
    o.row = bb.row;
    o.gain = bb.gain;
    o.threshold = bb.thr;
    o.n_left_search = bb.nl;
  }
}

// ------------------------------------------------------------------------------------------
// Segmented variant for nodes of <= S samples (S = 8, 16): the warp splits into 32/S segments of
// S lanes, each segment searches its own row (lane = sorted position), so one pass covers 32/S
// rows. Keys are the packed 64-bit sort keys; every candidate is evaluated exactly (one per
// lane). Each segment keeps its rows' best (rows in increasing order, strict '>'), and the
// segments' bests are reduced with the reference's rule (higher gain, then lower row).
// ------------------------------------------------------------------------------------------
template <int S, int KC>
__global__ void __launch_bounds__(128) k_exact_seg(
    const NodeIn* __restrict__ nodes, const uint32_t* __restrict__ list, int n_list, uint32_t R,
    int k, const uint32_t* __restrict__ row_ptr, const uint8_t* __restrict__ lab,
    const uint64_t* __restrict__ gbase, const float* __restrict__ G,
    const double* __restrict__ xl, NodeRes* __restrict__ res) {
  constexpr int NSEG = 32 / S;
  const int lane = threadIdx.x & 31;
  const int li = int(blockIdx.x) * 4 + (threadIdx.x >> 5);
  if (li >= n_list) return;  // whole warp
  const int sl = lane & (S - 1), seg = lane / S;
  const uint32_t node = list[li];
  const NodeIn nd = nodes[node];
  const uint32_t n = nd.n;
  const int y = uint32_t(sl) < n ? int(__ldg(lab + nd.begin + sl)) : -1;
  uint32_t tot[KC];
#pragma unroll
  for (int c = 0; c < KC; ++c) {
    uint32_t x = y == c ? 1u : 0u;
#pragma unroll
    for (int o = 1; o < S; o <<= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    tot[c] = x;
  }
  const uint32_t* rp = row_ptr + size_t(node) * (R + 1);
  const uint32_t Rp = vpitch(R);
  const float* Gn = G + gbase[node];
  const double dn = double(n);
  const double inv_n = 1.0 / dn;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  Best best{0.0, 0.f, 0, -1, 0.0, inv_n};
  for (uint32_t r0 = 0; r0 < R; r0 += NSEG) {
    const uint32_t r = r0 + uint32_t(seg);
    const bool act = r < R && __ldg(rp + r + 1) != __ldg(rp + r);  // split.hpp:308
    uint64_t key = ~0ull;
    if (act && uint32_t(sl) < n)
      key = (uint64_t(order_key(__ldg(Gn + uint64_t(sl) * Rp + r))) << 32) | uint64_t(uint32_t(y));
    // bitonic sort within the segment, ascending by sl
#pragma unroll
    for (int kk = 2; kk <= S; kk <<= 1) {
#pragma unroll
      for (int j = kk >> 1; j > 0; j >>= 1) {
        const uint64_t o = __shfl_xor_sync(0xffffffffu, key, j);
        const bool up = (sl & kk) == 0;
        const bool lower = (sl & j) == 0;
        const uint64_t mn = o < key ? o : key, mx = o < key ? key : o;
        key = (lower == up) ? mn : mx;
      }
    }
    // class counts of positions <= sl
    const int c = int(key & 0xffu);
    uint32_t left[KC];
#pragma unroll
    for (int cc = 0; cc < KC; ++cc) {
      uint32_t x = (uint32_t(sl) < n && c == cc) ? 1u : 0u;
#pragma unroll
      for (int o = 1; o < S; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, x, o, S);
        if (sl >= o) x += t;
      }
      left[cc] = x;
    }
    const uint64_t nxt = __shfl_down_sync(0xffffffffu, key, 1, S);
    const uint32_t p = uint32_t(sl);
    const bool cand = act && p + 1 < n &&
                      order_key_inv(uint32_t(key >> 32)) < order_key_inv(uint32_t(nxt >> 32));
    double X = inf;
    if (cand) X = impurity_sum<KC>(xl, left, tot, k, p + 1, n - (p + 1));
    double xmin = X;
#pragma unroll
    for (int o = 1; o < S; o <<= 1) xmin = fmin(xmin, __shfl_xor_sync(0xffffffffu, xmin, o));
    const double g = gain_from_x(nd.parent, xmin, dn);
    const bool upd = xmin < inf && !(best.row >= 0 && !(xmin < best.xmin)) && g > 0.0 &&
                     !(best.row >= 0 && !(g > best.gain));
    const double win = x_window_fast(nd.parent, xmin, dn, inv_n);
    uint32_t first = (cand && X <= win && (X == xmin || gain_from_x(nd.parent, X, dn) == g)) ? p : 0xffffffffu;
#pragma unroll
    for (int o = 1; o < S; o <<= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    const uint32_t fp = upd ? first : 0u;
    const int src = seg * S + int(min(fp, uint32_t(S - 2)));
    const uint64_t ka = __shfl_sync(0xffffffffu, key, src);
    const uint64_t kb = __shfl_sync(0xffffffffu, key, src + 1);
    if (upd) {
      best.xmin = xmin;
      best.row = int(r);
      best.gain = g;
      best.thr = midpoint_down(order_key_inv(uint32_t(ka >> 32)), order_key_inv(uint32_t(kb >> 32)));
      best.nl = fp + 1;
    }
  }
  // segments' bests -> lane 0 (higher gain, then lower row)
#pragma unroll
  for (int o = S; o < 32; o <<= 1) {
    const int orow = __shfl_xor_sync(0xffffffffu, best.row, o);
    const double og = __shfl_xor_sync(0xffffffffu, best.gain, o);
    const float ot = __shfl_xor_sync(0xffffffffu, best.thr, o);
    const uint32_t onl = __shfl_xor_sync(0xffffffffu, best.nl, o);
    if (orow >= 0 && (best.row < 0 || og > best.gain || (og == best.gain && orow < best.row))) {
      best.row = orow;
      best.gain = og;
      best.thr = ot;
      best.nl = onl;
    }
  }
  if (lane == 0) {
    NodeRes& out = res[node];
    out.row = best.row;
    out.gain = best.gain;
    out.threshold = best.thr;
    out.n_left_search = best.nl;
  }
}

// ------------------------------------------------------------------------------------------
// Team variant for nodes of 257..2048 samples: a team of W warps (E = 8 keys per lane) sorts one
// row together. Strides < 8 are intra-lane, < 256 shuffles, >= 256 go through shared memory
// between the team's warps (named barrier per team). CTA = 8 warps = 8/W teams; teams take rows
// round-robin, the CTA reduces the teams' bests (lowest row wins ties).
// ------------------------------------------------------------------------------------------
template <int W>
__device__ __forceinline__ void team_sync(int team) {
  if constexpr (W == 1) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(W * 32) : "memory");
  }
}

template <int W, int KC>
__global__ void __launch_bounds__(256, SOFG_TEAM_MINB) k_exact_team(
    const NodeIn* __restrict__ nodes, const uint32_t* __restrict__ list, int n_list, uint32_t R,
    int k, const uint32_t* __restrict__ terms, const uint32_t* __restrict__ row_ptr,
    const uint8_t* __restrict__ lab, const uint64_t* __restrict__ gbase,
    const float* __restrict__ G, const double* __restrict__ xl, const float* __restrict__ xlf,
    NodeRes* __restrict__ res, const float* __restrict__ rowlb,
    const unsigned long long* __restrict__ xstar) {
  constexpr int E = 8;
  constexpr int TEAMS = 8 / W;
  constexpr int P = 32 * E * W;  // positions per team
  // per team: ping-pong key/label arrays for the radix passes + per-warp digit histograms
  __shared__ uint32_t s_key[2][8 * 256];
  __shared__ uint8_t s_lab[2][8 * 256];
  __shared__ uint32_t s_hist[8][256];
  __shared__ uint32_t s_cnt[8][KC];
  __shared__ uint64_t s_first[8];
  __shared__ double s_xmin[8];
  __shared__ float s_xminf[8];
  __shared__ uint32_t s_pos[8];
  __shared__ uint32_t s_scan[8];
  __shared__ Best s_best[TEAMS];
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const int team = w / W;
  const int wt = w % W;
  const int tt = wt * 32 + lane;  // thread index inside the team
  uint32_t* keyA = s_key[0] + team * P;
  uint32_t* keyB = s_key[1] + team * P;
  uint8_t* labA = s_lab[0] + team * P;
  uint8_t* labB = s_lab[1] + team * P;
  const uint32_t node = list[blockIdx.x];
  const NodeIn nd = nodes[node];
  const uint32_t n = nd.n;
  const float* Gn = G + gbase[node];
  const int p0 = tt * E;  // blocked layout used by the scan phase
  const unsigned lt_mask = (1u << lane) - 1u;

  // node class totals (every team holds the full node)
  uint32_t cnt[KC];
#pragma unroll
  for (int c = 0; c < KC; ++c) cnt[c] = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const uint32_t p = uint32_t(p0 + e);
    if (p < n) {
      const int yy = lab[nd.begin + p];
#pragma unroll
      for (int c = 0; c < KC; ++c) cnt[c] += (c == yy);
    }
  }
#pragma unroll
  for (int c = 0; c < KC; ++c) {
    uint32_t x = cnt[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) s_cnt[w][c] = x;
  }
  __syncthreads();
  uint32_t tot[KC];
#pragma unroll
  for (int c = 0; c < KC; ++c) {
    uint32_t x = 0;
    for (int i = 0; i < W; ++i) x += s_cnt[team * W + i][c];
    tot[c] = x;
  }
  __syncthreads();

  const uint32_t* rp = row_ptr + size_t(node) * (R + 1);
  const uint32_t Rp = vpitch(R);
  Best best{0.0, 0.f, 0, -1, 0.0, 1.0 / double(n)};
  const double dn = double(n);
  const double inf = __longlong_as_double(0x7ff0000000000000ll);

  for (uint32_t r = uint32_t(team); r < R; r += uint32_t(TEAMS)) {
    const uint32_t tb = rp[r];
    const int nt = int(rp[r + 1] - tb);
    if (nt == 0) continue;  // uniform per team; split.hpp:308
    if (rowlb && pruned(rowlb, size_t(blockIdx.x) * R + r, xstar, blockIdx.x, best)) continue;
    // ---- projected values of row r (V block, sample-major) -> radix layout
    //      position q = wt*256 + e*32 + lane (warp-blocked, round-striped)
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const uint32_t q = uint32_t(wt * 256 + e * 32 + lane);
      keyA[q] = q < n ? order_key(__ldg(Gn + uint64_t(q) * Rp + r)) : 0xffffffffu;
      labA[q] = q < n ? __ldg(lab + nd.begin + q) : uint8_t(0);
    }
    team_sync<W>(team);
    // ---- LSD radix sort, 8-bit digits, stable (match.any ranking per 32-key round)
#pragma unroll 1
    for (int pass = 0; pass < 4; ++pass) {
      const int shift = pass * 8;
      uint32_t* src_k = (pass & 1) ? keyB : keyA;
      uint8_t* src_l = (pass & 1) ? labB : labA;
      uint32_t* dst_k = (pass & 1) ? keyA : keyB;
      uint8_t* dst_l = (pass & 1) ? labA : labB;
      uint32_t* hist = s_hist[w];
#pragma unroll
      for (int i = 0; i < 8; ++i) hist[i * 32 + lane] = 0;
      __syncwarp();
      uint32_t kk[E], rk[E];
      uint8_t ll[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int q = wt * 256 + e * 32 + lane;
        kk[e] = src_k[q];
        ll[e] = src_l[q];
        const uint32_t dg = (kk[e] >> shift) & 0xffu;
        const unsigned m = __match_any_sync(0xffffffffu, dg);
        const uint32_t before = hist[dg];
        rk[e] = before + __popc(m & lt_mask);
        __syncwarp();
        if ((m & lt_mask) == 0) hist[dg] = before + __popc(m);
        __syncwarp();
      }
      team_sync<W>(team);
      // exclusive scan over (digit, warp) in digit-major order: 256*W counters, 8 per thread
      {
        uint32_t v[8], sum = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int idx = tt * 8 + i;  // digit-major index
          v[i] = s_hist[team * W + (idx % W)][idx / W];
          sum += v[i];
        }
        uint32_t wtot;
        uint32_t ex = warp_excl_scan_u32(sum, lane, &wtot);
        if constexpr (W > 1) {
          if (lane == 0) s_scan[w] = wtot;
          team_sync<W>(team);
          for (int i = 0; i < wt; ++i) ex += s_scan[team * W + i];
        }
        team_sync<W>(team);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int idx = tt * 8 + i;
          s_hist[team * W + (idx % W)][idx / W] = ex;
          ex += v[i];
        }
      }
      team_sync<W>(team);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint32_t dg = (kk[e] >> shift) & 0xffu;
        const uint32_t pos = s_hist[w][dg] + rk[e];
        dst_k[pos] = kk[e];
        dst_l[pos] = ll[e];
      }
      team_sync<W>(team);
    }
    // sorted keys back in keyA/labA; blocked layout for the scan
    uint64_t key[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int q = p0 + e;
      key[e] = (uint64_t(keyA[q]) << 32) | uint64_t(labA[q]);
    }
    // ---- class prefix across the team
    uint32_t loc[KC], pre[KC];
#pragma unroll
    for (int c = 0; c < KC; ++c) loc[c] = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (uint32_t(p0 + e) < n) {
        const int c = int(key[e] & 0xffu);
#pragma unroll
        for (int cc = 0; cc < KC; ++cc) loc[cc] += (cc == c);
      }
    }
#pragma unroll
    for (int c = 0; c < KC; ++c) {
      uint32_t wtot;
      pre[c] = warp_excl_scan_u32(loc[c], lane, &wtot);
      if (lane == 0) s_cnt[w][c] = wtot;
    }
    if (lane == 0) s_first[w] = key[0];
    team_sync<W>(team);
#pragma unroll
    for (int c = 0; c < KC; ++c)
      for (int i = 0; i < wt; ++i) pre[c] += s_cnt[team * W + i][c];
    uint64_t next_first = __shfl_down_sync(0xffffffffu, key[0], 1);
    if (lane == 31) next_first = (wt + 1 < W) ? s_first[w + 1] : ~0ull;
    team_sync<W>(team);

    // pass 1 (float prefilter, see scan_row), team-wide minimum
    float Xf[E];
    float xminf = __int_as_float(0x7f800000);
    {
      uint32_t left[KC];
#pragma unroll
      for (int c = 0; c < KC; ++c) left[c] = pre[c];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        Xf[e] = __int_as_float(0x7f800000);
        const uint32_t p = uint32_t(p0 + e);
        if (p + 1 < n) {
          const int c = int(key[e] & 0xffu);
#pragma unroll
          for (int cc = 0; cc < KC; ++cc) left[cc] += (cc == c);
          const uint64_t kb = (e + 1 < E) ? key[(e + 1) % E] : next_first;
          if (order_key_inv(uint32_t(key[e] >> 32)) < order_key_inv(uint32_t(kb >> 32))) {
            if constexpr (KC == 2) {
              uint32_t lf[2] = {(p + 1) - left[1], left[1]};
              Xf[e] = impurity_sum_f<2>(xlf, lf, tot, k, p + 1, n - (p + 1));
            } else {
              Xf[e] = impurity_sum_f<KC>(xlf, left, tot, k, p + 1, n - (p + 1));
            }
            xminf = fminf(xminf, Xf[e]);
          }
        }
      }
    }
    xminf = warp_min_f32(xminf);
    if (lane == 0) s_xminf[w] = xminf;
    team_sync<W>(team);
    for (int i = 0; i < W; ++i) xminf = fminf(xminf, s_xminf[team * W + i]);
    const double eps = prefilter_eps(__ldg(xl + n), k);
    const bool row_live = xminf < __int_as_float(0x7f800000) &&
                          !(best.row >= 0 && double(xminf) - 2.0 * eps > best.xmin);
    const double lim = double(xminf) + 3.0 * eps;
    // pass 2: exact impurity of the prefiltered candidates
    double Xs[E];
    double xmin = inf;
    if (row_live) {  // uniform across the team
      uint32_t left[KC];
#pragma unroll
      for (int c = 0; c < KC; ++c) left[c] = pre[c];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        Xs[e] = inf;
        const uint32_t p = uint32_t(p0 + e);
        if (p + 1 < n) {
          const int c = int(key[e] & 0xffu);
#pragma unroll
          for (int cc = 0; cc < KC; ++cc) left[cc] += (cc == c);
          if (double(Xf[e]) <= lim) {
            const uint32_t nl = p + 1;
            if constexpr (KC == 2) {
              const uint32_t l1 = left[1], l0 = nl - l1;
              const double sl = __dadd_rn(__ldg(xl + l0), __ldg(xl + l1));
              const double sr = __dadd_rn(__ldg(xl + tot[0] - l0), __ldg(xl + tot[1] - l1));
              Xs[e] = __dsub_rn(__dadd_rn(__dsub_rn(__ldg(xl + nl), sl), __ldg(xl + (n - nl))), sr);
            } else {
              Xs[e] = impurity_sum<KC>(xl, left, tot, k, nl, n - nl);
            }
            xmin = fmin(xmin, Xs[e]);
          }
        }
      }
    }
    xmin = warp_min_f64(xmin);
    team_sync<W>(team);  // s_xminf reads done
    if (lane == 0) s_xmin[w] = xmin;
    team_sync<W>(team);
    for (int i = 0; i < W; ++i) xmin = fmin(xmin, s_xmin[team * W + i]);
    team_sync<W>(team);
    if (!(xmin < inf)) continue;
    if (best.row >= 0 && !(xmin < best.xmin)) continue;  // cannot beat an earlier row
    const double g = gain_from_x(nd.parent, xmin, dn);
    if (!(g > 0.0)) continue;
    if (best.row >= 0 && !(g > best.gain)) continue;
    const double win = x_window_fast(nd.parent, xmin, dn, best.inv_n);
    uint32_t first = 0xffffffffu;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const double X = Xs[e];
      if (first == 0xffffffffu && X <= win &&
          (X == xmin || gain_from_x(nd.parent, X, dn) == g))
        first = uint32_t(p0 + e);
    }
    first = warp_min_u32(first);
    if (lane == 0) s_pos[w] = first;
    team_sync<W>(team);
    uint32_t fp = first;
    for (int i = 0; i < W; ++i) fp = min(fp, s_pos[team * W + i]);
    // the two keys around the winning gap: sorted positions fp, fp+1 (still in keyA)
    const float a = order_key_inv(keyA[fp]);
    const float b = order_key_inv(keyA[fp + 1]);
    team_sync<W>(team);
    best.row = int(r);
    best.gain = g;
    best.xmin = xmin;
    best.thr = midpoint_down(a, b);
    best.nl = fp + 1;
  }
  if (wt == 0 && lane == 0) s_best[team] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    Best bb{0.0, 0.f, 0, -1, 0.0, 0.0};
    for (int i = 0; i < TEAMS; ++i) {
      const Best& c = s_best[i];
      if (c.row < 0) continue;
      if (bb.row < 0 || c.gain > bb.gain || (c.gain == bb.gain && c.row < bb.row)) bb = c;
    }
    NodeRes& o = res[node];
    o.row = bb.row;
    o.gain = bb.gain;
    o.threshold = bb.thr;
    o.n_left_search = bb.nl;
  }
}

template <int W, int KC>
cudaError_t launch_team(const NodeIn* nodes, const uint32_t* list, int n, uint32_t R, int k,
                        const uint32_t* terms, const uint32_t* row_ptr, const uint8_t* lab,
                        const uint64_t* gbase, const float* G, const double* xl, const float* xlf,
                        NodeRes* res, const float* rowlb, const unsigned long long* xstar,
                        cudaStream_t st) {
  k_exact_team<W, KC><<<n, 256, 0, st>>>(nodes, list, n, R, k, terms, row_ptr, lab, gbase, G, xl,
                                         xlf, res, rowlb, xstar);
  return cudaGetLastError();
}

template <int E, int GR, int WPN, int KC>
cudaError_t launch_bucket(const NodeIn* nodes, const uint32_t* list, int n, uint32_t R, int k,
                          const uint32_t* terms, const uint32_t* row_ptr, const uint8_t* lab,
                          const uint64_t* gbase, const float* G, const double* xl, const float* xlf,
                          NodeRes* res, const float* rowlb, const unsigned long long* xstar,
                          cudaStream_t st) {
  const int grid = WPN == 1 ? (n + 3) / 4 : n;
  k_exact_reg<E, GR, WPN, KC><<<grid, 128, 0, st>>>(nodes, list, n, R, k, terms, row_ptr, lab,
                                                     gbase, G, xl, xlf, res, rowlb, xstar);
  return cudaGetLastError();
}

template <int S, int KC>
cudaError_t launch_seg(const NodeIn* nodes, const uint32_t* list, int n, uint32_t R, int k,
                       const uint32_t* row_ptr, const uint8_t* lab, const uint64_t* gbase,
                       const float* G, const double* xl, NodeRes* res, cudaStream_t st) {
  k_exact_seg<S, KC><<<(n + 3) / 4, 128, 0, st>>>(nodes, list, n, R, k, row_ptr, lab, gbase, G, xl, res);
  return cudaGetLastError();
}

template <int KC>
cudaError_t launch_bucket_kc(int bucket, const NodeIn* nodes, const uint32_t* list, int n,
                             uint32_t R, int k, const uint32_t* terms, const uint32_t* row_ptr,
                             const uint8_t* lab, const uint64_t* gbase, const float* G,
                             const double* xl, const float* xlf, NodeRes* res, const float* rowlb,
                             const unsigned long long* xstar, cudaStream_t st) {
  switch (bucket - 2) {
    case -2: return launch_seg<8, KC>(nodes, list, n, R, k, row_ptr, lab, gbase, G, xl, res, st);
    case -1: return launch_seg<16, KC>(nodes, list, n, R, k, row_ptr, lab, gbase, G, xl, res, st);
    case 0: return launch_bucket<1, SOFG_GR32, 1, KC>(nodes, list, n, R, k, terms, row_ptr, lab, gbase, G, xl, xlf, res, rowlb, xstar, st);
    case 1: return launch_bucket<2, SOFG_GR64, 1, KC>(nodes, list, n, R, k, terms, row_ptr, lab, gbase, G, xl, xlf, res, rowlb, xstar, st);
    case 2: return launch_bucket<4, SOFG_GR128, 1, KC>(nodes, list, n, R, k, terms, row_ptr, lab, gbase, G, xl, xlf, res, rowlb, xstar, st);
    case 3: return launch_bucket<8, 1, 1, KC>(nodes, list, n, R, k, terms, row_ptr, lab, gbase, G, xl, xlf, res, rowlb, xstar, st);
    case 4: return launch_team<SOFG_TEAM512, KC>(nodes, list, n, R, k, terms, row_ptr, lab, gbase, G, xl, xlf, res, rowlb, xstar, st);  // (a register E = 16 sort measured slower)
    case 5: return launch_team<4, KC>(nodes, list, n, R, k, terms, row_ptr, lab, gbase, G, xl, xlf, res, rowlb, xstar, st);
    case 6: return launch_team<8, KC>(nodes, list, n, R, k, terms, row_ptr, lab, gbase, G, xl, xlf, res, rowlb, xstar, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace dev

cudaError_t launch_exact_prune(const NodeIn* nodes, const uint32_t* list, int n_list, uint32_t R,
                               const uint32_t* row_ptr, const uint8_t* lab, const uint64_t* gbase,
                               const float* G, const double* xl, float* rowlb,
                               unsigned long long* xstar, int buckets, int k, cudaStream_t st) {
  if (n_list == 0) return cudaSuccess;
  if (k < 2 || k > 4) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(xstar, 0x7f, sizeof(unsigned long long) * n_list, st);  // ~ +huge
  if (e != cudaSuccess) return e;
  const uint64_t warps = uint64_t(n_list) * ((R + 7) / 8);
  const unsigned grid = unsigned((warps + 3) / 4);
  if (k == 2) {
    if (buckets == 32)
      dev::k_exact_prune<32, 2><<<grid, 128, 0, st>>>(nodes, list, n_list, R, row_ptr, lab, gbase, G, xl, rowlb, xstar, k);
    else
      dev::k_exact_prune<64, 2><<<grid, 128, 0, st>>>(nodes, list, n_list, R, row_ptr, lab, gbase, G, xl, rowlb, xstar, k);
  } else {  // 3 or 4 classes
    if (buckets == 32)
      dev::k_exact_prune<32, 4><<<grid, 128, 0, st>>>(nodes, list, n_list, R, row_ptr, lab, gbase, G, xl, rowlb, xstar, k);
    else
      dev::k_exact_prune<64, 4><<<grid, 128, 0, st>>>(nodes, list, n_list, R, row_ptr, lab, gbase, G, xl, rowlb, xstar, k);
  }
  return cudaGetLastError();
}

int exact_bucket(uint32_t n) {
  int b = 0;
  uint32_t cap = 8;
  while (cap < n) {
    cap <<= 1;
    ++b;
  }
  return b;  // 0..8 for n <= 2048: 8, 16 (segmented), 32 .. 2048
}

cudaError_t launch_exact_bucket(int bucket, const NodeIn* nodes, const uint32_t* list, int n,
                                uint32_t R, int k, const uint32_t* terms,
                                const uint32_t* row_ptr, const uint8_t* lab, const uint64_t* gbase,
                                const float* G, const double* xl, const float* xlf, NodeRes* res,
                                const float* rowlb, const unsigned long long* xstar,
                                cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  if (k == 2)
    return dev::launch_bucket_kc<2>(bucket, nodes, list, n, R, k, terms, row_ptr, lab, gbase, G,
                                    xl, xlf, res, rowlb, xstar, st);
  return dev::launch_bucket_kc<kMaxClasses>(bucket, nodes, list, n, R, k, terms, row_ptr, lab,
                                            gbase, G, xl, xlf, res, rowlb, xstar, st);
}

}  // namespace sofg
