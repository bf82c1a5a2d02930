// Shared pieces of the wide-class splitters (wide.cu, exact_big.cu): more than kMaxClasses
// classes, class counts in shared memory, 32 candidates per warp step (see wide.cu).
#pragma once
#include <cuda_runtime.h>

#include "common.hpp"
#include "dev_util.cuh"

namespace sofg {
namespace dev {

constexpr int kWideThreads = 256;

__device__ __forceinline__ uint32_t lanemask_le(int lane) { return 0xffffffffu >> (31 - lane); }

// Impurity sums of 32 candidates of one warp, candidate of lane = position p (left = sorted
// positions [0, p]); lab = its label (valid only when `in`), base[c] = class-c count before this
// chunk, tot[c] = class totals. Advances base by the chunk. Returns X (valid when the lane's
// candidate is) in the reference's order: ((f(nl) - sum_c f(l_c)) + f(nr)) - sum_c f(r_c).
__device__ __forceinline__ double wide_chunk_x(bool in, int lab, uint32_t nl, uint32_t n, int k,
                                               uint32_t* base, const uint32_t* tot,
                                               const double* __restrict__ xl, int lane) {
  double sl = 0.0, sr = 0.0;
  const uint32_t le = lanemask_le(lane);
  for (int c = 0; c < k; ++c) {
    const uint32_t m = __ballot_sync(0xffffffffu, in && lab == c);
    const uint32_t b = base[c];
    const uint32_t l = b + __popc(m & le);
    sl = __dadd_rn(sl, __ldg(xl + l));
    sr = __dadd_rn(sr, __ldg(xl + (tot[c] - l)));
    __syncwarp();
    if (lane == 0) base[c] = b + __popc(m);
    __syncwarp();
  }
  if (!in || nl >= n) return __longlong_as_double(0x7ff0000000000000ll);  // no candidate (+inf)
  const uint32_t nr = n - nl;
  return __dsub_rn(__dadd_rn(__dsub_rn(__ldg(xl + nl), sl), __ldg(xl + nr)), sr);
}

// ------------------------------------------------------------------------------------------
// Exact scan of one sorted row by a whole CTA (8 warps, warp w takes positions [n w / 8,
// n (w + 1) / 8)). key_at(p) = the packed key at sorted position p. s_base: [8][k], s_tot: [k],
// s_x: n doubles or nullptr (recompute in the second pass).
template <class KeyAt>
__device__ RowRes wide_exact_scan(const KeyAt& key_at, uint32_t n, int k, double parent,
                                  const double* __restrict__ xl, uint32_t* s_base, uint32_t* s_run,
                                  uint32_t* s_tot, double* s_x, double* s_red, uint32_t* s_ured) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int NW = kWideThreads / 32;
  const uint32_t p0 = uint32_t(uint64_t(n) * w / NW), p1 = uint32_t(uint64_t(n) * (w + 1) / NW);
  for (int i = threadIdx.x; i < NW * k; i += kWideThreads) s_base[i] = 0;
  __syncthreads();
  for (uint32_t p = p0 + lane; p < p1; p += 32) atomicAdd(&s_base[w * k + int(key_at(p) & 0xffu)], 1u);
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += kWideThreads) {  // per-warp exclusive prefix, totals
    uint32_t run = 0;
    for (int ww = 0; ww < NW; ++ww) {
      const uint32_t x = s_base[ww * k + c];
      s_base[ww * k + c] = run;
      run += x;
    }
    s_tot[c] = run;
  }
  __syncthreads();
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  const double dn = double(n);
  // every candidate gap of this warp's range, in order; the first pass computes (and keeps, when
  // s_x is given) the impurity sums, the second reads them back or recomputes them
  auto pass = [&](bool first_pass, auto&& visit) {
    uint32_t* run = s_run + w * k;
    for (int c = lane; c < k; c += 32) run[c] = s_base[w * k + c];
    __syncwarp();
    for (uint32_t q = p0; q < p1; q += 32) {
      const uint32_t p = q + uint32_t(lane);
      const bool in = p < p1;
      uint64_t ka = 0, kb = 0;
      if (in) {
        ka = key_at(p);
        if (p + 1 < n) kb = key_at(p + 1);
      }
      const bool cand = in && p + 1 < n && order_key_inv(uint32_t(ka >> 32)) < order_key_inv(uint32_t(kb >> 32));
      double X;
      if (s_x && !first_pass) {
        X = cand ? s_x[p] : inf;
      } else {
        X = wide_chunk_x(in, int(ka & 0xffu), p + 1, n, k, run, s_tot, xl, lane);
        if (s_x && in) s_x[p] = cand ? X : inf;
      }
      if (cand) visit(p, X);
    }
  };
  double xmin = inf;  // pass 1: minimum impurity
  pass(true, [&](uint32_t, double X) { xmin = fmin(xmin, X); });
  xmin = warp_min_f64(xmin);
  if (lane == 0) s_red[w] = xmin;
  __syncthreads();
  xmin = s_red[0];
  for (int i = 1; i < NW; ++i) xmin = fmin(xmin, s_red[i]);
  RowRes res{};
  if (!(xmin < inf)) return res;
  const double g = gain_from_x(parent, xmin, dn);
  if (!(g > 0.0)) return res;
  const double win = x_window(parent, xmin, dn);
  uint32_t first = 0xffffffffu;  // pass 2: first position whose gain equals the best
  pass(false, [&](uint32_t p, double X) {
    if (first == 0xffffffffu && X <= win && gain_from_x(parent, X, dn) == g) first = p;
  });
  first = warp_min_u32(first);
  __syncthreads();  // s_red reuse
  if (lane == 0) s_ured[w] = first;
  __syncthreads();
  uint32_t fp = s_ured[0];
  for (int i = 1; i < NW; ++i) fp = min(fp, s_ured[i]);
  const uint64_t ka = key_at(fp), kb = key_at(fp + 1);
  res.valid = 1;
  res.gain = g;
  res.threshold = midpoint_down(order_key_inv(uint32_t(ka >> 32)), order_key_inv(uint32_t(kb >> 32)));
  res.n_left = fp + 1;
  return res;
}

struct WideShared {  // carve-up of the dynamic shared memory of the exact kernels
  uint32_t* base;  // [8][k]
  uint32_t* run;   // [8][k]
  uint32_t* tot;   // [k]
  double* red;     // [8]
  uint32_t* ured;  // [8]
  unsigned char* rest;
};
__device__ __forceinline__ WideShared wide_carve(unsigned char* sm, int k) {
  WideShared s;
  s.red = reinterpret_cast<double*>(sm);
  s.ured = reinterpret_cast<uint32_t*>(s.red + 8);
  s.base = s.ured + 8;
  s.run = s.base + 8 * k;
  s.tot = s.run + 8 * k;
  s.rest = reinterpret_cast<unsigned char*>(s.tot + ((k + 3) & ~3));
  return s;
}
__host__ __device__ inline size_t wide_carve_bytes(int k) { return 64 + 4 * 16 + 4 * (17 * size_t(k) + 4) + 16; }

}  // namespace dev
}  // namespace sofg
