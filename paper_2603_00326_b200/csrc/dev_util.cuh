// Device helpers shared by the split-finding kernels: bit-exact restatements of the reference's
// scalar helpers plus warp-level sorting / scanning primitives.
#pragma once
#include <cstdint>
#include <type_traits>

#include "common.hpp"

namespace sofg {
namespace dev {

// split.hpp:126-134 — order-preserving float -> u32 map.
// Read-only load with a 64-byte L2 fill: for strided reads (one 4-byte value per 384-byte sample
// block: the partition's winning row) the default fill of a missed line is 128 bytes; 64 halves
// the DRAM bytes (tools/mb/sector_mb.cu: 128 -> 64 B per value, 1.25 -> 1.00 ms; partition 58 ->
// 54 ms per step). Not for the boundary picks: their neighbouring rows reuse the wider fill.
__device__ __forceinline__ float ldg_l2_64(const float* p) {
  float v;
  asm("ld.global.nc.L2::64B.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ uint32_t order_key(float v) {
  const uint32_t u = __float_as_uint(v);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float order_key_inv(uint32_t k) {
  const uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}

// histogram.hpp:23-28 as the reference's default build computes it (g++ -O2 -march=native
// contracts a + (b - a) / 2 into vfmadd132ss): fma(b - a, 0.5f, a), clamped below b.
__device__ __forceinline__ float midpoint_down(float a, float b) {
  const float t = __fmaf_rn(__fsub_rn(b, a), 0.5f, a);
  return (t < b) ? t : a;
}

// Scattered 4-byte gathers from the column-major table. The cache operator matters: the
// read-only path promotes L1 misses to whole lines, which multiplies HBM traffic for isolated
// samples. SOFG_GATHER selects the operator (0 = ld.global.nc, 1 = .nc.L1::no_allocate,
// 2 = .cg (L2 only), 3 = .cs (streaming)).
#ifndef SOFG_GATHER
#define SOFG_GATHER 2
#endif
__device__ __forceinline__ float gather(const float* p) {
#if SOFG_GATHER == 0
  return __ldg(p);
#elif SOFG_GATHER == 1
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
#elif SOFG_GATHER == 2
  return __ldcg(p);
#else
  return __ldcs(p);
#endif
}

// projection.hpp:86-108 for one sample: terms in ascending feature order, double accumulation,
// first term assigns, later terms add, rounded to float once. Weights are +-1 so w*x is exact.
__device__ __forceinline__ float project_sample(const float* __restrict__ X, uint64_t ld,
                                                const uint32_t* __restrict__ terms, int nt,
                                                uint32_t sample) {
  if (nt == 0) return 0.f;
  double acc = 0.0;
  for (int t = 0; t < nt; ++t) {
    const uint32_t tm = terms[t];
    const float x = gather(X + uint64_t(tm >> 1) * ld + sample);
    const double dx = (tm & 1u) ? -double(x) : double(x);
    acc = (t == 0) ? dx : __dadd_rn(acc, dx);
  }
  return __double2float_rn(acc);
}

// The same value from the wave's gathered terms (csp.cu): Gn is the node's G block (term q of the
// node at Gn[q*n + j]); the row's terms are q0..q0+nt-1 with signs in rt[t] & 1.
__device__ __forceinline__ float combine_g(const float* __restrict__ Gn, uint32_t n,
                                           const uint32_t* __restrict__ rt, int nt, uint32_t q0,
                                           uint32_t j) {
  if (nt == 0) return 0.f;
  double acc = 0.0;
  for (int t = 0; t < nt; ++t) {
    const float x = Gn[uint64_t(q0 + uint32_t(t)) * n + j];
    const double dx = (rt[t] & 1u) ? -double(x) : double(x);
    acc = (t == 0) ? dx : __dadd_rn(acc, dx);
  }
  return __double2float_rn(acc);
}

// Warp-cooperative bitonic sort of a[0..P), P a power of two >= 2, ascending.
template <class K>
__device__ __forceinline__ void warp_bitonic_sort(K* a, int P, int lane) {
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < P; i += 32) {
        const int p = i ^ j;
        if (p > i) {
          const K x = a[i], y = a[p];
          const bool up = (i & k) == 0;
          if ((x > y) == up) {
            a[i] = y;
            a[p] = x;
          }
        }
      }
      __syncwarp();
    }
  }
}

// Register bitonic sort of 32*E keys held E per lane in blocked layout (lane l holds sorted
// positions [l*E, (l+1)*E)), ascending: intra-lane compare-exchange for strides < E, shuffles for
// strides >= E.
template <int E, class K, bool COMPACT = false>
__device__ __forceinline__ void reg_bitonic_sort_k(K (&key)[E], int lane) {
  constexpr int P = 32 * E;
  if constexpr (COMPACT) {
    // Stage loops as runtime loops (compact code for large kernels, where the fully unrolled
    // network for E >= 8 overflows the instruction cache); only the register indexing is unrolled.
#pragma unroll 1
    for (int k = 2; k <= P; k <<= 1) {
#pragma unroll 1
      for (int j = k >> 1; j >= E; j >>= 1) {  // partner in another lane
        const int lm = j / E;
        const bool lower = (lane & lm) == 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const K o = __shfl_xor_sync(0xffffffffu, key[e], lm);
          const bool up = ((lane * E + e) & k) == 0;
          const K mn = o < key[e] ? o : key[e];
          const K mx = o < key[e] ? key[e] : o;
          key[e] = (lower == up) ? mn : mx;
        }
      }
#pragma unroll
      for (int j = (E >> 1); j > 0; j >>= 1) {  // partner in this lane
        if (j < k) {
#pragma unroll
          for (int e = 0; e < E; ++e) {
            if ((e & j) == 0) {
              const bool up = ((lane * E + e) & k) == 0;
              const K a = key[e], b = key[e | j];
              const bool sw = (a > b) == up;
              key[e] = sw ? b : a;
              key[e | j] = sw ? a : b;
            }
          }
        }
      }
    }
  } else {
    // the fully unrolled network (every index and direction a constant)
#pragma unroll
    for (int k = 2; k <= P; k <<= 1) {
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        if (j >= E) {
          const int lm = j / E;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const K o = __shfl_xor_sync(0xffffffffu, key[e], lm);
            const int i = lane * E + e;
            const bool up = (i & k) == 0;
            const bool lower = (lane & lm) == 0;
            const K mn = o < key[e] ? o : key[e];
            const K mx = o < key[e] ? key[e] : o;
            key[e] = (lower == up) ? mn : mx;
          }
        } else {
#pragma unroll
          for (int e = 0; e < E; ++e) {
            if ((e & j) == 0) {
              const int i = lane * E + e;
              const bool up = (i & k) == 0;
              const K a = key[e], b = key[e | j];
              const bool sw = (a > b) == up;
              key[e] = sw ? b : a;
              key[e | j] = sw ? a : b;
            }
          }
        }
      }
    }
  }
}

// Sort a[0..P) in (warp-private) shared memory, P a power of two in [32, 512], through registers
// (larger P: the shared-memory network).
template <class K>
__device__ __forceinline__ void warp_sort_via_regs(K* a, int P, int lane) {
  auto run = [&](auto eval) {
    constexpr int E = decltype(eval)::value;
    K k[E];
#pragma unroll
    for (int e = 0; e < E; ++e) k[e] = a[lane * E + e];
    reg_bitonic_sort_k<E, K>(k, lane);
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; ++e) a[lane * E + e] = k[e];
    __syncwarp();
  };
  switch (P) {
    case 32: run(std::integral_constant<int, 1>{}); break;
    case 64: run(std::integral_constant<int, 2>{}); break;
    case 128: run(std::integral_constant<int, 4>{}); break;
    case 256: run(std::integral_constant<int, 8>{}); break;
    case 512: run(std::integral_constant<int, 16>{}); break;
    default: warp_bitonic_sort(a, P, lane);
  }
}

// Register bitonic sort of one key per lane (32 keys), ascending by lane.
template <class K>
__device__ __forceinline__ K warp_sort32(K v, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const K o = __shfl_xor_sync(0xffffffffu, v, j);
      const bool lower = (lane & j) == 0;
      const bool up = (lane & k) == 0;
      // keep min when (lower && up) || (!lower && !up)
      const bool take_min = (lower == up);
      v = take_min ? (o < v ? o : v) : (o > v ? o : v);
    }
  }
  return v;
}

__device__ __forceinline__ uint32_t warp_excl_scan_u32(uint32_t v, int lane, uint32_t* total) {
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  *total = __shfl_sync(0xffffffffu, x, 31);
  return x - v;
}

__device__ __forceinline__ double warp_min_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_min_f32(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ uint32_t warp_min_u32(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Impurity sum of a candidate split: X = f(nl) - sum_c f(l_c) + f(nr) - sum_c f(r_c) with
// f = xlogx, in the reference's operation order (split.hpp:66-76). gain = parent - X / n.
// Division and subtraction are monotone, so the best gain is attained at min X; the exact
// first-maximum position is then resolved among candidates whose X lies within a window of the
// minimum (see first_best_in_window).
template <int KC>
__device__ __forceinline__ double impurity_sum(const double* __restrict__ xl, const uint32_t* left,
                                               const uint32_t* total, int k, uint32_t nl,
                                               uint32_t nr) {
  double sl = 0.0, sr = 0.0;
#pragma unroll
  for (int c = 0; c < KC; ++c) {
    if (c < k) {
      sl = __dadd_rn(sl, xl[left[c]]);
      sr = __dadd_rn(sr, xl[total[c] - left[c]]);
    }
  }
  return __dsub_rn(__dadd_rn(__dsub_rn(xl[nl], sl), xl[nr]), sr);
}

// Impurity sum of a candidate in float from the float copy of the xlogx table (prefilter only).
// Same operation structure as impurity_sum; |Xf - X| <= prefilter_eps(xl[n], k).
template <int KC>
__device__ __forceinline__ float impurity_sum_f(const float* __restrict__ xlf, const uint32_t* left,
                                                const uint32_t* tot, int k, uint32_t nl,
                                                uint32_t nr) {
  float sl = 0.f, sr = 0.f;
  if constexpr (KC == 2) {
    sl = __ldg(xlf + left[0]) + __ldg(xlf + left[1]);
    sr = __ldg(xlf + tot[0] - left[0]) + __ldg(xlf + tot[1] - left[1]);
  } else {
#pragma unroll
    for (int c = 0; c < KC; ++c)
      if (c < k) {
        sl += __ldg(xlf + left[c]);
        sr += __ldg(xlf + tot[c] - left[c]);
      }
  }
  return ((__ldg(xlf + nl) - sl) + __ldg(xlf + nr)) - sr;
}
// Bound on |Xf - X|: 2k+2 table values each within 2^-24 relative of xl[n] (the largest table
// entry used), and 2k+1 float operations on partial sums bounded by 2 xl[n] each; doubled margin.
__device__ __forceinline__ double prefilter_eps(double xln, int k) {
  return double(2 * (2 * k + 2) + 4 * (2 * k + 1)) * xln * 0x1p-24 + 0x1p-60;
}

__device__ __forceinline__ double gain_from_x(double parent, double X, double n) {
  return __dsub_rn(parent, __ddiv_rn(X, n));
}

// Window around Xmin that contains every X whose gain rounds to the same double as Xmin's.
// |q1 - q2| <= 2 ulp(max(parent, q)) for equal results; scaled back by n with a 2^10 margin.
__device__ __forceinline__ double x_window(double parent, double xmin, double n) {
  const double q = xmin / n;
  const double mag = fmax(fabs(parent), fabs(q));
  return xmin + (mag * n + fabs(xmin)) * 0x1p-40 + 1e-300;
}

// Same window with q approximated by xmin * (1/n): the window only has to contain the candidates
// whose exact gain can round to the best one, and the 2^-40 margin dwarfs the approximation.
__device__ __forceinline__ double x_window_fast(double parent, double xmin, double n, double inv_n) {
  const double q = xmin * inv_n;
  const double mag = fmax(fabs(parent), fabs(q));
  return xmin + (mag * n + fabs(xmin)) * 0x1p-40 + 1e-300;
}

}  // namespace dev
}  // namespace sofg
