#include "host_rng.hpp"

#include <algorithm>
#include <cmath>
#include <iterator>

namespace sofg {
namespace host {

namespace {
// Counting forward iterator over [0, n): std::sample sees a forward population (the same
// selection-sampling branch the reference's vector iterator takes) without an iota array.
struct CountIt {
  using iterator_category = std::forward_iterator_tag;
  using value_type = uint32_t;
  using difference_type = std::ptrdiff_t;
  using pointer = const uint32_t*;
  using reference = uint32_t;
  uint32_t v;
  uint32_t operator*() const { return v; }
  CountIt& operator++() {
    ++v;
    return *this;
  }
  CountIt operator++(int) {
    CountIt t = *this;
    ++v;
    return t;
  }
  bool operator==(const CountIt& o) const { return v == o.v; }
  bool operator!=(const CountIt& o) const { return v != o.v; }
};

// Output iterator writing into a preallocated buffer.
struct PutIt {
  using iterator_category = std::output_iterator_tag;
  using value_type = void;
  using difference_type = std::ptrdiff_t;
  using pointer = void;
  using reference = void;
  uint32_t* p;
  PutIt& operator*() { return *this; }
  PutIt& operator=(uint32_t x) {
    *p = x;
    return *this;
  }
  PutIt& operator++() {
    ++p;
    return *this;
  }
  PutIt operator++(int) {
    PutIt t = *this;
    ++p;
    return t;
  }
};
}  // namespace

std::vector<uint32_t> bootstrap_indices(uint64_t n, double fraction, uint64_t seed) {
  uint64_t k = uint64_t(std::llround(fraction * double(n)));  // dataset.hpp:338-340
  k = std::clamp<uint64_t>(k, 1, n);
  std::mt19937_64 g(split_mix64(seed));
  if (n == 0) return {};
  // libstdc++'s std::sample for forward iterators (selection sampling, stl_algo.h __sample):
  // while two indices fit one draw (n^2 <= 2^64 - 1), pairs (p0, p1) = divmod(x, u - 1) with
  // x = uniform_int_distribution{0, u(u-1) - 1}(g), u the unsampled count, whose 64-bit engine
  // path is Lemire's multiply-shift (uniform_int_dist.h _S_nd). Restated here so the pair split
  // needs no division: with x = hi64(r * u(u-1)) for the accepted engine output r,
  // x / (u-1) = hi64(r * u) exactly (nested floor division), and x % (u-1) = x - that * (u-1).
  std::vector<uint32_t> out(k + 1);
  uint64_t uns = n, need = k, cnt = 0;
  uint32_t idx = 0;
  using u128 = unsigned __int128;
  if (~0ull / uns >= uns) {
    while (need != 0 && uns >= 2) {
      const uint64_t b0 = uns, b1 = uns - 1, range = b0 * b1;
      uint64_t r = g();
      u128 prod = u128(r) * range;
      if (uint64_t(prod) < range) {
        const uint64_t thr = (0 - range) % range;
        while (uint64_t(prod) < thr) {
          r = g();
          prod = u128(r) * range;
        }
      }
      const uint64_t x = uint64_t(prod >> 64);
      const uint64_t p0 = uint64_t((u128(r) * b0) >> 64);
      const uint64_t p1 = x - p0 * b1;
      --uns;
      out[cnt] = idx++;
      const uint64_t s0 = p0 < need ? 1u : 0u;
      cnt += s0;
      need -= s0;
      if (need == 0) break;
      --uns;
      out[cnt] = idx++;
      const uint64_t s1 = p1 < need ? 1u : 0u;
      cnt += s1;
      need -= s1;
    }
  }
  std::uniform_int_distribution<std::ptrdiff_t> d;
  using P = std::uniform_int_distribution<std::ptrdiff_t>::param_type;
  for (; need != 0; ++idx) {
    --uns;
    if (uint64_t(d(g, P{0, std::ptrdiff_t(uns)})) < need) {
      out[cnt++] = idx;
      --need;
    }
  }
  out.resize(cnt);
  return out;
}

double entropy(const uint32_t* c, int k) {
  double n = 0.0;
  for (int i = 0; i < k; ++i) n += c[i];
  if (n == 0.0) return 0.0;
  double h = 0.0;
  for (int i = 0; i < k; ++i) {
    if (c[i] == 0) continue;
    const double p = double(c[i]) / n;
    h = std::fma(-p, std::log2(p), h);
  }
  return h;
}

std::vector<double> xlogx_table(uint64_t n) {
  std::vector<double> t(n + 1, 0.0);
  for (uint64_t c = 2; c <= n; ++c) {
    const double x = double(c);
    t[c] = x * std::log2(x);
  }
  return t;
}

}  // namespace host
}  // namespace sofg
