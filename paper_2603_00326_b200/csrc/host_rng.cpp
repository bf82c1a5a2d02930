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
  std::vector<uint32_t> out(k);
  std::mt19937_64 g(split_mix64(seed));
  PutIt end = std::sample(CountIt{0}, CountIt{uint32_t(n)}, PutIt{out.data()}, std::ptrdiff_t(k), g);
  out.resize(size_t(end.p - out.data()));
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
