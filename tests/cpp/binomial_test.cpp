// FastBinomial (host_rng.hpp) against libstdc++ std::binomial_distribution<long long>: the same
// draw and the same number of engine outputs consumed, for the projection-count parameters of
// the reference's defaults (cells = ceil(1.5 sqrt d) * d, density = round(3 sqrt d) / cells,
// projection.hpp:37-47) over a range of d, dense densities, the "easy" waiting-time regime
// (t p < 8) and p > 0.5, from fresh engines and after skipped outputs (retries).
// Build + run: tests/test_host_binomial.py. Exit status 1 on any mismatch.
#include <cmath>
#include <cstdio>
#include <random>

#include "host_rng.hpp"

using namespace sofg::host;

struct Counting {
  std::mt19937_64 g;
  uint64_t n = 0;
  using result_type = uint64_t;
  static constexpr uint64_t min() { return 0; }
  static constexpr uint64_t max() { return ~0ull; }
  uint64_t operator()() {
    ++n;
    return g();
  }
};

int main(int argc, char** argv) {
  const size_t per = argc > 1 ? size_t(atol(argv[1])) : 20000;
  struct P {
    long long t;
    double p;
  };
  std::vector<P> ps;
  for (long long d : {1, 2, 3, 4, 5, 6, 8, 10, 16, 64, 100, 512, 1024, 4096, 16384, 65536}) {
    const double sd = std::sqrt(double(d));
    const long long R = (long long)std::ceil(1.5 * sd);
    const long long e = std::llround(3.0 * sd);
    ps.push_back({R * d, std::min(1.0, double(e) / double(R * d))});
    ps.push_back({R * d, 1e-3});
    ps.push_back({R * d, 0.25});
  }
  ps.push_back({393216, 0.7});
  ps.push_back({1000, 0.004});  // t p = 4: waiting-time method
  ps.push_back({50, 0.999});
  size_t bad = 0, total = 0;
  for (const P& q : ps) {
    if (q.p > 1.0 || q.t <= 0) continue;
    const FastBinomial fb(q.t, q.p);
    const std::binomial_distribution<long long>::param_type prm(q.t, q.p);
    for (size_t i = 0; i < per; ++i) {
      const uint64_t seed = derive_seed(uint64_t(q.t) * 31 + 7, i);
      const uint64_t skip = i % 3 == 0 ? i % 29 : 0;
      Counting a{std::mt19937_64(split_mix64(seed))}, b{std::mt19937_64(split_mix64(seed))};
      for (uint64_t s = 0; s < skip; ++s) {
        a();
        b();
      }
      std::binomial_distribution<long long> d(prm);
      const long long za = d(a);
      const long long zb = fb(b);
      ++total;
      if (za != zb || a.n != b.n) {
        if (bad < 10)
          std::printf("mismatch t=%lld p=%g seed=%llu: std %lld (%llu outputs) fast %lld (%llu)\n", q.t, q.p,
                      (unsigned long long)seed, za, (unsigned long long)a.n, zb, (unsigned long long)b.n);
        ++bad;
      }
    }
    // the batch path (fresh engines, primed together) against the same draws
    std::vector<uint64_t> seeds(per);
    for (size_t i = 0; i < per; ++i) seeds[i] = derive_seed(uint64_t(q.t) * 17 + 3, i);
    std::vector<uint32_t> z(per), used(per);
    const BinomialDraw bd(uint64_t(q.t), q.p);
    bd.batch(seeds.data(), per, z.data(), used.data());
    for (size_t i = 0; i < per; ++i) {
      Counting a{std::mt19937_64(split_mix64(seeds[i]))};
      std::binomial_distribution<long long> d(prm);
      const long long za = d(a);
      ++total;
      if (uint32_t(za) != z[i] || a.n != used[i]) ++bad;
    }
  }
  std::printf("binomial draws compared: %zu, mismatches: %zu\n", total, bad);
  return bad ? 1 : 0;
}
