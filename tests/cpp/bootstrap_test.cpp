// bootstrap_indices (host_rng.cpp: the libstdc++ selection-sampling restatement on a vectorised
// mt19937_64) against the reference's own call, std::sample over iota(n) with
// std::mt19937_64(split_mix64(seed)) (dataset.hpp:332-349), for many (n, fraction, seed) — up to
// ~500 engine blocks per case, so the vectorised twist and tempering are checked word for word.
// Build + run: tests/test_host_binomial.py. Exit status 1 on any mismatch.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <numeric>
#include <random>
#include <vector>

#include "host_rng.hpp"

using namespace sofg::host;

int main() {
  size_t bad = 0, cases = 0;
  const uint64_t ns[] = {1, 2, 3, 7, 64, 1000, 4097, 65537, 300000};
  const double fracs[] = {0.0001, 0.1, 0.5, 0.632, 0.99, 1.0};
  for (uint64_t n : ns)
    for (double f : fracs)
      for (uint64_t seed = 1; seed <= 6; ++seed) {
        const uint64_t s = derive_seed(seed * 7919, n);
        uint64_t k = uint64_t(std::llround(f * double(n)));
        k = std::clamp<uint64_t>(k, 1, n);
        std::vector<uint32_t> pop(n), ref;
        std::iota(pop.begin(), pop.end(), 0u);
        std::mt19937_64 g(split_mix64(s));
        std::sample(pop.begin(), pop.end(), std::back_inserter(ref), std::ptrdiff_t(k), g);
        const std::vector<uint32_t> got = bootstrap_indices(n, f, s);
        ++cases;
        if (got != ref) {
          ++bad;
          if (bad < 5) std::printf("mismatch n=%llu f=%g seed=%llu\n", (unsigned long long)n, f, (unsigned long long)seed);
        }
      }
  std::printf("bootstrap cases: %zu, mismatches: %zu\n", cases, bad);
  return bad ? 1 : 0;
}
