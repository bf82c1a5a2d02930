// Host side of the per-node random stream.
//
// The reference seeds one std::mt19937_64 per node (make_rng, reference random.hpp:26) and draws
// the projection nonzero count with std::binomial_distribution<long long> (projection.hpp:66-67),
// whose rejection sampler uses glibc log/lgamma/exp — so that single draw stays on the host, on
// the same libstdc++/libm as the reference. Everything after it (Floyd cells, coins, boundary
// picks) is integer-only and is regenerated on the device from (seed, outputs consumed).
//
// LazyMt64 produces exactly std::mt19937_64's output sequence but only computes the seeding
// recurrence as far as the requested outputs need it: output i < 156 of the first block depends
// on seed words i, i+1 and i+156, so the handful of outputs a binomial draw consumes costs ~160
// recurrence steps instead of 312 + a full twist.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <new>
#include <random>
#include <vector>

namespace sofg {
namespace host {

inline uint64_t split_mix64(uint64_t z) {  // reference random.hpp:13-18
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
inline uint64_t derive_seed(uint64_t seed, uint64_t key) {  // random.hpp:22-24
  return split_mix64(seed ^ split_mix64(key + 0x632be59bd9b4e019ull));
}

class LazyMt64 {
 public:
  using result_type = uint64_t;
  static constexpr result_type min() { return 0; }
  static constexpr result_type max() { return ~0ull; }

  explicit LazyMt64(uint64_t node_seed) {
    s_[0] = split_mix64(node_seed);
    seeded_ = 1;
  }

  result_type operator()() {
    if (count_ < kN) {
      const int i = int(count_);
      uint64_t w;
      if (i < kN - kM) {
        need(i + kM);
        w = mix(s_[i], s_[i + 1], s_[i + kM]);
      } else {
        need(kN - 1);
        const uint64_t nxt = (i + 1 < kN) ? s_[i + 1] : b_[0];
        w = mix(s_[i], nxt, b_[i - (kN - kM)]);
      }
      b_[i] = w;
      ++count_;
      return temper(w);
    }
    const int i = int(count_ % kN);
    if (i == 0) twist_in_place();
    ++count_;
    return temper(b_[i]);
  }

  uint64_t consumed() const { return count_; }

  // Advance the seeding recurrence of M engines to word `upto` in lockstep: the chains are
  // independent, so the multiplies overlap (the recurrence is one dependent chain per engine).
  template <int M>
  static void prime(LazyMt64* g, int upto) {
    int from = g[0].seeded_;
    for (int j = 1; j < M; ++j) from = std::min(from, g[j].seeded_);
    uint64_t p[M];
    for (int j = 0; j < M; ++j) p[j] = g[j].s_[from - 1];
    for (int i = from; i <= upto; ++i) {
#pragma GCC unroll 8
      for (int j = 0; j < M; ++j) {
        p[j] = 6364136223846793005ull * (p[j] ^ (p[j] >> 62)) + uint64_t(i);
        g[j].s_[i] = p[j];
      }
    }
    for (int j = 0; j < M; ++j) g[j].seeded_ = upto + 1;
  }

  static constexpr int kBatch = 8;  // engines primed together by BinomialDraw::batch

 private:
  static constexpr int kN = 312, kM = 156;
  static uint64_t mix(uint64_t cur, uint64_t nxt, uint64_t far) {
    const uint64_t y = (cur & 0xFFFFFFFF80000000ull) | (nxt & 0x7FFFFFFFull);
    return far ^ (y >> 1) ^ ((y & 1ull) ? 0xB5026F5AA96619E9ull : 0ull);
  }
  static uint64_t temper(uint64_t y) {
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    return y ^ (y >> 43);
  }
  void need(int upto) {
    while (seeded_ <= upto) {
      const uint64_t p = s_[seeded_ - 1];
      s_[seeded_] = 6364136223846793005ull * (p ^ (p >> 62)) + uint64_t(seeded_);
      ++seeded_;
    }
  }
  void twist_in_place() {
    for (int k = 0; k < kN - kM; ++k) b_[k] = mix(b_[k], b_[k + 1], b_[k + kM]);
    for (int k = kN - kM; k < kN - 1; ++k) b_[k] = mix(b_[k], b_[k + 1], b_[k - (kN - kM)]);
    b_[kN - 1] = mix(b_[kN - 1], b_[0], b_[kM - 1]);
  }

  uint64_t s_[kN];  // seeding recurrence words (computed on demand)
  uint64_t b_[kN];  // current raw block
  int seeded_ = 0;
  uint64_t count_ = 0;
};

// Binomial nonzero count of one projection matrix: the reference constructs a fresh
// std::binomial_distribution<long long>(cells, density) per matrix (projection.hpp:66-67), so no
// normal variate carries over between nodes. FastBinomial restates that draw — libstdc++ 13
// binomial_distribution::operator() (bits/random.tcc:1563-1680, Devroye's rejection method, and
// _M_waiting :1532-1551) — for one fixed parameter:
//  * the parameter block is the library's own (param_type::_M_initialize, read back from a
//    genuine param_type object), not recomputed;
//  * every uniform, normal, log and exponential is the same libstdc++/glibc call in the same
//    order with the same expressions (so the compiler contracts them the same way);
//  * the acceptance test's lgamma(np + x + 1) + lgamma(t - (np + x) + 1) depends only on the
//    integer x: it is tabulated once per parameter (the same glibc lgamma values) for the x the
//    sampler produces in practice, and computed inline outside that window. Besides the two calls
//    per draw this removes glibc lgamma's store to the process-global `signgam`, which made
//    concurrent draws contend for one cache line (16 host threads: 47 ns per draw with
//    std::binomial_distribution vs 10 ns, tools/mb/binom_mb.cpp on the B200 host).
// tests/cpp/binomial_test.cpp checks it against std::binomial_distribution draw for draw
// (values and engine outputs consumed).
class FastBinomial {
 public:
  FastBinomial(long long t, double p) {
    const std::binomial_distribution<long long>::param_type prm(t, p);
    static_assert(sizeof(Mirror) == sizeof(prm), "libstdc++ binomial param_type layout");
    std::memcpy(&m_, &prm, sizeof(m_));
    if (!m_.easy) {
      const double p12 = m_.p <= 0.5 ? m_.p : 1.0 - m_.p;
      np_ = std::floor(m_.t * p12);
      lo_ = -std::min<long long>(kWin, (long long)np_);
      const long long hi = std::min<long long>(kWin, m_.t - (long long)np_);
      lfx_.resize(size_t(hi - lo_ + 1));
      for (long long x = lo_; x <= hi; ++x) lfx_[size_t(x - lo_)] = lfx_direct(double(x));
    }
  }

  template <class G>
  long long operator()(G& g) const {
    long long ret;
    const long long t = m_.t;
    const double p = m_.p;
    const double p12 = p <= 0.5 ? p : 1.0 - p;
    if (!m_.easy) {
      double x = 0.0;
      const double naf = (1 - std::numeric_limits<double>::epsilon()) / 2;
      const double thr = std::numeric_limits<long long>::max() + naf;
      const double np = std::floor(t * p12);
      const double spi_2 = 1.2533141373155002512078826424055226L;  // sqrt(pi / 2)
      const double a1 = m_.a1;
      const double a12 = a1 + m_.s2 * spi_2;
      const double a123 = m_.a123;
      const double s1s = m_.s1 * m_.s1;
      const double s2s = m_.s2 * m_.s2;
      std::normal_distribution<double> nd;  // binomial_distribution::_M_nd of a fresh object
      bool reject;
      do {
        const double u = m_.s * canon(g);
        double v = 0.0;
        if (u <= a1) {
          const double n = nd(g);
          const double y = m_.s1 * std::abs(n);
          reject = y >= m_.d1;
          if (!reject) {
            const double e = -std::log(1.0 - canon(g));
            x = std::floor(y);
            v = -e - n * n / 2 + m_.c;
          }
        } else if (u <= a12) {
          const double n = nd(g);
          const double y = m_.s2 * std::abs(n);
          reject = y >= m_.d2;
          if (!reject) {
            const double e = -std::log(1.0 - canon(g));
            x = std::floor(-y);
            v = -e - n * n / 2;
          }
        } else if (u <= a123) {
          const double e1 = -std::log(1.0 - canon(g));
          const double e2 = -std::log(1.0 - canon(g));
          const double y = m_.d1 + 2 * s1s * e1 / m_.d1;
          x = std::floor(y);
          v = (-e2 + m_.d1 * (1 / (t - np) - y / (2 * s1s)));
          reject = false;
        } else {
          const double e1 = -std::log(1.0 - canon(g));
          const double e2 = -std::log(1.0 - canon(g));
          const double y = m_.d2 + 2 * s2s * e1 / m_.d2;
          x = std::floor(-y);
          v = -e2 - m_.d2 * y / (2 * s2s);
          reject = false;
        }
        reject = reject || x < -np || x > t - np;
        if (!reject) {
          const double lfx = lfx_of(x);
          reject = v > m_.lf - lfx + x * m_.lp1p;
        }
        reject |= x + np >= thr;
      } while (reject);
      x += np + naf;
      const long long z = waiting(g, t - (long long)(x), m_.q);
      ret = (long long)(x) + z;
    } else {
      ret = waiting(g, t, m_.q);
    }
    if (p12 != p) ret = t - ret;
    return ret;
  }

 private:
  struct Mirror {  // binomial_distribution<long long>::param_type (bits/random.h), in order
    long long t;
    double p, q, d1, d2, s1, s2, c, a1, a123, s, lf, lp1p;
    bool easy;
  };
  static constexpr long long kWin = 4096;
  template <class G>
  static double canon(G& g) {  // __detail::_Adaptor<G, double>
    return std::generate_canonical<double, std::numeric_limits<double>::digits>(g);
  }
  template <class G>
  static long long waiting(G& g, long long t, double q) {
    long long x = 0;
    double sum = 0.0;
    do {
      if (t == x) return x;
      const double e = -std::log(1.0 - canon(g));
      sum += e / (t - x);
      x += 1;
    } while (sum <= q);
    return x - 1;
  }
  double lfx_direct(double x) const { return std::lgamma(np_ + x + 1) + std::lgamma(m_.t - (np_ + x) + 1); }
  double lfx_of(double x) const {
    const long long xi = (long long)x;  // an integer (floor) inside [-np, t - np]
    const long long i = xi - lo_;
    if (i >= 0 && i < (long long)lfx_.size()) return lfx_[size_t(i)];
    return lfx_direct(x);
  }
  Mirror m_;
  double np_ = 0.0;
  long long lo_ = 0;
  std::vector<double> lfx_;
};

// Binomial draws of fresh engines make_rng(seed): the projection nonzero count of a matrix.
struct BinomialDraw {
  FastBinomial dist;
  BinomialDraw(uint64_t cells, double density) : dist((long long)cells, density) {}

  // Draws for m fresh engines make_rng(seeds[i]) (no skipped outputs), a batch at a time with
  // their seeding recurrences primed together (a draw typically reads outputs 0..6).
  void batch(const uint64_t* seeds, size_t m, uint32_t* z, uint32_t* used) const {
    constexpr int M = LazyMt64::kBatch;
    for (size_t i0 = 0; i0 < m; i0 += M) {
      const int c = int(std::min<size_t>(M, m - i0));
      alignas(64) unsigned char mem[M * sizeof(LazyMt64)];
      LazyMt64* g = reinterpret_cast<LazyMt64*>(mem);
      for (int j = 0; j < M; ++j) new (g + j) LazyMt64(seeds[i0 + size_t(j < c ? j : 0)]);
      LazyMt64::prime<M>(g, 156 + 8);
      for (int j = 0; j < c; ++j) {
        z[i0 + size_t(j)] = uint32_t(dist(g[j]));
        used[i0 + size_t(j)] = uint32_t(g[j].consumed());
      }
    }
  }

  // Draw for engine make_rng(seed) after `skip` outputs. Returns z; *used = skip + consumed.
  uint64_t operator()(uint64_t seed, uint64_t skip, uint64_t* used) const {
    LazyMt64 g(seed);
    for (uint64_t i = 0; i < skip; ++i) g();
    const long long z = dist(g);
    *used = g.consumed();
    return uint64_t(z);
  }
};

// bootstrap_sample (reference dataset.hpp:332-349): std::sample selection sampling over iota(n)
// with make_rng(seed); sorted output. Same libstdc++ algorithm as the reference by construction.
std::vector<uint32_t> bootstrap_indices(uint64_t n, double fraction, uint64_t seed);

// Entropy in bits of class counts (reference split.hpp:20-31), with the contraction the
// reference's default -march=native build applies: h = fma(-p, log2(p), h).
double entropy(const uint32_t* counts, int k);

// xlogx table entries c * log2(c) (split.hpp:55-62), c = 0..n.
std::vector<double> xlogx_table(uint64_t n);

}  // namespace host
}  // namespace sofg
