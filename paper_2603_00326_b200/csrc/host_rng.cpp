#include "host_rng.hpp"

#include <immintrin.h>

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

// std::mt19937_64 with its block twist and tempering vectorised (AVX2, 4 words per instruction):
// the same seeding, the same 312-word blocks (libstdc++ random.tcc _M_gen_rand), the same outputs
// (tests/cpp/bootstrap_test.cpp checks it against std::mt19937_64 and bootstrap_indices against
// std::sample). The scalar library generator was half of bootstrap_indices' time.
class BlockMt64 {
 public:
  using result_type = uint64_t;
  static constexpr result_type min() { return 0; }
  static constexpr result_type max() { return ~0ull; }
  explicit BlockMt64(uint64_t s) {
    mt_[0] = s;
    for (int i = 1; i < kN; ++i) mt_[i] = 6364136223846793005ull * (mt_[i - 1] ^ (mt_[i - 1] >> 62)) + uint64_t(i);
  }
  result_type operator()() {
    if (pos_ == kN) refill();
    return out_[pos_++];
  }

 private:
  static constexpr int kN = 312, kM = 156;
  static constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull, kLower = 0x7FFFFFFFull, kA = 0xB5026F5AA96619E9ull;
  static uint64_t mix(uint64_t cur, uint64_t nxt, uint64_t far) {
    const uint64_t y = (cur & kUpper) | (nxt & kLower);
    return far ^ (y >> 1) ^ ((y & 1ull) ? kA : 0ull);
  }
  static __m256i mix4(__m256i cur, __m256i nxt, __m256i far) {
    const __m256i y = _mm256_or_si256(_mm256_and_si256(cur, _mm256_set1_epi64x(int64_t(kUpper))),
                                      _mm256_and_si256(nxt, _mm256_set1_epi64x(int64_t(kLower))));
    const __m256i odd = _mm256_sub_epi64(_mm256_setzero_si256(), _mm256_and_si256(y, _mm256_set1_epi64x(1)));
    return _mm256_xor_si256(_mm256_xor_si256(far, _mm256_srli_epi64(y, 1)),
                            _mm256_and_si256(odd, _mm256_set1_epi64x(int64_t(kA))));
  }
  __m256i ld(int i) const { return _mm256_loadu_si256(reinterpret_cast<const __m256i*>(mt_ + i)); }
  void refill() {
    static_assert((kN - kM) % 4 == 0, "first twist phase in whole vectors");
    int k = 0;
    for (; k < kN - kM; k += 4)  // reads k+1.. and k+156.. before they are rewritten
      _mm256_storeu_si256(reinterpret_cast<__m256i*>(mt_ + k), mix4(ld(k), ld(k + 1), ld(k + kM)));
    for (; k + 4 <= kN - 1; k += 4)  // mt_[k - 156] rewritten above; k + 1.. not yet
      _mm256_storeu_si256(reinterpret_cast<__m256i*>(mt_ + k), mix4(ld(k), ld(k + 1), ld(k - (kN - kM))));
    for (; k < kN - 1; ++k) mt_[k] = mix(mt_[k], mt_[k + 1], mt_[k - (kN - kM)]);
    mt_[kN - 1] = mix(mt_[kN - 1], mt_[0], mt_[kM - 1]);
    for (int i = 0; i < kN; i += 4) {  // tempering (random.tcc operator())
      __m256i y = ld(i);
      y = _mm256_xor_si256(y, _mm256_and_si256(_mm256_srli_epi64(y, 29), _mm256_set1_epi64x(0x5555555555555555ll)));
      y = _mm256_xor_si256(y, _mm256_and_si256(_mm256_slli_epi64(y, 17), _mm256_set1_epi64x(0x71D67FFFEDA60000ll)));
      y = _mm256_xor_si256(y, _mm256_and_si256(_mm256_slli_epi64(y, 37), _mm256_set1_epi64x(int64_t(0xFFF7EEE000000000ull))));
      y = _mm256_xor_si256(y, _mm256_srli_epi64(y, 43));
      _mm256_storeu_si256(reinterpret_cast<__m256i*>(out_ + i), y);
    }
    pos_ = 0;
  }
  alignas(32) uint64_t mt_[kN];
  alignas(32) uint64_t out_[kN];
  int pos_ = kN;
};
}  // namespace

std::vector<uint32_t> bootstrap_indices(uint64_t n, double fraction, uint64_t seed) {
  uint64_t k = uint64_t(std::llround(fraction * double(n)));  // dataset.hpp:338-340
  k = std::clamp<uint64_t>(k, 1, n);
  BlockMt64 g(split_mix64(seed));  // = std::mt19937_64(split_mix64(seed)) (random.hpp:26)
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
