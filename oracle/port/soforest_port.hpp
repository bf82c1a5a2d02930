// TEST INFRASTRUCTURE ONLY — CPU oracle ("port" kind).
//
// A plain C++ restatement of the reference learner's algorithm (soforest, arXiv 2603.00326,
// /root/reference/proj/include/soforest/*.hpp), written from the reference's behaviour. It is
// the checker for the CUDA path: only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline leg may load it. It is pinned against the compiled reference itself
// (oracle/_ref, see oracle/Makefile) and against the reference tests' known answers
// (tests/test_oracle_*.py).
//
// Third-party arithmetic on this path, pinned by toolchain:
//   * libstdc++ 13 <random>: std::mt19937_64, std::binomial_distribution<long long>,
//     std::uniform_int_distribution (Lemire, bits/uniform_int_dist.h:257-281),
//     std::normal_distribution, std::sample.
//   * glibc libm: log2 (entropy / xlogx), log/lgamma/exp/sqrt (binomial, normal).
//   * FMA contraction of the reference's default build (-O2 -march=native): entropy() contracts
//     to vfnmadd231sd and midpoint_down() to vfmadd132ss (checked with g++ -S); restated here
//     with explicit std::fma so the oracle is flag-independent.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <iterator>
#include <numeric>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace port {

using Engine = std::mt19937_64;  // random.hpp:10

// random.hpp:13-18 — SplitMix64 output function.
inline uint64_t split_mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
// random.hpp:22-24
inline uint64_t derive_seed(uint64_t seed, uint64_t key) {
  return split_mix64(seed ^ split_mix64(key + 0x632be59bd9b4e019ull));
}
// random.hpp:26
inline Engine make_rng(uint64_t seed) { return Engine(split_mix64(seed)); }

// Counts engine outputs so tests can report stream positions.
struct CountingEngine {
  using result_type = uint64_t;
  Engine& e;
  uint64_t count = 0;
  static constexpr result_type min() { return Engine::min(); }
  static constexpr result_type max() { return Engine::max(); }
  result_type operator()() {
    ++count;
    return e();
  }
};

// random.hpp:31-45 — Floyd subset sampling; the result is the sorted set.
template <class G>
void floyd(uint64_t n, uint64_t k, G& g, std::vector<uint64_t>& set) {
  set.clear();
  if (k == 0) return;
  k = std::min(k, n);
  for (uint64_t j = n - k; j < n; ++j) {
    const uint64_t t = std::uniform_int_distribution<uint64_t>(0, j)(g);
    auto it = std::lower_bound(set.begin(), set.end(), t);
    if (it != set.end() && *it == t)
      set.push_back(j);  // j is larger than everything present
    else
      set.insert(it, t);
  }
}

// ---------------------------------------------------------------- dataset (dataset.hpp)
struct Dataset {
  uint64_t n = 0, d = 0;
  int32_t k = 0;
  const float* X = nullptr;  // column-major
  const int32_t* y = nullptr;
  float at(uint64_t sample, uint64_t f) const { return X[f * n + sample]; }
  const float* col(uint64_t f) const { return X + f * n; }
};

// dataset.hpp:306-329 — one engine, row-major draw order, class = i % 2.
inline void generate_trunk(uint64_t n, uint64_t d, uint64_t seed, float* X, int32_t* y) {
  if (n < 2) throw std::invalid_argument("n_samples must be at least 2");
  if (d == 0) throw std::invalid_argument("n_features must be positive");
  std::vector<double> mu(d);
  for (uint64_t f = 0; f < d; ++f) mu[f] = 1.0 / std::sqrt(double(f + 1));
  Engine g = make_rng(seed);
  std::normal_distribution<double> normal(0.0, 1.0);
  for (uint64_t i = 0; i < n; ++i) {
    const int32_t c = int32_t(i % 2);
    y[i] = c;
    const double s = c == 0 ? 1.0 : -1.0;
    for (uint64_t f = 0; f < d; ++f) X[f * n + i] = float(s * mu[f] + normal(g));
  }
}

// dataset.hpp:332-349 — selection sampling over iota(n) via std::sample, sorted output.
inline std::vector<uint32_t> bootstrap(uint64_t n, double fraction, uint64_t seed) {
  if (!(fraction > 0.0) || fraction > 1.0)
    throw std::invalid_argument("bootstrap fraction must be in (0, 1]");
  uint64_t k = uint64_t(std::llround(fraction * double(n)));
  k = std::clamp<uint64_t>(k, 1, n);
  std::vector<uint32_t> all(n), out;
  std::iota(all.begin(), all.end(), 0u);
  out.reserve(k);
  Engine g = make_rng(seed);
  std::sample(all.begin(), all.end(), std::back_inserter(out), k, g);
  return out;
}

// ---------------------------------------------------------------- projection.hpp
struct ProjConfig {
  uint64_t d = 0, rows = 0, expected = 0;
  double density = 0.0;
};
// projection.hpp:39-50
inline ProjConfig proj_config(uint64_t d) {
  if (d == 0) throw std::invalid_argument("n_features must be positive");
  const double r = std::sqrt(double(d));
  ProjConfig c;
  c.d = d;
  c.rows = uint64_t(std::ceil(1.5 * r));
  c.expected = uint64_t(std::llround(3.0 * r));
  c.density = std::min(1.0, double(c.expected) / (double(c.rows) * double(d)));
  return c;
}

struct Term {
  uint32_t feature;
  float weight;
  bool operator==(const Term& o) const { return feature == o.feature && weight == o.weight; }
};
using Row = std::vector<Term>;
using Matrix = std::vector<Row>;

// projection.hpp:57-82 — z ~ Binomial(cells, density); Floyd over cells; one coin per chosen
// cell in ascending cell order.
template <class G>
Matrix sample_matrix(const ProjConfig& c, G& g) {
  if (c.d == 0 || c.rows == 0) throw std::invalid_argument("projection config is empty");
  if (!(c.density >= 0.0) || c.density > 1.0)
    throw std::invalid_argument("cell density must be in [0, 1]");
  const uint64_t cells = c.rows * c.d;
  std::binomial_distribution<long long> nnz((long long)cells, c.density);
  const uint64_t z = uint64_t(nnz(g));
  Matrix m(c.rows);
  std::vector<uint64_t> chosen;
  floyd(cells, z, g, chosen);
  std::uniform_int_distribution<int> coin(0, 1);
  for (uint64_t cell : chosen) m[cell / c.d].push_back({uint32_t(cell % c.d), coin(g) ? 1.f : -1.f});
  return m;
}

// projection.hpp:86-108 — double accumulation in term order, first term assigns.
inline void apply(const Dataset& D, const Row& row, const uint32_t* active, uint64_t n,
                  float* out) {
  if (row.empty()) {
    std::fill(out, out + n, 0.f);
    return;
  }
  std::vector<double> acc(n);
  for (size_t t = 0; t < row.size(); ++t) {
    const float* col = D.col(row[t].feature);
    const double w = double(row[t].weight);
    for (uint64_t j = 0; j < n; ++j) {
      const double x = w * double(col[active[j]]);
      acc[j] = t == 0 ? x : acc[j] + x;
    }
  }
  for (uint64_t j = 0; j < n; ++j) out[j] = float(acc[j]);
}

// ---------------------------------------------------------------- histogram.hpp
// histogram.hpp:23-28 as compiled by the reference's default flags: fma(b - a, 0.5f, a).
inline float midpoint_down(float a, float b) {
  float t = std::fma(b - a, 0.5f, a);
  if (!(t < b)) t = a;
  return t;
}

// histogram.hpp:37-61
template <class G>
uint64_t sample_boundaries(const float* v, uint64_t n, uint64_t bins, G& g, float* out) {
  if (bins < 1) throw std::invalid_argument("bin_count must be positive");
  if (n < 2 || bins < 2) return 0;
  const uint64_t m = std::min(bins, n);
  std::vector<float> drawn(m);
  if (m == n) {
    std::copy(v, v + n, drawn.begin());
  } else {
    std::vector<uint64_t> picks;
    floyd(n, m, g, picks);
    for (uint64_t i = 0; i < m; ++i) drawn[i] = v[picks[i]];
  }
  std::sort(drawn.begin(), drawn.end());
  uint64_t nb = 0;
  for (uint64_t i = 1; i < m; ++i)
    if (drawn[i - 1] < drawn[i]) out[nb++] = midpoint_down(drawn[i - 1], drawn[i]);
  return nb;
}

// histogram.hpp:72-75 (and the two-level equivalent, :118-173): #boundaries <= v.
inline uint64_t bin_of(const float* b, uint64_t nb, float v) {
  return uint64_t(std::upper_bound(b, b + nb, v) - b);
}

// histogram.hpp:180-206, bin-major counts[bin*k + class].
inline void build_histogram(const float* v, const int32_t* y, uint64_t n, const float* b,
                            uint64_t nb, int32_t k, uint32_t* counts) {
  std::fill(counts, counts + (nb + 1) * uint64_t(k), 0u);
  for (uint64_t j = 0; j < n; ++j) counts[bin_of(b, nb, v[j]) * k + y[j]]++;
}

// ---------------------------------------------------------------- split.hpp
// split.hpp:20-31 with the reference build's contraction h = fma(-p, log2 p, h).
inline double entropy(const uint32_t* c, int32_t k) {
  double n = 0.0;
  for (int32_t i = 0; i < k; ++i) n += c[i];
  if (n == 0.0) return 0.0;
  double h = 0.0;
  for (int32_t i = 0; i < k; ++i) {
    if (c[i] == 0) continue;
    const double p = double(c[i]) / n;
    h = std::fma(-p, std::log2(p), h);
  }
  return h;
}

// split.hpp:55-62
inline double xlogx(uint64_t c) {
  static thread_local std::vector<double> tab{0.0, 0.0};
  while (tab.size() <= c) {
    const double x = double(tab.size());
    tab.push_back(x * std::log2(x));
  }
  return tab[c];
}

// split.hpp:66-76
inline double gain_of(const uint32_t* left, const uint32_t* total, int32_t k, uint64_t nl,
                      uint64_t nr, double parent) {
  double sl = 0.0, sr = 0.0;
  for (int32_t c = 0; c < k; ++c) {
    sl += xlogx(left[c]);
    sr += xlogx(total[c] - left[c]);
  }
  return parent - (xlogx(nl) - sl + xlogx(nr) - sr) / double(nl + nr);
}

struct Split {
  uint64_t row = 0;
  float threshold = 0.f;
  double gain = 0.0;
  uint32_t n_left = 0, n_right = 0;
};

// split.hpp:84-120
inline std::optional<Split> best_split_histogram(const float* b, uint64_t nb, const uint32_t* counts,
                                                 int32_t k, uint64_t row = 0) {
  if (nb == 0) return std::nullopt;
  std::vector<uint32_t> total(k, 0), left(k, 0);
  for (uint64_t bin = 0; bin <= nb; ++bin)
    for (int32_t c = 0; c < k; ++c) total[c] += counts[bin * k + c];
  double n = 0.0;
  for (uint32_t t : total) n += t;
  if (n < 2.0) return std::nullopt;
  const double parent = entropy(total.data(), k);
  std::optional<Split> best;
  uint64_t nl = 0;
  for (uint64_t bin = 0; bin < nb; ++bin) {
    for (int32_t c = 0; c < k; ++c) {
      left[c] += counts[bin * k + c];
      nl += counts[bin * k + c];
    }
    const uint64_t nr = uint64_t(n) - nl;
    if (nl == 0 || nr == 0) continue;
    const double g = gain_of(left.data(), total.data(), k, nl, nr, parent);
    if (g > 0.0 && (!best || g > best->gain)) best = Split{row, b[bin], g, uint32_t(nl), uint32_t(nr)};
  }
  return best;
}

// split.hpp:126-134
inline uint32_t order_key(float v) {
  uint32_t u;
  std::memcpy(&u, &v, 4);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
inline float order_key_inverse(uint32_t key) {
  const uint32_t u = (key & 0x80000000u) ? (key & 0x7fffffffu) : ~key;
  float v;
  std::memcpy(&v, &u, 4);
  return v;
}

// split.hpp:142-194 (float specialisation: packed 64-bit keys, value groups by float compare).
inline std::optional<Split> best_split_exact(const float* v, const int32_t* y, uint64_t n,
                                             int32_t k, uint64_t row = 0) {
  if (n < 2) return std::nullopt;
  std::vector<uint32_t> total(k, 0), left(k, 0);
  for (uint64_t j = 0; j < n; ++j) total[y[j]]++;
  const double parent = entropy(total.data(), k);
  std::vector<uint64_t> key(n);
  for (uint64_t j = 0; j < n; ++j) key[j] = (uint64_t(order_key(v[j])) << 32) | uint32_t(y[j]);
  std::sort(key.begin(), key.end());
  std::optional<Split> best;
  for (uint64_t j = 1; j < n; ++j) {
    left[int32_t(key[j - 1] & 0xffffffffu)]++;
    const float a = order_key_inverse(uint32_t(key[j - 1] >> 32));
    const float b = order_key_inverse(uint32_t(key[j] >> 32));
    if (!(a < b)) continue;
    const double g = gain_of(left.data(), total.data(), k, j, n - j, parent);
    if (g > 0.0 && (!best || g > best->gain))
      best = Split{row, midpoint_down(a, b), g, uint32_t(j), uint32_t(n - j)};
  }
  return best;
}

enum Method { kExact = 0, kHistogram = 1 };

// split.hpp:229-317 — all rows projected, then per-row search; strict '>' keeps the lowest row.
// `values` receives the row-major [R][n] projections (the reference's scratch.values).
template <class G>
std::optional<Split> find_node_split(const Dataset& D, const uint32_t* active, uint64_t n,
                                     const Matrix& m, Method method, uint64_t bins, G& g,
                                     std::vector<float>& values) {
  const uint64_t R = m.size();
  const int32_t k = D.k;
  if (n < 2) return std::nullopt;
  if (bins < 2) throw std::invalid_argument("bin_count must be at least 2");
  std::vector<int32_t> y(n);
  for (uint64_t j = 0; j < n; ++j) y[j] = D.y[active[j]];
  values.assign(R * n, 0.f);
  for (uint64_t r = 0; r < R; ++r) apply(D, m[r], active, n, values.data() + r * n);

  std::optional<Split> best;
  auto consider = [&](const std::optional<Split>& c) {
    if (c && (!best || c->gain > best->gain)) best = c;
  };
  if (method == kHistogram) {
    const uint64_t maxb = bins - 1;
    std::vector<float> bnd(R * maxb);
    std::vector<uint64_t> nb(R);
    for (uint64_t r = 0; r < R; ++r)  // every row draws, even empty ones (split.hpp:272-276)
      nb[r] = sample_boundaries(values.data() + r * n, n, bins, g, bnd.data() + r * maxb);
    std::vector<uint32_t> counts;
    for (uint64_t r = 0; r < R; ++r) {
      if (nb[r] == 0) continue;
      counts.assign((nb[r] + 1) * k, 0);
      build_histogram(values.data() + r * n, y.data(), n, bnd.data() + r * maxb, nb[r], k,
                      counts.data());
      consider(best_split_histogram(bnd.data() + r * maxb, nb[r], counts.data(), k, r));
    }
  } else {
    for (uint64_t r = 0; r < R; ++r) {
      if (m[r].empty()) continue;  // split.hpp:308
      consider(best_split_exact(values.data() + r * n, y.data(), n, k, r));
    }
  }
  return best;
}

// ---------------------------------------------------------------- forest.hpp
struct Config {
  uint64_t n_trees = 100;
  int mode = 2;  // 0 exact-only, 1 histogram-only, 2 dynamic
  uint64_t bin_count = 256;
  std::optional<uint64_t> breakeven;
  double bootstrap_fraction = 0.632;
  std::optional<uint64_t> max_depth;
  uint64_t min_samples_split = 2;
  uint64_t max_split_retries = 1;
  uint64_t n_workers = 1;
  uint64_t seed = 0;
  uint64_t num_projections = 0;  // extension (D3)
  double cell_density = 0.0;     // extension (D3)
};

struct Node {
  Row projection;
  float threshold = 0.f;
  int32_t left = -1, right = -1, predicted_class = -1;
};
struct Tree {
  std::vector<Node> nodes;
};

inline ProjConfig effective_proj_config(const Config& cfg, uint64_t d) {
  ProjConfig pc = proj_config(d);
  if (cfg.num_projections) pc.rows = cfg.num_projections;
  if (cfg.cell_density > 0.0) pc.density = cfg.cell_density;
  return pc;
}

// forest.hpp:157-240 — depth-first growth; node ids in split order, children pushed right
// then left, each node's engine is make_rng(node seed), children seeds derive(seed, 1/2).
inline Tree grow(const Dataset& D, const Config& cfg, const ProjConfig& pc, uint64_t breakeven,
                 std::vector<uint32_t> idx, uint64_t root_seed, uint64_t root_depth) {
  struct Item {
    int32_t node;
    uint32_t begin, end, depth;
    uint64_t seed;
  };
  Tree tree;
  tree.nodes.emplace_back();
  std::vector<Item> stack{{0, 0, uint32_t(idx.size()), uint32_t(root_depth), root_seed}};
  std::vector<uint32_t> totals(D.k);
  std::vector<float> values;
  std::vector<uint32_t> spill;
  while (!stack.empty()) {
    const Item it = stack.back();
    stack.pop_back();
    const uint64_t n = it.end - it.begin;
    const uint32_t* active = idx.data() + it.begin;
    std::fill(totals.begin(), totals.end(), 0u);
    for (uint64_t j = 0; j < n; ++j) totals[D.y[active[j]]]++;
    const uint32_t top = *std::max_element(totals.begin(), totals.end());
    const bool splittable = top < n && n >= cfg.min_samples_split && n >= 2 &&
                            (!cfg.max_depth || it.depth < *cfg.max_depth);
    bool split_done = false;
    if (splittable) {
      Engine g = make_rng(it.seed);
      Method method = cfg.mode == 0   ? kExact
                      : cfg.mode == 1 ? kHistogram
                                      : (n > breakeven ? kHistogram : kExact);  // split.hpp:46-48
      for (uint64_t attempt = 0; attempt <= cfg.max_split_retries && !split_done; ++attempt) {
        Matrix m = sample_matrix(pc, g);
        auto s = find_node_split(D, active, n, m, method, cfg.bin_count, g, values);
        if (!s) continue;
        const float* v = values.data() + s->row * n;
        spill.clear();
        uint32_t w = it.begin;
        for (uint64_t j = 0; j < n; ++j) {
          const uint32_t sample = idx[it.begin + j];
          if (v[j] <= s->threshold)
            idx[w++] = sample;
          else
            spill.push_back(sample);
        }
        const uint32_t nl = w - it.begin;
        if (nl == 0 || nl == n) continue;  // forest.hpp:211: degenerate, try again
        std::copy(spill.begin(), spill.end(), idx.begin() + w);
        const int32_t l = int32_t(tree.nodes.size());
        Node& p = tree.nodes[it.node];
        p.projection = m[s->row];
        p.threshold = s->threshold;
        p.left = l;
        p.right = l + 1;
        tree.nodes.emplace_back();
        tree.nodes.emplace_back();
        stack.push_back({l + 1, it.begin + nl, it.end, it.depth + 1, derive_seed(it.seed, 2)});
        stack.push_back({l, it.begin, it.begin + nl, it.depth + 1, derive_seed(it.seed, 1)});
        split_done = true;
      }
    }
    if (!split_done)
      tree.nodes[it.node].predicted_class =
          int32_t(std::max_element(totals.begin(), totals.end()) - totals.begin());
  }
  return tree;
}

inline void validate(const Dataset& D, const Config& cfg) {  // forest.hpp:270-276
  if (cfg.n_trees < 1) throw std::invalid_argument("n_trees must be positive");
  if (cfg.bin_count < 2) throw std::invalid_argument("bin_count must be at least 2");
  if (cfg.min_samples_split < 2) throw std::invalid_argument("min_samples_split must be at least 2");
  if (!(cfg.bootstrap_fraction > 0.0) || cfg.bootstrap_fraction > 1.0)
    throw std::invalid_argument("bootstrap fraction must be in (0, 1]");
  if (D.n < 2) throw std::invalid_argument("need at least 2 samples");
  if (D.k < 2) throw std::invalid_argument("need at least 2 classes");
}

constexpr uint64_t kFallbackBreakeven = 1024;  // calibrate.hpp:43

// forest.hpp:250-262
inline Tree train_tree(const Dataset& D, const std::vector<uint32_t>& active, const Config& cfg,
                       uint64_t seed, uint64_t depth) {
  if (active.empty()) throw std::invalid_argument("active sample set is empty");
  for (uint32_t s : active)
    if (s >= D.n) throw std::out_of_range("sample index out of range");
  return grow(D, cfg, effective_proj_config(cfg, D.d), cfg.breakeven.value_or(kFallbackBreakeven),
              active, seed, depth);
}

// forest.hpp:267-313; calibration is out of scope for the oracle: a breakeven must be given
// (or the fallback 1024 is used), matching how parity runs pin the semantic threshold (D2).
inline std::vector<Tree> train_forest(const Dataset& D, const Config& cfg, uint64_t* breakeven_out) {
  validate(D, cfg);
  const uint64_t be = cfg.mode == 2 ? cfg.breakeven.value_or(kFallbackBreakeven) : 0;
  if (breakeven_out) *breakeven_out = be;
  const ProjConfig pc = effective_proj_config(cfg, D.d);
  std::vector<Tree> trees(cfg.n_trees);
  const uint64_t W = std::max<uint64_t>(1, std::min(cfg.n_workers, cfg.n_trees));
  auto work = [&](uint64_t w) {
    for (uint64_t t = w; t < cfg.n_trees; t += W) {  // parallel.hpp:31 strided map
      const uint64_t ts = derive_seed(cfg.seed, t + 1);
      trees[t] = grow(D, cfg, pc, be, bootstrap(D.n, cfg.bootstrap_fraction, derive_seed(ts, 0)),
                      derive_seed(ts, 1), 0);
    }
  };
  if (W == 1) {
    work(0);
  } else {
    std::vector<std::thread> th;
    for (uint64_t w = 0; w < W; ++w) th.emplace_back(work, w);
    for (auto& t : th) t.join();
  }
  return trees;
}

// forest.hpp:88-102
inline int32_t predict_tree(const Tree& t, const float* x) {
  const Node* nd = &t.nodes[0];
  while (nd->left >= 0) {
    double acc = 0.0;
    bool first = true;
    for (const Term& term : nd->projection) {
      const double p = double(term.weight) * double(x[term.feature]);
      acc = first ? p : acc + p;
      first = false;
    }
    nd = &t.nodes[float(acc) <= nd->threshold ? nd->left : nd->right];
  }
  return nd->predicted_class;
}

}  // namespace port
