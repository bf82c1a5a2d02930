// TEST INFRASTRUCTURE ONLY — C ABI over the *reference itself*.
//
// Compiled by oracle/Makefile against the unmodified reference headers
// (/root/reference/proj/include, header-only C++20) into oracle/_ref/libsoforest_ref.so. Nothing
// here re-implements the algorithm: every entry point forwards to the reference's own function.
// The one exception is the ProjectionConfig extension (the reference hard-wires
// ProjectionConfig::for_features at forest.hpp:257,295), which drives the reference's own
// sample_projection_matrix / find_node_split / bootstrap_sample through a depth-first loop that
// mirrors TreeGrower::grow_from (forest.hpp:157-240).
#include <sstream>
#include <soforest/bench.hpp>
#include <soforest/soforest.hpp>

#include <cstring>
#include <thread>
#include <optional>

#include "forest_flat.hpp"

using namespace soforest;

ORC_COMMON_EXPORTS

// predict through the reference's own soforest::predict (forest.hpp:110-121) on a Forest rebuilt
// from the flat arrays; rows in parallel.
extern "C" int orc_predict(const orc_forest* f, const float* rows, uint64_t n_rows, uint64_t n_features,
                           int32_t* out_label, double* out_votes) {
  return orc_guard([&] {
    Forest forest;
    forest.n_features = std::uint32_t(f->n_features);
    forest.class_count = f->class_count;
    const uint64_t T = f->tree_off.size() - 1;
    forest.trees.resize(T);
    for (uint64_t t = 0; t < T; ++t)
      for (int64_t q = f->tree_off[t]; q < f->tree_off[t + 1]; ++q) {
        TreeNode<float> nd;
        nd.left = f->left[q];
        nd.right = f->right[q];
        nd.predicted_class = f->pred[q];
        nd.threshold = f->thr[q];
        for (int64_t u = f->term_off[q]; u < f->term_off[q + 1]; ++u)
          nd.projection.push_back({f->feat[u], f->weight[u]});
        forest.trees[t].nodes.push_back(std::move(nd));
      }
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    parallel_for(n_rows, hw, [&](std::size_t i, std::size_t) {
      const Prediction p = soforest::predict(forest, std::span<const float>(rows + i * n_features, n_features));
      out_label[i] = p.label;
      if (out_votes) std::memcpy(out_votes + i * f->class_count, p.votes.data(), 8 * f->class_count);
    });
  });
}

namespace {

ColumnarDataset make_data(const float* X, const int32_t* y, uint64_t n, uint64_t d, int32_t k) {
  std::vector<std::vector<float>> cols(d);
  for (uint64_t f = 0; f < d; ++f) cols[f].assign(X + f * n, X + (f + 1) * n);
  std::vector<int32_t> labels(y, y + n);
  std::vector<std::string> names;
  for (int32_t c = 0; c < k; ++c) names.push_back(std::to_string(c));
  return ColumnarDataset(std::move(cols), std::move(labels), std::move(names));
}

TrainConfig to_cfg(const orc_config* c) {
  TrainConfig t;
  t.n_trees = c->n_trees;
  t.mode = c->mode == 0 ? SplitMode::kExactOnly
           : c->mode == 1 ? SplitMode::kHistogramOnly
                          : SplitMode::kDynamic;
  t.bin_count = c->bin_count;
  t.two_level_binning = c->two_level_binning != 0;
  if (c->has_breakeven) t.breakeven = c->breakeven;
  t.bootstrap_fraction = c->bootstrap_fraction;
  if (c->has_max_depth) t.max_depth = c->max_depth;
  t.min_samples_split = c->min_samples_split;
  t.max_split_retries = c->max_split_retries;
  t.n_workers = c->n_workers;
  t.seed = c->seed;
  return t;
}

bool custom_projection(const orc_config* c) { return c->num_projections || c->cell_density > 0.0; }

ProjectionConfig projection_for(const orc_config* c, uint64_t d) {
  ProjectionConfig p = ProjectionConfig::for_features(d);
  if (c->num_projections) p.num_projections = c->num_projections;
  if (c->cell_density > 0.0) p.cell_density = c->cell_density;
  return p;
}

// TreeGrower::grow_from (forest.hpp:157-240) with a caller-supplied ProjectionConfig; calls the
// reference's own kernels (sample_projection_matrix, find_node_split).
Tree<float> grow_custom(const ColumnarDataset& data, const TrainConfig& cfg,
                        const ProjectionConfig& pcfg, std::size_t breakeven,
                        std::vector<std::uint32_t> idx, std::uint64_t root_seed,
                        std::uint32_t root_depth) {
  struct Work {
    std::int32_t node;
    std::uint32_t begin, end, depth;
    std::uint64_t seed;
  };
  Tree<float> tree;
  tree.nodes.emplace_back();
  std::vector<Work> stack{{0, 0, std::uint32_t(idx.size()), root_depth, root_seed}};
  std::vector<std::uint32_t> totals(data.class_count());
  SplitScratch<float> scratch;
  std::vector<std::uint32_t> spill;
  while (!stack.empty()) {
    Work w = stack.back();
    stack.pop_back();
    const std::size_t n = w.end - w.begin;
    std::span<const std::uint32_t> active(idx.data() + w.begin, n);
    std::fill(totals.begin(), totals.end(), 0u);
    for (auto s : active) totals[data.labels()[s]]++;
    const auto top = *std::max_element(totals.begin(), totals.end());
    bool split = false;
    if (top < n && n >= cfg.min_samples_split && n >= 2 &&
        (!cfg.max_depth || w.depth < *cfg.max_depth)) {
      Rng engine = make_rng(w.seed);
      SplitMethod m = cfg.mode == SplitMode::kExactOnly       ? SplitMethod::kExact
                      : cfg.mode == SplitMode::kHistogramOnly ? SplitMethod::kHistogram
                                                              : choose_method(n, breakeven);
      NodeSplitOptions opt{m, cfg.bin_count, cfg.two_level_binning};
      for (std::size_t a = 0; a <= cfg.max_split_retries && !split; ++a) {
        auto proj = sample_projection_matrix<float>(pcfg, engine);
        auto s = find_node_split(data, active, proj, opt, engine, scratch);
        if (!s) continue;
        const float* v = scratch.values.data() + s->candidate.projection_index * n;
        spill.clear();
        std::uint32_t wr = w.begin;
        for (std::size_t j = 0; j < n; ++j) {
          const auto smp = idx[w.begin + j];
          if (v[j] <= s->candidate.threshold)
            idx[wr++] = smp;
          else
            spill.push_back(smp);
        }
        const std::uint32_t nl = wr - w.begin;
        if (nl == 0 || nl == n) continue;
        std::copy(spill.begin(), spill.end(), idx.begin() + wr);
        const auto l = std::int32_t(tree.nodes.size());
        tree.nodes[w.node].projection = s->projection;
        tree.nodes[w.node].threshold = s->candidate.threshold;
        tree.nodes[w.node].left = l;
        tree.nodes[w.node].right = l + 1;
        tree.nodes.emplace_back();
        tree.nodes.emplace_back();
        stack.push_back({l + 1, w.begin + nl, w.end, w.depth + 1, derive_seed(w.seed, 2)});
        stack.push_back({l, w.begin, w.begin + nl, w.depth + 1, derive_seed(w.seed, 1)});
        split = true;
      }
    }
    if (!split)
      tree.nodes[w.node].predicted_class =
          std::int32_t(std::max_element(totals.begin(), totals.end()) - totals.begin());
  }
  return tree;
}

struct CountingRng {
  using result_type = Rng::result_type;
  Rng& e;
  uint64_t count = 0;
  static constexpr result_type min() { return Rng::min(); }
  static constexpr result_type max() { return Rng::max(); }
  result_type operator()() {
    ++count;
    return e();
  }
};

orc_split to_c(const std::optional<SplitCandidate<float>>& s) {
  orc_split o{};
  if (!s) return o;
  o.found = 1;
  o.projection_index = int32_t(s->projection_index);
  o.threshold = s->threshold;
  o.n_left = s->n_left;
  o.n_right = s->n_right;
  o.gain = s->gain;
  return o;
}

}  // namespace

extern "C" const char* orc_impl_name(void) { return "reference"; }

struct orc_dataset {
  ColumnarDataset data;
};

extern "C" int orc_dataset_create(const float* X, const int32_t* y, uint64_t n, uint64_t d,
                                  int32_t k, orc_dataset** out) {
  return orc_guard([&] { *out = new orc_dataset{make_data(X, y, n, d, k)}; });
}
extern "C" void orc_dataset_free(orc_dataset* ds) { delete ds; }

static void train_forest_impl(const ColumnarDataset& data, const orc_config* c, orc_forest** out);

extern "C" int orc_train_forest(const float* X, const int32_t* y, uint64_t n, uint64_t d,
                                int32_t k, const orc_config* c, orc_forest** out) {
  return orc_guard([&] { train_forest_impl(make_data(X, y, n, d, k), c, out); });
}

extern "C" int orc_train_forest_ds(const orc_dataset* ds, const orc_config* c, orc_forest** out) {
  return orc_guard([&] { train_forest_impl(ds->data, c, out); });
}

static void train_forest_impl(const ColumnarDataset& data, const orc_config* c, orc_forest** out) {
  const uint64_t d = data.n_features();
  const int32_t k = data.class_count();
  {
    const TrainConfig cfg = to_cfg(c);
    auto* f = new orc_forest;
    f->class_count = k;
    f->n_features = d;
    if (!custom_projection(c)) {
      Forest forest = train_forest(data, cfg);  // forest.hpp:267
      f->breakeven = forest.breakeven;
      for (const auto& t : forest.trees) f->add_tree(t);
    } else {
      // Same validation and seed derivation as train_forest (forest.hpp:270-306).
      Forest probe = train_forest(data, [&] {
        TrainConfig one = cfg;
        one.n_trees = 1;
        one.n_workers = 1;
        one.max_depth = 0;
        return one;
      }());
      f->breakeven = probe.breakeven;
      const ProjectionConfig pcfg = projection_for(c, d);
      std::vector<Tree<float>> trees(cfg.n_trees);
      parallel_for(cfg.n_trees, cfg.n_workers, [&](std::size_t t, std::size_t) {
        const std::uint64_t ts = derive_seed(cfg.seed, t + 1);
        SampleIndexSet boot = bootstrap_sample(data, cfg.bootstrap_fraction, derive_seed(ts, 0));
        trees[t] = grow_custom(data, cfg, pcfg, f->breakeven, std::move(boot.indices),
                               derive_seed(ts, 1), 0);
      });
      for (const auto& t : trees) f->add_tree(t);
    }
    *out = f;
  }
}

static void train_tree_impl(const ColumnarDataset& data, const uint32_t* active, uint64_t n_active,
                            const orc_config* c, uint64_t seed, uint64_t depth, orc_forest** out) {
  SampleIndexSet s;
  s.indices.assign(active, active + n_active);
  auto* f = new orc_forest;
  f->class_count = data.class_count();
  f->n_features = data.n_features();
  if (!custom_projection(c)) {
    f->add_tree(train_tree(data, s, to_cfg(c), seed, depth));  // forest.hpp:250
  } else {
    const TrainConfig cfg = to_cfg(c);
    f->add_tree(grow_custom(data, cfg, projection_for(c, data.n_features()),
                            cfg.breakeven ? *cfg.breakeven : kFallbackBreakeven,
                            std::move(s.indices), seed, std::uint32_t(depth)));
  }
  *out = f;
}

extern "C" int orc_train_tree(const float* X, const int32_t* y, uint64_t n, uint64_t d, int32_t k,
                              const uint32_t* active, uint64_t n_active, const orc_config* c,
                              uint64_t seed, uint64_t depth, orc_forest** out) {
  return orc_guard([&] { train_tree_impl(make_data(X, y, n, d, k), active, n_active, c, seed, depth, out); });
}

extern "C" int orc_train_tree_ds(const orc_dataset* ds, const uint32_t* active, uint64_t n_active,
                                 const orc_config* c, uint64_t seed, uint64_t depth, orc_forest** out) {
  return orc_guard([&] { train_tree_impl(ds->data, active, n_active, c, seed, depth, out); });
}

extern "C" uint64_t orc_split_mix64(uint64_t x) { return split_mix64(x); }
extern "C" uint64_t orc_derive_seed(uint64_t s, uint64_t k) { return derive_seed(s, k); }
extern "C" void orc_rng_outputs(uint64_t seed, uint64_t skip, uint64_t count, uint64_t* out) {
  Rng g = make_rng(seed);
  g.discard(skip);
  for (uint64_t i = 0; i < count; ++i) out[i] = g();
}

extern "C" int orc_generate_trunk(uint64_t n, uint64_t d, uint64_t seed, float* X, int32_t* y) {
  return orc_guard([&] {
    ColumnarDataset data = generate_trunk<float>(n, d, seed);
    for (uint64_t f = 0; f < d; ++f) std::memcpy(X + f * n, data.column(f).data(), n * 4);
    std::memcpy(y, data.labels().data(), n * 4);
  });
}

extern "C" uint64_t orc_bootstrap(uint64_t n, double fraction, uint64_t seed, uint32_t* out) {
  // bootstrap_sample only reads n_samples(); a label-only dataset keeps this cheap.
  std::vector<std::vector<float>> cols;
  std::vector<int32_t> labels(n, 0);
  ColumnarDataset d(std::move(cols), std::move(labels), {"0"});
  SampleIndexSet s = bootstrap_sample(d, fraction, seed);
  std::copy(s.indices.begin(), s.indices.end(), out);
  return s.indices.size();
}

extern "C" void orc_projection_config(uint64_t d, uint64_t* R, uint64_t* e, double* dens) {
  ProjectionConfig c = ProjectionConfig::for_features(d);
  *R = c.num_projections;
  *e = c.expected_nonzeros;
  *dens = c.cell_density;
}

extern "C" int64_t orc_sample_projection(uint64_t d, uint64_t R, double density, uint64_t seed,
                                         uint64_t skip, uint32_t* row_ptr, uint32_t* feat,
                                         float* weight, uint64_t cap, uint64_t* consumed) {
  ProjectionConfig c;
  c.n_features = d;
  c.num_projections = R;
  c.cell_density = density;
  Rng e = make_rng(seed);
  e.discard(skip);
  // sample_projection_matrix takes Rng& — count outputs by diffing against a twin engine.
  Rng twin = e;
  ProjectionMatrix<float> m = sample_projection_matrix<float>(c, e);
  uint64_t used = 0;
  while (!(twin == e)) {
    twin();
    ++used;
  }
  *consumed = used;
  uint64_t nnz = 0;
  row_ptr[0] = 0;
  for (uint64_t r = 0; r < R; ++r) {
    for (const auto& t : m.rows[r]) {
      if (nnz >= cap) return -1;
      feat[nnz] = t.feature;
      weight[nnz] = t.weight;
      ++nnz;
    }
    row_ptr[r + 1] = uint32_t(nnz);
  }
  return int64_t(nnz);
}

extern "C" uint64_t orc_binomial_draw(uint64_t cells, double density, uint64_t seed, uint64_t skip,
                                      uint64_t* consumed) {
  Rng e = make_rng(seed);
  e.discard(skip);
  CountingRng g{e};
  std::binomial_distribution<long long> b((long long)cells, density);  // projection.hpp:66
  const uint64_t z = uint64_t(b(g));
  *consumed = g.count;
  return z;
}

extern "C" void orc_apply_projection(const float* X, uint64_t n, const uint32_t* feat,
                                     const float* w, uint64_t nt, const uint32_t* active,
                                     uint64_t na, float* out) {
  uint64_t d = 0;
  for (uint64_t t = 0; t < nt; ++t) d = std::max<uint64_t>(d, feat[t] + 1);
  std::vector<int32_t> y(n, 0);
  const ColumnarDataset data = make_data(X, y.data(), n, d, 1);
  SparseRow<float> row;
  for (uint64_t t = 0; t < nt; ++t) row.push_back({feat[t], w[t]});
  std::vector<double> acc;
  apply_projection(data, row, std::span<const std::uint32_t>(active, na), std::span<float>(out, na),
                   acc);
}

extern "C" uint64_t orc_sample_boundaries(const float* v, uint64_t n, uint64_t bins, uint64_t seed,
                                          uint64_t skip, float* out, uint64_t* consumed) {
  Rng e = make_rng(seed);
  e.discard(skip);
  Rng twin = e;
  const uint64_t nb = sample_boundaries(std::span<const float>(v, n), bins, e, out);
  uint64_t used = 0;
  while (!(twin == e)) {
    twin();
    ++used;
  }
  *consumed = used;
  return nb;
}

extern "C" void orc_build_histogram(const float* v, const int32_t* y, uint64_t n, const float* b,
                                    uint64_t nb, int32_t k, uint32_t* counts) {
  build_histogram(std::span<const float>(v, n), std::span<const int32_t>(y, n),
                  std::span<const float>(b, nb), k, std::span<uint32_t>(counts, (nb + 1) * k));
}

extern "C" double orc_entropy(const uint32_t* c, int32_t k) {
  return entropy(std::span<const uint32_t>(c, k));
}

extern "C" orc_split orc_best_split_exact(const float* v, const int32_t* y, uint64_t n, int32_t k) {
  return to_c(best_split_exact(std::span<const float>(v, n), std::span<const int32_t>(y, n), k));
}

extern "C" orc_split orc_best_split_histogram(const float* b, uint64_t nb, const uint32_t* counts,
                                              int32_t k) {
  return to_c(best_split_histogram(std::span<const float>(b, nb),
                                   std::span<const uint32_t>(counts, (nb + 1) * k), k));
}

extern "C" orc_split orc_find_node_split(const float* X, const int32_t* y, uint64_t n, int32_t k,
                                         const uint32_t* active, uint64_t na,
                                         const uint32_t* row_ptr, uint64_t R, const uint32_t* feat,
                                         const float* w, int32_t method, uint64_t bins,
                                         uint64_t seed, uint64_t skip, uint64_t* consumed,
                                         float* winner_values) {
  uint64_t d = 1;
  for (uint64_t q = 0; q < row_ptr[R]; ++q) d = std::max<uint64_t>(d, feat[q] + 1);
  const ColumnarDataset data = make_data(X, y, n, d, k);
  ProjectionMatrix<float> m;
  m.rows.resize(R);
  for (uint64_t r = 0; r < R; ++r)
    for (uint32_t q = row_ptr[r]; q < row_ptr[r + 1]; ++q) m.rows[r].push_back({feat[q], w[q]});
  Rng e = make_rng(seed);
  e.discard(skip);
  Rng twin = e;
  SplitScratch<float> scratch;
  NodeSplitOptions opt{method == 1 ? SplitMethod::kHistogram : SplitMethod::kExact, bins, true};
  auto s = find_node_split(data, std::span<const std::uint32_t>(active, na), m, opt, e, scratch);
  uint64_t used = 0;
  while (!(twin == e)) {
    twin();
    ++used;
  }
  *consumed = used;
  if (!s) return orc_split{};
  if (winner_values)
    std::memcpy(winner_values, scratch.values.data() + s->candidate.projection_index * na, na * 4);
  return to_c(s->candidate);
}

// ---- model I/O (model_io.hpp:124-283): the reference's own writer, for byte-identity tests ----
#include "soforest/model_io.hpp"

extern "C" int orc_train_save_model(const float* X, const int32_t* y, uint64_t n, uint64_t d,
                                    int32_t k, const orc_config* c, const char* path) {
  return orc_guard([&] {
    const Forest forest = train_forest(make_data(X, y, n, d, k), to_cfg(c));  // forest.hpp:267
    save_model(forest, path);                                                 // model_io.hpp:124
  });
}

extern "C" int orc_load_model_summary(const char* path, uint64_t* n_trees, uint64_t* n_nodes) {
  return orc_guard([&] {
    const Forest f = load_model<float>(path);  // model_io.hpp:186 (validating loader)
    *n_trees = f.trees.size();
    uint64_t nodes = 0;
    for (const auto& t : f.trees) nodes += t.nodes.size();
    *n_nodes = nodes;
  });
}

// Forest::breakeven and Forest::calibration as the reference loader reads them (model_io.hpp:252-253).
extern "C" int orc_load_model_calibration(const char* path, uint64_t* breakeven, int32_t* has_cal,
                                          uint64_t* cal_breakeven, uint64_t* n_samples, int32_t* fallback) {
  return orc_guard([&] {
    const Forest f = load_model<float>(path);
    *breakeven = f.breakeven;
    *has_cal = f.calibration.has_value();
    *cal_breakeven = f.calibration ? f.calibration->breakeven : 0;
    *n_samples = f.calibration ? f.calibration->samples.size() : 0;
    *fallback = f.calibration ? f.calibration->fallback : 0;
  });
}

// TrainInstrumentation::by_depth node and sample counts of a reference train_forest run
// (forest.hpp:237, timing.hpp:58-63); returns the number of depths (<= cap written).
extern "C" int orc_train_forest_depths(const float* X, const int32_t* y, uint64_t n, uint64_t d, int32_t k,
                                       const orc_config* c, uint64_t* nodes, uint64_t* samples, uint64_t cap,
                                       uint64_t* n_depths) {
  return orc_guard([&] {
    TrainInstrumentation instr;
    (void)train_forest(make_data(X, y, n, d, k), to_cfg(c), &instr);
    *n_depths = instr.by_depth.size();
    for (uint64_t i = 0; i < std::min<uint64_t>(cap, instr.by_depth.size()); ++i) {
      nodes[i] = instr.by_depth[i].nodes;
      samples[i] = instr.by_depth[i].samples;
    }
  });
}

// bench.hpp:36-40 number formatting (std::to_chars), for the CSV schema tests.
extern "C" uint64_t orc_csv_number(double v, char* out, uint64_t cap) {
  std::ostringstream os;
  soforest::detail::csv_number(os, v);
  const std::string s = os.str();
  const uint64_t n = std::min<uint64_t>(s.size(), cap ? cap - 1 : 0);
  std::memcpy(out, s.data(), n);
  if (cap) out[n] = 0;
  return s.size();
}
