// soforest::gpu — the B200 trainer as a drop-in for the reference learner's C++ API, on the
// reference's OWN types (soforest, proj/include/soforest). Header-only over the C ABI (sofg.h):
// include it where the reference headers are on the include path and link libsofg.so.
//
//   reference (proj/include/soforest)                        here (same signature, GPU)
//   train_forest(data, cfg, instr)        forest.hpp:267-313  soforest::gpu::train_forest(data, cfg, instr)
//   train_tree(data, active, cfg, seed,   forest.hpp:250-262  soforest::gpu::train_tree(...)
//              depth, instr)
//   calibrate_crossover<T>(opt)           calibrate.hpp:135   soforest::gpu::Session::calibrate_crossover(opt)
//   predict(forest, sample)               forest.hpp:110-121  soforest::predict (unchanged: the forest IS a
//                                                             BasicForest<float>); batched GPU predict:
//                                                             soforest::gpu::Session::predict
//   bench_depth_profile / bench_phase_    bench.hpp:53-123    soforest::gpu::bench_* (same row types;
//   profile / bench_mode_comparison                           soforest::write_csv writes the same CSV)
//
// The returned BasicForest<float> is the reference's type, field for field (n_features,
// class_count, label_names, config, breakeven, calibration, trees), so soforest::predict,
// soforest::save_model and the CLI consume it unchanged. Trees are bit-identical to the
// reference's for the same data and TrainConfig (seeds, breakeven). Errors are the reference's:
// std::invalid_argument / std::out_of_range with the reference's messages, std::runtime_error for
// CUDA failures; there is no CPU fallback.
//
// Only T = float (the reference's ColumnarDataset, and its benchmark type) is supported on the GPU.
#pragma once

#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include <soforest/bench.hpp>
#include <soforest/forest.hpp>

#include "../sofg.h"

namespace soforest::gpu {

namespace detail {

[[noreturn]] inline void rethrow(int rc) {
  std::string m = sofg_last_error();
  for (const char* prefix : {"invalid_argument: ", "out_of_range: ", "runtime_error: "}) {
    const std::size_t len = std::strlen(prefix);
    if (m.compare(0, len, prefix) == 0) {
      m.erase(0, len);  // the C ABI tags the exception class; rethrow with the reference's text
      break;
    }
  }
  if (rc == 1) throw std::invalid_argument(m);
  if (rc == 2) throw std::out_of_range(m);
  throw std::runtime_error(m);
}

inline void check(int rc) {
  if (rc) rethrow(rc);
}

inline int default_device() {
  const char* e = std::getenv("SOFG_DEVICE");
  return e ? std::atoi(e) : 0;
}

inline sofg_train_config to_c(const TrainConfig& t) {
  sofg_train_config c;
  sofg_default_config(&c);
  c.n_trees = t.n_trees;
  c.mode = t.mode == SplitMode::kExactOnly ? 0 : t.mode == SplitMode::kHistogramOnly ? 1 : 2;
  c.two_level_binning = t.two_level_binning;
  c.bin_count = t.bin_count;
  c.has_breakeven = t.breakeven.has_value();
  c.breakeven = t.breakeven.value_or(0);
  c.has_max_depth = t.max_depth.has_value();
  c.max_depth = t.max_depth.value_or(0);
  c.bootstrap_fraction = t.bootstrap_fraction;
  c.min_samples_split = t.min_samples_split;
  c.max_split_retries = t.max_split_retries;
  c.n_workers = t.n_workers;
  c.seed = t.seed;
  c.calibration.n_min = t.calibration.n_min;
  c.calibration.n_max = t.calibration.n_max;
  c.calibration.budget_seconds = t.calibration.budget_seconds;
  c.calibration.bin_count = t.calibration.bin_count;
  c.calibration.two_level = t.calibration.two_level;
  c.calibration.repetitions = t.calibration.repetitions;
  c.calibration.seed = t.calibration.seed;
  return c;
}

inline CrossoverCalibration from_c(const sofg_calibration& c) {
  CrossoverCalibration out;
  out.breakeven = c.breakeven;
  out.elapsed_seconds = c.elapsed_seconds;
  out.fallback = c.fallback != 0;
  for (uint64_t i = 0; i < c.n_samples; ++i)
    out.samples.push_back({c.samples[i].n, c.samples[i].exact_seconds, c.samples[i].histogram_seconds});
  return out;
}

// The library's flat forest (node ids in the reference's depth-first order) as reference trees.
inline std::vector<Tree<float>> trees_of(const sofg_forest* f) {
  const void* a[8];
  sofg_forest_arrays(f, a);
  const auto* tree_off = static_cast<const int64_t*>(a[0]);
  const auto* left = static_cast<const int32_t*>(a[1]);
  const auto* right = static_cast<const int32_t*>(a[2]);
  const auto* pred = static_cast<const int32_t*>(a[3]);
  const auto* thr = static_cast<const float*>(a[4]);
  const auto* term_off = static_cast<const int64_t*>(a[5]);
  const auto* feat = static_cast<const uint32_t*>(a[6]);
  const auto* weight = static_cast<const float*>(a[7]);
  std::vector<Tree<float>> out(sofg_forest_num_trees(f));
  for (std::size_t t = 0; t < out.size(); ++t) {
    auto& nodes = out[t].nodes;
    nodes.resize(std::size_t(tree_off[t + 1] - tree_off[t]));
    for (std::size_t i = 0; i < nodes.size(); ++i) {
      const std::size_t q = std::size_t(tree_off[t]) + i;
      TreeNode<float>& nd = nodes[i];
      nd.left = left[q];
      nd.right = right[q];
      nd.predicted_class = pred[q];
      nd.threshold = thr[q];
      for (int64_t u = term_off[q]; u < term_off[q + 1]; ++u)
        nd.projection.push_back({feat[u], weight[u]});
    }
  }
  return out;
}

// Adds a run's per-depth accounting to `instr` the way train_forest merges its workers'
// (forest.hpp:309-312): by_depth and phases accumulate, total_seconds is the run's.
inline void merge_instrumentation(const sofg_forest* f, TrainInstrumentation& instr) {
  const uint64_t nd = sofg_forest_instrumentation(f, nullptr, nullptr, nullptr, 0, nullptr, nullptr, nullptr);
  std::vector<double> sec(nd);
  std::vector<uint64_t> nodes(nd), samples(nd);
  sofg_phase_times ph[kDepthBuckets];
  double split = 0.0, total = 0.0;
  sofg_forest_instrumentation(f, sec.data(), nodes.data(), samples.data(), nd, ph, &split, &total);
  TrainInstrumentation run;
  run.by_depth.resize(nd);
  for (uint64_t d = 0; d < nd; ++d) run.by_depth[d] = {sec[d], nodes[d], samples[d]};
  for (std::size_t b = 0; b < kDepthBuckets; ++b)
    run.phases[b] = {ph[b].sample_projections, ph[b].apply_projections, ph[b].build_histograms,
                     ph[b].evaluate_splits};
  run.split_seconds = split;
  instr.merge(run);
  instr.total_seconds = total;
}

struct ForestHandle {
  sofg_forest* f = nullptr;
  ForestHandle() = default;
  ForestHandle(const ForestHandle&) = delete;
  ForestHandle& operator=(const ForestHandle&) = delete;
  ~ForestHandle() { sofg_forest_free(f); }
};

// forest.hpp:270-276, in the reference's order and words, before anything touches the GPU.
template <typename T>
void validate(const BasicColumnarDataset<T>& data, const TrainConfig& cfg) {
  if (cfg.n_trees < 1) throw std::invalid_argument("n_trees must be positive");
  if (cfg.bin_count < 2) throw std::invalid_argument("bin_count must be at least 2");
  if (cfg.min_samples_split < 2) throw std::invalid_argument("min_samples_split must be at least 2");
  if (!(cfg.bootstrap_fraction > 0.0) || cfg.bootstrap_fraction > 1.0)
    throw std::invalid_argument("bootstrap fraction must be in (0, 1]");
  if (data.n_samples() < 2) throw std::invalid_argument("need at least 2 samples");
  if (data.class_count() < 2) throw std::invalid_argument("need at least 2 classes");
}

}  // namespace detail

// One GPU context with a resident dataset. Reuse a Session to train several forests (or probe,
// predict) on one dataset without re-uploading it; one host thread per Session.
class Session {
 public:
  explicit Session(int device = detail::default_device()) { detail::check(sofg_create(device, &ctx_)); }
  ~Session() { sofg_destroy(ctx_); }
  Session(const Session&) = delete;
  Session& operator=(const Session&) = delete;

  // Uploads the table (column by column, the reference's layout) and labels to HBM.
  void upload(const ColumnarDataset& data) {
    std::vector<const float*> cols(data.n_features());
    for (std::size_t f = 0; f < cols.size(); ++f) cols[f] = data.column(f).data();
    detail::check(sofg_upload_columns(ctx_, cols.data(), data.n_samples(), data.n_features(),
                                      data.labels().data(), data.class_count()));
    n_features_ = static_cast<std::uint32_t>(data.n_features());
    class_count_ = data.class_count();
    label_names_ = data.label_names();
  }

  // train_forest on the resident dataset (forest.hpp:267-313).
  Forest train_forest(const TrainConfig& cfg, TrainInstrumentation* instr = nullptr) {
    sofg_train_config c = detail::to_c(cfg);
    c.instrument = instr != nullptr;
    detail::ForestHandle h;
    detail::check(sofg_train_forest(ctx_, &c, &h.f));
    Forest forest;
    forest.n_features = n_features_;
    forest.class_count = class_count_;
    forest.label_names = label_names_;
    forest.config = cfg;
    forest.breakeven = sofg_forest_breakeven(h.f);
    sofg_calibration cal;
    if (sofg_forest_calibration(h.f, &cal)) forest.calibration = detail::from_c(cal);
    forest.trees = detail::trees_of(h.f);
    if (instr) detail::merge_instrumentation(h.f, *instr);
    return forest;
  }

  // train_tree on the resident dataset (forest.hpp:250-262).
  Tree<float> train_tree(const SampleIndexSet& active, const TrainConfig& cfg, std::uint64_t seed,
                         std::size_t depth = 0, TrainInstrumentation* instr = nullptr) {
    sofg_train_config c = detail::to_c(cfg);
    c.instrument = instr != nullptr;
    detail::ForestHandle h;
    detail::check(sofg_train_tree(ctx_, active.indices.data(), active.indices.size(), &c, seed, depth, &h.f));
    if (instr) detail::merge_instrumentation(h.f, *instr);
    return std::move(detail::trees_of(h.f).at(0));
  }

  // calibrate_crossover (calibrate.hpp:51-196): the reference's search with GPU probes.
  CrossoverCalibration calibrate_crossover(const CalibrationOptions& opt = {}) {
    TrainConfig cfg;
    cfg.calibration = opt;
    const sofg_train_config c = detail::to_c(cfg);
    sofg_calibration out;
    detail::check(sofg_calibrate(ctx_, &c, &out));
    return detail::from_c(out);
  }

  // predict (forest.hpp:110-121) for n_rows row-major samples in one GPU launch.
  std::vector<Prediction> predict(const Forest& forest, std::span<const float> rows) {
    if (forest.n_features == 0 || rows.size() % forest.n_features != 0)
      throw std::invalid_argument("row buffer is not a whole number of samples");
    const std::size_t n_rows = rows.size() / forest.n_features;
    std::vector<int64_t> tree_off{0}, term_off{0};
    std::vector<int32_t> left, right, pred;
    std::vector<float> thr, weight;
    std::vector<uint32_t> feat;
    for (const auto& t : forest.trees) {
      for (const auto& nd : t.nodes) {
        left.push_back(nd.left);
        right.push_back(nd.right);
        pred.push_back(nd.predicted_class);
        thr.push_back(nd.threshold);
        for (const auto& term : nd.projection) {
          feat.push_back(term.feature);
          weight.push_back(term.weight);
        }
        term_off.push_back(int64_t(feat.size()));
      }
      tree_off.push_back(int64_t(left.size()));
    }
    detail::ForestHandle h;
    detail::check(sofg_forest_import(forest.trees.size(), forest.n_features, forest.class_count, tree_off.data(),
                                     left.data(), right.data(), pred.data(), thr.data(), term_off.data(),
                                     feat.data(), weight.data(), &h.f));
    std::vector<int32_t> labels(n_rows);
    std::vector<double> votes(n_rows * std::size_t(forest.class_count));
    detail::check(sofg_predict(ctx_, h.f, rows.data(), n_rows, forest.n_features, labels.data(), votes.data()));
    std::vector<Prediction> out(n_rows);
    for (std::size_t i = 0; i < n_rows; ++i) {
      out[i].label = labels[i];
      out[i].votes.assign(votes.begin() + std::ptrdiff_t(i * forest.class_count),
                          votes.begin() + std::ptrdiff_t((i + 1) * forest.class_count));
    }
    return out;
  }

  sofg_ctx* handle() const { return ctx_; }

 private:
  sofg_ctx* ctx_ = nullptr;
  std::uint32_t n_features_ = 0;
  std::int32_t class_count_ = 0;
  std::vector<std::string> label_names_;
};

// ---- the reference's free functions, same signatures -------------------------------------

template <typename T>
BasicForest<T> train_forest(const BasicColumnarDataset<T>& data, const TrainConfig& cfg,
                            TrainInstrumentation* instr = nullptr) {
  static_assert(std::is_same_v<T, float>, "the GPU trainer computes in float (ColumnarDataset)");
  detail::validate(data, cfg);
  Session s;
  s.upload(data);
  return s.train_forest(cfg, instr);
}

template <typename T>
Tree<T> train_tree(const BasicColumnarDataset<T>& data, const SampleIndexSet& active, const TrainConfig& cfg,
                   std::uint64_t seed, std::size_t depth = 0, TrainInstrumentation* instr = nullptr) {
  static_assert(std::is_same_v<T, float>, "the GPU trainer computes in float (ColumnarDataset)");
  if (active.indices.empty()) throw std::invalid_argument("active sample set is empty");  // forest.hpp:254
  for (std::uint32_t s : active.indices)
    if (s >= data.n_samples()) throw std::out_of_range("sample index out of range");  // :256
  Session s;
  s.upload(data);
  return s.train_tree(active, cfg, seed, depth, instr);
}

// ---- bench.hpp:53-123 on the GPU: same rows, so soforest::write_csv emits the same CSV --------

namespace detail {
// bench.hpp:47-51: Dynamic runs of one harness call share one calibration.
inline TrainConfig resolved(Session& s, const TrainConfig& base) {
  TrainConfig cfg = base;
  if (!cfg.breakeven) cfg.breakeven = s.calibrate_crossover(cfg.calibration).breakeven;
  return cfg;
}
}  // namespace detail

template <typename T>
std::vector<DepthProfileRow> bench_depth_profile(const BasicColumnarDataset<T>& data, const TrainConfig& base) {
  Session s;
  s.upload(data);
  const TrainConfig cfg = detail::resolved(s, base);
  std::vector<DepthProfileRow> rows;
  for (SplitMode mode : {SplitMode::kExactOnly, SplitMode::kHistogramOnly, SplitMode::kDynamic}) {
    TrainConfig c = cfg;
    c.mode = mode;
    TrainInstrumentation instr;
    s.train_forest(c, &instr);
    for (std::size_t d = 0; d < instr.by_depth.size(); ++d) {
      const DepthAccum& a = instr.by_depth[d];
      rows.push_back({d, split_mode_name(mode), a.seconds, a.nodes, a.samples});
    }
  }
  return rows;
}

template <typename T>
std::vector<PhaseProfileRow> bench_phase_profile(const BasicColumnarDataset<T>& data, const TrainConfig& base) {
  Session s;
  s.upload(data);
  const TrainConfig cfg = detail::resolved(s, base);
  TrainInstrumentation instr;
  s.train_forest(cfg, &instr);
  std::vector<PhaseProfileRow> rows;
  for (std::size_t b = 0; b < kDepthBuckets; ++b) {
    const SplitPhaseTimes& p = instr.phases[b];
    const char* bucket = depth_bucket_name(b);
    rows.push_back({"sample_projections", bucket, p.sample_projections});
    rows.push_back({"apply_projections", bucket, p.apply_projections});
    rows.push_back({"build_histograms", bucket, p.build_histograms});
    rows.push_back({"evaluate_splits", bucket, p.evaluate_splits});
  }
  return rows;
}

template <typename T>
std::vector<ModeComparisonRow> bench_mode_comparison(const BasicColumnarDataset<T>& data, const TrainConfig& base) {
  Session s;
  s.upload(data);
  const TrainConfig cfg = detail::resolved(s, base);
  struct Run {
    const char* name;
    SplitMode mode;
    bool two_level;
  };
  constexpr Run runs[] = {
      {"exact", SplitMode::kExactOnly, true},
      {"histogram", SplitMode::kHistogramOnly, true},
      {"dynamic_scalar", SplitMode::kDynamic, false},
      {"dynamic_two_level", SplitMode::kDynamic, true},
  };
  std::vector<ModeComparisonRow> rows;
  for (const Run& run : runs) {
    TrainConfig c = cfg;
    c.mode = run.mode;
    c.two_level_binning = run.two_level;
    Stopwatch clock;
    s.train_forest(c);
    rows.push_back({run.name, clock.seconds(), 0.0});
  }
  const double exact_seconds = rows[0].seconds;
  for (auto& row : rows) row.normalized = row.seconds / exact_seconds;
  return rows;
}

}  // namespace soforest::gpu
