// C++ API of the B200 sparse-oblique forest trainer — mirrors the reference learner's public
// train/predict surface (soforest, /root/reference/proj/include/soforest/forest.hpp) so a caller
// of soforest::train_forest can switch to sofg::train_forest with the same arguments and get the
// same trees (bit-exact, same seeds). Implemented in paper_2603_00326_b200/lib/libsofg.so on top
// of the C ABI in include/sofg.h.
//
//   reference                                   here
//   soforest::BasicColumnarDataset<float>       sofg::ColumnarDataset   (dataset.hpp:23-69)
//   soforest::TrainConfig                       sofg::TrainConfig       (forest.hpp:38-53)
//   soforest::Tree / TreeNode / Forest          sofg::Tree / TreeNode / Forest (forest.hpp:55-83)
//   soforest::train_forest(data, cfg)           sofg::train_forest(data, cfg)  (forest.hpp:267)
//   soforest::train_tree(data, active, cfg, s)  sofg::train_tree(...)          (forest.hpp:250)
//   soforest::predict(forest, sample)           sofg::predict(forest, sample)  (forest.hpp:110)
#pragma once
#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace sofg {

enum class SplitMode { kExactOnly, kHistogramOnly, kDynamic };

inline constexpr std::size_t kFallbackBreakeven = 1024;  // reference calibrate.hpp:43

struct TrainConfig {
  std::size_t n_trees = 100;
  SplitMode mode = SplitMode::kDynamic;
  std::size_t bin_count = 256;
  bool two_level_binning = true;           // accepted for parity; binning is exact either way
  std::optional<std::size_t> breakeven;    // Dynamic only; the reference calibrates when absent,
                                           // this trainer uses kFallbackBreakeven
  double bootstrap_fraction = 0.632;
  std::optional<std::size_t> max_depth;
  std::size_t min_samples_split = 2;
  std::size_t max_split_retries = 1;
  std::size_t n_workers = 1;               // host threads (0 = all cores)
  std::uint64_t seed = 0;
  // extensions (not in the reference)
  std::size_t num_projections = 0;         // 0: ProjectionConfig::for_features(d)
  double cell_density = 0.0;               // <= 0: for_features(d) density
  std::size_t batch_trees = 0;             // trees grown together per level launch (0 = auto)
  int device = 0;
};

struct ProjectionTerm {
  std::uint32_t feature = 0;
  float weight = 0.f;
  bool operator==(const ProjectionTerm&) const = default;
};
using SparseRow = std::vector<ProjectionTerm>;

struct TreeNode {
  SparseRow projection;
  float threshold = 0.f;
  std::int32_t left = -1;
  std::int32_t right = -1;
  std::int32_t predicted_class = -1;
  bool is_leaf() const { return left < 0; }
  bool operator==(const TreeNode&) const = default;
};

struct Tree {
  std::vector<TreeNode> nodes;
  bool operator==(const Tree&) const = default;
};

struct Forest {
  std::uint32_t n_features = 0;
  std::int32_t class_count = 0;
  std::vector<std::string> label_names;
  TrainConfig config{};
  std::size_t breakeven = 0;
  std::vector<Tree> trees;
};

// Feature-major table, one contiguous column per feature (reference dataset.hpp:23-69).
class ColumnarDataset {
 public:
  ColumnarDataset() = default;
  ColumnarDataset(std::vector<std::vector<float>> columns, std::vector<std::int32_t> labels,
                  std::vector<std::string> label_names);
  std::size_t n_samples() const { return labels_.size(); }
  std::size_t n_features() const { return columns_.size(); }
  std::int32_t class_count() const { return std::int32_t(label_names_.size()); }
  std::span<const float> column(std::size_t f) const { return columns_[f]; }
  std::span<const std::int32_t> labels() const { return labels_; }
  const std::vector<std::string>& label_names() const { return label_names_; }

 private:
  std::vector<std::vector<float>> columns_;
  std::vector<std::int32_t> labels_;
  std::vector<std::string> label_names_;
};

struct SampleIndexSet {
  std::vector<std::uint32_t> indices;
};

struct Prediction {
  std::int32_t label = -1;
  std::vector<double> votes;
};

Forest train_forest(const ColumnarDataset& data, const TrainConfig& cfg);
Tree train_tree(const ColumnarDataset& data, const SampleIndexSet& active, const TrainConfig& cfg,
                std::uint64_t seed, std::size_t depth = 0);
Prediction predict(const Forest& forest, std::span<const float> sample);

}  // namespace sofg
