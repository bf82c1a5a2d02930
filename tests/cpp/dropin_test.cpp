// TEST INFRASTRUCTURE — the C++ drop-in (include/sofg/soforest_gpu.hpp) checked against the
// reference learner itself, on the reference's own types. Built by `make -C oracle dropin` against
// the reference headers (proj/include) and libsofg.so into oracle/_ref/dropin_test; run on a GPU
// box by tests/test_gpu_dropin.py. Every check mirrors a reference call site:
//   train_forest   forest.hpp:267 (Tree== as forest_test.cpp:172-204), error messages :270-276
//   train_tree     forest.hpp:250-262 (derived stream, forest_test.cpp:172-185), errors :254-256
//   predict        forest.hpp:110-121 on the GPU forest; batched GPU predict
//   save_model / load_model   model_io.hpp:124-283 (bytes identical to the reference's file)
//   TrainInstrumentation      timing.hpp:39-79 (by_depth nodes/samples)
//   calibration    forest.hpp:285-293 (record stored, serialized, reloaded)
//   bench.hpp      depth / phase / mode profiles, CSV schema via soforest::write_csv
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <sstream>
#include <string>

#include <soforest/bench.hpp>
#include <soforest/model_io.hpp>
#include <soforest/soforest.hpp>

#include "sofg/soforest_gpu.hpp"

namespace {

int g_fail = 0;
#define CHECK(cond)                                                     \
  do {                                                                  \
    if (!(cond)) {                                                      \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++g_fail;                                                         \
    }                                                                   \
  } while (0)

template <class E, class F>
void expect_throw(F&& f, const std::string& msg) {
  try {
    f();
    std::fprintf(stderr, "FAIL: expected exception '%s'\n", msg.c_str());
    ++g_fail;
  } catch (const E& e) {
    if (std::string(e.what()) != msg) {
      std::fprintf(stderr, "FAIL: message '%s' != '%s'\n", e.what(), msg.c_str());
      ++g_fail;
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "FAIL: wrong exception type for '%s': %s\n", msg.c_str(), e.what());
    ++g_fail;
  }
}

std::string file_bytes(const std::string& p) {
  std::ifstream in(p, std::ios::binary);
  return std::string(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
}

}  // namespace

int main(int argc, char** argv) {
  using namespace soforest;
  const std::string tmp = argc > 1 ? argv[1] : std::filesystem::temp_directory_path().string();
  const ColumnarDataset data = generate_trunk<float>(6000, 24, 3);
  const ColumnarDataset holdout = generate_trunk<float>(2000, 24, 4);

  TrainConfig cfg;
  cfg.n_trees = 6;
  cfg.mode = SplitMode::kDynamic;
  cfg.breakeven = 300;
  cfg.seed = 7;
  cfg.n_workers = 4;

  // ---- train_forest: same trees, same forest fields -----------------------------------------
  TrainInstrumentation gi, ci;
  const Forest g = gpu::train_forest(data, cfg, &gi);
  const Forest c = train_forest(data, cfg, &ci);
  CHECK(g.trees.size() == c.trees.size());
  for (std::size_t t = 0; t < c.trees.size(); ++t) CHECK(g.trees[t] == c.trees[t]);
  CHECK(g.n_features == c.n_features && g.class_count == c.class_count);
  CHECK(g.label_names == c.label_names && g.config == c.config && g.breakeven == c.breakeven);
  CHECK(!g.calibration.has_value());
  // instrumentation: node and sample counts per depth are functions of the trees
  CHECK(gi.by_depth.size() == ci.by_depth.size());
  for (std::size_t d = 0; d < std::min(gi.by_depth.size(), ci.by_depth.size()); ++d) {
    CHECK(gi.by_depth[d].nodes == ci.by_depth[d].nodes);
    CHECK(gi.by_depth[d].samples == ci.by_depth[d].samples);
  }
  CHECK(gi.split_seconds > 0.0 && gi.total_seconds >= gi.split_seconds);

  // ---- predict: the reference's predict on the GPU forest, and the batched GPU predict --------
  {
    gpu::Session s;
    std::vector<float> rows;
    for (std::size_t i = 0; i < holdout.n_samples(); ++i) {
      const std::vector<float> r = holdout.row(i);
      rows.insert(rows.end(), r.begin(), r.end());
    }
    const std::vector<Prediction> gp = s.predict(g, rows);
    for (std::size_t i = 0; i < holdout.n_samples(); ++i) {
      const std::vector<float> r = holdout.row(i);
      const Prediction a = predict(g, std::span<const float>(r));
      const Prediction b = predict(c, std::span<const float>(r));
      CHECK(a.label == b.label && a.votes == b.votes);
      CHECK(gp[i].label == a.label && gp[i].votes == a.votes);
    }
  }

  // ---- save_model: byte-identical files; load_model accepts ours -----------------------------
  {
    const std::string pg = tmp + "/dropin_gpu.model", pc = tmp + "/dropin_cpu.model";
    save_model(g, pg);
    save_model(c, pc);
    CHECK(file_bytes(pg) == file_bytes(pc));
    const Forest back = load_model<float>(pg);
    for (std::size_t t = 0; t < c.trees.size(); ++t) CHECK(back.trees[t] == c.trees[t]);
  }

  // ---- train_tree on a derived stream (forest_test.cpp:172-185) ------------------------------
  {
    const std::uint64_t ts = derive_seed(cfg.seed, 3);
    const SampleIndexSet boot = bootstrap_sample(data, cfg.bootstrap_fraction, derive_seed(ts, 0));
    TrainInstrumentation ti;
    const Tree<float> gt = gpu::train_tree(data, boot, cfg, derive_seed(ts, 1), 0, &ti);
    CHECK(gt == train_tree(data, boot, cfg, derive_seed(ts, 1)));
    CHECK(gt == c.trees[2]);
    CHECK(!ti.by_depth.empty() && ti.by_depth[0].nodes == 1 && ti.by_depth[0].samples == boot.size());
    SampleIndexSet sub{{5, 9, 40, 41, 77, 300, 301, 1000, 4000, 5999}};
    CHECK(gpu::train_tree(data, sub, cfg, 99, 2) == train_tree(data, sub, cfg, 99, 2));
  }

  // ---- errors: the reference's exception types and messages --------------------------------
  {
    TrainConfig bad = cfg;
    bad.n_trees = 0;
    expect_throw<std::invalid_argument>([&] { gpu::train_forest(data, bad); }, "n_trees must be positive");
    bad = cfg;
    bad.bin_count = 1;
    expect_throw<std::invalid_argument>([&] { gpu::train_forest(data, bad); }, "bin_count must be at least 2");
    bad = cfg;
    bad.bootstrap_fraction = 1.5;
    expect_throw<std::invalid_argument>([&] { gpu::train_forest(data, bad); },
                                        "bootstrap fraction must be in (0, 1]");
    expect_throw<std::invalid_argument>([&] { gpu::train_tree(data, SampleIndexSet{}, cfg, 1); },
                                        "active sample set is empty");
    expect_throw<std::out_of_range>([&] { gpu::train_tree(data, SampleIndexSet{{1, 6000}}, cfg, 1); },
                                    "sample index out of range");
    const ColumnarDataset one({{1.f, 2.f, 3.f}}, {0, 0, 0}, {"only"});
    expect_throw<std::invalid_argument>([&] { gpu::train_forest(one, cfg); }, "need at least 2 classes");
  }

  // ---- calibration: Dynamic without a breakeven calibrates and records (forest.hpp:285-293) ---
  {
    TrainConfig cal_cfg = cfg;
    cal_cfg.breakeven.reset();
    cal_cfg.n_trees = 3;
    const Forest gc = gpu::train_forest(data, cal_cfg);
    CHECK(gc.calibration.has_value());
    if (gc.calibration) {
      CHECK(gc.breakeven == gc.calibration->breakeven);
      CHECK(!gc.calibration->samples.empty() && gc.calibration->samples.front().n == cal_cfg.calibration.n_min);
      // one sample only when the histogram probe already won at n_min (calibrate.hpp:84)
      if (gc.calibration->samples.size() == 1) CHECK(gc.breakeven == cal_cfg.calibration.n_min);
    }
    TrainConfig at = cal_cfg;
    at.breakeven = gc.breakeven;
    const Forest cc = train_forest(data, at);
    for (std::size_t t = 0; t < cc.trees.size(); ++t) CHECK(gc.trees[t] == cc.trees[t]);
    const std::string p = tmp + "/dropin_cal.model";
    save_model(gc, p);
    const Forest back = load_model<float>(p);
    CHECK(back.calibration.has_value() && back.breakeven == gc.breakeven);
    if (back.calibration && gc.calibration) CHECK(back.calibration->samples.size() == gc.calibration->samples.size());
  }

  // ---- bench.hpp profiles: same rows (nodes / samples per depth) and the same CSV schema -------
  {
    TrainConfig b = cfg;
    b.n_trees = 3;
    const auto gd = gpu::bench_depth_profile(data, b);
    const auto cd = bench_depth_profile(data, b);
    CHECK(gd.size() == cd.size());
    for (std::size_t i = 0; i < std::min(gd.size(), cd.size()); ++i) {
      CHECK(gd[i].depth == cd[i].depth && gd[i].mode == cd[i].mode);
      CHECK(gd[i].nodes == cd[i].nodes && gd[i].samples == cd[i].samples);
    }
    const auto gp = gpu::bench_phase_profile(data, b);
    const auto cp = bench_phase_profile(data, b);
    CHECK(gp.size() == cp.size());
    for (std::size_t i = 0; i < std::min(gp.size(), cp.size()); ++i)
      CHECK(gp[i].phase == cp[i].phase && gp[i].depth_bucket == cp[i].depth_bucket);
    const auto gm = gpu::bench_mode_comparison(data, b);
    CHECK(gm.size() == 4 && gm[0].mode == "exact" && gm[0].normalized == 1.0 && gm[3].mode == "dynamic_two_level");
    std::ostringstream a, bb, cc2;
    write_csv(gd, a);
    write_csv(gp, bb);
    write_csv(gm, cc2);
    CHECK(a.str().rfind("depth,mode,seconds,nodes,samples\n", 0) == 0);
    CHECK(bb.str().rfind("phase,depth_bucket,seconds\n", 0) == 0);
    CHECK(cc2.str().rfind("mode,seconds,normalized\n", 0) == 0);
    std::ofstream(tmp + "/dropin_depth_profile.csv") << a.str();
    std::ofstream(tmp + "/dropin_phase_profile.csv") << bb.str();
    std::ofstream(tmp + "/dropin_mode_comparison.csv") << cc2.str();
  }

  if (g_fail) {
    std::fprintf(stderr, "dropin_test: %d check(s) failed\n", g_fail);
    return 1;
  }
  std::printf("dropin_test: all checks passed (%zu trees bit-identical, files byte-identical)\n", c.trees.size());
  return 0;
}
