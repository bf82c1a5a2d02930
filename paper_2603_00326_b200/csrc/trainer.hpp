// Level-wise frontier scheduler: grows a batch of trees one depth at a time, every open node of
// the depth searched and partitioned by one wave of kernels (engine.hpp). Replaces the
// reference's depth-first per-node loop detail::TreeGrower::grow_from (forest.hpp:157-240) while
// reproducing its trees exactly: per-node engines depend only on the node seed
// (forest.hpp:183,226,228), so level order does not change any random stream, and node ids are
// restored by replaying the reference's depth-first split order at the end.
#pragma once
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <memory>
#include <type_traits>
#include <mutex>
#include <optional>
#include <thread>
#include <vector>

#include "engine.hpp"

namespace sofg {

// std::vector whose resize() leaves trivially-constructible elements uninitialized (the forest
// arrays are written in parallel right after sizing; zero-filling them first is a serial pass).
template <class T, class A = std::allocator<T>>
struct default_init_allocator : A {
  using A::A;
  template <class U>
  struct rebind {
    using other = default_init_allocator<U, typename std::allocator_traits<A>::template rebind_alloc<U>>;
  };
  template <class U>
  void construct(U* p) noexcept(std::is_nothrow_default_constructible<U>::value) {
    ::new (static_cast<void*>(p)) U;
  }
  template <class U, class... Args>
  void construct(U* p, Args&&... args) {
    std::allocator_traits<A>::construct(static_cast<A&>(*this), p, std::forward<Args>(args)...);
  }
};
template <class T>
using pod_vector = std::vector<T, default_init_allocator<T>>;

struct FlatForest {
  pod_vector<int64_t> tree_off{0};
  pod_vector<int32_t> left, right, pred;
  pod_vector<float> thr;
  pod_vector<int64_t> term_off{0};
  pod_vector<uint32_t> feat;
  pod_vector<float> weight;
  uint64_t breakeven = 0;
  int32_t class_count = 0;
  uint64_t n_features = 0;
  uint64_t n_trees() const { return tree_off.size() - 1; }
};

// Freed forests' arrays are kept (up to two) and handed to the next training's output, so a
// step does not fault in hundreds of MB of fresh pages for its forest.
void recycle_forest(FlatForest&& f);
void adopt_recycled(FlatForest& out);

// Per-depth accounting of a training run, the GPU counterpart of soforest::TrainInstrumentation
// (timing.hpp:39-79): every tree node (internal and leaf) is counted at its depth with its sample
// count; seconds are the device time of the waves at that depth (CUDA events; a wave is every open
// node of the depth across the tree batch), and the split phases are summed per depth bucket
// (timing.hpp:50-56: depth / 5, capped at 3).
struct DepthProfile {
  static constexpr int kBuckets = 4;
  std::vector<double> seconds;
  std::vector<uint64_t> nodes, samples;
  double phases[kBuckets][4] = {};  // sample_projections, apply_projections, build_histograms, evaluate_splits
  double split_seconds = 0.0;
  void add(size_t depth, double s, uint64_t n_nodes, uint64_t n_samples) {
    if (seconds.size() <= depth) {
      seconds.resize(depth + 1, 0.0);
      nodes.resize(depth + 1, 0);
      samples.resize(depth + 1, 0);
    }
    seconds[depth] += s;
    nodes[depth] += n_nodes;
    samples[depth] += n_samples;
  }
  static int bucket(size_t depth) { return int(std::min<size_t>(depth / 5, kBuckets - 1)); }
};

struct TrainParams {
  int mode = 2;  // 0 exact-only, 1 histogram-only, 2 dynamic
  uint64_t bins = 256;
  bool two_level = true;   // two_level_binning
  uint64_t breakeven = 1024;
  std::optional<uint64_t> max_depth;
  uint64_t min_samples_split = 2;
  uint64_t max_split_retries = 1;
  uint32_t R = 0;          // projection rows
  double density = 0.0;    // cell density
  uint64_t batch_trees = 0;
  int host_threads = 0;
  DepthProfile* profile = nullptr;  // filled when set (requires WaveRunner::collect_stats)
  // Background host work run in the waits for a wave (levels whose kernels outlast the host's
  // work): called repeatedly while the wave is in flight, each call one bounded chunk; returns
  // false when nothing is left.
  std::function<bool()> idle_work;
};

// Minimal fork-join pool for the per-node host work (binomial draws, bootstraps).
class ThreadPool {
 public:
  explicit ThreadPool(int n);
  ~ThreadPool();
  int size() const { return int(workers_.size()) + 1; }
  // f(i) for i in [0, n), caller participates.
  void parallel_for(size_t n, const std::function<void(size_t)>& f);
  // Splits [0, n) into contiguous chunks (at least `grain` items each) and runs
  // f(chunk, begin, end) in parallel; returns the chunk boundaries (size chunks + 1).
  std::vector<size_t> chunks(size_t n, size_t grain,
                             const std::function<void(size_t, size_t, size_t)>& f);

 private:
  void worker();
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(size_t)>* job_ = nullptr;
  size_t job_n_ = 0;
  std::atomic<size_t> next_{0};
  int active_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

struct HostTimes {
  double ms_binomial = 0, ms_bootstrap = 0, ms_total = 0;
  double ms_roots = 0, ms_prep = 0, ms_submit = 0, ms_spec = 0, ms_wait = 0, ms_post = 0,
         ms_final = 0, ms_book = 0;
  uint64_t levels = 0;
};

// Grows one tree per root (sorted active set + root seed) at depth offset root_depth and
// appends them, renumbered in the reference's node order, to `out`.
void grow_trees(WaveRunner& eng, const TrainParams& P, ThreadPool& pool,
                const std::vector<std::vector<uint32_t>>& roots,
                const std::vector<uint64_t>& root_seeds, uint32_t root_depth, FlatForest& out,
                HostTimes& times);

}  // namespace sofg
