// C ABI (include/sofg.h) and C++ API (include/sofg/soforest_gpu.hpp) over the level-wise trainer.
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <thread>
#include <memory>
#include <mutex>
#include <string>

#include "../../include/sofg.h"
#include "calibrate.hpp"
#include "engine.hpp"
#include "host_rng.hpp"
#include "kernels.hpp"
#include "trainer.hpp"

// Bootstrap samples computed ahead in the host's idle time during training (the waits for long
// waves): the next batch of the same call, or the tree range a following call with the same
// seed would train next. Tree t's sample is a pure function of (n, fraction, seed, t)
// (forest.hpp:153,305), so a prefetched sample is the one the call would compute.
struct BootAhead {
  uint64_t n = 0, seed = 0, t0 = 0, t1 = 0, next = 0;
  double frac = 0.0;
  std::vector<std::vector<uint32_t>> roots;  // trees [t0, t1); filled for [t0, next)
  void plan(uint64_t n_, double f, uint64_t s, uint64_t a, uint64_t b) {
    if (n == n_ && frac == f && seed == s && t0 == a && t1 == b) return;  // keep what is done
    n = n_;
    frac = f;
    seed = s;
    t0 = a;
    t1 = b;
    next = a;
    roots.assign(size_t(b - a), {});
  }
  bool take(uint64_t n_, double f, uint64_t s, uint64_t t, std::vector<uint32_t>& out) {
    if (n != n_ || frac != f || seed != s || t < t0 || t >= next) return false;
    std::vector<uint32_t>& r = roots[size_t(t - t0)];
    if (r.empty()) return false;
    out.swap(r);
    return true;
  }
};

// Per device, over all contexts of the process: trainings in progress, and table uploads some
// call is waiting for (see upload: how many slices a feeder keeps in flight).
std::atomic<int> g_training[64];
std::atomic<int> g_waited[64];
struct TrainingMark {
  int dev;
  explicit TrainingMark(int d) : dev(d & 63) { g_training[dev].fetch_add(1); }
  ~TrainingMark() { g_training[dev].fetch_sub(1); }
};

struct sofg_ctx {
  BootAhead ahead;
  std::unique_ptr<sofg::WaveRunner> eng;
  std::unique_ptr<sofg::ThreadPool> pool;
  int pool_threads = 0;
  sofg::HostTimes times;
  int stats_mode = 0;
  // Page-locked table uploads are fed to the copy engine in slices by this thread (one slice in
  // flight), so other contexts' small copies on the same GPU are not queued behind a 16 GB copy;
  // every later call on the context joins it first (its device work is stream-ordered after it).
  std::thread feeder;
  std::exception_ptr feeder_error;
  std::atomic<bool> feeder_waited{false};  // a call of this context is waiting for the feeder
  int feeder_dev = 0;
  void join_feeder() {
    if (feeder.joinable()) {
      feeder_waited = true;
      g_waited[feeder_dev & 63].fetch_add(1);
      feeder.join();
      g_waited[feeder_dev & 63].fetch_sub(1);
      feeder_waited = false;
    }
    if (feeder_error) {
      std::exception_ptr e = feeder_error;
      feeder_error = nullptr;
      std::rethrow_exception(e);
    }
  }
  ~sofg_ctx() {
    if (feeder.joinable()) feeder.join();
  }
};

struct sofg_forest {
  sofg::FlatForest f;
  bool has_cal = false;
  sofg_calibration cal{};
  bool has_prof = false;
  sofg::DepthProfile prof;
  double total_seconds = 0.0;
};

using sofg::cuda_check;
using sofg::DevBuf;
using sofg::launch_generate_trunk;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = std::string("invalid_argument: ") + e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = std::string("out_of_range: ") + e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = std::string("runtime_error: ") + e.what();
    return 3;
  }
}

void require_ctx(sofg_ctx* c) {
  if (!c || !c->eng) throw std::invalid_argument("null context");
}
void require_data(sofg_ctx* c) {
  require_ctx(c);
  c->join_feeder();
  if (!c->eng->data().loaded()) throw std::invalid_argument("no dataset uploaded");
}

int hw_threads() {
  const unsigned h = std::thread::hardware_concurrency();
  return h ? int(h) : 4;
}

sofg::ThreadPool& pool_for(sofg_ctx* c, uint64_t n_workers) {
  int want = n_workers ? int(n_workers) : hw_threads();
  want = std::max(1, std::min(want, hw_threads()));
  if (!c->pool || c->pool_threads != want) {
    c->eng->set_pool(nullptr);
    c->pool.reset(new sofg::ThreadPool(want));
    c->pool_threads = want;
  }
  c->eng->set_pool(c->pool.get());
  return *c->pool;
}

// xlogx tables (split.hpp:55-62) indexed by node size: entries 0..m. A node's size is at most its
// active set's length, which may exceed n_samples when an explicit active set repeats indices
// (train_tree / find_node_split), so the tables grow to the largest set seen.
void ensure_xlogx(sofg::DeviceData& D, uint64_t m, cudaStream_t st) {
  if (D.xl_n >= m && D.xl.p) return;
  const std::vector<double> xl = sofg::host::xlogx_table(m);
  std::vector<float> xlf(xl.begin(), xl.end());
  cuda_check(cudaStreamSynchronize(st), "sync tables");  // queued waves may read the old tables
  D.xl.exact(m + 1);
  D.xlf.exact(m + 1);
  cuda_check(cudaMemcpyAsync(D.xl.p, xl.data(), 8 * (m + 1), cudaMemcpyHostToDevice, st), "H2D xlogx");
  cuda_check(cudaMemcpyAsync(D.xlf.p, xlf.data(), 4 * (m + 1), cudaMemcpyHostToDevice, st),
             "H2D xlogx f32");
  cuda_check(cudaStreamSynchronize(st), "sync tables");  // the host vectors die here
  D.xl_n = m;
}

// Dataset staging into HBM: ld = n rounded up to 32 samples (128 B column alignment).
// copy_X returns 0: synchronous copy (pageable), 1: enqueued on the context's stream, 2: deferred
// to the feeder thread, which copies `pending_src` (column-major [d][n], page-locked) in slices.
void upload(sofg_ctx* c, uint64_t n, uint64_t d, const int32_t* labels, int32_t k,
            const std::function<int(float* dev, uint64_t ld)>& copy_X, const float* pending_src = nullptr) {
  if (n < 1 || d < 1) throw std::invalid_argument("empty dataset");
  if (n >= (1ull << 31)) throw std::invalid_argument("n_samples must be < 2^31");
  if (k < 1) throw std::invalid_argument("class_count must be positive");
  if (k > sofg::kMaxClassesWide)
    throw std::invalid_argument("class_count > " + std::to_string(sofg::kMaxClassesWide) +
                                " is not supported by the GPU splitter");
  for (uint64_t i = 0; i < n; ++i)  // dataset.hpp:41-44
    if (labels[i] < 0 || labels[i] >= k) throw std::invalid_argument("label id out of range");
  sofg::DeviceData& D = c->eng->data();
  cuda_check(cudaSetDevice(c->eng->device()), "cudaSetDevice");
  D.n = n;
  D.d = d;
  D.k = k;
  D.ld = (n + 31) / 32 * 32;
  D.X.exact(D.ld * d);
  // Pageable host -> device copies (legacy stream) can return before their DMA has landed, and
  // the engine's stream does not order against the legacy stream: wait for those. Copies from
  // page-locked memory are enqueued on the engine stream instead and left in flight — training
  // starts with host-side work (bootstrap sampling) that overlaps them.
  const int copied = copy_X(D.X.p, D.ld);
  if (copied == 0) cuda_check(cudaDeviceSynchronize(), "upload sync");
  cudaStream_t st = c->eng->stream();
  // Row-major copy for the sample-major projection sweep (sweep.cu); rows padded to 128 B. The
  // previous allocation is reused when it is large enough (a 16 GB free + malloc per upload costs
  // hundreds of ms).
  D.ldr = (d + 1 + 31) / 32 * 32;  // >= one zero pad column (the sweep's empty-row term)
  // The copy is an accelerator, not a requirement: when it would not leave room for the wave
  // buffers (projected rows, level buffers: ~16 GB kept free) or its allocation fails, the table
  // stays column-major only and every wave uses the gather producer (same results).
  bool row_table = std::getenv("SOFG_NO_ROW_TABLE") == nullptr;
  if (row_table && !(D.XR.p && D.XR.cap >= n * D.ldr)) {
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const size_t need = n * D.ldr * 4, reserve = size_t(16) << 30;
    const size_t avail = free_b + (D.XR.p ? D.XR.cap * 4 : 0);
    if (avail < need + reserve) row_table = false;
  }
  if (row_table) {
    try {
      D.XR.exact(n * D.ldr);
    } catch (const sofg::CudaError&) {
      cudaGetLastError();
      row_table = false;
    }
  }
  if (!row_table) D.XR.release();
  if (copied == 2) {  // sliced page-locked copy on the feeder thread, then the transpose
    sofg::DeviceData* Dp = &D;
    const float* src = pending_src;
    const int dev = c->eng->device();
    c->feeder_dev = dev;
    c->feeder = std::thread([c, Dp, src, n, d, st, dev, row_table] {
      try {
        cuda_check(cudaSetDevice(dev), "cudaSetDevice");
        // Slices in flight: two when a call of this context waits for the table, or when nothing
        // else uses the GPU, so the copy engine always has the next slice queued (one in flight
        // leaves it idle while this thread wakes up: 16 GB in ~480 ms instead of ~300 at 32 MB
        // slices); one while another context trains, whose per-wave copies otherwise starve
        // behind the queued slices (measured: +300 ms per concurrent 100-tree step); none while
        // another context's call waits for its own table (both would take twice as long).
        // Blocking-sync events: the thread sleeps between slices instead of spinning on a core
        // the trainers' host pools use.
        cudaEvent_t ev[2];
        for (cudaEvent_t& e : ev)
          cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventBlockingSync), "event");
        static const uint64_t slice_mb = std::getenv("SOFG_UPLOAD_SLICE_MB") ? std::strtoull(std::getenv("SOFG_UPLOAD_SLICE_MB"), nullptr, 10) : 32;
        const uint64_t cols = std::max<uint64_t>(1, (slice_mb << 20) / (4 * n));
        uint64_t i = 0;
        const int dv = dev & 63;
        for (uint64_t f0 = 0; f0 < d; f0 += cols, ++i) {
          while (!c->feeder_waited.load() && g_waited[dv].load() > 0)  // another table is awaited
            std::this_thread::sleep_for(std::chrono::microseconds(100));
          const uint64_t w = std::min(cols, d - f0);
          cuda_check(cudaMemcpy2DAsync(Dp->X.p + f0 * Dp->ld, Dp->ld * 4, src + f0 * n, n * 4, n * 4, w,
                                       cudaMemcpyHostToDevice, st),
                     "H2D table slice");
          cuda_check(cudaEventRecord(ev[i & 1], st), "event");
          if (!c->feeder_waited.load() && g_training[dv].load() > 0)
            cuda_check(cudaEventSynchronize(ev[i & 1]), "slice sync");  // this slice: one in flight
          else if (i > 0)
            cuda_check(cudaEventSynchronize(ev[(i - 1) & 1]), "slice sync");
        }
        if (i > 0) cuda_check(cudaEventSynchronize(ev[(i - 1) & 1]), "slice sync");
        for (cudaEvent_t& e : ev) cudaEventDestroy(e);
        if (row_table)
          cuda_check(sofg::launch_transpose_rows(Dp->X.p, Dp->ld, n, d, Dp->XR.p, Dp->ldr, st), "transpose_rows");
      } catch (...) {
        c->feeder_error = std::current_exception();
      }
    });
  } else if (row_table) {
    cuda_check(sofg::launch_transpose_rows(D.X.p, D.ld, n, d, D.XR.p, D.ldr, st), "transpose_rows");
  }
  D.labels_host.assign(labels, labels + n);
  // labels through page-locked staging, on the engine stream (the staging is rewritten only
  // after its previous copy has completed)
  if (!D.lab_ev) cuda_check(cudaEventCreateWithFlags(&D.lab_ev, cudaEventDisableTiming), "event");
  cuda_check(cudaEventSynchronize(D.lab_ev), "label staging");
  uint8_t* l8 = D.lab_stage.ensure(n);
  for (uint64_t i = 0; i < n; ++i) l8[i] = uint8_t(labels[i]);
  D.lab.exact(n);
  cuda_check(cudaMemcpyAsync(D.lab.p, l8, n, cudaMemcpyHostToDevice, st), "H2D labels");
  cuda_check(cudaEventRecord(D.lab_ev, st), "event");
  ensure_xlogx(D, n, st);
}

struct PCfg {
  uint32_t R;
  double density;
};
PCfg projection_config(uint64_t d, uint64_t num_projections, double cell_density) {
  // ProjectionConfig::for_features (projection.hpp:39-50)
  const double sd = std::sqrt(double(d));
  PCfg p;
  p.R = uint32_t(std::ceil(1.5 * sd));
  const double e = double(std::llround(3.0 * sd));
  p.density = std::min(1.0, e / (double(p.R) * double(d)));
  if (num_projections) p.R = uint32_t(num_projections);
  if (cell_density > 0.0) p.density = cell_density;
  return p;
}

// Histogram bin counts the GPU splitter takes: up to kMaxBins; the shared-memory counters of the
// wide-class / large-bin counting kernel (wide.cu) bound bins x classes there.
void check_bins(uint64_t bins, int k) {
  if (bins < 2) throw std::invalid_argument("bin_count must be at least 2");
  if (bins > uint64_t(sofg::kMaxBins))
    throw std::invalid_argument("bin_count > " + std::to_string(sofg::kMaxBins) +
                                " is not supported by the GPU histogram splitter");
  if ((k > sofg::kMaxClasses || bins > 1024) && sofg::hist_wide_smem(uint32_t(bins), k) > size_t(sofg::kSmemOptin))
    throw std::invalid_argument("bin_count x class_count too large for the GPU histogram splitter");
}

void validate_cfg(const sofg_train_config* cfg, const sofg::DeviceData& D) {  // forest.hpp:270-276
  if (cfg->n_trees < 1) throw std::invalid_argument("n_trees must be positive");
  if (cfg->bin_count < 2) throw std::invalid_argument("bin_count must be at least 2");
  if (cfg->min_samples_split < 2)
    throw std::invalid_argument("min_samples_split must be at least 2");
  if (!(cfg->bootstrap_fraction > 0.0) || cfg->bootstrap_fraction > 1.0)
    throw std::invalid_argument("bootstrap fraction must be in (0, 1]");
  if (D.n < 2) throw std::invalid_argument("need at least 2 samples");
  if (D.k < 2) throw std::invalid_argument("need at least 2 classes");
  check_bins(cfg->bin_count, D.k);
  if (cfg->mode < 0 || cfg->mode > 2) throw std::invalid_argument("unknown split mode");
}

sofg::TrainParams params_for(const sofg_train_config* cfg, const sofg::DeviceData& D,
                             bool forest) {
  sofg::TrainParams P;
  P.mode = cfg->mode;
  P.bins = cfg->bin_count;
  P.two_level = cfg->two_level_binning != 0;
  // train_forest stores the resolved breakeven only for Dynamic (forest.hpp:285-293);
  // train_tree uses cfg.breakeven or the fallback regardless of mode (forest.hpp:258).
  P.breakeven = cfg->has_breakeven ? cfg->breakeven : sofg::kFallbackBreakeven;
  (void)forest;
  if (cfg->has_max_depth) P.max_depth = cfg->max_depth;
  P.min_samples_split = cfg->min_samples_split;
  P.max_split_retries = cfg->max_split_retries;
  const PCfg pc = projection_config(D.d, cfg->num_projections, cfg->cell_density);
  P.R = pc.R;
  P.density = pc.density;
  P.batch_trees = cfg->batch_trees;
  return P;
}

uint64_t auto_batch(uint64_t n_root, uint64_t n_trees, const sofg::TrainParams& P, uint64_t d) {
  const uint64_t n0 = std::max<uint64_t>(n_root, 1);
  // level buffers: 2 x (4 B id + 1 B label) per root sample + the inverse map; keep under ~8 GB
  uint64_t cap = std::max<uint64_t>(1, (8ull << 30) / (14 * n0));
  // projected rows of the widest (root) level: n0 x Rp floats per tree; keep under ~40 GB
  cap = std::min<uint64_t>(cap, std::max<uint64_t>(1, (40ull << 30) / (n0 * sofg::vpitch(P.R) * 4)));
  // terms per wave stay < 2^31: the widest level has far fewer than n0/32 open nodes per tree
  const double ez = std::max(1.0, double(P.R) * double(d) * P.density);
  cap = std::min<uint64_t>(cap, std::max<uint64_t>(1, uint64_t(2147483648.0 / (std::max(1.0, n0 / 32.0) * ez))));
  return std::min(n_trees, cap);
}

sofg::CalOptions cal_options(const sofg_calibration_options& o) {
  sofg::CalOptions c;
  c.n_min = o.n_min;
  c.n_max = o.n_max;
  c.budget_seconds = o.budget_seconds;
  c.bin_count = o.bin_count;
  c.two_level = o.two_level != 0;
  c.repetitions = o.repetitions;
  c.seed = o.seed;
  return c;
}

void run_calibration(sofg_ctx* c, const sofg_train_config* cfg, const sofg::TrainParams& P,
                     sofg_calibration* out) {
  const sofg::CalOptions opt = cal_options(cfg->calibration);
  if (opt.n_max >= (1ull << 31)) throw std::invalid_argument("calibration n_max too large");
  ensure_xlogx(c->eng->data(), opt.n_max, c->eng->stream());
  sofg::ThreadPool& pool = pool_for(c, cfg->n_workers);
  const sofg::CalResult r = sofg::calibrate_crossover(*c->eng, pool, P, opt);
  std::memset(out, 0, sizeof(*out));
  out->breakeven = r.breakeven;
  out->elapsed_seconds = r.elapsed_seconds;
  out->fallback = r.fallback;
  out->n_samples = std::min<uint64_t>(r.samples.size(), SOFG_MAX_CAL_SAMPLES);
  for (uint64_t i = 0; i < out->n_samples; ++i)
    out->samples[i] = {r.samples[i].n, r.samples[i].exact_seconds, r.samples[i].histogram_seconds};
}

}  // namespace

// =============================================================================== C ABI
extern "C" {

void sofg_default_config(sofg_train_config* c) {
  std::memset(c, 0, sizeof(*c));
  c->n_trees = 100;
  c->mode = 2;
  c->two_level_binning = 1;
  c->bin_count = 256;
  c->bootstrap_fraction = 0.632;
  c->min_samples_split = 2;
  c->max_split_retries = 1;
  c->n_workers = 1;
  c->calibration.n_min = 64;  // calibrate.hpp:22-32
  c->calibration.n_max = 65536;
  c->calibration.budget_seconds = 0.1;
  c->calibration.bin_count = 256;
  c->calibration.two_level = 1;
  c->calibration.repetitions = 5;
  c->calibration.seed = 0xca11b8a7e5eedull;
}

const char* sofg_last_error(void) { return g_err.c_str(); }
const char* sofg_version(void) { return "sofg 0.1 (sm_100a)"; }

int sofg_create(int device, sofg_ctx** out) {
  return guard([&] {
    int n = 0;
    cuda_check(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
    if (device < 0 || device >= n) throw std::invalid_argument("no such CUDA device");
    auto* c = new sofg_ctx;
    try {
      c->eng.reset(new sofg::WaveRunner(device));
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

int sofg_destroy(sofg_ctx* c) {
  return guard([&] { delete c; });
}

int sofg_upload_dataset(sofg_ctx* c, const float* X, uint64_t n, uint64_t d, const int32_t* y,
                        int32_t k) {
  return guard([&] {
    require_ctx(c);
    c->join_feeder();
    cudaPointerAttributes at{};
    const bool pinned = cudaPointerGetAttributes(&at, X) == cudaSuccess && at.type == cudaMemoryTypeHost;
    cudaGetLastError();  // clear a failed attribute query (plain pageable memory)
    upload(c, n, d, y, k, [&](float* dev, uint64_t ld) {
      if (pinned) return 2;  // sliced on the feeder thread
      cuda_check(cudaMemcpy2D(dev, ld * 4, X, n * 4, n * 4, d, cudaMemcpyHostToDevice), "H2D table");
      return 0;
    }, pinned ? X : nullptr);
  });
}

int sofg_upload_columns(sofg_ctx* c, const float* const* cols, uint64_t n, uint64_t d,
                        const int32_t* y, int32_t k) {
  return guard([&] {
    require_ctx(c);
    c->join_feeder();
    upload(c, n, d, y, k, [&](float* dev, uint64_t ld) {
      for (uint64_t f = 0; f < d; ++f)
        cuda_check(cudaMemcpyAsync(dev + f * ld, cols[f], n * 4, cudaMemcpyHostToDevice,
                                   c->eng->stream()),
                   "H2D column");
      cuda_check(cudaStreamSynchronize(c->eng->stream()), "sync columns");
      return 1;
    });
  });
}

int sofg_generate_trunk(sofg_ctx* c, uint64_t n, uint64_t d, int32_t k, uint64_t seed) {
  return guard([&] {
    require_ctx(c);
    c->join_feeder();
    if (n < 2) throw std::invalid_argument("n_samples must be at least 2");
    if (d == 0) throw std::invalid_argument("n_features must be positive");
    if (k < 1 || k > sofg::kMaxClassesWide) throw std::invalid_argument("class_count out of range");
    std::vector<int32_t> y(n);
    for (uint64_t i = 0; i < n; ++i) y[i] = int32_t(i % uint64_t(k));
    upload(c, n, d, y.data(), k, [&](float* dev, uint64_t ld) {
      DevBuf<uint8_t> tmp;
      tmp.exact(n);
      cuda_check(launch_generate_trunk(dev, ld, tmp.p, n, d, k, seed, c->eng->stream()),
                 "generate_trunk");
      cuda_check(cudaStreamSynchronize(c->eng->stream()), "sync generate");
      return 1;
    });
  });
}

int sofg_download_dataset(sofg_ctx* c, float* X, int32_t* y) {
  return guard([&] {
    require_data(c);
    const sofg::DeviceData& D = c->eng->data();
    cuda_check(cudaStreamSynchronize(c->eng->stream()), "sync upload");  // an upload may be in flight
    if (X)
      cuda_check(cudaMemcpy2D(X, D.n * 4, D.X.p, D.ld * 4, D.n * 4, D.d, cudaMemcpyDeviceToHost),
                 "D2H table");
    if (y) std::memcpy(y, D.labels_host.data(), 4 * D.n);
  });
}

int sofg_train_forest(sofg_ctx* c, const sofg_train_config* cfg, sofg_forest** out) {
  return guard([&] {
    require_data(c);
    const TrainingMark busy(c->eng->device());
    const sofg::DeviceData& D = c->eng->data();
    validate_cfg(cfg, D);
    sofg::TrainParams P = params_for(cfg, D, true);
    const uint64_t tb = cfg->tree_begin;
    const uint64_t te = cfg->tree_end ? std::min(cfg->tree_end, cfg->n_trees) : cfg->n_trees;
    if (tb > te) throw std::invalid_argument("tree_begin > tree_end");
    const auto t_start = std::chrono::steady_clock::now();
    auto* res = new sofg_forest;
    std::unique_ptr<sofg_forest> guard_res(res);
    res->f.class_count = D.k;
    res->f.n_features = D.d;
    if (cfg->mode == 2 && !cfg->has_breakeven) {  // forest.hpp:285-293: calibrate when absent
      run_calibration(c, cfg, P, &res->cal);
      res->has_cal = true;
      P.breakeven = res->cal.breakeven;
    }
    res->f.breakeven = cfg->mode == 2 ? P.breakeven : 0;
    sofg::ThreadPool& pool = pool_for(c, cfg->n_workers);
    const bool had_stats = c->eng->collect_stats;
    if (cfg->instrument) {  // TrainInstrumentation: per-wave CUDA-event timing for this call
      res->has_prof = true;
      P.profile = &res->prof;
      c->eng->collect_stats = true;
    }
    struct StatsRestore {
      sofg_ctx* c;
      bool on;
      ~StatsRestore() { c->eng->collect_stats = on; }
    } stats_restore{c, had_stats};
    uint64_t k0 = uint64_t(std::llround(cfg->bootstrap_fraction * double(D.n)));
    k0 = std::clamp<uint64_t>(k0, 1, D.n);
    const uint64_t batch = P.batch_trees ? P.batch_trees : auto_batch(k0, te - tb, P, D.d);
    for (uint64_t t0 = tb; t0 < te; t0 += batch) {
      const uint64_t t1 = std::min(te, t0 + batch);
      const size_t B = size_t(t1 - t0);
      std::vector<std::vector<uint32_t>> roots(B);
      std::vector<uint64_t> seeds(B);
      const auto tbs = std::chrono::steady_clock::now();
      BootAhead& ah = c->ahead;
      pool.parallel_for(B, [&](size_t b) {
        const uint64_t ts = sofg::host::derive_seed(cfg->seed, t0 + b + 1);  // forest.hpp:305
        if (!ah.take(D.n, cfg->bootstrap_fraction, cfg->seed, t0 + b, roots[b]))
          roots[b] = sofg::host::bootstrap_indices(D.n, cfg->bootstrap_fraction,
                                                   sofg::host::derive_seed(ts, 0));
        seeds[b] = sofg::host::derive_seed(ts, 1);
      });
      c->times.ms_bootstrap +=
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tbs).count();
      // the next batch's samples (this call's, else the range a next call would train)
      const uint64_t n0 = t1 < te ? t1 : te, n1 = t1 < te ? std::min(te, t1 + batch) : te + (t1 - t0);
      ah.plan(D.n, cfg->bootstrap_fraction, cfg->seed, n0, n1);
      sofg::TrainParams Pb = P;
      if (!std::getenv("SOFG_NO_BOOT_AHEAD"))
        Pb.idle_work = [&ah, &pool]() {
          if (ah.next >= ah.t1) return false;
          const uint64_t a = ah.next, b = std::min(ah.t1, a + uint64_t(pool.size()));
          pool.parallel_for(size_t(b - a), [&](size_t i) {
            const uint64_t ts = sofg::host::derive_seed(ah.seed, a + i + 1);
            ah.roots[size_t(a + i - ah.t0)] = sofg::host::bootstrap_indices(ah.n, ah.frac, sofg::host::derive_seed(ts, 0));
          });
          ah.next = b;
          return ah.next < ah.t1;
        };
      sofg::grow_trees(*c->eng, Pb, pool, roots, seeds, 0, res->f, c->times);
    }
    res->total_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    *out = guard_res.release();
  });
}

int sofg_calibrate(sofg_ctx* c, const sofg_train_config* cfg, sofg_calibration* out) {
  return guard([&] {
    require_data(c);
    if (!out) throw std::invalid_argument("null output");
    const sofg::DeviceData& D = c->eng->data();
    validate_cfg(cfg, D);
    const sofg::TrainParams P = params_for(cfg, D, true);
    run_calibration(c, cfg, P, out);
  });
}

int sofg_train_tree(sofg_ctx* c, const uint32_t* active, uint64_t n_active,
                    const sofg_train_config* cfg, uint64_t seed, uint64_t depth,
                    sofg_forest** out) {
  return guard([&] {
    require_data(c);
    const sofg::DeviceData& D = c->eng->data();
    if (n_active == 0) throw std::invalid_argument("active sample set is empty");  // forest.hpp:254
    for (uint64_t i = 0; i < n_active; ++i)
      if (active[i] >= D.n) throw std::out_of_range("sample index out of range");  // :256
    check_bins(cfg->bin_count, D.k);
    sofg::TrainParams P = params_for(cfg, D, false);
    ensure_xlogx(c->eng->data(), n_active, c->eng->stream());
    sofg::ThreadPool& pool = pool_for(c, cfg->n_workers);
    auto* res = new sofg_forest;
    std::unique_ptr<sofg_forest> guard_res(res);
    res->f.class_count = D.k;
    res->f.n_features = D.d;
    const auto t_start = std::chrono::steady_clock::now();
    const bool had_stats = c->eng->collect_stats;
    if (cfg->instrument) {
      res->has_prof = true;
      P.profile = &res->prof;
      c->eng->collect_stats = true;
    }
    struct StatsRestore {
      sofg_ctx* c;
      bool on;
      ~StatsRestore() { c->eng->collect_stats = on; }
    } stats_restore{c, had_stats};
    std::vector<std::vector<uint32_t>> roots{std::vector<uint32_t>(active, active + n_active)};
    std::vector<uint64_t> seeds{seed};
    sofg::grow_trees(*c->eng, P, pool, roots, seeds, uint32_t(depth), res->f, c->times);
    res->total_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    *out = guard_res.release();
  });
}

uint64_t sofg_forest_num_trees(const sofg_forest* f) { return f->f.n_trees(); }
uint64_t sofg_forest_num_nodes(const sofg_forest* f) { return f->f.left.size(); }
uint64_t sofg_forest_num_terms(const sofg_forest* f) { return f->f.feat.size(); }
uint64_t sofg_forest_breakeven(const sofg_forest* f) { return f->f.breakeven; }

int sofg_forest_calibration(const sofg_forest* f, sofg_calibration* out) {
  if (!f || !f->has_cal) return 0;
  if (out) *out = f->cal;
  return 1;
}

uint64_t sofg_forest_instrumentation(const sofg_forest* f, double* seconds, uint64_t* nodes,
                                     uint64_t* samples, uint64_t cap, sofg_phase_times* phases,
                                     double* split_seconds, double* total_seconds) {
  if (!f || !f->has_prof) return 0;
  const sofg::DepthProfile& p = f->prof;
  const uint64_t nd = p.seconds.size();
  for (uint64_t i = 0; i < std::min(nd, cap); ++i) {
    if (seconds) seconds[i] = p.seconds[i];
    if (nodes) nodes[i] = p.nodes[i];
    if (samples) samples[i] = p.samples[i];
  }
  if (phases)
    for (int b = 0; b < sofg::DepthProfile::kBuckets; ++b)
      phases[b] = {p.phases[b][0], p.phases[b][1], p.phases[b][2], p.phases[b][3]};
  if (split_seconds) *split_seconds = p.split_seconds;
  if (total_seconds) *total_seconds = f->total_seconds;
  return nd;
}

void sofg_forest_arrays(const sofg_forest* fo, const void** a) {
  const sofg::FlatForest& f = fo->f;
  a[0] = f.tree_off.data();
  a[1] = f.left.data();
  a[2] = f.right.data();
  a[3] = f.pred.data();
  a[4] = f.thr.data();
  a[5] = f.term_off.data();
  a[6] = f.feat.data();
  a[7] = f.weight.data();
}

void sofg_forest_export(const sofg_forest* fo, int64_t* tree_off, int32_t* left, int32_t* right,
                        int32_t* pred, float* thr, int64_t* term_off, uint32_t* feat,
                        float* weight) {
  const sofg::FlatForest& f = fo->f;
  // parallel copies (hundreds of MB for a 100-tree forest at 1M x 4096)
  struct Part {
    void* dst;
    const void* src;
    size_t bytes;
  };
  const Part parts[] = {{tree_off, f.tree_off.data(), 8 * f.tree_off.size()},
                        {left, f.left.data(), 4 * f.left.size()},
                        {right, f.right.data(), 4 * f.right.size()},
                        {pred, f.pred.data(), 4 * f.pred.size()},
                        {thr, f.thr.data(), 4 * f.thr.size()},
                        {term_off, f.term_off.data(), 8 * f.term_off.size()},
                        {feat, f.feat.data(), 4 * f.feat.size()},
                        {weight, f.weight.data(), 4 * f.weight.size()}};
  size_t total = 0;
  for (const Part& p : parts) total += p.bytes;
  const int nt = total > (size_t(64) << 20) ? std::max(1, std::min(8, hw_threads())) : 1;
  auto run = [&](int t) {
    for (const Part& p : parts) {
      if (!p.dst || !p.bytes) continue;
      const size_t b0 = p.bytes * size_t(t) / size_t(nt) & ~size_t(63);
      const size_t b1 = t + 1 == nt ? p.bytes : (p.bytes * size_t(t + 1) / size_t(nt) & ~size_t(63));
      if (b1 > b0) std::memcpy(static_cast<char*>(p.dst) + b0, static_cast<const char*>(p.src) + b0, b1 - b0);
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nt; ++t) th.emplace_back(run, t);
  run(0);
  for (auto& x : th) x.join();
}

int sofg_forest_import(uint64_t n_trees, uint64_t n_features, int32_t k, const int64_t* tree_off,
                       const int32_t* left, const int32_t* right, const int32_t* pred,
                       const float* thr, const int64_t* term_off, const uint32_t* feat,
                       const float* weight, sofg_forest** out) {
  return guard([&] {
    // Structural checks of the reference loader (model_io.hpp:255-277), plus child ids above the
    // parent's (every trained tree satisfies it: ids are assigned at split time, depth first), so
    // a malformed forest cannot send sofg_predict's traversal out of bounds or into a cycle.
    if (k < 1) throw std::invalid_argument("class_count must be positive");
    if (!tree_off || tree_off[0] != 0) throw std::invalid_argument("tree_off[0] must be 0");
    for (uint64_t t = 0; t < n_trees; ++t)
      if (tree_off[t + 1] <= tree_off[t]) throw std::invalid_argument("empty tree");
    const uint64_t N = uint64_t(tree_off[n_trees]);
    if (term_off[0] != 0) throw std::invalid_argument("term_off[0] must be 0");
    for (uint64_t q = 0; q < N; ++q)
      if (term_off[q + 1] < term_off[q]) throw std::invalid_argument("term offsets not monotone");
    const uint64_t Q = uint64_t(term_off[N]);
    for (uint64_t u = 0; u < Q; ++u)
      if (feat[u] >= n_features) throw std::invalid_argument("projection feature out of range");
    for (uint64_t t = 0; t < n_trees; ++t) {
      const int64_t size = tree_off[t + 1] - tree_off[t];
      for (int64_t i = 0; i < size; ++i) {
        const uint64_t q = uint64_t(tree_off[t] + i);
        if (left[q] < 0) {
          if (pred[q] < 0 || pred[q] >= k) throw std::invalid_argument("leaf class out of range");
        } else if (left[q] <= i || right[q] <= i || left[q] >= size || right[q] >= size ||
                   term_off[q + 1] == term_off[q]) {
          throw std::invalid_argument("malformed internal node");
        }
      }
    }
    auto* r = new sofg_forest;
    sofg::FlatForest& f = r->f;
    f.tree_off.assign(tree_off, tree_off + n_trees + 1);
    f.left.assign(left, left + N);
    f.right.assign(right, right + N);
    f.pred.assign(pred, pred + N);
    f.thr.assign(thr, thr + N);
    f.term_off.assign(term_off, term_off + N + 1);
    f.feat.assign(feat, feat + Q);
    f.weight.assign(weight, weight + Q);
    f.class_count = k;
    f.n_features = n_features;
    *out = r;
  });
}

void sofg_forest_free(sofg_forest* f) {
  if (!f) return;
  sofg::recycle_forest(std::move(f->f));
  delete f;
}

int sofg_predict(sofg_ctx* c, const sofg_forest* fo, const float* rows, uint64_t n_rows,
                 uint64_t d, int32_t* labels, double* votes) {
  return guard([&] {
    require_ctx(c);
    c->join_feeder();
    const sofg::FlatForest& f = fo->f;
    if (d != f.n_features)
      throw std::invalid_argument("sample has " + std::to_string(d) + " features, model expects " +
                                  std::to_string(f.n_features));  // forest.hpp:112-113
    const int k = f.class_count;
    const int T = int(f.n_trees());
    if (n_rows == 0) return;
    cudaStream_t st = c->eng->stream();
    cuda_check(cudaSetDevice(c->eng->device()), "cudaSetDevice");
    DevBuf<float> drows;
    DevBuf<int64_t> dto, dqo;
    DevBuf<int32_t> dl, dr, dp;
    DevBuf<float> dt;
    DevBuf<uint32_t> dq, dv;
    std::vector<uint32_t> terms(f.feat.size());
    for (size_t q = 0; q < terms.size(); ++q)
      terms[q] = sofg::encode_term(f.feat[q], f.weight[q] < 0.f);
    auto up = [&](auto& buf, const auto& vec) {
      using T0 = typename std::decay_t<decltype(vec)>::value_type;
      buf.exact(vec.size());
      if (!vec.empty())
        cuda_check(cudaMemcpyAsync(buf.p, vec.data(), sizeof(T0) * vec.size(),
                                   cudaMemcpyHostToDevice, st),
                   "H2D forest");
    };
    drows.exact(n_rows * d);
    cuda_check(cudaMemcpyAsync(drows.p, rows, 4 * n_rows * d, cudaMemcpyHostToDevice, st), "H2D rows");
    up(dto, f.tree_off);
    up(dl, f.left);
    up(dr, f.right);
    up(dp, f.pred);
    up(dt, f.thr);
    up(dqo, f.term_off);
    up(dq, terms);
    dv.exact(n_rows * uint64_t(k));
    cuda_check(cudaMemsetAsync(dv.p, 0, 4 * n_rows * uint64_t(k), st), "memset votes");
    cuda_check(sofg::launch_predict(drows.p, n_rows, d, dto.p, T, dl.p, dr.p, dp.p, dt.p, dqo.p,
                                    dq.p, k, dv.p, st),
               "predict");
    std::vector<uint32_t> hv(n_rows * uint64_t(k));
    cuda_check(cudaMemcpyAsync(hv.data(), dv.p, 4 * hv.size(), cudaMemcpyDeviceToHost, st), "D2H votes");
    cuda_check(cudaStreamSynchronize(st), "sync predict");
    for (uint64_t i = 0; i < n_rows; ++i) {
      int32_t best = 0;
      for (int cc = 0; cc < k; ++cc) {
        const double v = double(hv[i * k + cc]) / double(T);  // forest.hpp:116
        if (votes) votes[i * k + cc] = v;
        if (hv[i * k + cc] > hv[i * k + best]) best = cc;
      }
      labels[i] = best;
    }
  });
}

int sofg_apply_projection(sofg_ctx* c, const uint32_t* feat, const float* weight, uint64_t nt,
                          const uint32_t* active, uint64_t n, float* out) {
  return guard([&] {
    require_data(c);
    const sofg::DeviceData& D = c->eng->data();
    for (uint64_t i = 0; i < n; ++i)
      if (active[i] >= D.n) throw std::out_of_range("sample index out of range");
    std::vector<uint32_t> t(nt);
    for (uint64_t q = 0; q < nt; ++q) {
      if (feat[q] >= D.d) throw std::out_of_range("feature index out of range");
      t[q] = sofg::encode_term(feat[q], weight[q] < 0.f);
    }
    if (n == 0) return;
    cudaStream_t st = c->eng->stream();
    DevBuf<uint32_t> dt, da;
    DevBuf<float> dout;
    dt.exact(nt);
    da.exact(n);
    dout.exact(n);
    if (nt) cuda_check(cudaMemcpyAsync(dt.p, t.data(), 4 * nt, cudaMemcpyHostToDevice, st), "H2D");
    cuda_check(cudaMemcpyAsync(da.p, active, 4 * n, cudaMemcpyHostToDevice, st), "H2D");
    cuda_check(sofg::launch_apply_projection(D.X.p, D.ld, dt.p, int(nt), da.p, n, dout.p, st),
               "apply_projection");
    cuda_check(cudaMemcpyAsync(out, dout.p, 4 * n, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "sync");
  });
}

int sofg_bootstrap_sample(uint64_t n, double fraction, uint64_t seed, uint32_t* out, uint64_t* count) {
  return guard([&] {
    if (!out || !count) throw std::invalid_argument("null output");
    if (n == 0) throw std::invalid_argument("empty dataset");
    if (!(fraction > 0.0) || fraction > 1.0)
      throw std::invalid_argument("bootstrap fraction must be in (0, 1]");  // dataset.hpp:335-336
    if (n > 0xFFFFFFFFull) throw std::invalid_argument("n_samples exceeds 2^32");
    const std::vector<uint32_t> v = sofg::host::bootstrap_indices(n, fraction, seed);
    std::memcpy(out, v.data(), 4 * v.size());
    *count = v.size();
  });
}

int sofg_sample_projection(sofg_ctx* c, uint64_t d, uint64_t R, double density,
                           const uint64_t* seeds, const uint64_t* skip, uint64_t n_nodes,
                           uint32_t* row_ptr, uint32_t* feat, float* weight, uint64_t cap,
                           uint64_t* consumed) {
  return guard([&] {
    require_ctx(c);
    if (d == 0 || R == 0) throw std::invalid_argument("projection config is empty");
    if (!(density >= 0.0) || density > 1.0)
      throw std::invalid_argument("cell density must be in [0, 1]");
    if (R * d >= (1ull << 32)) throw std::invalid_argument("projection matrix has >= 2^32 cells");
    sofg::host::BinomialDraw binom(R * d, density);
    std::vector<sofg::NodeIn> nodes(n_nodes);
    uint64_t off = 0, zmax = 32;
    for (uint64_t i = 0; i < n_nodes; ++i) {
      uint64_t used;
      const uint64_t z = binom(seeds[i], skip[i], &used);
      if (z > cap) throw std::invalid_argument("projection nonzeros exceed output capacity");
      nodes[i] = sofg::NodeIn{};
      nodes[i].seed = seeds[i];
      nodes[i].z = uint32_t(z);
      nodes[i].pos = uint32_t(used);
      nodes[i].term_off = uint32_t(off);
      off += z;
      zmax = std::max(zmax, z);
    }
    cudaStream_t st = c->eng->stream();
    sofg::Scratch scratch;  // freed after the stream synchronization below
    DevBuf<sofg::NodeIn> dn;
    DevBuf<uint32_t> dterms, drp, dpos;
    dn.exact(n_nodes);
    dterms.exact(off + 1);
    drp.exact(n_nodes * (R + 1));
    dpos.exact(n_nodes);
    cuda_check(cudaMemcpyAsync(dn.p, nodes.data(), sizeof(sofg::NodeIn) * n_nodes,
                               cudaMemcpyHostToDevice, st),
               "H2D nodes");
    cuda_check(sofg::launch_sample_projection(dn.p, int(n_nodes), uint32_t(d), uint32_t(R),
                                              uint32_t(zmax), dterms.p, drp.p, dpos.p, scratch, st),
               "sample_projection");
    std::vector<uint32_t> ht(off + 1), hrp(n_nodes * (R + 1)), hpos(n_nodes);
    cuda_check(cudaMemcpyAsync(ht.data(), dterms.p, 4 * (off + 1), cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaMemcpyAsync(hrp.data(), drp.p, 4 * hrp.size(), cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaMemcpyAsync(hpos.data(), dpos.p, 4 * n_nodes, cudaMemcpyDeviceToHost, st), "D2H");
    cuda_check(cudaStreamSynchronize(st), "sync sample");
    for (uint64_t i = 0; i < n_nodes; ++i) {
      for (uint64_t r = 0; r <= R; ++r) row_ptr[i * (R + 1) + r] = hrp[i * (R + 1) + r];
      for (uint32_t q = 0; q < nodes[i].z; ++q) {
        const uint32_t t = ht[nodes[i].term_off + q];
        feat[i * cap + q] = t >> 1;
        weight[i * cap + q] = (t & 1u) ? -1.f : 1.f;
      }
      consumed[i] = uint64_t(hpos[i]) - skip[i];
    }
  });
}

int sofg_find_node_split(sofg_ctx* c, const uint32_t* active, uint64_t n, const uint32_t* row_ptr,
                         uint64_t R, const uint32_t* feat, const float* weight, int32_t method,
                         uint64_t bins, uint64_t seed, uint64_t skip, sofg_split* out) {
  return guard([&] {
    require_data(c);
    const sofg::DeviceData& D = c->eng->data();
    std::memset(out, 0, sizeof(*out));
    if (n < 2) return;  // split.hpp:238
    check_bins(bins, D.k);
    for (uint64_t i = 0; i < n; ++i)
      if (active[i] >= D.n) throw std::out_of_range("sample index out of range");
    ensure_xlogx(c->eng->data(), n, c->eng->stream());
    const uint64_t nnz = row_ptr[R];
    sofg::WaveSpec w;
    w.R = uint32_t(R);
    w.d = uint32_t(D.d);
    w.bins = uint32_t(bins);
    w.k = D.k;
    w.given_csr = true;
    w.given_terms.resize(nnz);
    for (uint64_t q = 0; q < nnz; ++q) {
      if (feat[q] >= D.d) throw std::out_of_range("feature index out of range");
      w.given_terms[q] = sofg::encode_term(feat[q], weight[q] < 0.f);
    }
    w.given_row_ptr.assign(row_ptr, row_ptr + R + 1);
    w.given_pos = {uint32_t(skip)};
    std::vector<uint32_t> counts(size_t(D.k), 0u);
    std::vector<uint8_t> l8(n);
    for (uint64_t i = 0; i < n; ++i) {
      l8[i] = uint8_t(D.labels_host[active[i]]);
      counts[l8[i]]++;
    }
    sofg::NodeIn nd{};
    nd.seed = seed;
    nd.begin = 0;
    nd.n = uint32_t(n);
    nd.z = uint32_t(nnz);
    nd.pos = uint32_t(skip);
    nd.flags = sofg::kNodeGivenCsr | (method == 1 ? sofg::kNodeHist : 0u);
    nd.parent = sofg::host::entropy(counts.data(), D.k);
    w.nodes = {nd};
    cudaStream_t st = c->eng->stream();
    DevBuf<uint32_t> di, dio;
    DevBuf<uint8_t> dl, dlo;
    di.exact(n);
    dio.exact(n);
    dl.exact(n);
    dlo.exact(n);
    cuda_check(cudaMemcpyAsync(di.p, active, 4 * n, cudaMemcpyHostToDevice, st), "H2D");
    cuda_check(cudaMemcpyAsync(dl.p, l8.data(), n, cudaMemcpyHostToDevice, st), "H2D");
    w.idx_in = di.p;
    w.lab_in = dl.p;
    w.idx_out = dio.p;
    w.lab_out = dlo.p;
    std::vector<sofg::NodeRes> res;
    c->eng->run(w, res);
    const sofg::NodeRes& r = res[0];
    out->found = r.row >= 0;
    out->projection_index = r.row;
    out->threshold = r.threshold;
    out->gain = r.gain;
    out->n_left = r.n_left_search;
    out->n_right = r.row >= 0 ? uint32_t(n) - r.n_left_search : 0;
    out->n_left_partition = r.n_left;
    out->consumed = uint64_t(r.pos_after) - skip;
  });
}

void* sofg_stream(sofg_ctx* c) { return c && c->eng ? (void*)c->eng->stream() : nullptr; }

void* sofg_host_alloc(uint64_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, bytes) != cudaSuccess) return nullptr;
  return p;
}

void sofg_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int sofg_set_stats(sofg_ctx* c, int enable) {
  return guard([&] {
    require_ctx(c);
    c->stats_mode = enable;
    c->eng->collect_stats = enable != 0;
    c->eng->sector_accounting = enable >= 2;
  });
}

int sofg_get_stats(sofg_ctx* c, sofg_stats* o) {
  return guard([&] {
    require_ctx(c);
    std::memset(o, 0, sizeof(*o));
    const sofg::WaveStats& s = c->eng->stats;
    o->ms_sample = s.ms_sample;
    o->ms_hist_rng = s.ms_hist_rng;
    o->ms_hist_count = s.ms_hist_count;
    o->ms_exact = s.ms_exact;
    o->ms_partition = s.ms_partition;
    o->ms_waves_total = s.ms_total;
    o->ms_host_binomial = c->times.ms_binomial;
    o->ms_host_bootstrap = c->times.ms_bootstrap;
    o->ms_train_total = c->times.ms_total;
    o->waves = s.waves;
    o->nodes = s.nodes;
    o->hist_nodes = s.hist_nodes;
    o->exact_nodes = s.exact_nodes;
    o->kernel_launches = s.launches;
    o->levels = c->times.levels;
    o->hist_count_launches = s.hist_count_launches;
    o->exact_launches = s.exact_launches;
    o->hist_strict_bytes = s.hist_strict_bytes;
    o->exact_strict_bytes = s.exact_strict_bytes;
    o->hist_sector_bytes = s.hist_sector_bytes;
    o->exact_sector_bytes = s.exact_sector_bytes;
    o->ms_host_roots = c->times.ms_roots;
    o->ms_host_prep = c->times.ms_prep;
    o->ms_host_submit = c->times.ms_submit;
    o->ms_host_spec = c->times.ms_spec;
    o->ms_host_wait = c->times.ms_wait;
    o->ms_host_post = c->times.ms_post;
    o->ms_host_final = c->times.ms_final;
    o->sweep_waves = s.sweep_waves;
    o->gather_waves = s.gather_waves;
    o->sweep_alg_bytes = s.sweep_alg_bytes;
    o->sweep_cta_threads = s.sweep_cta_threads;
    o->sweep_entry_bytes = s.sweep_entry_bytes;
  });
}

namespace {
const sofg::WaveStats& merged_stats(sofg_ctx* c) { return c->eng->stats; }
}  // namespace

int sofg_stats_kernels(sofg_ctx* c) { return c && c->eng ? int(merged_stats(c).per_kernel.size()) : 0; }

int sofg_stats_kernel(sofg_ctx* c, int i, const char** name, double* ms, uint64_t* launches) {
  return guard([&] {
    require_ctx(c);
    const auto& v = merged_stats(c).per_kernel;
    if (i < 0 || size_t(i) >= v.size()) throw std::out_of_range("kernel stat index");
    *name = v[size_t(i)].name;
    *ms = v[size_t(i)].ms;
    *launches = v[size_t(i)].launches;
  });
}

int sofg_reset_stats(sofg_ctx* c) {
  return guard([&] {
    require_ctx(c);
    c->eng->stats = sofg::WaveStats{};
    c->times = sofg::HostTimes{};
  });
}

}  // extern "C"
