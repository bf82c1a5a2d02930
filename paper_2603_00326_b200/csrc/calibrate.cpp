#include "calibrate.hpp"

#include <algorithm>
#include <chrono>
#include <functional>
#include <stdexcept>
#include <string>

#include "host_rng.hpp"

namespace sofg {

namespace {

using Clock = std::chrono::steady_clock;

// One probe wave: M nodes of n samples of the resident table, every node split by `hist` or the
// exact method. Sample ids are a fixed multiplicative-hash walk of the table (repeats allowed: the
// gather projection, both splitters and the partition take any active list), so every repetition
// at a given n times the same work.
class WaveProbe {
 public:
  WaveProbe(WaveRunner& eng, ThreadPool& pool, const TrainParams& P, const CalOptions& opt)
      : eng_(eng), P_(P), opt_(opt), binom_(uint64_t(P.R) * eng.data().d, P.density) {
    eng.set_pool(&pool);
  }

  double operator()(uint64_t n, bool hist) {
    prepare(n);
    for (NodeIn& nd : w_.nodes) nd.flags = hist ? kNodeHist : 0u;
    std::vector<NodeRes> res;
    eng_.run(w_, res);
    sink_ += res.empty() ? 0.0 : res[0].gain;
    return 1e-3 * double(eng_.last_split_ms()) / double(w_.nodes.size());
  }
  double sink() const { return sink_; }

 private:
  void prepare(uint64_t n) {
    if (n == n_) return;
    n_ = n;
    const DeviceData& D = eng_.data();
    const uint64_t M = std::clamp<uint64_t>((uint64_t(1) << 18) / std::max<uint64_t>(n, 1), 1, 4096);
    const uint64_t total = M * n;
    std::vector<uint32_t> ids(total);
    std::vector<uint8_t> lab(total);
    w_ = WaveSpec{};
    w_.R = P_.R;
    w_.d = uint32_t(D.d);
    w_.bins = uint32_t(opt_.bin_count);
    w_.two_level = opt_.two_level;
    w_.k = D.k;
    w_.force_mode = 0;  // no inverse map: the gather projection producer
    w_.nodes.resize(M);
    std::vector<uint32_t> z(M), used(M);
    std::vector<uint64_t> seeds(M);
    for (uint64_t i = 0; i < M; ++i) seeds[i] = host::derive_seed(opt_.seed, (n << 16) + i);
    binom_.batch(seeds.data(), M, z.data(), used.data());
    uint64_t term_off = 0;
    for (uint64_t i = 0; i < M; ++i) {
      std::vector<uint32_t> counts(size_t(D.k), 0u);
      for (uint64_t j = 0; j < n; ++j) {
        const uint64_t q = i * n + j;
        const uint32_t s = uint32_t((q * 0x9E3779B97F4A7C15ull >> 17) % D.n);
        ids[q] = s;
        lab[q] = uint8_t(D.labels_host[s]);
        counts[lab[q]]++;
      }
      NodeIn& nd = w_.nodes[i];
      nd = NodeIn{};
      nd.seed = seeds[i];
      nd.begin = uint32_t(i * n);
      nd.n = uint32_t(n);
      nd.z = z[i];
      nd.pos = used[i];
      nd.term_off = uint32_t(term_off);
      nd.parent = host::entropy(counts.data(), D.k);
      term_off += z[i];
    }
    cudaStream_t st = eng_.stream();
    idx_[0].ensure(total);
    idx_[1].ensure(total);
    lab_[0].ensure(total);
    lab_[1].ensure(total);
    cuda_check(cudaMemcpyAsync(idx_[0].p, ids.data(), 4 * total, cudaMemcpyHostToDevice, st), "H2D probe ids");
    cuda_check(cudaMemcpyAsync(lab_[0].p, lab.data(), total, cudaMemcpyHostToDevice, st), "H2D probe labels");
    cuda_check(cudaStreamSynchronize(st), "probe upload");
    w_.idx_in = idx_[0].p;
    w_.lab_in = lab_[0].p;
    w_.idx_out = idx_[1].p;
    w_.lab_out = lab_[1].p;
  }

  WaveRunner& eng_;
  const TrainParams& P_;
  const CalOptions& opt_;
  host::BinomialDraw binom_;
  WaveSpec w_;
  uint64_t n_ = 0;
  DevBuf<uint32_t> idx_[2];
  DevBuf<uint8_t> lab_[2];
  double sink_ = 0.0;
};

}  // namespace

CalResult calibrate_crossover(WaveRunner& eng, ThreadPool& pool, const TrainParams& P, const CalOptions& opt) {
  if (opt.n_min < 2 || opt.n_min >= opt.n_max) throw std::invalid_argument("need 2 <= n_min < n_max");
  if (opt.repetitions < 1) throw std::invalid_argument("repetitions must be positive");
  if (opt.bin_count < 2 || opt.bin_count > uint64_t(kMaxBins))
    throw std::invalid_argument("calibration bin_count must be in [2, " + std::to_string(kMaxBins) + "]");

  // probes need CUDA-event timing; the caller's statistics are left as they were
  const bool had_stats = eng.collect_stats, had_sectors = eng.sector_accounting;
  const WaveStats saved = eng.stats;
  eng.collect_stats = true;
  eng.sector_accounting = false;
  WaveProbe probe(eng, pool, P, opt);
  auto restore = [&] {
    eng.collect_stats = had_stats;
    eng.sector_accounting = had_sectors;
    eng.stats = saved;
  };

  CalResult out;
  try {
    // untimed warm-up of both paths (calibrate.hpp:188-193)
    const uint64_t warm_n = std::min<uint64_t>(opt.n_max, 512);
    probe(warm_n, false);
    probe(warm_n, true);

    // ---- the reference's search (calibrate.hpp:62-112) -------------------------------------
    const auto t0 = Clock::now();
    auto seconds = [&] { return std::chrono::duration<double>(Clock::now() - t0).count(); };
    const double soft = opt.budget_seconds, hard = 2.0 * opt.budget_seconds;
    auto median = [](std::vector<double>& v) {
      std::sort(v.begin(), v.end());
      return v[v.size() / 2];
    };
    auto measure = [&](uint64_t n) {
      std::vector<double> es, hs;
      for (uint64_t rep = 0; rep < opt.repetitions; ++rep) {
        es.push_back(probe(n, false));
        hs.push_back(probe(n, true));
        if (seconds() > soft) break;
      }
      const CalSample s{n, median(es), median(hs)};
      out.samples.push_back(s);
      return s;
    };
    auto finalize = [&](uint64_t breakeven) {
      out.breakeven = breakeven;
      std::sort(out.samples.begin(), out.samples.end(),
                [](const CalSample& a, const CalSample& b) { return a.n < b.n; });
      out.elapsed_seconds = seconds();
    };
    auto wins = [](const CalSample& s) { return s.histogram_seconds < s.exact_seconds; };

    const CalSample at_min = measure(opt.n_min);
    if (wins(at_min)) {
      finalize(opt.n_min);
    } else if (seconds() > hard) {
      out.fallback = true;
      finalize(kFallbackBreakeven);
    } else {
      const CalSample at_max = measure(opt.n_max);
      if (!wins(at_max)) {
        finalize(opt.n_max + 1);
      } else {
        uint64_t lo = opt.n_min, hi = opt.n_max;
        while (hi - lo > 1) {
          if (seconds() > hard) break;
          const uint64_t mid = lo + (hi - lo) / 2;
          if (wins(measure(mid)))
            hi = mid;
          else
            lo = mid;
        }
        finalize(hi - 1);
      }
    }
  } catch (...) {
    restore();
    throw;
  }
  restore();
  return out;
}

}  // namespace sofg
