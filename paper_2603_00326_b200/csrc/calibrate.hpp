// B200 crossover calibration of the dynamic split switch (reference calibrate.hpp).
//
// The reference times one exact and one histogram split search of a synthetic two-class node of n
// values on the CPU and binary-searches n for the crossover (calibrate.hpp:51-112 search,
// :135-196 probes). On the GPU a single node is launch-latency bound, so a probe here is one wave:
// M nodes of n samples each (M * n ~ 2^18, the batched analogue of probe_batch_size,
// calibrate.hpp:125-130) drawn from the resident table, all split by the same method through the
// production kernels; the probe value is the wave's split-search device time (CUDA events from the
// end of the projection stage to the start of the partition) divided by M. The search itself —
// probe at n_min, then n_max, then bisection, soft/hard budgets, median of repetitions, fallback
// 1024 — is the reference's.
#pragma once
#include <cstdint>
#include <vector>

#include "engine.hpp"
#include "trainer.hpp"

namespace sofg {

struct CalOptions {  // soforest::CalibrationOptions (calibrate.hpp:22-32), same defaults
  uint64_t n_min = 64;
  uint64_t n_max = 65536;
  double budget_seconds = 0.1;
  uint64_t bin_count = 256;
  bool two_level = true;
  uint64_t repetitions = 5;
  uint64_t seed = 0xca11b8a7e5eedull;
};

struct CalSample {  // soforest::CrossoverSample (calibrate.hpp:16-20)
  uint64_t n = 0;
  double exact_seconds = 0.0;
  double histogram_seconds = 0.0;
};

struct CalResult {  // soforest::CrossoverCalibration (calibrate.hpp:34-41)
  uint64_t breakeven = 1024;
  std::vector<CalSample> samples;  // sorted by n
  double elapsed_seconds = 0.0;
  bool fallback = false;
};

// Requires the dataset resident on `eng` and its xlogx tables covering opt.n_max; P supplies the
// projection configuration (R, density). Throws std::invalid_argument on bad options
// (calibrate.hpp:58-60).
CalResult calibrate_crossover(WaveRunner& eng, ThreadPool& pool, const TrainParams& P, const CalOptions& opt);

}  // namespace sofg
