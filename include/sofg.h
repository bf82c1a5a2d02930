/*
 * sofg — C ABI of the B200-native sparse-oblique forest trainer (libsofg.so).
 *
 * The reference (soforest, arXiv 2603.00326) is a header-only C++ library with no plugin or FFI
 * layer; its drop-in boundary is the train/predict API of proj/include/soforest/forest.hpp. Each
 * entry point below replaces one reference function (cited), taking plain pointers and sizes so
 * any FFI (ctypes, cgo, JNI, N-API) can bind it; see INTEGRATION.md.
 *
 * Conventions
 *   - every call returns 0 on success, non-zero on failure; sofg_last_error() (thread-local)
 *     describes the failure and keeps the reference's exception class as a prefix:
 *       1 "invalid_argument: ..."  (std::invalid_argument in the reference)
 *       2 "out_of_range: ..."      (std::out_of_range)
 *       3 "runtime_error: ..."     (CUDA / resource failures)
 *   - X is column-major float32: column f at X[f * n_samples .. (f+1) * n_samples)
 *     (the reference's BasicColumnarDataset<float> columns, dataset.hpp:23-69)
 *   - a context owns one GPU (one host thread per context); contexts are independent.
 *   - no CPU fallback: if the CUDA kernels cannot run, calls fail.
 */
#ifndef SOFG_H
#define SOFG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sofg_ctx sofg_ctx;
typedef struct sofg_forest sofg_forest;

/* Mirrors soforest::CalibrationOptions (calibrate.hpp:22-32); same fields and defaults. */
typedef struct sofg_calibration_options {
  uint64_t n_min;              /* 64 */
  uint64_t n_max;              /* 65536 */
  double budget_seconds;       /* 0.1 (soft; hard stop at twice that) */
  uint64_t bin_count;          /* 256 */
  int32_t two_level;           /* 1 (accepted; binning is exact either way) */
  int32_t _pad;
  uint64_t repetitions;        /* 5: median of this many runs per probe */
  uint64_t seed;               /* 0xca11b8a7e5eed */
} sofg_calibration_options;

/* Mirrors soforest::CrossoverSample / CrossoverCalibration (calibrate.hpp:16-41). */
typedef struct sofg_crossover_sample {
  uint64_t n;
  double exact_seconds;        /* per-node split-search device time, exact method */
  double histogram_seconds;    /* same, histogram method */
} sofg_crossover_sample;

#define SOFG_MAX_CAL_SAMPLES 64
typedef struct sofg_calibration {
  uint64_t breakeven;          /* largest n still split exactly */
  double elapsed_seconds;
  int32_t fallback;            /* budget exhausted before a usable measurement (breakeven 1024) */
  int32_t _pad;
  uint64_t n_samples;
  sofg_crossover_sample samples[SOFG_MAX_CAL_SAMPLES];  /* sorted by n */
} sofg_calibration;

/* Mirrors soforest::SplitPhaseTimes (timing.hpp:23-28), seconds. */
typedef struct sofg_phase_times {
  double sample_projections, apply_projections, build_histograms, evaluate_splits;
} sofg_phase_times;

/* Mirrors soforest::TrainConfig (forest.hpp:38-53); same field meaning and defaults. */
typedef struct sofg_train_config {
  uint64_t n_trees;            /* 100 */
  int32_t mode;                /* 0 exact-only, 1 histogram-only, 2 dynamic (forest.hpp:20) */
  int32_t two_level_binning;   /* accepted, results identical either way (histogram.hpp:118) */
  uint64_t bin_count;          /* 256, 2..8192 (bins x classes bounded) */
  int32_t has_breakeven;       /* Dynamic: histogram iff n > breakeven (split.hpp:46-48) */
  int32_t has_max_depth;
  uint64_t breakeven;          /* absent: train_forest calibrates on the GPU (forest.hpp:285-293);
                                  train_tree uses 1024 (forest.hpp:258) */
  uint64_t max_depth;
  double bootstrap_fraction;   /* 0.632 */
  uint64_t min_samples_split;  /* 2 */
  uint64_t max_split_retries;  /* 1 */
  uint64_t n_workers;          /* host threads for the per-node binomial draws (0 = all) */
  uint64_t seed;               /* 0 */
  /* extensions */
  uint64_t num_projections;    /* 0: ProjectionConfig::for_features (projection.hpp:39-50) */
  double cell_density;         /* <= 0: for_features density */
  uint64_t batch_trees;        /* trees grown together per level (0 = all / memory bound) */
  uint64_t tree_begin;         /* train trees [tree_begin, tree_end) of the forest (sharding) */
  uint64_t tree_end;           /* 0 = n_trees */
  /* soforest::TrainConfig::calibration (forest.hpp:52): used when Dynamic has no breakeven */
  sofg_calibration_options calibration;
  int32_t instrument;          /* 1: record soforest::TrainInstrumentation in the forest */
  int32_t _pad2;
} sofg_train_config;

void sofg_default_config(sofg_train_config* cfg);
const char* sofg_last_error(void);
const char* sofg_version(void);

/* ---- context / dataset ------------------------------------------------------------------ */
int sofg_create(int device, sofg_ctx** out);
int sofg_destroy(sofg_ctx* ctx);
/* Upload a dataset (replaces constructing BasicColumnarDataset<float>, dataset.hpp:28-45).
 * labels: int32 in [0, class_count). Validates like the reference constructor; class_count <= 64
 * (more than 8 classes run the wide-class splitters, wide.cu; the reference has no bound).
 * X page-locked (e.g. from sofg_host_alloc): returns at once; a context thread feeds the copy to
 * the GPU in ~32 MB slices (two in flight when a call waits for it or the GPU is otherwise idle;
 * one while another context of the process trains on the same GPU, so that context's copies are
 * not queued behind it; paused while another context's call waits for its own table) and the next
 * call on this context waits for it; keep X unchanged until the next
 * training / download call on this context returns. Pageable X: the copy has landed when this
 * returns. */
int sofg_upload_dataset(sofg_ctx* ctx, const float* X, uint64_t n_samples, uint64_t n_features,
                        const int32_t* labels, int32_t class_count);
/* Same, one pointer per column (the reference's vector<vector<float>> layout). */
int sofg_upload_columns(sofg_ctx* ctx, const float* const* columns, uint64_t n_samples,
                        uint64_t n_features, const int32_t* labels, int32_t class_count);
/* Synthetic trunk-model table generated directly in HBM (bench input; not bit-identical to
 * the reference's serial generate_trunk, dataset.hpp:306-329 — same model). */
int sofg_generate_trunk(sofg_ctx* ctx, uint64_t n_samples, uint64_t n_features,
                        int32_t class_count, uint64_t seed);
/* Copy the resident table back (column-major) and the labels; either pointer may be NULL. */
int sofg_download_dataset(sofg_ctx* ctx, float* X, int32_t* labels);

/* ---- training ------------------------------------------------------------------------------ */
/* train_forest (forest.hpp:267-313): trees tree_begin..tree_end-1 of the forest defined by cfg
 * (tree t is a pure function of (data, cfg, t), forest.hpp:264-266, so shards concatenate). */
int sofg_train_forest(sofg_ctx* ctx, const sofg_train_config* cfg, sofg_forest** out);
/* calibrate_crossover (calibrate.hpp:51-196): the reference's breakeven search with GPU probes —
 * each probe is one wave of nodes of n samples of the resident table split by one method, timed
 * with CUDA events. Uses cfg->calibration and cfg's projection settings. */
int sofg_calibrate(sofg_ctx* ctx, const sofg_train_config* cfg, sofg_calibration* out);
/* train_tree (forest.hpp:250-262): one tree grown from an explicit sorted active set. */
int sofg_train_tree(sofg_ctx* ctx, const uint32_t* active, uint64_t n_active,
                    const sofg_train_config* cfg, uint64_t seed, uint64_t depth,
                    sofg_forest** out);

/* ---- forest access (layout shared with the CPU oracle, oracle/oracle_capi.h) --------------- */
uint64_t sofg_forest_num_trees(const sofg_forest* f);
uint64_t sofg_forest_num_nodes(const sofg_forest* f);
uint64_t sofg_forest_num_terms(const sofg_forest* f);
uint64_t sofg_forest_breakeven(const sofg_forest* f);
/* Forest::calibration (forest.hpp:81): 1 and *out filled when train_forest calibrated, else 0. */
int sofg_forest_calibration(const sofg_forest* f, sofg_calibration* out);
/* soforest::TrainInstrumentation (timing.hpp:39-79) of a run with cfg.instrument = 1: per depth
 * (every node, internal or leaf, at its depth) seconds / nodes / samples, the four split phases
 * per depth bucket (depth / 5, capped at 3), split_seconds and total_seconds. Returns the number
 * of depths (0 when not instrumented); arrays with room for `cap` depths, any may be NULL. */
uint64_t sofg_forest_instrumentation(const sofg_forest* f, double* seconds, uint64_t* nodes,
                                     uint64_t* samples, uint64_t cap, sofg_phase_times* phases4,
                                     double* split_seconds, double* total_seconds);
void sofg_forest_export(const sofg_forest* f, int64_t* tree_off, int32_t* left, int32_t* right,
                        int32_t* pred, float* thr, int64_t* term_off, uint32_t* feat,
                        float* weight);
/* Zero-copy access: pointers to the forest's own arrays (valid until sofg_forest_free), in the
 * order tree_off, left, right, pred, thr, term_off, feat, weight. */
void sofg_forest_arrays(const sofg_forest* f, const void** arrays8);
/* Build a forest from flat arrays (e.g. an oracle forest) for sofg_predict. */
int sofg_forest_import(uint64_t n_trees, uint64_t n_features, int32_t class_count,
                       const int64_t* tree_off, const int32_t* left, const int32_t* right,
                       const int32_t* pred, const float* thr, const int64_t* term_off,
                       const uint32_t* feat, const float* weight, sofg_forest** out);
void sofg_forest_free(sofg_forest* f);

/* predict (forest.hpp:110-121) for n_rows row-major host samples on the GPU.
 * labels[n_rows]; votes[n_rows * class_count] (may be NULL). */
int sofg_predict(sofg_ctx* ctx, const sofg_forest* f, const float* rows, uint64_t n_rows,
                 uint64_t n_features, int32_t* labels, double* votes);

/* ---- per-function entry points (kernel-level parity with the reference) -------------------- */
/* bootstrap_sample (dataset.hpp:332-349): round(fraction * n) distinct sorted row indices drawn
 * with make_rng(seed) (the caller passes the tree's derive_seed(tree_seed, 0)). Host-only (no
 * device needed); out has room for n entries; *count = entries written. */
int sofg_bootstrap_sample(uint64_t n, double fraction, uint64_t seed, uint32_t* out, uint64_t* count);
/* apply_projection (projection.hpp:86-108) on the resident table. */
int sofg_apply_projection(sofg_ctx* ctx, const uint32_t* feat, const float* weight,
                          uint64_t n_terms, const uint32_t* active, uint64_t n_active,
                          float* out);
/* sample_projection_matrix (projection.hpp:57-82) for n_nodes engines make_rng(seeds[i]) after
 * skip[i] outputs: host binomial + device Floyd/coins. row_ptr[n_nodes][R+1] (node-local),
 * feat/weight[n_nodes][cap], consumed[n_nodes] = outputs used by the call. */
int sofg_sample_projection(sofg_ctx* ctx, uint64_t n_features, uint64_t num_projections,
                           double cell_density, const uint64_t* seeds, const uint64_t* skip,
                           uint64_t n_nodes, uint32_t* row_ptr, uint32_t* feat, float* weight,
                           uint64_t cap, uint64_t* consumed);
/* find_node_split (split.hpp:229-317) for one node on the device with a caller-supplied
 * projection matrix and engine = make_rng(seed) after `skip` outputs. */
typedef struct sofg_split {
  int32_t found;
  int32_t projection_index;
  float threshold;
  uint32_t n_left;   /* as reported by the split search */
  uint32_t n_right;
  uint32_t n_left_partition; /* values <= threshold (forest.hpp:205) */
  double gain;
  uint64_t consumed; /* engine outputs used (boundary picks) */
} sofg_split;
int sofg_find_node_split(sofg_ctx* ctx, const uint32_t* active, uint64_t n_active,
                         const uint32_t* row_ptr, uint64_t n_rows, const uint32_t* feat,
                         const float* weight, int32_t method, uint64_t bin_count, uint64_t seed,
                         uint64_t skip, sofg_split* out);

/* The context's CUDA stream (cudaStream_t) — for timing with events on the launching stream. */
void* sofg_stream(sofg_ctx* ctx);
/* Page-locked host buffers for end-to-end transfers (cudaMallocHost / cudaFreeHost). */
void* sofg_host_alloc(uint64_t bytes);
void sofg_host_free(void* p);

/* ---- instrumentation ----------------------------------------------------------------------- */
typedef struct sofg_stats {
  double ms_sample, ms_hist_rng, ms_hist_count, ms_exact, ms_partition, ms_waves_total;
  double ms_host_binomial, ms_host_bootstrap, ms_train_total;
  uint64_t waves, nodes, hist_nodes, exact_nodes, kernel_launches, levels;
  uint64_t hist_count_launches, exact_launches;
  double hist_strict_bytes, exact_strict_bytes, hist_sector_bytes, exact_sector_bytes;
  /* host-side phases of the level loop (ms) */
  double ms_host_roots, ms_host_prep, ms_host_submit, ms_host_spec, ms_host_wait, ms_host_post,
      ms_host_final;
  /* projection stage: waves swept over the row-major table vs gathered, and the sweep's
     algorithmic bytes (table rows streamed + projected rows written + term lists read) */
  uint64_t sweep_waves, gather_waves;
  double sweep_alg_bytes;
  /* sweep kernel variant of the widest sweep wave: CTA threads and term-entry bytes (2 or 4) */
  uint32_t sweep_cta_threads, sweep_entry_bytes;
} sofg_stats;
/* enable: 1 = CUDA-event timing per phase (+ sector accounting when 2); 0 = off */
int sofg_set_stats(sofg_ctx* ctx, int enable);
int sofg_get_stats(sofg_ctx* ctx, sofg_stats* out);
int sofg_reset_stats(sofg_ctx* ctx);
/* Per-launch-site CUDA-event times (stats mode): number of sites, then name/ms/launches of i. */
int sofg_stats_kernels(sofg_ctx* ctx);
int sofg_stats_kernel(sofg_ctx* ctx, int i, const char** name, double* ms, uint64_t* launches);

#ifdef __cplusplus
}
#endif
#endif
