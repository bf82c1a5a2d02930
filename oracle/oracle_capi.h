/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle.
 *
 * One C ABI, two implementations:
 *   oracle/port/      -> oracle/liboracle_port.so   (a C++ restatement of the reference algorithm)
 *   oracle/ref_capi.cpp -> oracle/_ref/libsoforest_ref.so (the reference headers themselves,
 *                          compiled from /root/reference/proj/include by oracle/Makefile)
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load these libraries, and only as the checker or the CPU baseline — never as the product path.
 *
 * Data conventions (shared with include/sofg.h):
 *   X       column-major float32, column f occupies X[f*n_samples .. (f+1)*n_samples)
 *   labels  int32 class ids in [0, class_count)
 *   forest  exported as flat arrays (see orc_forest_export)
 */
#ifndef SOFG_ORACLE_CAPI_H
#define SOFG_ORACLE_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors soforest::TrainConfig (/root/reference/proj/include/soforest/forest.hpp:38-53). */
typedef struct orc_config {
  uint64_t n_trees;
  int32_t mode; /* 0 exact-only, 1 histogram-only, 2 dynamic (forest.hpp:20) */
  int32_t two_level_binning;
  uint64_t bin_count;
  int32_t has_breakeven;
  int32_t has_max_depth;
  uint64_t breakeven;
  uint64_t max_depth;
  double bootstrap_fraction;
  uint64_t min_samples_split;
  uint64_t max_split_retries;
  uint64_t n_workers;
  uint64_t seed;
  /* Extension: override ProjectionConfig. 0 / <=0 keeps for_features(d). */
  uint64_t num_projections;
  double cell_density;
} orc_config;

typedef struct orc_forest orc_forest;

const char* orc_last_error(void);
const char* orc_impl_name(void);

/* train_forest (forest.hpp:267-313). Returns 0 on success. */
int orc_train_forest(const float* X, const int32_t* labels, uint64_t n_samples, uint64_t n_features,
                     int32_t class_count, const orc_config* cfg, orc_forest** out);
/* Same, with the table converted once (timing excludes the copy into the reference's
 * vector-of-columns dataset). */
typedef struct orc_dataset orc_dataset;
int orc_dataset_create(const float* X, const int32_t* labels, uint64_t n_samples,
                       uint64_t n_features, int32_t class_count, orc_dataset** out);
void orc_dataset_free(orc_dataset* ds);
int orc_train_forest_ds(const orc_dataset* ds, const orc_config* cfg, orc_forest** out);
/* train_tree (forest.hpp:250-262): grow one tree from an explicit active set. */
int orc_train_tree(const float* X, const int32_t* labels, uint64_t n_samples, uint64_t n_features,
                   int32_t class_count, const uint32_t* active, uint64_t n_active,
                   const orc_config* cfg, uint64_t seed, uint64_t depth, orc_forest** out);
/* Same on a dataset handle (no per-call copy of the table). */
int orc_train_tree_ds(const orc_dataset* ds, const uint32_t* active, uint64_t n_active,
                      const orc_config* cfg, uint64_t seed, uint64_t depth, orc_forest** out);

uint64_t orc_forest_num_trees(const orc_forest* f);
uint64_t orc_forest_num_nodes(const orc_forest* f);
uint64_t orc_forest_num_terms(const orc_forest* f);
uint64_t orc_forest_breakeven(const orc_forest* f);
/* tree_off[n_trees+1], left/right/pred/thr[n_nodes], term_off[n_nodes+1], feat/weight[n_terms] */
void orc_forest_export(const orc_forest* f, int64_t* tree_off, int32_t* left, int32_t* right,
                       int32_t* pred, float* thr, int64_t* term_off, uint32_t* feat, float* weight);
void orc_forest_free(orc_forest* f);

/* Flat arrays (the layout orc_forest_export writes) -> forest handle, e.g. trees assembled from
 * several orc_train_tree calls, for orc_predict. */
int orc_forest_import(uint64_t n_trees, uint64_t n_features, int32_t class_count,
                      const int64_t* tree_off, const int32_t* left, const int32_t* right,
                      const int32_t* pred, const float* thr, const int64_t* term_off,
                      const uint32_t* feat, const float* weight, orc_forest** out);
/* predict (forest.hpp:110-121) for n_rows row-major samples; out_label[n_rows],
 * out_votes[n_rows*class_count] (may be NULL). */
int orc_predict(const orc_forest* f, const float* rows, uint64_t n_rows, uint64_t n_features,
                int32_t* out_label, double* out_votes);

/* ---- primitives (per-function parity / golden tests) ---- */
uint64_t orc_split_mix64(uint64_t x);
uint64_t orc_derive_seed(uint64_t seed, uint64_t key);
/* First `count` outputs of make_rng(seed) after discarding `skip` outputs. */
void orc_rng_outputs(uint64_t seed, uint64_t skip, uint64_t count, uint64_t* out);

/* generate_trunk (dataset.hpp:306-329); X column-major [d][n], labels[n]. */
int orc_generate_trunk(uint64_t n_samples, uint64_t n_features, uint64_t seed, float* X,
                       int32_t* labels);
/* bootstrap_sample (dataset.hpp:332-349); out has llround(fraction*n) clamped entries. */
uint64_t orc_bootstrap(uint64_t n_samples, double fraction, uint64_t seed, uint32_t* out);

/* ProjectionConfig::for_features (projection.hpp:39-50). */
void orc_projection_config(uint64_t d, uint64_t* num_projections, uint64_t* expected_nonzeros,
                           double* cell_density);
/* sample_projection_matrix (projection.hpp:57-82) from make_rng(seed) after `skip` draws.
 * row_ptr[R+1]; feat/weight capacity `cap`; returns nnz (or -1 if cap too small).
 * *consumed = engine outputs consumed by the call (binomial + Floyd + coins). */
int64_t orc_sample_projection(uint64_t n_features, uint64_t num_projections, double cell_density,
                              uint64_t seed, uint64_t skip, uint32_t* row_ptr, uint32_t* feat,
                              float* weight, uint64_t cap, uint64_t* consumed);
/* Binomial part only: z and the outputs it consumed. */
uint64_t orc_binomial_draw(uint64_t cells, double density, uint64_t seed, uint64_t skip,
                           uint64_t* consumed);

/* apply_projection (projection.hpp:86-108). */
void orc_apply_projection(const float* X, uint64_t n_samples, const uint32_t* feat,
                          const float* weight, uint64_t n_terms, const uint32_t* active,
                          uint64_t n_active, float* out);

/* sample_boundaries (histogram.hpp:37-61) on make_rng(seed) after `skip`; out capacity bin_count-1. */
uint64_t orc_sample_boundaries(const float* values, uint64_t n, uint64_t bin_count, uint64_t seed,
                               uint64_t skip, float* out, uint64_t* consumed);
/* build_histogram (histogram.hpp:180-206); counts[(nb+1)*k]. */
void orc_build_histogram(const float* values, const int32_t* labels, uint64_t n,
                         const float* boundaries, uint64_t nb, int32_t k, uint32_t* counts);

typedef struct orc_split {
  int32_t found;
  int32_t projection_index;
  float threshold;
  uint32_t n_left;
  uint32_t n_right;
  uint32_t _pad;
  double gain;
} orc_split;

double orc_entropy(const uint32_t* counts, int32_t k);
orc_split orc_best_split_exact(const float* values, const int32_t* labels, uint64_t n, int32_t k);
orc_split orc_best_split_histogram(const float* boundaries, uint64_t nb, const uint32_t* counts,
                                   int32_t k);

/* find_node_split (split.hpp:229-317) over an explicit CSR projection matrix, engine =
 * make_rng(seed) after `skip` outputs. method 0 exact / 1 histogram. *consumed = outputs used.
 * winner_values (optional, size n_active) receives the winning row's projected values. */
orc_split orc_find_node_split(const float* X, const int32_t* labels, uint64_t n_samples,
                              int32_t k, const uint32_t* active, uint64_t n_active,
                              const uint32_t* row_ptr, uint64_t n_rows, const uint32_t* feat,
                              const float* weight, int32_t method, uint64_t bin_count,
                              uint64_t seed, uint64_t skip, uint64_t* consumed,
                              float* winner_values);

/* ---- model I/O (reference build only; model_io.hpp) ---- */
/* train_forest + save_model(forest, path) with the reference's writer. */
int orc_train_save_model(const float* X, const int32_t* labels, uint64_t n_samples,
                         uint64_t n_features, int32_t class_count, const orc_config* cfg,
                         const char* path);
/* load_model(path) with the reference's validating loader; totals of the loaded forest. */
int orc_load_model_summary(const char* path, uint64_t* n_trees, uint64_t* n_nodes);
int orc_train_forest_depths(const float* X, const int32_t* labels, uint64_t n_samples, uint64_t n_features,
                            int32_t class_count, const orc_config* cfg, uint64_t* nodes, uint64_t* samples,
                            uint64_t cap, uint64_t* n_depths);
uint64_t orc_csv_number(double v, char* out, uint64_t cap);
int orc_load_model_calibration(const char* path, uint64_t* breakeven, int32_t* has_cal,
                               uint64_t* cal_breakeven, uint64_t* n_samples, int32_t* fallback);

#ifdef __cplusplus
}
#endif
#endif
