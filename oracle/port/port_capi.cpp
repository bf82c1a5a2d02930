// TEST INFRASTRUCTURE ONLY — C ABI over the restated oracle (oracle/port/soforest_port.hpp).
#include <algorithm>
#include <cstring>

#include "../forest_flat.hpp"
#include "soforest_port.hpp"

using namespace port;

ORC_COMMON_EXPORTS

extern "C" int orc_predict(const orc_forest* f, const float* rows, uint64_t n_rows, uint64_t n_features,
                           int32_t* out_label, double* out_votes) {
  return orc_guard([&] {
    if (n_features != f->n_features) throw std::invalid_argument("feature count mismatch");
    for (uint64_t i = 0; i < n_rows; ++i)
      out_label[i] = f->predict_row(rows + i * n_features, out_votes ? out_votes + i * f->class_count : nullptr);
  });
}

static Config to_cfg(const orc_config* c) {
  Config k;
  k.n_trees = c->n_trees;
  k.mode = c->mode;
  k.bin_count = c->bin_count;
  if (c->has_breakeven) k.breakeven = c->breakeven;
  k.bootstrap_fraction = c->bootstrap_fraction;
  if (c->has_max_depth) k.max_depth = c->max_depth;
  k.min_samples_split = c->min_samples_split;
  k.max_split_retries = c->max_split_retries;
  k.n_workers = c->n_workers;
  k.seed = c->seed;
  k.num_projections = c->num_projections;
  k.cell_density = c->cell_density;
  return k;
}

static Dataset to_data(const float* X, const int32_t* y, uint64_t n, uint64_t d, int32_t k) {
  Dataset D;
  D.X = X;
  D.y = y;
  D.n = n;
  D.d = d;
  D.k = k;
  return D;
}

extern "C" const char* orc_impl_name(void) { return "port"; }

extern "C" int orc_train_forest(const float* X, const int32_t* y, uint64_t n, uint64_t d,
                                int32_t k, const orc_config* c, orc_forest** out) {
  return orc_guard([&] {
    const Dataset D = to_data(X, y, n, d, k);
    uint64_t be = 0;
    auto trees = train_forest(D, to_cfg(c), &be);
    auto* f = new orc_forest;
    f->breakeven = be;
    f->class_count = k;
    f->n_features = d;
    for (auto& t : trees) f->add_tree(t);
    *out = f;
  });
}

struct orc_dataset {
  std::vector<float> X;
  std::vector<int32_t> y;
  Dataset D;
};

extern "C" int orc_dataset_create(const float* X, const int32_t* y, uint64_t n, uint64_t d,
                                  int32_t k, orc_dataset** out) {
  return orc_guard([&] {
    auto* ds = new orc_dataset;
    ds->X.assign(X, X + n * d);
    ds->y.assign(y, y + n);
    ds->D = to_data(ds->X.data(), ds->y.data(), n, d, k);
    *out = ds;
  });
}
extern "C" void orc_dataset_free(orc_dataset* ds) { delete ds; }

extern "C" int orc_train_forest_ds(const orc_dataset* ds, const orc_config* c, orc_forest** out) {
  return orc_train_forest(ds->D.X, ds->D.y, ds->D.n, ds->D.d, ds->D.k, c, out);
}

extern "C" int orc_train_tree(const float* X, const int32_t* y, uint64_t n, uint64_t d, int32_t k,
                              const uint32_t* active, uint64_t n_active, const orc_config* c,
                              uint64_t seed, uint64_t depth, orc_forest** out) {
  return orc_guard([&] {
    const Dataset D = to_data(X, y, n, d, k);
    std::vector<uint32_t> a(active, active + n_active);
    Tree t = train_tree(D, a, to_cfg(c), seed, depth);
    auto* f = new orc_forest;
    f->class_count = k;
    f->n_features = d;
    f->add_tree(t);
    *out = f;
  });
}

extern "C" int orc_train_tree_ds(const orc_dataset* ds, const uint32_t* active, uint64_t n_active,
                                 const orc_config* c, uint64_t seed, uint64_t depth, orc_forest** out) {
  return orc_train_tree(ds->D.X, ds->D.y, ds->D.n, ds->D.d, ds->D.k, active, n_active, c, seed, depth, out);
}

extern "C" uint64_t orc_split_mix64(uint64_t x) { return split_mix64(x); }
extern "C" uint64_t orc_derive_seed(uint64_t s, uint64_t k) { return derive_seed(s, k); }
extern "C" void orc_rng_outputs(uint64_t seed, uint64_t skip, uint64_t count, uint64_t* out) {
  Engine g = make_rng(seed);
  g.discard(skip);
  for (uint64_t i = 0; i < count; ++i) out[i] = g();
}

extern "C" int orc_generate_trunk(uint64_t n, uint64_t d, uint64_t seed, float* X, int32_t* y) {
  return orc_guard([&] { generate_trunk(n, d, seed, X, y); });
}

extern "C" uint64_t orc_bootstrap(uint64_t n, double fraction, uint64_t seed, uint32_t* out) {
  auto v = bootstrap(n, fraction, seed);
  std::copy(v.begin(), v.end(), out);
  return v.size();
}

extern "C" void orc_projection_config(uint64_t d, uint64_t* R, uint64_t* e, double* dens) {
  ProjConfig c = proj_config(d);
  *R = c.rows;
  *e = c.expected;
  *dens = c.density;
}

extern "C" int64_t orc_sample_projection(uint64_t d, uint64_t R, double density, uint64_t seed,
                                         uint64_t skip, uint32_t* row_ptr, uint32_t* feat,
                                         float* weight, uint64_t cap, uint64_t* consumed) {
  Engine e = make_rng(seed);
  e.discard(skip);
  CountingEngine g{e};
  ProjConfig c;
  c.d = d;
  c.rows = R;
  c.density = density;
  Matrix m = sample_matrix(c, g);
  *consumed = g.count;
  uint64_t nnz = 0;
  row_ptr[0] = 0;
  for (uint64_t r = 0; r < R; ++r) {
    for (const Term& t : m[r]) {
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
  Engine e = make_rng(seed);
  e.discard(skip);
  CountingEngine g{e};
  std::binomial_distribution<long long> b((long long)cells, density);
  const uint64_t z = uint64_t(b(g));
  *consumed = g.count;
  return z;
}

extern "C" void orc_apply_projection(const float* X, uint64_t n, const uint32_t* feat,
                                     const float* w, uint64_t nt, const uint32_t* active,
                                     uint64_t na, float* out) {
  Dataset D = to_data(X, nullptr, n, 0, 0);
  Row row;
  for (uint64_t t = 0; t < nt; ++t) row.push_back({feat[t], w[t]});
  apply(D, row, active, na, out);
}

extern "C" uint64_t orc_sample_boundaries(const float* v, uint64_t n, uint64_t bins, uint64_t seed,
                                          uint64_t skip, float* out, uint64_t* consumed) {
  Engine e = make_rng(seed);
  e.discard(skip);
  CountingEngine g{e};
  const uint64_t nb = sample_boundaries(v, n, bins, g, out);
  *consumed = g.count;
  return nb;
}

extern "C" void orc_build_histogram(const float* v, const int32_t* y, uint64_t n, const float* b,
                                    uint64_t nb, int32_t k, uint32_t* counts) {
  build_histogram(v, y, n, b, nb, k, counts);
}

extern "C" double orc_entropy(const uint32_t* c, int32_t k) { return entropy(c, k); }

static orc_split to_c(const std::optional<Split>& s) {
  orc_split o{};
  if (!s) return o;
  o.found = 1;
  o.projection_index = int32_t(s->row);
  o.threshold = s->threshold;
  o.n_left = s->n_left;
  o.n_right = s->n_right;
  o.gain = s->gain;
  return o;
}

extern "C" orc_split orc_best_split_exact(const float* v, const int32_t* y, uint64_t n, int32_t k) {
  return to_c(best_split_exact(v, y, n, k));
}
extern "C" orc_split orc_best_split_histogram(const float* b, uint64_t nb, const uint32_t* counts,
                                              int32_t k) {
  return to_c(best_split_histogram(b, nb, counts, k));
}

extern "C" orc_split orc_find_node_split(const float* X, const int32_t* y, uint64_t n, int32_t k,
                                         const uint32_t* active, uint64_t na,
                                         const uint32_t* row_ptr, uint64_t R, const uint32_t* feat,
                                         const float* w, int32_t method, uint64_t bins,
                                         uint64_t seed, uint64_t skip, uint64_t* consumed,
                                         float* winner_values) {
  Dataset D = to_data(X, y, n, 0, k);
  Matrix m(R);
  for (uint64_t r = 0; r < R; ++r)
    for (uint32_t q = row_ptr[r]; q < row_ptr[r + 1]; ++q) m[r].push_back({feat[q], w[q]});
  Engine e = make_rng(seed);
  e.discard(skip);
  CountingEngine g{e};
  std::vector<float> values;
  auto s = find_node_split(D, active, na, m, method == 1 ? kHistogram : kExact, bins, g, values);
  *consumed = g.count;
  if (s && winner_values) std::memcpy(winner_values, values.data() + s->row * na, na * 4);
  return to_c(s);
}
