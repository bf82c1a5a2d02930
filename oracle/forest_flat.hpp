// TEST INFRASTRUCTURE ONLY — flat forest container shared by the two oracle C ABIs.
#pragma once
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "oracle_capi.h"

struct orc_forest {
  std::vector<int64_t> tree_off{0};
  std::vector<int32_t> left, right, pred;
  std::vector<float> thr;
  std::vector<int64_t> term_off{0};
  std::vector<uint32_t> feat;
  std::vector<float> weight;
  uint64_t breakeven = 0;
  int32_t class_count = 0;
  uint64_t n_features = 0;

  // Appends one tree; `Node` exposes projection (feature/weight terms), threshold, left, right,
  // predicted_class.
  template <class TreeT>
  void add_tree(const TreeT& t) {
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

  // Reference predict semantics (forest.hpp:88-121) over the flat arrays.
  int32_t predict_row(const float* x, double* votes) const {
    std::vector<double> v(class_count, 0.0);
    const uint64_t T = tree_off.size() - 1;
    for (uint64_t t = 0; t < T; ++t) {
      int64_t nd = tree_off[t];
      while (left[nd] >= 0) {
        double acc = 0.0;
        bool first = true;
        for (int64_t q = term_off[nd]; q < term_off[nd + 1]; ++q) {
          const double p = double(weight[q]) * double(x[feat[q]]);
          acc = first ? p : acc + p;
          first = false;
        }
        nd = tree_off[t] + (float(acc) <= thr[nd] ? left[nd] : right[nd]);
      }
      v[pred[nd]] += 1.0;
    }
    int32_t best = 0;
    for (int32_t c = 0; c < class_count; ++c) {
      v[c] /= double(T);
      if (v[c] > v[best]) best = c;
    }
    if (votes) std::memcpy(votes, v.data(), sizeof(double) * class_count);
    return best;
  }
};

inline thread_local std::string g_orc_err;

template <class F>
int orc_guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_orc_err = std::string("invalid_argument: ") + e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_orc_err = std::string("out_of_range: ") + e.what();
    return 2;
  } catch (const std::exception& e) {
    g_orc_err = std::string("error: ") + e.what();
    return 3;
  }
}

#define ORC_COMMON_EXPORTS                                                                     \
  extern "C" const char* orc_last_error(void) { return g_orc_err.c_str(); }                    \
  extern "C" uint64_t orc_forest_num_trees(const orc_forest* f) { return f->tree_off.size() - 1; } \
  extern "C" uint64_t orc_forest_num_nodes(const orc_forest* f) { return f->left.size(); }     \
  extern "C" uint64_t orc_forest_num_terms(const orc_forest* f) { return f->feat.size(); }     \
  extern "C" uint64_t orc_forest_breakeven(const orc_forest* f) { return f->breakeven; }       \
  extern "C" void orc_forest_export(const orc_forest* f, int64_t* tree_off, int32_t* left,     \
                                    int32_t* right, int32_t* pred, float* thr, int64_t* term_off, \
                                    uint32_t* feat, float* weight) {                           \
    std::memcpy(tree_off, f->tree_off.data(), f->tree_off.size() * 8);                         \
    std::memcpy(left, f->left.data(), f->left.size() * 4);                                     \
    std::memcpy(right, f->right.data(), f->right.size() * 4);                                  \
    std::memcpy(pred, f->pred.data(), f->pred.size() * 4);                                     \
    std::memcpy(thr, f->thr.data(), f->thr.size() * 4);                                        \
    std::memcpy(term_off, f->term_off.data(), f->term_off.size() * 8);                         \
    std::memcpy(feat, f->feat.data(), f->feat.size() * 4);                                     \
    std::memcpy(weight, f->weight.data(), f->weight.size() * 4);                               \
  }                                                                                            \
  extern "C" void orc_forest_free(orc_forest* f) { delete f; }                                 \
  extern "C" int orc_forest_import(uint64_t n_trees, uint64_t n_features, int32_t k,            \
                                   const int64_t* tree_off, const int32_t* left,               \
                                   const int32_t* right, const int32_t* pred, const float* thr, \
                                   const int64_t* term_off, const uint32_t* feat,              \
                                   const float* weight, orc_forest** out) {                    \
    return orc_guard([&] {                                                                     \
      auto* f = new orc_forest;                                                                \
      const uint64_t N = uint64_t(tree_off[n_trees]), Q = uint64_t(term_off[N]);               \
      f->tree_off.assign(tree_off, tree_off + n_trees + 1);                                    \
      f->left.assign(left, left + N);                                                          \
      f->right.assign(right, right + N);                                                       \
      f->pred.assign(pred, pred + N);                                                          \
      f->thr.assign(thr, thr + N);                                                             \
      f->term_off.assign(term_off, term_off + N + 1);                                          \
      f->feat.assign(feat, feat + Q);                                                          \
      f->weight.assign(weight, weight + Q);                                                    \
      f->class_count = k;                                                                      \
      f->n_features = n_features;                                                              \
      *out = f;                                                                                \
    });                                                                                        \
  }
