// Host-callable launchers for the sm_100a kernels (all asynchronous on `st`).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "common.hpp"

namespace sofg {

// sample.cu
cudaError_t launch_sample_projection(const NodeIn* nodes, int n_nodes, uint32_t d, uint32_t R,
                                     uint32_t zmax, uint32_t* terms, uint32_t* row_ptr,
                                     uint32_t* pos_after, cudaStream_t st);
cudaError_t launch_hist_draws(const NodeIn* nodes, const uint32_t* hist_nodes, int n_hist,
                              uint32_t R, uint32_t bins, const uint32_t* pos_after_proj,
                              uint32_t* draws, uint32_t* pos_split, cudaStream_t st);
cudaError_t launch_hist_boundaries(const NodeIn* nodes, const uint32_t* hist_nodes, int n_hist,
                                   uint32_t R, uint32_t bins, const uint32_t* draws,
                                   const uint32_t* terms, const uint32_t* row_ptr,
                                   const uint64_t* gbase, const float* G, float* bnd,
                                   uint32_t* nb, cudaStream_t st);

// split.cu
size_t hist_count_smem(uint32_t bins, int k, int chunk_cap);
cudaError_t launch_hist_count(const NodeIn* nodes, const uint32_t* node_hist_slot,
                              const HistWork* work, int n_work, const uint32_t* multi_slot,
                              uint32_t R, uint32_t bins, int k, int chunk_cap,
                              const uint32_t* terms, const uint32_t* row_ptr, const uint8_t* lab,
                              const uint64_t* gbase, const float* G, const float* bnd,
                              const uint32_t* nb, const double* xl, uint32_t* gcnt,
                              uint32_t* done, RowRes* rowres, cudaStream_t st);
cudaError_t launch_hist_select(const uint32_t* hist_nodes, int n_hist, uint32_t R,
                               const RowRes* rowres, NodeRes* res, cudaStream_t st);
// csp.cu — column-sweep gather into G (per node: z x n raw values, term-major)
uint64_t csp_items(uint32_t n, uint32_t z);
cudaError_t launch_csp(const NodeIn* nodes, int n_nodes, const uint64_t* gbase,
                       const uint32_t* terms, uint32_t d, uint64_t n_items, uint32_t* cnt,
                       uint64_t* items, const uint32_t* idx, const float* X, uint64_t ld, float* G,
                       cudaStream_t st);

// exact.cu — register-resident exact splitter, bucketed by node size (<= 2048 samples)
int exact_bucket(uint32_t n);
cudaError_t launch_exact_bucket(int bucket, const NodeIn* nodes, const uint32_t* list, int n,
                                uint32_t R, int k, const uint32_t* terms,
                                const uint32_t* row_ptr, const uint8_t* lab, const uint64_t* gbase,
                                const float* G, const double* xl, NodeRes* res, cudaStream_t st);

// partition.cu
cudaError_t launch_partition(const NodeIn* nodes, int n_nodes, const Tile* tiles, int n_tiles,
                             const uint32_t* tile_first, uint32_t R, int k, const uint32_t* terms,
                             const uint32_t* row_ptr, const uint32_t* pos_proj,
                             const uint32_t* pos_split, const uint32_t* idx_in,
                             const uint8_t* lab_in, uint32_t* idx_out, uint8_t* lab_out,
                             const uint64_t* gbase, const float* G, NodeRes* res, uint32_t* flags,
                             uint32_t* tile_left, cudaStream_t st);

cudaError_t launch_sector_count(const NodeIn* nodes, const Tile* tiles, int n_tiles,
                                const uint32_t* idx, NodeRes* res, cudaStream_t st);

// misc.cu
cudaError_t launch_generate_trunk(float* X, uint64_t ld, uint8_t* labels, uint64_t n, uint64_t d,
                                  int k, uint64_t seed, cudaStream_t st);
cudaError_t launch_apply_projection(const float* X, uint64_t ld, const uint32_t* terms, int nt,
                                    const uint32_t* active, uint64_t n, float* out,
                                    cudaStream_t st);
cudaError_t launch_predict(const float* rows, uint64_t n_rows, uint64_t d, const int64_t* tree_off,
                           int n_trees, const int32_t* left, const int32_t* right,
                           const int32_t* pred, const float* thr, const int64_t* term_off,
                           const uint32_t* terms, int k, uint32_t* votes, cudaStream_t st);

}  // namespace sofg
