// Host-callable launchers for the sm_100a kernels (all asynchronous on `st`).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "common.hpp"

namespace sofg {

// Dynamic shared-memory opt-in, always set to the sm_100 maximum: the attribute is per kernel and
// process-wide, so per-launch values would race between the host threads of concurrent tree groups.
constexpr int kSmemOptin = 226 * 1024;  // 227 KB opt-in minus room for static __shared__

// Grow-only device scratch owned by a WaveRunner (so by one device and one stream): launchers whose
// temporaries are sized at launch time take numbered slots from it. Growing a slot waits for the
// stream first (an earlier launch may still read the old block).
class Scratch {
 public:
  static constexpr int kSlots = 10;
  enum : int { kSampleKeys = 0, kSampleAux = 1, kBigFirst = 2 };  // exact_big uses 2..8
  Scratch() = default;
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  ~Scratch();
  void* get(int slot, size_t bytes, cudaStream_t st);  // nullptr on allocation failure

 private:
  void* p_[kSlots] = {};
  size_t cap_[kSlots] = {};
};

// sample.cu
cudaError_t launch_sample_projection(const NodeIn* nodes, int n_nodes, uint32_t d, uint32_t R,
                                     uint32_t zmax, uint32_t* terms, uint32_t* row_ptr,
                                     uint32_t* pos_after, Scratch& scratch, cudaStream_t st);
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
                              uint32_t R, uint32_t bins, int k, int chunk_cap, int two_level,
                              const uint32_t* terms, const uint32_t* row_ptr, const uint8_t* lab,
                              const uint64_t* gbase, const float* G, const float* bnd,
                              const uint32_t* nb, const double* xl, uint32_t* gcnt,
                              uint32_t* done, RowRes* rowres, cudaStream_t st);
// lane = row counting (two classes, <= 256 bins), CTA = 32 rows x chunk (HistWork.row0 % 32 == 0)
bool hist_count_lane_rows(uint32_t R, uint32_t bins, int k);
size_t hist_count_lr_smem(uint32_t bins, int chunk_cap);
cudaError_t launch_hist_count_lr(const NodeIn* nodes, const uint32_t* node_hist_slot, const HistWork* work,
                                 int n_work, const uint32_t* multi_slot, uint32_t R, uint32_t bins, int chunk_cap,
                                 int two_level, const uint8_t* lab, const uint64_t* gbase, const float* G,
                                 const float* bnd, const uint32_t* nb, const double* xl, uint32_t* gcnt,
                                 uint32_t* done, RowRes* rowres, cudaStream_t st);
cudaError_t launch_hist_select(const uint32_t* hist_nodes, int n_hist, uint32_t R,
                               const RowRes* rowres, NodeRes* res, cudaStream_t st);
// sweep.cu — projection stage: node rows into V (per node n x Rp floats, sample-major)
cudaError_t launch_transpose_rows(const float* X, uint64_t ld, uint64_t n, uint64_t d, float* XR,
                                  uint64_t ldr, cudaStream_t st);
cudaError_t launch_inv_init(const uint32_t* idx, const uint64_t* off, uint32_t B,
                            uint64_t n_samples, uint64_t max_per_tree, uint32_t* inv,
                            cudaStream_t st);
cudaError_t launch_pos_fill(const NodeIn* nodes, const Tile* tiles, int n_tiles, uint64_t total,
                            uint32_t* pos_node, cudaStream_t st);
size_t aug_bytes(uint64_t total_terms, uint32_t n_nodes, uint32_t R, uint32_t d);
// pnode (optional, 16 bytes per node): what a pair record of the node needs, in one load —
// {V block of the node's position 0 (/ 8, mod 2^32), term-list block offset, quarter boundaries}
cudaError_t launch_aug_build(const NodeIn* nodes, int n_nodes, const uint32_t* terms,
                             const uint32_t* row_ptr, uint32_t R, uint32_t d, void* aug,
                             uint16_t* qsplit, const uint64_t* vbase, uint32_t* pnode, cudaStream_t st);
size_t row_sweep_smem(uint64_t ldr, uint32_t B, uint32_t R);
void row_sweep_variant(uint32_t B, uint32_t d, uint32_t* cta_threads, uint32_t* entry_bytes);
bool aug_narrow(uint32_t d);  // 16-bit term entries (d < 8192)
// sweep_pipe.cu — pipelined sweep: per-sample pair lists, then a warp-specialised persistent kernel
bool row_sweep_pipe_fits(uint64_t ldr, uint32_t B, uint32_t R);
size_t pair_rec_bytes();
cudaError_t launch_pair_build(const uint32_t* inv, uint32_t B, uint32_t N, const uint32_t* pos_node,
                              const uint32_t* pnode, uint32_t R, uint32_t d, void* recs, uint32_t* pcnt,
                              int n_sm, cudaStream_t st);
cudaError_t launch_row_sweep_pipe(const float* XR, uint64_t ldr, uint32_t N, const void* recs,
                                  const uint32_t* pcnt, uint32_t B, const void* aug, uint32_t R,
                                  uint32_t d, float* V, int n_sm, cudaStream_t st);
cudaError_t launch_row_sweep(const float* XR, uint64_t ldr, uint32_t N, const uint32_t* inv,
                             uint32_t B, const uint32_t* pos_node, const NodeIn* nodes,
                             const uint64_t* vbase, const void* aug, const uint16_t* qsplit, uint32_t R,
                             uint32_t d, float* V, int n_sm, cudaStream_t st);
cudaError_t launch_project_gather(const NodeIn* nodes, const Tile* tiles, int n_tiles,
                                  const uint64_t* vbase, const uint32_t* terms,
                                  const uint32_t* row_ptr, uint32_t R, uint32_t zmax,
                                  const uint32_t* idx, const float* X, uint64_t ld, float* V,
                                  cudaStream_t st);

// exact.cu — register-resident exact splitter, bucketed by node size (<= 2048 samples)
constexpr int kExactBuckets = 9;  // n <= 8, 16, 32, ..., 2048
int exact_bucket(uint32_t n);
cudaError_t launch_exact_bucket(int bucket, const NodeIn* nodes, const uint32_t* list, int n,
                                uint32_t R, int k, const uint32_t* terms,
                                const uint32_t* row_ptr, const uint8_t* lab, const uint64_t* gbase,
                                const float* G, const double* xl, const float* xlf, NodeRes* res,
                                const float* rowlb, const unsigned long long* xstar,
                                cudaStream_t st);
// Branch-and-bound row bounds for exact nodes (two classes): rowlb[li*R + r], xstar[li].
cudaError_t launch_exact_prune(const NodeIn* nodes, const uint32_t* list, int n_list, uint32_t R,
                               const uint32_t* row_ptr, const uint8_t* lab, const uint64_t* gbase,
                               const float* G, const double* xl, float* rowlb,
                               unsigned long long* xstar, int buckets, int k, cudaStream_t st);

// exact_big.cu — exact splits of nodes above kExactSmemMax (device-wide segmented sort)
cudaError_t launch_exact_big(const NodeIn* nodes, const NodeIn* h_nodes, const uint32_t* h_list,
                             int n, uint32_t R, int k, const uint32_t* row_ptr, const uint8_t* lab,
                             const uint64_t* vbase, const float* V, const double* xl, NodeRes* res,
                             Scratch& scratch, cudaStream_t st);

// partition.cu
cudaError_t launch_partition(const NodeIn* nodes, int n_nodes, const Tile* tiles, int n_tiles,
                             const uint32_t* tile_first, uint32_t R, int k, const uint32_t* terms,
                             const uint32_t* row_ptr, const uint32_t* pos_proj,
                             const uint32_t* pos_split, const uint32_t* idx_in,
                             const uint8_t* lab_in, uint32_t* idx_out, uint8_t* lab_out,
                             const uint64_t* gbase, const float* G, NodeRes* res, uint32_t* flags,
                             uint32_t* tile_left, uint32_t* inv, uint32_t B, uint32_t* class_left,
                             cudaStream_t st);  // class_left: [node][k] left class counts (zeroed by the caller)

cudaError_t launch_win_terms(const NodeIn* nodes, const NodeRes* res, const uint32_t* row_ptr,
                             const uint32_t* terms, uint32_t R, const uint32_t* list, int n_list,
                             const uint32_t* off, uint32_t* out, cudaStream_t st);
cudaError_t launch_sector_count(const NodeIn* nodes, const Tile* tiles, int n_tiles,
                                const uint32_t* idx, NodeRes* res, cudaStream_t st);

// misc.cu
// Tree b's sorted sample ids from its bitmap bits[b * W, (b + 1) * W) into ids[off[b] ...].
cudaError_t launch_bits_to_ids(const uint32_t* bits, uint64_t W, uint32_t B, const uint64_t* off, uint32_t* ids,
                               cudaStream_t st);
// lab_out[p] = labels[idx[p]]; counts[b * k + c] = class-c count of tree b's root segment
cudaError_t launch_root_labels(const uint32_t* idx, const uint64_t* off, uint32_t B,
                               uint64_t max_per_tree, const uint8_t* labels, uint8_t* lab_out,
                               int k, uint32_t* counts, cudaStream_t st);
cudaError_t launch_generate_trunk(float* X, uint64_t ld, uint8_t* labels, uint64_t n, uint64_t d,
                                  int k, uint64_t seed, cudaStream_t st);
cudaError_t launch_apply_projection(const float* X, uint64_t ld, const uint32_t* terms, int nt,
                                    const uint32_t* active, uint64_t n, float* out,
                                    cudaStream_t st);
cudaError_t launch_predict(const float* rows, uint64_t n_rows, uint64_t d, const int64_t* tree_off,
                           int n_trees, const int32_t* left, const int32_t* right,
                           const int32_t* pred, const float* thr, const int64_t* term_off,
                           const uint32_t* terms, int k, uint32_t* votes, cudaStream_t st);

// wide.cu: more than kMaxClasses classes (RowRes per (node, row); k_hist_select picks the row)
size_t exact_wide_smem(uint32_t nmax, int k);
cudaError_t launch_exact_wide(const NodeIn* nodes, const uint32_t* list, int n_list, uint32_t nmax, uint32_t R,
                              int k, const uint32_t* row_ptr, const uint8_t* lab, const uint64_t* gbase,
                              const float* G, const double* xl, RowRes* rowres, cudaStream_t st);
size_t hist_wide_smem(uint32_t bins, int k);
// work items: one per (node, row = row0, chunk of <= 65535 samples)
cudaError_t launch_hist_wide(const NodeIn* nodes, const uint32_t* node_hist_slot, const HistWork* work, int n_work,
                             const uint32_t* multi_slot, uint32_t R, uint32_t bins, int k, int two_level,
                             const uint8_t* lab, const uint64_t* gbase, const float* G, const float* bnd,
                             const uint32_t* nb, const double* xl, uint32_t* gcnt, uint32_t* done, RowRes* rowres,
                             cudaStream_t st);

}  // namespace sofg
