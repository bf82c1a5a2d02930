// Device context and the per-wave launch sequence.
#pragma once
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.hpp"
#include "kernels.hpp"

namespace sofg {

class ThreadPool;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t cap = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  T* ensure(size_t n) {
    if (n <= cap && p) return p;
    if (p && std::getenv("SOFG_GROW_LOG")) std::fprintf(stderr, "[grow] device %zu -> %zu bytes\n", cap * sizeof(T), n * sizeof(T));
    release();  // cudaFree synchronizes the device: grow rarely (x2 up to 256 MB, +1/8 above)
    const size_t want = n < 64 ? 64 : (n * sizeof(T) <= (size_t(256) << 20) ? 2 * n : n + n / 8);
    alloc(want);
    return p;
  }
  T* exact(size_t n) {  // no slack (large one-off buffers)
    if (n <= cap && p) return p;
    release();
    alloc(n ? n : 1);
    return p;
  }

 private:
  void alloc(size_t n) {
    void* q = nullptr;
    const cudaError_t e = cudaMalloc(&q, n * sizeof(T));
    if (e != cudaSuccess) {
      cudaGetLastError();  // clear the sticky-free allocation error
      cuda_check(e, "cudaMalloc");
    }
    p = static_cast<T*>(q);
    cap = n;
  }
};

template <class T>
struct PinnedBuf {
  T* p = nullptr;
  size_t cap = 0;
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  T* ensure(size_t n) {
    if (n <= cap && p) return p;
    if (p && std::getenv("SOFG_GROW_LOG")) std::fprintf(stderr, "[grow] pinned %zu -> %zu bytes\n", cap * sizeof(T), n * sizeof(T));
    if (p) cudaFreeHost(p);
    p = nullptr;
    const size_t want = n < 64 ? 64 : 2 * n;  // pinning is slow (~ms per 10 MB): grow rarely
    cuda_check(cudaMallocHost(&p, want * sizeof(T)), "cudaMallocHost");
    cap = want;
    return p;
  }
};

// Dataset resident in HBM: column-major float table with a 32-sample-aligned leading dimension,
// u8 labels, and the reference's xlogx table up to n.
struct DeviceData {
  DevBuf<float> X;
  DevBuf<float> XR;  // row-major copy [n][ldr] for the sample-major projection sweep (sweep.cu)
  uint64_t ldr = 0;
  DevBuf<uint8_t> lab;
  DevBuf<double> xl;
  DevBuf<float> xlf;  // float(xl[i]): prefilter table (exact values are always re-evaluated in double)
  uint64_t xl_n = 0;  // sample count the xlogx tables were built for
  PinnedBuf<uint8_t> lab_stage;     // page-locked staging of the labels (asynchronous upload)
  cudaEvent_t lab_ev = nullptr;     // the staging's last copy
  DeviceData() = default;
  DeviceData(const DeviceData&) = delete;
  DeviceData& operator=(const DeviceData&) = delete;
  ~DeviceData() {
    if (lab_ev) cudaEventDestroy(lab_ev);
  }
  uint64_t n = 0, d = 0, ld = 0;
  int k = 0;
  std::vector<int32_t> labels_host;  // for root class counts
  bool loaded() const { return n > 0; }
};

// One wave: a set of open nodes searched and partitioned together.
struct WaveSpec {
  uint32_t R = 0, d = 0, bins = 256;
  int k = 2;
  int chunk_cap = 8192;
  bool two_level = true;  // TrainConfig::two_level_binning (decides the NaN bin, split.hpp:281-283)
  std::vector<NodeIn> nodes;
  // optional host-supplied projection matrices (kNodeGivenCsr on every node)
  bool given_csr = false;
  std::vector<uint32_t> given_terms;    // concatenated, node i at nodes[i].term_off
  std::vector<uint32_t> given_row_ptr;  // [nodes][R+1]
  std::vector<uint32_t> given_pos;      // stream position after the matrix (per node)
  // level buffers
  const uint32_t* idx_in = nullptr;
  const uint8_t* lab_in = nullptr;
  uint32_t* idx_out = nullptr;
  uint8_t* lab_out = nullptr;
  // inverse map of the batch (sweep.cu): inv[s*B + tree] = level position of sample s in tree,
  // maintained by the partition. nullptr: the projection stage gathers instead of sweeping.
  uint32_t* inv = nullptr;
  uint32_t B = 0;
  uint64_t total = 0;  // level buffer length (positions)
  int force_mode = -1;  // -1 auto, 0 gather, 1 sweep (tests / experiments)
};

struct KernelTime {
  const char* name;
  double ms;
  uint64_t launches;
};

struct WaveStats {
  double ms_sample = 0, ms_hist_rng = 0, ms_hist_count = 0, ms_exact = 0, ms_partition = 0;
  double ms_total = 0;
  uint64_t waves = 0, nodes = 0, hist_nodes = 0, exact_nodes = 0;
  uint64_t launches = 0;
  // algorithmic gather bytes (useful 4 B per gathered value; 32 B-sector model)
  double hist_strict_bytes = 0, hist_sector_bytes = 0, exact_strict_bytes = 0,
         exact_sector_bytes = 0;
  uint64_t hist_count_launches = 0, exact_launches = 0;
  uint64_t sweep_waves = 0, gather_waves = 0;
  double sweep_alg_bytes = 0;  // table rows streamed + V written + term lists read (sweep waves)
  uint32_t sweep_cta_threads = 0, sweep_entry_bytes = 0;  // variant of the widest sweep wave
  uint64_t sweep_widest_nodes = 0;
  std::vector<KernelTime> per_kernel;  // CUDA-event time per launch site (stats mode)
  void merge(const WaveStats& o) {
    ms_sample += o.ms_sample; ms_hist_rng += o.ms_hist_rng; ms_hist_count += o.ms_hist_count;
    ms_exact += o.ms_exact; ms_partition += o.ms_partition; ms_total += o.ms_total;
    waves += o.waves; nodes += o.nodes; hist_nodes += o.hist_nodes; exact_nodes += o.exact_nodes;
    launches += o.launches; hist_strict_bytes += o.hist_strict_bytes;
    hist_sector_bytes += o.hist_sector_bytes; exact_strict_bytes += o.exact_strict_bytes;
    exact_sector_bytes += o.exact_sector_bytes; hist_count_launches += o.hist_count_launches;
    exact_launches += o.exact_launches; sweep_waves += o.sweep_waves; gather_waves += o.gather_waves;
    sweep_alg_bytes += o.sweep_alg_bytes;
    if (o.sweep_widest_nodes > sweep_widest_nodes) {
      sweep_widest_nodes = o.sweep_widest_nodes;
      sweep_cta_threads = o.sweep_cta_threads;
      sweep_entry_bytes = o.sweep_entry_bytes;
    }
    for (const auto& k : o.per_kernel) {
      bool found = false;
      for (auto& m : per_kernel)
        if (m.name == k.name) {
          m.ms += k.ms;
          m.launches += k.launches;
          found = true;
        }
      if (!found) per_kernel.push_back(k);
    }
  }
  void add_kernel(const char* name, double ms) {
    for (auto& k : per_kernel)
      if (k.name == name) {
        k.ms += ms;
        k.launches++;
        return;
      }
    per_kernel.push_back({name, ms, 1});
  }
};

class WaveRunner {
 public:
  // Runners created with a shared DeviceData train on the same resident table on their own stream
  // (several tree groups in flight on one GPU).
  // `stream`, when given, is shared (not owned): runners on one stream execute their waves in
  // submission order, and collect() waits on this runner's own completion event only.
  explicit WaveRunner(int device, std::shared_ptr<DeviceData> data = nullptr,
                      cudaStream_t stream = nullptr);
  ~WaveRunner();
  WaveRunner(const WaveRunner&) = delete;
  WaveRunner& operator=(const WaveRunner&) = delete;

  cudaStream_t stream() const { return st_; }
  int device() const { return device_; }
  DeviceData& data() { return *data_; }
  const DeviceData& data() const { return *data_; }
  std::shared_ptr<DeviceData> shared_data() const { return data_; }

  // Searches and partitions every node of `w`; res[i] receives node i's result.
  void run(const WaveSpec& w, std::vector<NodeRes>& res) {
    submit(w);
    collect(w, res);
  }
  // Asynchronous halves of run(): submit() enqueues the wave's copies and kernels and returns;
  // collect() waits for them and copies the node results out. `w` must stay alive in between.
  void submit(const WaveSpec& w);
  void collect(const WaveSpec& w, std::vector<NodeRes>& res);
  // Same wait, no copy: the node results in page-locked memory, valid until the next submit().
  const NodeRes* collect_view(const WaveSpec& w);
  // The partition's left class counts of the collected wave, [node][k]; valid as long as the
  // results of collect_view are.
  const uint32_t* class_counts_view() const { return h_cl_p_; }
  // Only the wait for the wave (no host pool use): callers sharing a pool wait first, then
  // take their host turn and call collect_view().
  bool last_was_sweep() const { return pend_sweep_; }
  float last_wave_ms() const { return last_wave_ms_; }  // device time of the last collected wave (stats on)
  // Device time of the last collected wave (stats on) by the reference's split phases
  // (timing.hpp:23-28): 0 sample_projections, 1 apply_projections, 2 build_histograms (boundary
  // sampling + binning), 3 evaluate_splits (histogram scan / exact splitters); partition excluded.
  const float* last_phase_ms() const { return last_phase_ms_; }
  float last_split_ms() const { return last_phase_ms_[2] + last_phase_ms_[3]; }
  void wait_wave();
  bool wave_done() const { return pend_n_ == 0 || cudaEventQuery(done_ev_) == cudaSuccess; }
  // Page-locked staging reused across calls (root segments).
  PinnedBuf<unsigned char> staging;
  // Terms of node `node`'s winning row in the last collected wave, for rows longer than the
  // kWinTermsMax terms NodeRes carries inline (fetched in one batch by collect()).
  // Returns a pointer to the row's n_terms entries (valid until the next collect).
  const uint32_t* fetch_row_terms(const WaveSpec& w, uint32_t node, uint32_t row) const;

  void set_pool(ThreadPool* p) { pool_ = p; }

  WaveStats stats;
  bool collect_stats = false;   // CUDA-event timing per phase + sector accounting
  bool sector_accounting = false;

  // Level state of grow_trees (kept across calls so no allocation synchronizes the device).
  DevBuf<uint32_t> lvl_idx[2];
  DevBuf<uint8_t> lvl_lab[2];
  DevBuf<uint32_t> inv;
  DevBuf<uint64_t> tree_off;
  DevBuf<uint32_t> root_counts;
  DevBuf<uint32_t> root_bits;  // root sets as bitmaps (one bit per dataset row, per tree)

 private:
  int device_;
  ThreadPool* pool_ = nullptr;
  cudaStream_t st_ = nullptr;
  bool own_stream_ = true;
  cudaEvent_t done_ev_ = nullptr;  // end of this runner's last submitted wave
  cudaEvent_t ev_[6]{};
  // fine-grained per-launch timing (stats mode)
  static constexpr int kMaxMarks = 32;
  cudaEvent_t mk_[kMaxMarks + 1]{};
  const char* mk_name_[kMaxMarks]{};
  int n_marks_ = 0;
  void mark(const char* name);
  std::shared_ptr<DeviceData> data_;

  // packed host->device inputs
  PinnedBuf<unsigned char> h_in_;
  DevBuf<unsigned char> d_in_;
  PinnedBuf<NodeRes> h_res_buf_[2];  // alternate per wave: a wave's results stay readable while
  int h_res_cur_ = 0;                 // the next wave's are copied back
  NodeRes* h_res_p_ = nullptr;
  PinnedBuf<uint32_t> h_cl_buf_[2];   // left class counts [N][k], same alternation
  uint32_t* h_cl_p_ = nullptr;
  DevBuf<uint32_t> cl_;
  DevBuf<RowRes> rowres_ex_;          // wide classes: exact results per (node, row)
  // device scratch
  DevBuf<uint32_t> terms_, row_ptr_, pos_proj_, pos_split_, draws_, nb_, flags_, tile_left_,
      gcnt_, done_, sectors_;
  DevBuf<float> bnd_;
  DevBuf<RowRes> rowres_;
  DevBuf<NodeRes> res_;
  DevBuf<float> V_;          // projected rows of the wave (sweep.cu)
  DevBuf<uint32_t> pos_node_;  // level position -> wave node (sweep mode)
  DevBuf<unsigned char> aug_;  // augmented term lists (sweep mode)
  DevBuf<uint16_t> qsplit_;    // per node: the term lists' quarter boundaries (sweep mode)
  DevBuf<uint32_t> pnode_;     // per node: 16-byte pair-record template (pipelined sweep)
  DevBuf<unsigned char> recs_;  // per-sample pair lists (pipelined sweep)
  DevBuf<uint32_t> pcnt_;       // pairs per sample (pipelined sweep)
  Scratch scratch_;                    // launch-sized temporaries (dense projections, exact_big)
  DevBuf<float> rowlb_;                // exact branch-and-bound: per (node, row) lower bounds
  DevBuf<unsigned long long> xstar_;   // and per node the best pivot-candidate impurity
  int n_sm_ = 148;
  const uint32_t* last_terms_ = nullptr;
  const NodeIn* last_nodes_ = nullptr;
  // long winning rows of the last wave (host copies): node -> [long_off_[k], long_off_[k+1])
  std::vector<uint32_t> long_pos_, long_off_, long_terms_;
  PinnedBuf<uint32_t> h_long_;
  DevBuf<uint32_t> d_long_;
  const uint32_t* last_rp_ = nullptr;
  // submit -> collect state
  NodeRes* pend_dres_ = nullptr;
  int pend_n_ = 0, pend_launches_ = 0;
  float last_wave_ms_ = 0.f;
  float last_phase_ms_[4] = {};
  size_t pend_hist_ = 0, pend_exact_ = 0;
  bool pend_sweep_ = false;
  double pend_sweep_bytes_ = 0;
};

}  // namespace sofg
