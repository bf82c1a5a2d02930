#include "engine.hpp"

#ifndef SOFG_PRUNE32_MAXB
#define SOFG_PRUNE32_MAXB 4  // exact buckets pruned with 32 value buckets (4: n <= 128), 64 above
#endif

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>

#include "kernels.hpp"
#include "trainer.hpp"

namespace sofg {

WaveRunner::WaveRunner(int device, std::shared_ptr<DeviceData> data, cudaStream_t stream)
    : device_(device), data_(data ? std::move(data) : std::make_shared<DeviceData>()) {
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  // The split search is a scattered 4-byte gather: ask L2 to fetch single 32-byte sectors from
  // HBM instead of larger granules (override with SOFG_L2_FETCH=0..128 for experiments).
  {
    size_t gran = 32;
    if (const char* e = std::getenv("SOFG_L2_FETCH")) gran = size_t(std::atoi(e));
    cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
    cudaGetLastError();
  }
  if (stream) {
    st_ = stream;
    own_stream_ = false;
  } else {
    cuda_check(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking), "cudaStreamCreate");
  }
  cuda_check(cudaEventCreateWithFlags(&done_ev_, cudaEventDisableTiming), "cudaEventCreate");
  cudaDeviceGetAttribute(&n_sm_, cudaDevAttrMultiProcessorCount, device);
  for (auto& e : ev_) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
  for (auto& e : mk_) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
}

void WaveRunner::mark(const char* name) {
  if (!collect_stats || n_marks_ >= kMaxMarks) return;
  mk_name_[n_marks_] = name;
  cudaEventRecord(mk_[n_marks_ + 1], st_);
  ++n_marks_;
}

WaveRunner::~WaveRunner() {
  cudaSetDevice(device_);
  for (auto& e : ev_)
    if (e) cudaEventDestroy(e);
  for (auto& e : mk_)
    if (e) cudaEventDestroy(e);
  if (done_ev_) cudaEventDestroy(done_ev_);
  if (st_ && own_stream_) cudaStreamDestroy(st_);
}

Scratch::~Scratch() {
  for (void* p : p_)
    if (p) cudaFree(p);
}

void* Scratch::get(int slot, size_t bytes, cudaStream_t st) {
  if (bytes <= cap_[slot] && p_[slot]) return p_[slot];
  if (p_[slot]) {
    cudaStreamSynchronize(st);  // launches already queued may still read the old block
    cudaFree(p_[slot]);
  }
  p_[slot] = nullptr;
  cap_[slot] = 0;
  const size_t want = bytes + bytes / 4 + 256;
  if (cudaMalloc(&p_[slot], want) != cudaSuccess) {
    cudaGetLastError();
    p_[slot] = nullptr;
    return nullptr;
  }
  cap_[slot] = want;
  return p_[slot];
}

namespace {
struct Packer {
  std::vector<size_t> off;
  size_t total = 0;
  size_t add(size_t bytes) {
    total = (total + 255) & ~size_t(255);
    const size_t o = total;
    total += bytes;
    off.push_back(o);
    return o;
  }
};
// Launch site -> reference split phase (timing.hpp:23-28); -1 = outside the split search.
int phase_of(const char* site) {
  const std::string s(site);
  if (s == "sample_projection") return 0;
  if (s == "sweep_prep" || s == "pair_build" || s == "row_sweep" || s == "project_gather") return 1;
  if (s == "hist_draws" || s == "hist_boundaries" || s == "hist_count") return 2;
  if (s == "partition") return -1;
  return 3;  // hist_select, exact_prune, exact buckets, exact_big
}
int pow2_at_least(int x, int lo) {
  int p = lo;
  while (p < x) p <<= 1;
  return p;
}
}  // namespace

void WaveRunner::submit(const WaveSpec& w) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  const DeviceData& D = *data_;
  const int N = int(w.nodes.size());
  pend_n_ = N;
  if (N == 0) return;
  const uint32_t R = w.R;
  const int k = w.k;
  const uint32_t bins = w.bins;
  const int bpad = pow2_at_least(int(bins), 32);

  // ---- derived work lists (built straight into the page-locked staging buffer) ------------
  // Per node: histogram work items (row groups x chunks), partition tiles, exact bucket, G block
  // offset and gather-item count. Two parallel passes over node chunks: counts, then fills.
  // Histogram counting: two classes and <= 256 bins go to the lane = row kernel for every node
  // size (32 rows per CTA, chunks of lr_chunk samples merged in global counters: 241 -> 177 ms per
  // 1M x 4096 step against the lane = sample kernel above 64K samples); other class / bin counts to
  // the lane = sample kernel (8 rows per CTA, chunks of chunk_cap), more than 8 classes to wide.cu.
  static const int lr_env = std::getenv("SOFG_HIST_LR") ? std::atoi(std::getenv("SOFG_HIST_LR")) : -1;
  // Nodes above lr_chunk samples are counted in chunks of lr_chunk (u16 packed counters per CTA),
  // merged in the global counters like the lane = sample kernel's multi-chunk nodes.
  static const uint32_t lr_chunk_env =
      std::getenv("SOFG_HIST_LR_CHUNK") ? uint32_t(std::atoi(std::getenv("SOFG_HIST_LR_CHUNK"))) : 32768u;
  const bool wide = k > kMaxClasses;  // wide.cu kernels, class counts in side arrays
  // histogram counting by wide.cu also above 1024 bins (the register / lane = row kernels' limit)
  const bool wide_hist = wide || bins > 1024;
  constexpr uint32_t kWideChunk = 65535;  // u16 counters per CTA
  const bool lr_ok = !wide_hist && k == 2 && bins <= 256 && (lr_env >= 0 ? lr_env != 0 : hist_count_lane_rows(R, bins, k));
  const uint32_t lr_max = lr_ok ? 0xffffffffu : 0u;
  const uint32_t lr_chunk = std::max(1024u, std::min(lr_chunk_env, 65504u));
  const uint32_t groups = (R + kHistRowsPerCta - 1) / kHistRowsPerCta;
  const uint32_t groups_lr = (R + 31) / 32;
  const uint32_t cap = uint32_t(w.chunk_cap);
  struct Cnt {
    uint64_t hist = 0, multi = 0, work = 0, work_lr = 0, tiles = 0, g = 0, items = 0;
    uint32_t lr_len = 0;  // longest lane = row chunk
    uint32_t exact_nmax = 0;  // largest shared-memory exact node
    uint64_t exact[kExactBuckets] = {};
    uint32_t zmax = 32;
    uint64_t terms_end = 0;
    uint64_t big = 0;
  };
  ThreadPool* pool = pool_;
  std::vector<Cnt> cc;
  std::vector<size_t> cb;
  auto run_chunks = [&](const std::function<void(size_t, size_t, size_t)>& f) {
    if (pool && N >= 4096) {
      cb = pool->chunks(size_t(N), 2048, f);
    } else {
      cb = {0, size_t(N)};
      f(0, 0, size_t(N));
    }
  };
  // pass 1: counts (chunk layout fixed by the first call)
  {
    std::vector<Cnt> tmp(pool ? size_t(pool->size()) * 4 + 1 : 1);
    run_chunks([&](size_t c, size_t b0, size_t b1) {
      Cnt& t = tmp[c];
      for (size_t i = b0; i < b1; ++i) {
        const NodeIn& nd = w.nodes[i];
        t.zmax = std::max(t.zmax, nd.z);
        t.terms_end = std::max<uint64_t>(t.terms_end, uint64_t(nd.term_off) + nd.z);
        if (nd.flags & kNodeHist) {
          t.hist++;
          if (wide_hist) {  // one item per (row, chunk of <= 65535 samples): wide.cu
            const uint32_t chunks = (nd.n + kWideChunk - 1) / kWideChunk;
            if (chunks > 1) t.multi++;
            t.work += uint64_t(R) * chunks;
          } else if (nd.n <= lr_max) {
            const uint32_t chunks = (nd.n + lr_chunk - 1) / lr_chunk;
            if (chunks > 1) t.multi++;
            t.work_lr += uint64_t(groups_lr) * chunks;
            t.lr_len = std::max(t.lr_len, std::min(nd.n, lr_chunk));
          } else {
            const uint32_t chunks = (nd.n + cap - 1) / cap;
            if (chunks > 1) t.multi++;
            t.work += uint64_t(groups) * chunks;
          }
        } else if (nd.n > uint32_t(kExactSmemMax)) {
          t.big++;  // device-wide segmented sort path (exact_big.cu)
        } else {
          t.exact[exact_bucket(nd.n)]++;
          t.exact_nmax = std::max(t.exact_nmax, nd.n);
        }
        t.tiles += (nd.n + kTileElems - 1) / kTileElems;
        t.g += uint64_t(vpitch(R)) * nd.n;
        t.items += uint64_t(nd.z) * nd.n;
      }
    });
    cc.assign(tmp.begin(), tmp.begin() + (cb.size() - 1));
  }
  const size_t C = cc.size();
  Cnt tot;
  std::vector<Cnt> off(C);
  uint64_t exact_total = 0;
  for (size_t c = 0; c < C; ++c) {
    off[c].hist = tot.hist;
    off[c].multi = tot.multi;
    off[c].work = tot.work;
    off[c].work_lr = tot.work_lr;
    off[c].tiles = tot.tiles;
    off[c].g = tot.g;
    tot.hist += cc[c].hist;
    tot.multi += cc[c].multi;
    tot.work += cc[c].work;
    tot.work_lr += cc[c].work_lr;
    tot.tiles += cc[c].tiles;
    tot.g += cc[c].g;
    tot.items += cc[c].items;
    tot.big += cc[c].big;
    tot.zmax = std::max(tot.zmax, cc[c].zmax);
    tot.lr_len = std::max(tot.lr_len, cc[c].lr_len);
    tot.exact_nmax = std::max(tot.exact_nmax, cc[c].exact_nmax);
    tot.terms_end = std::max(tot.terms_end, cc[c].terms_end);
  }
  uint64_t bucket_base[kExactBuckets + 1] = {0};
  for (int bk = 0; bk < kExactBuckets; ++bk) {
    uint64_t acc = 0;
    for (size_t c = 0; c < C; ++c) acc += cc[c].exact[bk];
    bucket_base[bk + 1] = bucket_base[bk] + acc;
  }
  exact_total = bucket_base[kExactBuckets];
  for (int bk = 0; bk < kExactBuckets; ++bk) {
    uint64_t run = bucket_base[bk];
    for (size_t c = 0; c < C; ++c) {
      off[c].exact[bk] = run;
      run += cc[c].exact[bk];
    }
  }
  const uint32_t zmax = tot.zmax, n_multi = uint32_t(tot.multi);
  const uint64_t g_total = tot.g, sum_nz = tot.items;
  uint64_t total_terms = w.given_csr ? w.given_terms.size() : tot.terms_end;
  const size_t nh = size_t(tot.hist);
  const size_t n_tiles = size_t(tot.tiles), n_work_old = size_t(tot.work), n_work = n_work_old + size_t(tot.work_lr);

  // ---- pack inputs -----------------------------------------------------------------------
  Packer pk;
  const size_t o_nodes = pk.add(sizeof(NodeIn) * N);
  const size_t o_hist = pk.add(4 * nh);
  const size_t o_exact = pk.add(4 * exact_total);
  const size_t o_gbase = pk.add(8 * size_t(N));
  const size_t o_hslot = pk.add(4 * size_t(N));
  const size_t o_mslot = pk.add(4 * size_t(N));
  const size_t o_work = pk.add(sizeof(HistWork) * n_work);
  const size_t o_tiles = pk.add(sizeof(Tile) * n_tiles);
  const size_t o_tfirst = pk.add(4 * (size_t(N) + 1));
  size_t o_gterms = 0, o_grp = 0, o_gpos = 0;
  if (w.given_csr) {
    o_gterms = pk.add(4 * w.given_terms.size());
    o_grp = pk.add(4 * w.given_row_ptr.size());
    o_gpos = pk.add(4 * w.given_pos.size());
  }
  unsigned char* hb = h_in_.ensure(pk.total);
  NodeIn* p_nodes = reinterpret_cast<NodeIn*>(hb + o_nodes);
  uint32_t* p_hist = reinterpret_cast<uint32_t*>(hb + o_hist);
  uint32_t* p_exact = reinterpret_cast<uint32_t*>(hb + o_exact);
  uint64_t* p_gbase = reinterpret_cast<uint64_t*>(hb + o_gbase);
  uint32_t* p_hslot = reinterpret_cast<uint32_t*>(hb + o_hslot);
  uint32_t* p_mslot = reinterpret_cast<uint32_t*>(hb + o_mslot);
  HistWork* p_work = reinterpret_cast<HistWork*>(hb + o_work);
  Tile* p_tiles = reinterpret_cast<Tile*>(hb + o_tiles);
  uint32_t* p_tfirst = reinterpret_cast<uint32_t*>(hb + o_tfirst);
  // pass 2: fills, same chunk boundaries
  auto fill = [&](size_t c, size_t b0, size_t b1) {
    Cnt o = off[c];
    for (size_t i = b0; i < b1; ++i) {
      const NodeIn& nd = w.nodes[i];
      p_nodes[i] = nd;
      p_gbase[i] = o.g;
      o.g += uint64_t(vpitch(R)) * nd.n;
      p_tfirst[i] = uint32_t(o.tiles);
      for (uint32_t s0 = 0, t = 0; s0 < nd.n; s0 += kTileElems, ++t)
        p_tiles[o.tiles++] = {uint32_t(i), s0, std::min(nd.n - s0, uint32_t(kTileElems)), t};
      p_mslot[i] = ~0u;
      p_hslot[i] = ~0u;
      if (nd.flags & kNodeHist) {
        p_hslot[i] = uint32_t(o.hist);
        p_hist[o.hist++] = uint32_t(i);
        if (wide_hist) {
          const uint32_t chunks = (nd.n + kWideChunk - 1) / kWideChunk;
          if (chunks > 1) p_mslot[i] = uint32_t(o.multi++);
          for (uint32_t r = 0; r < R; ++r)
            for (uint32_t ch = 0; ch < chunks; ++ch) {
              const uint32_t s0 = ch * kWideChunk;
              p_work[o.work++] = {uint32_t(i), r, s0, std::min(nd.n - s0, kWideChunk), ch, chunks};
            }
        } else if (nd.n <= lr_max) {  // lane = row items after the lane = sample ones
          const uint32_t chunks = (nd.n + lr_chunk - 1) / lr_chunk;
          if (chunks > 1) p_mslot[i] = uint32_t(o.multi++);
          for (uint32_t g = 0; g < groups_lr; ++g)
            for (uint32_t ch = 0; ch < chunks; ++ch) {
              const uint32_t s0 = ch * lr_chunk;
              p_work[n_work_old + o.work_lr++] = {uint32_t(i), g * 32u, s0, std::min(nd.n - s0, lr_chunk), ch,
                                                  chunks};
            }
        } else {
          const uint32_t chunks = (nd.n + cap - 1) / cap;
          if (chunks > 1) p_mslot[i] = uint32_t(o.multi++);
          for (uint32_t g = 0; g < groups; ++g)
            for (uint32_t ch = 0; ch < chunks; ++ch) {
              const uint32_t s0 = ch * cap;
              p_work[o.work++] = {uint32_t(i), g * kHistRowsPerCta, s0, std::min(nd.n - s0, cap), ch,
                                  chunks};
            }
        }
      } else if (nd.n <= uint32_t(kExactSmemMax)) {
        p_exact[o.exact[exact_bucket(nd.n)]++] = uint32_t(i);
      }
    }
  };
  if (cb.size() > 2) {
    pool->parallel_for(cb.size() - 1, [&](size_t c) { fill(c, cb[c], cb[c + 1]); });
  } else {
    fill(0, 0, size_t(N));
  }
  p_tfirst[N] = uint32_t(n_tiles);
  if (w.given_csr) {
    std::memcpy(hb + o_gterms, w.given_terms.data(), 4 * w.given_terms.size());
    std::memcpy(hb + o_grp, w.given_row_ptr.data(), 4 * w.given_row_ptr.size());
    std::memcpy(hb + o_gpos, w.given_pos.data(), 4 * w.given_pos.size());
  }
  unsigned char* db = d_in_.ensure(pk.total);
  cuda_check(cudaMemcpyAsync(db, hb, pk.total, cudaMemcpyHostToDevice, st_), "H2D wave");
  auto dp = [&](size_t off2) { return db + off2; };
  const NodeIn* d_nodes = reinterpret_cast<const NodeIn*>(dp(o_nodes));
  const uint32_t* d_hist = reinterpret_cast<const uint32_t*>(dp(o_hist));
  const uint32_t* d_exact = reinterpret_cast<const uint32_t*>(dp(o_exact));
  const uint64_t* d_gbase = reinterpret_cast<const uint64_t*>(dp(o_gbase));
  const uint32_t* d_hslot = reinterpret_cast<const uint32_t*>(dp(o_hslot));
  const uint32_t* d_mslot = reinterpret_cast<const uint32_t*>(dp(o_mslot));
  const HistWork* d_work = reinterpret_cast<const HistWork*>(dp(o_work));
  const Tile* d_tiles = reinterpret_cast<const Tile*>(dp(o_tiles));
  const uint32_t* d_tfirst = reinterpret_cast<const uint32_t*>(dp(o_tfirst));
  std::vector<size_t> exact_b_count(kExactBuckets);
  for (int bk = 0; bk < kExactBuckets; ++bk) exact_b_count[size_t(bk)] = size_t(bucket_base[bk + 1] - bucket_base[bk]);

  // ---- scratch ---------------------------------------------------------------------------
  uint32_t* d_terms;
  uint32_t* d_rp;
  uint32_t* d_pos_proj;
  if (w.given_csr) {
    d_terms = reinterpret_cast<uint32_t*>(dp(o_gterms));
    d_rp = reinterpret_cast<uint32_t*>(dp(o_grp));
    d_pos_proj = reinterpret_cast<uint32_t*>(dp(o_gpos));
  } else {
    d_terms = terms_.ensure(total_terms + 1);
    d_rp = row_ptr_.ensure(size_t(N) * (R + 1));
    d_pos_proj = pos_proj_.ensure(size_t(N));
  }
  last_terms_ = d_terms;
  last_rp_ = d_rp;
  last_nodes_ = d_nodes;
  uint32_t* d_pos_split = pos_split_.ensure(size_t(N));
  uint32_t* d_draws = draws_.ensure(std::max<size_t>(1, nh * R * bins));
  float* d_bnd = bnd_.ensure(std::max<size_t>(1, nh * R * (bins - 1)));
  uint32_t* d_nb = nb_.ensure(std::max<size_t>(1, nh * R));
  RowRes* d_rowres = rowres_.ensure(std::max<size_t>(1, nh * R));
  // multi-chunk counters: [slot][R][bpad][2] (lane = row), [slot][R][bins][k] (wide), [slot][R][bpad][k]
  const size_t gcnt_n = size_t(n_multi) * R * std::max<size_t>(bpad, bins) * size_t(k);
  const size_t done_n = size_t(n_multi) * std::max<size_t>(groups, R);
  uint32_t* d_gcnt = gcnt_.ensure(std::max<size_t>(1, gcnt_n));
  uint32_t* d_done = done_.ensure(std::max<size_t>(1, done_n));
  // wide: the partition's left class counts [N][k] (NodeRes carries kMaxClasses), exact row results
  uint32_t* d_cl = cl_.ensure(size_t(N) * size_t(k));
  RowRes* d_rowres_ex = wide ? rowres_ex_.ensure(std::max<size_t>(1, size_t(exact_total) * R)) : nullptr;
  NodeRes* d_res = res_.ensure(size_t(N));
  float* d_G = V_.ensure(std::max<uint64_t>(1, g_total));
  // Projection stage: sweep the row-major table when the wave's gathers would touch a sizeable
  // part of it (a full sweep streams n*d*4 bytes; gathers cost one 32 B sector per term value).
  static const double sweep_frac = std::getenv("SOFG_SWEEP_FRAC") ? std::atof(std::getenv("SOFG_SWEEP_FRAC")) : 0.05;  // measured: 0.25 -> 55.9, 0.1 -> 56.8, 0.05 -> 56.9 trees/s
  bool sweep = w.inv && D.XR.p && w.B > 0 &&
               row_sweep_smem(D.ldr, w.B, R) <= size_t(227) * 1024 &&
               double(sum_nz) >= sweep_frac * double(D.n) * double(D.d);
  if (w.force_mode == 0) sweep = false;
  if (w.force_mode == 1 && w.inv && D.XR.p) sweep = true;
  uint32_t* d_pos_node = sweep ? pos_node_.ensure(std::max<uint64_t>(1, w.total)) : nullptr;
  uint32_t* d_flags = flags_.ensure(std::max<size_t>(1, n_tiles * 32));
  uint32_t* d_tleft = tile_left_.ensure(std::max<size_t>(1, n_tiles));

  cuda_check(cudaMemsetAsync(d_res, 0, sizeof(NodeRes) * N, st_), "memset res");
  if (n_multi) {
    cuda_check(cudaMemsetAsync(d_gcnt, 0, 4 * gcnt_n, st_), "memset gcnt");
    cuda_check(cudaMemsetAsync(d_done, 0, 4 * done_n, st_), "memset done");
  }
  cuda_check(cudaMemsetAsync(d_cl, 0, 4 * size_t(N) * size_t(k), st_), "memset class counts");

  const bool timing = collect_stats;
  if (sector_accounting)
    cuda_check(launch_sector_count(d_nodes, d_tiles, int(n_tiles), w.idx_in, d_res, st_),
               "sector_count");
  if (timing) {
    cudaEventRecord(ev_[0], st_);
    cudaEventRecord(mk_[0], st_);
  }
  n_marks_ = 0;
  int launches = 0;
  if (!w.given_csr) {
    cuda_check(launch_sample_projection(d_nodes, N, w.d, R, zmax, d_terms, d_rp, d_pos_proj, scratch_, st_),
               "sample_projection");
    ++launches;
    mark("sample_projection");
  }
  if (sweep) {
    cuda_check(launch_pos_fill(d_nodes, d_tiles, int(n_tiles), w.total, d_pos_node, st_), "pos_fill");
    const size_t abytes = aug_bytes(total_terms, uint32_t(N), R, w.d);
    void* d_aug = aug_.ensure(abytes);
    pend_sweep_bytes_ = double(D.n) * double(D.ldr) * 4.0 + double(g_total) * 4.0 + double(abytes);
    uint16_t* d_qs = qsplit_.ensure(size_t(N) * 4);
    // Pipelined sweep (sweep_pipe.cu) when samples carry enough pairs to fill a ticket stream;
    // the chunked kernel below it for sparse waves.
    static const double pipe_min = std::getenv("SOFG_SWEEP_PIPE_MIN") ? std::atof(std::getenv("SOFG_SWEEP_PIPE_MIN")) : 16.0;
    const double pairs_per_sample = double(g_total / vpitch(R)) / double(D.n);
    // (pair records hold 32-bit V block (/ 8) and term-list offsets)
    const bool pipe = pairs_per_sample >= pipe_min && row_sweep_pipe_fits(D.ldr, w.B, R) &&
                      g_total / 8 < (uint64_t(1) << 32) && abytes / (aug_narrow(w.d) ? 2 : 4) < (uint64_t(1) << 32);
    uint32_t* d_pn = pipe ? pnode_.ensure(size_t(N) * 4) : nullptr;
    cuda_check(launch_aug_build(d_nodes, N, d_terms, d_rp, R, w.d, d_aug, d_qs, d_gbase, d_pn, st_), "aug_build");
    mark("sweep_prep");
    if (uint64_t(N) > stats.sweep_widest_nodes) {
      stats.sweep_widest_nodes = uint64_t(N);
      row_sweep_variant(w.B, w.d, &stats.sweep_cta_threads, &stats.sweep_entry_bytes);
    }
    if (pipe) {
      const uint32_t PB = (w.B + 1u) & ~1u;
      void* d_recs = recs_.ensure(size_t(D.n) * PB * pair_rec_bytes());
      uint32_t* d_pcnt = pcnt_.ensure(size_t(D.n));
      cuda_check(launch_pair_build(w.inv, w.B, uint32_t(D.n), d_pos_node, d_pn, R, w.d, d_recs, d_pcnt, n_sm_, st_),
                 "pair_build");
      mark("pair_build");
      cuda_check(launch_row_sweep_pipe(D.XR.p, D.ldr, uint32_t(D.n), d_recs, d_pcnt, w.B, d_aug, R, w.d, d_G,
                                       n_sm_, st_),
                 "row_sweep_pipe");
      launches += 4;
    } else {
      cuda_check(launch_row_sweep(D.XR.p, D.ldr, uint32_t(D.n), w.inv, w.B, d_pos_node, d_nodes,
                                  d_gbase, d_aug, d_qs, R, w.d, d_G, n_sm_, st_),
                 "row_sweep");
      launches += 3;
    }
    mark("row_sweep");
  } else {
    cuda_check(launch_project_gather(d_nodes, d_tiles, int(n_tiles), d_gbase, d_terms, d_rp, R,
                                     zmax, w.idx_in, D.X.p, D.ld, d_G, st_),
               "project_gather");
    launches += 1;
    mark("project_gather");
  }
  pend_sweep_ = sweep;
  if (timing) cudaEventRecord(ev_[1], st_);
  if (nh) {
    cuda_check(launch_hist_draws(d_nodes, d_hist, int(nh), R, bins, d_pos_proj, d_draws,
                                 d_pos_split, st_),
               "hist_draws");
    mark("hist_draws");
    cuda_check(launch_hist_boundaries(d_nodes, d_hist, int(nh), R, bins, d_draws, d_terms, d_rp,
                                      d_gbase, d_G, d_bnd, d_nb, st_),
               "hist_boundaries");
    launches += 2;
    mark("hist_boundaries");
  }
  if (timing) cudaEventRecord(ev_[2], st_);
  if (nh) {
    if (n_work > n_work_old)
      cuda_check(launch_hist_count_lr(d_nodes, d_hslot, d_work + n_work_old, int(n_work - n_work_old), d_mslot, R,
                                      bins, int(std::max(tot.lr_len, 32u)), w.two_level ? 1 : 0, w.lab_in, d_gbase, d_G, d_bnd, d_nb,
                                      D.xl.p, d_gcnt, d_done, d_rowres, st_),
                 "hist_count_lr");
    if (n_work_old && wide_hist)
      cuda_check(launch_hist_wide(d_nodes, d_hslot, d_work, int(n_work_old), d_mslot, R, bins, k, w.two_level ? 1 : 0,
                                  w.lab_in, d_gbase, d_G, d_bnd, d_nb, D.xl.p, d_gcnt, d_done, d_rowres, st_),
                 "hist_wide");
    else if (n_work_old)
      cuda_check(launch_hist_count(d_nodes, d_hslot, d_work, int(n_work_old), d_mslot, R, bins, k,
                                   w.chunk_cap, w.two_level ? 1 : 0, d_terms, d_rp, w.lab_in, d_gbase, d_G, d_bnd, d_nb,
                                   D.xl.p, d_gcnt, d_done, d_rowres, st_),
                 "hist_count");
    mark("hist_count");
    cuda_check(launch_hist_select(d_hist, int(nh), R, d_rowres, d_res, st_), "hist_select");
    launches += 2;
    mark("hist_select");
  }
  if (timing) cudaEventRecord(ev_[3], st_);
  {
    // Exact nodes above 64 samples (two classes): per-row bounds first, so rows that cannot
    // hold the node's best split are not sorted (k_exact_prune, exact.cu).
    static const int kPruneFrom = std::getenv("SOFG_PRUNE_FROM") ? std::atoi(std::getenv("SOFG_PRUNE_FROM")) : 4;  // bucket of n <= 128
    size_t prune_off = 0, prune_n = 0;
    for (int b = 0; b < kExactBuckets; ++b) {
      if (b < kPruneFrom) prune_off += exact_b_count[size_t(b)];
      else prune_n += exact_b_count[size_t(b)];
    }
    const bool prune = k <= 4 && prune_n > 0 && !(std::getenv("SOFG_PRUNE") && std::atoi(std::getenv("SOFG_PRUNE")) == 0);
    float* d_rowlb = nullptr;
    unsigned long long* d_xstar = nullptr;
    if (prune) {
      d_rowlb = rowlb_.ensure(prune_n * R);
      d_xstar = xstar_.ensure(prune_n);
      // 32 value buckets per row for n <= 128 (bounds tight enough, half the cost), 64 above
      size_t n_small = 0;
      for (int b = kPruneFrom; b <= SOFG_PRUNE32_MAXB; ++b) n_small += exact_b_count[size_t(b)];
      cuda_check(launch_exact_prune(d_nodes, d_exact + prune_off, int(n_small), R, d_rp, w.lab_in,
                                    d_gbase, d_G, D.xl.p, d_rowlb, d_xstar, 32, k, st_),
                 "exact_prune");
      cuda_check(launch_exact_prune(d_nodes, d_exact + prune_off + n_small, int(prune_n - n_small), R,
                                    d_rp, w.lab_in, d_gbase, d_G, D.xl.p, d_rowlb + n_small * R,
                                    d_xstar + n_small, 64, k, st_),
                 "exact_prune");
      ++launches;
      mark("exact_prune");
    }
    if (wide && exact_total) {  // every shared-memory exact node at once, then its best row
      cuda_check(launch_exact_wide(d_nodes, d_exact, int(exact_total), tot.exact_nmax, R, k, d_rp, w.lab_in, d_gbase,
                                   d_G, D.xl.p, d_rowres_ex, st_),
                 "exact_wide");
      cuda_check(launch_hist_select(d_exact, int(exact_total), R, d_rowres_ex, d_res, st_), "exact_wide_select");
      launches += 2;
      mark("exact_wide");
    }
    size_t off = 0;
    for (int b = 0; b < kExactBuckets && !wide; ++b) {
      const size_t m = exact_b_count[size_t(b)];
      if (!m) continue;
      const bool pb = prune && b >= kPruneFrom;
      cuda_check(launch_exact_bucket(b, d_nodes, d_exact + off, int(m), R, k, d_terms, d_rp,
                                     w.lab_in, d_gbase, d_G, D.xl.p, D.xlf.p, d_res,
                                     pb ? d_rowlb + (off - prune_off) * R : nullptr,
                                     pb ? d_xstar + (off - prune_off) : nullptr, st_),
                 "exact_bucket");
      off += m;
      ++launches;
      static const char* kBucketName[kExactBuckets] = {"exact_n<=8", "exact_n<=16", "exact_n<=32", "exact_n<=64", "exact_n<=128",
                                           "exact_n<=256", "exact_n<=512", "exact_n<=1024",
                                           "exact_n<=2048"};
      mark(kBucketName[b]);
    }
  }
  if (tot.big) {
    std::vector<uint32_t> big;
    big.reserve(size_t(tot.big));
    for (int i = 0; i < N; ++i)
      if (!(w.nodes[size_t(i)].flags & kNodeHist) && w.nodes[size_t(i)].n > uint32_t(kExactSmemMax))
        big.push_back(uint32_t(i));
    cuda_check(launch_exact_big(d_nodes, w.nodes.data(), big.data(), int(big.size()), R, k, d_rp,
                                w.lab_in, d_gbase, d_G, D.xl.p, d_res, scratch_, st_),
               "exact_big");
    launches += 4;
    mark("exact_big");
  }
  if (timing) cudaEventRecord(ev_[4], st_);
  cuda_check(launch_partition(d_nodes, N, d_tiles, int(n_tiles), d_tfirst, R, k, d_terms,
                              d_rp, d_pos_proj, d_pos_split, w.idx_in, w.lab_in, w.idx_out,
                              w.lab_out, d_gbase, d_G, d_res, d_flags, d_tleft, w.inv, w.B, d_cl, st_),
             "partition");
  launches += 3;
  mark("partition");
  if (timing) cudaEventRecord(ev_[5], st_);

  h_res_cur_ ^= 1;
  NodeRes* hr = h_res_buf_[h_res_cur_].ensure(size_t(N));
  h_res_p_ = hr;
  cuda_check(cudaMemcpyAsync(hr, d_res, sizeof(NodeRes) * N, cudaMemcpyDeviceToHost, st_),
             "D2H res");
  {
    uint32_t* hc = h_cl_buf_[h_res_cur_].ensure(size_t(N) * size_t(k));
    h_cl_p_ = hc;
    cuda_check(cudaMemcpyAsync(hc, d_cl, 4 * size_t(N) * size_t(k), cudaMemcpyDeviceToHost, st_), "D2H class counts");
  }
  cuda_check(cudaEventRecord(done_ev_, st_), "record wave end");
  pend_dres_ = d_res;
  pend_launches_ = launches;
  pend_hist_ = nh;
  pend_exact_ = size_t(exact_total);
}

void WaveRunner::collect(const WaveSpec& w, std::vector<NodeRes>& res) {
  const NodeRes* r = collect_view(w);
  res.assign(r, r + pend_n_);
}

void WaveRunner::wait_wave() {
  if (pend_n_ > 0) cuda_check(cudaEventSynchronize(done_ev_), "wave sync");
}

const NodeRes* WaveRunner::collect_view(const WaveSpec& w) {
  const int N = pend_n_;
  if (N == 0) return h_res_p_;
  cuda_check(cudaEventSynchronize(done_ev_), "wave sync");
  const NodeRes* res = h_res_p_;
  // winning rows longer than NodeRes carries inline: one gather + one D2H for the whole wave
  long_off_.assign(1, 0u);
  std::vector<uint32_t> list;
  {
    auto is_long = [&](size_t i) { return res[i].row >= 0 && res[i].n_terms > uint32_t(kWinTermsMax); };
    if (pool_ && N >= 65536) {  // the scan reads one line per result: split it over the host pool
      std::vector<std::vector<uint32_t>> part(size_t(pool_->size()) * 4 + 1);
      const std::vector<size_t> cb = pool_->chunks(size_t(N), 16384, [&](size_t c, size_t b0, size_t b1) {
        for (size_t i = b0; i < b1; ++i)
          if (is_long(i)) part[c].push_back(uint32_t(i));
      });
      for (size_t c = 0; c + 1 < cb.size(); ++c) list.insert(list.end(), part[c].begin(), part[c].end());
    } else {
      for (int i = 0; i < N; ++i)
        if (is_long(size_t(i))) list.push_back(uint32_t(i));
    }
    for (const uint32_t i : list) long_off_.push_back(long_off_.back() + res[i].n_terms);
  }
  if (!list.empty()) {
    long_pos_.assign(size_t(N), ~0u);
    for (size_t k = 0; k < list.size(); ++k) long_pos_[list[k]] = uint32_t(k);
    const size_t L = list.size(), T = long_off_.back();
    uint32_t* hb = h_long_.ensure(2 * L + 1 + T);
    std::memcpy(hb, list.data(), 4 * L);
    std::memcpy(hb + L, long_off_.data(), 4 * (L + 1));
    uint32_t* db = d_long_.ensure(2 * L + 1 + T);
    cuda_check(cudaMemcpyAsync(db, hb, 4 * (2 * L + 1), cudaMemcpyHostToDevice, st_), "H2D long rows");
    cuda_check(launch_win_terms(last_nodes_, pend_dres_, last_rp_, last_terms_, w.R, db, int(L),
                                db + L, db + 2 * L + 1, st_),
               "win_terms");
    cuda_check(cudaMemcpyAsync(hb + 2 * L + 1, db + 2 * L + 1, 4 * T, cudaMemcpyDeviceToHost, st_),
               "D2H long rows");
    cuda_check(cudaEventRecord(done_ev_, st_), "record long rows");
    cuda_check(cudaEventSynchronize(done_ev_), "long rows sync");
    long_terms_.assign(hb + 2 * L + 1, hb + 2 * L + 1 + T);
  } else {
    long_pos_.clear();
  }
  const size_t nh = pend_hist_;
  const int launches = pend_launches_;
  const bool timing = collect_stats;
  stats.waves++;
  stats.nodes += uint64_t(N);
  stats.hist_nodes += nh;
  stats.exact_nodes += pend_exact_;
  stats.launches += uint64_t(launches);
  if (nh) stats.hist_count_launches++;
  (pend_sweep_ ? stats.sweep_waves : stats.gather_waves)++;
  if (pend_sweep_) stats.sweep_alg_bytes += pend_sweep_bytes_;
  if (pend_exact_) stats.exact_launches++;
  if (timing) {
    float t[5];
    for (int i = 0; i < 5; ++i) cudaEventElapsedTime(&t[i], ev_[i], ev_[i + 1]);
    stats.ms_sample += t[0];
    stats.ms_hist_rng += t[1];
    stats.ms_hist_count += t[2];
    stats.ms_exact += t[3];
    stats.ms_partition += t[4];
    float tt;
    cudaEventElapsedTime(&tt, ev_[0], ev_[5]);
    stats.ms_total += tt;
    last_wave_ms_ = tt;
    static const bool wave_log = std::getenv("SOFG_LEVEL_LOG") != nullptr;
    for (float& p : last_phase_ms_) p = 0.f;
    for (int i = 0; i < n_marks_; ++i) {
      float dt;
      cudaEventElapsedTime(&dt, mk_[i], mk_[i + 1]);
      stats.add_kernel(mk_name_[i], dt);
      const int ph = phase_of(mk_name_[i]);
      if (ph >= 0) last_phase_ms_[ph] += dt;
      if (wave_log) std::fprintf(stderr, "%s%s %.2f", i ? ", " : "  [wave] ", mk_name_[i], double(dt));
    }
    if (wave_log && n_marks_) std::fprintf(stderr, "\n");
    for (int i = 0; i < N; ++i) {
      const NodeIn& nd = w.nodes[size_t(i)];
      const double strict = 4.0 * double(nd.n) * double(nd.z);
      const double sector = 32.0 * double(res[size_t(i)].sectors) * double(nd.z);
      if (nd.flags & kNodeHist) {
        stats.hist_strict_bytes += strict;
        stats.hist_sector_bytes += sector;
      } else {
        stats.exact_strict_bytes += strict;
        stats.exact_sector_bytes += sector;
      }
    }
  }
  return res;
}

const uint32_t* WaveRunner::fetch_row_terms(const WaveSpec& w, uint32_t node, uint32_t row) const {
  (void)w;
  (void)row;
  if (node >= long_pos_.size() || long_pos_[node] == ~0u)
    throw std::logic_error("winning row terms were not fetched");
  return long_terms_.data() + long_off_[long_pos_[node]];
}

}  // namespace sofg
