#include "engine.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "kernels.hpp"

namespace sofg {

WaveRunner::WaveRunner(int device) : device_(device) {
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  // The split search is a scattered 4-byte gather: ask L2 to fetch single 32-byte sectors from
  // HBM instead of larger granules (override with SOFG_L2_FETCH=0..128 for experiments).
  {
    size_t gran = 32;
    if (const char* e = std::getenv("SOFG_L2_FETCH")) gran = size_t(std::atoi(e));
    cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
    cudaGetLastError();
  }
  cuda_check(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking), "cudaStreamCreate");
  for (auto& e : ev_) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
}

WaveRunner::~WaveRunner() {
  cudaSetDevice(device_);
  for (auto& e : ev_)
    if (e) cudaEventDestroy(e);
  if (st_) cudaStreamDestroy(st_);
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
int pow2_at_least(int x, int lo) {
  int p = lo;
  while (p < x) p <<= 1;
  return p;
}
}  // namespace

void WaveRunner::submit(const WaveSpec& w) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  const DeviceData& D = data_;
  const int N = int(w.nodes.size());
  pend_n_ = N;
  if (N == 0) return;
  const uint32_t R = w.R;
  const int k = w.k;
  const uint32_t bins = w.bins;
  const int bpad = pow2_at_least(int(bins), 32);

  // ---- derived work lists --------------------------------------------------------------
  std::vector<uint32_t> hist, exact, hist_slot(size_t(N), ~0u), multi_slot(size_t(N), ~0u);
  std::vector<uint32_t> exact_b[7];
  std::vector<HistWork> work;
  std::vector<Tile> tiles;
  std::vector<uint32_t> tile_first(size_t(N) + 1, 0);
  uint32_t zmax = 32, n_multi = 0;
  std::vector<uint64_t> gbase(static_cast<size_t>(N));
  uint64_t g_total = 0, n_items = 0;
  uint64_t total_terms = 0;
  const uint32_t groups = (R + kHistRowsPerCta - 1) / kHistRowsPerCta;
  for (int i = 0; i < N; ++i) {
    const NodeIn& nd = w.nodes[size_t(i)];
    zmax = std::max(zmax, nd.z);
    total_terms = std::max<uint64_t>(total_terms, uint64_t(nd.term_off) + nd.z);
    if (nd.flags & kNodeHist) {
      hist_slot[size_t(i)] = uint32_t(hist.size());
      hist.push_back(uint32_t(i));
      const uint32_t chunks = (nd.n + uint32_t(w.chunk_cap) - 1) / uint32_t(w.chunk_cap);
      if (chunks > 1) multi_slot[size_t(i)] = n_multi++;
      for (uint32_t g = 0; g < groups; ++g)
        for (uint32_t c = 0; c < chunks; ++c) {
          const uint32_t s = c * uint32_t(w.chunk_cap);
          work.push_back({uint32_t(i), g * kHistRowsPerCta, s, std::min(nd.n - s, uint32_t(w.chunk_cap)),
                          c, chunks});
        }
    } else {
      if (nd.n > uint32_t(kExactSmemMax))
        throw std::invalid_argument("exact split of a node with " + std::to_string(nd.n) +
                                    " samples exceeds the GPU exact splitter (" +
                                    std::to_string(kExactSmemMax) + "); use a breakeven <= " +
                                    std::to_string(kExactSmemMax));
      exact_b[size_t(exact_bucket(nd.n))].push_back(uint32_t(i));
    }
    gbase[size_t(i)] = g_total;
    g_total += uint64_t(nd.z) * nd.n;
    n_items += csp_items(nd.n, nd.z);
    tile_first[size_t(i)] = uint32_t(tiles.size());
    for (uint32_t s = 0, t = 0; s < nd.n; s += kTileElems, ++t)
      tiles.push_back({uint32_t(i), s, std::min(nd.n - s, uint32_t(kTileElems)), t});
  }
  tile_first[size_t(N)] = uint32_t(tiles.size());
  if (w.given_csr) total_terms = w.given_terms.size();

  // ---- pack inputs -----------------------------------------------------------------------
  Packer pk;
  const size_t o_nodes = pk.add(sizeof(NodeIn) * N);
  const size_t o_hist = pk.add(4 * hist.size());
  for (auto& v : exact_b) exact.insert(exact.end(), v.begin(), v.end());
  const size_t o_exact = pk.add(4 * exact.size());
  const size_t o_gbase = pk.add(8 * size_t(N));
  const size_t o_hslot = pk.add(4 * size_t(N));
  const size_t o_mslot = pk.add(4 * size_t(N));
  const size_t o_work = pk.add(sizeof(HistWork) * work.size());
  const size_t o_tiles = pk.add(sizeof(Tile) * tiles.size());
  const size_t o_tfirst = pk.add(4 * tile_first.size());
  size_t o_gterms = 0, o_grp = 0, o_gpos = 0;
  if (w.given_csr) {
    o_gterms = pk.add(4 * w.given_terms.size());
    o_grp = pk.add(4 * w.given_row_ptr.size());
    o_gpos = pk.add(4 * w.given_pos.size());
  }
  unsigned char* hb = h_in_.ensure(pk.total);
  auto put = [&](size_t off, const void* src, size_t bytes) {
    if (bytes) std::memcpy(hb + off, src, bytes);
  };
  put(o_nodes, w.nodes.data(), sizeof(NodeIn) * N);
  put(o_hist, hist.data(), 4 * hist.size());
  put(o_exact, exact.data(), 4 * exact.size());
  put(o_gbase, gbase.data(), 8 * size_t(N));
  put(o_hslot, hist_slot.data(), 4 * size_t(N));
  put(o_mslot, multi_slot.data(), 4 * size_t(N));
  put(o_work, work.data(), sizeof(HistWork) * work.size());
  put(o_tiles, tiles.data(), sizeof(Tile) * tiles.size());
  put(o_tfirst, tile_first.data(), 4 * tile_first.size());
  if (w.given_csr) {
    put(o_gterms, w.given_terms.data(), 4 * w.given_terms.size());
    put(o_grp, w.given_row_ptr.data(), 4 * w.given_row_ptr.size());
    put(o_gpos, w.given_pos.data(), 4 * w.given_pos.size());
  }
  unsigned char* db = d_in_.ensure(pk.total);
  cuda_check(cudaMemcpyAsync(db, hb, pk.total, cudaMemcpyHostToDevice, st_), "H2D wave");
  auto dp = [&](size_t off) { return db + off; };
  const NodeIn* d_nodes = reinterpret_cast<const NodeIn*>(dp(o_nodes));
  const uint32_t* d_hist = reinterpret_cast<const uint32_t*>(dp(o_hist));
  const uint32_t* d_exact = reinterpret_cast<const uint32_t*>(dp(o_exact));
  const uint64_t* d_gbase = reinterpret_cast<const uint64_t*>(dp(o_gbase));
  const uint32_t* d_hslot = reinterpret_cast<const uint32_t*>(dp(o_hslot));
  const uint32_t* d_mslot = reinterpret_cast<const uint32_t*>(dp(o_mslot));
  const HistWork* d_work = reinterpret_cast<const HistWork*>(dp(o_work));
  const Tile* d_tiles = reinterpret_cast<const Tile*>(dp(o_tiles));
  const uint32_t* d_tfirst = reinterpret_cast<const uint32_t*>(dp(o_tfirst));

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
  uint32_t* d_pos_split = pos_split_.ensure(size_t(N));
  const size_t nh = hist.size();
  uint32_t* d_draws = draws_.ensure(std::max<size_t>(1, nh * R * bins));
  float* d_bnd = bnd_.ensure(std::max<size_t>(1, nh * R * (bins - 1)));
  uint32_t* d_nb = nb_.ensure(std::max<size_t>(1, nh * R));
  RowRes* d_rowres = rowres_.ensure(std::max<size_t>(1, nh * R));
  uint32_t* d_gcnt = gcnt_.ensure(std::max<size_t>(1, size_t(n_multi) * R * bpad * k));
  uint32_t* d_done = done_.ensure(std::max<size_t>(1, size_t(n_multi) * groups));
  NodeRes* d_res = res_.ensure(size_t(N));
  float* d_G = G_.ensure(std::max<uint64_t>(1, g_total));
  uint64_t* d_items = items_.ensure(std::max<uint64_t>(1, n_items));
  uint32_t* d_fcnt = fcnt_.ensure(w.d);
  uint32_t* d_flags = flags_.ensure(std::max<size_t>(1, tiles.size() * 32));
  uint32_t* d_tleft = tile_left_.ensure(std::max<size_t>(1, tiles.size()));

  cuda_check(cudaMemsetAsync(d_res, 0, sizeof(NodeRes) * N, st_), "memset res");
  if (n_multi) {
    cuda_check(cudaMemsetAsync(d_gcnt, 0, 4 * size_t(n_multi) * R * bpad * k, st_), "memset gcnt");
    cuda_check(cudaMemsetAsync(d_done, 0, 4 * size_t(n_multi) * groups, st_), "memset done");
  }

  const bool timing = collect_stats;
  if (sector_accounting)
    cuda_check(launch_sector_count(d_nodes, d_tiles, int(tiles.size()), w.idx_in, d_res, st_),
               "sector_count");
  if (timing) cudaEventRecord(ev_[0], st_);
  int launches = 0;
  if (!w.given_csr) {
    cuda_check(launch_sample_projection(d_nodes, N, w.d, R, zmax, d_terms, d_rp, d_pos_proj, st_),
               "sample_projection");
    ++launches;
  }
  cuda_check(launch_csp(d_nodes, N, d_gbase, d_terms, w.d, n_items, d_fcnt, d_items, w.idx_in,
                        D.X.p, D.ld, d_G, st_),
             "column_sweep_gather");
  launches += 4;
  if (timing) cudaEventRecord(ev_[1], st_);
  if (nh) {
    cuda_check(launch_hist_draws(d_nodes, d_hist, int(nh), R, bins, d_pos_proj, d_draws,
                                 d_pos_split, st_),
               "hist_draws");
    cuda_check(launch_hist_boundaries(d_nodes, d_hist, int(nh), R, bins, d_draws, d_terms, d_rp,
                                      d_gbase, d_G, d_bnd, d_nb, st_),
               "hist_boundaries");
    launches += 2;
  }
  if (timing) cudaEventRecord(ev_[2], st_);
  if (nh) {
    cuda_check(launch_hist_count(d_nodes, d_hslot, d_work, int(work.size()), d_mslot, R, bins, k,
                                 w.chunk_cap, d_terms, d_rp, w.lab_in, d_gbase, d_G, d_bnd, d_nb,
                                 D.xl.p, d_gcnt, d_done, d_rowres, st_),
               "hist_count");
    cuda_check(launch_hist_select(d_hist, int(nh), R, d_rowres, d_res, st_), "hist_select");
    launches += 2;
  }
  if (timing) cudaEventRecord(ev_[3], st_);
  {
    size_t off = 0;
    for (int b = 0; b < 7; ++b) {
      const size_t m = exact_b[b].size();
      if (!m) continue;
      cuda_check(launch_exact_bucket(b, d_nodes, d_exact + off, int(m), R, k, d_terms, d_rp,
                                     w.lab_in, d_gbase, d_G, D.xl.p, d_res, st_),
                 "exact_bucket");
      off += m;
      ++launches;
    }
  }
  if (timing) cudaEventRecord(ev_[4], st_);
  cuda_check(launch_partition(d_nodes, N, d_tiles, int(tiles.size()), d_tfirst, R, k, d_terms,
                              d_rp, d_pos_proj, d_pos_split, w.idx_in, w.lab_in, w.idx_out,
                              w.lab_out, d_gbase, d_G, d_res, d_flags, d_tleft, st_),
             "partition");
  launches += 3;
  if (timing) cudaEventRecord(ev_[5], st_);

  NodeRes* hr = h_res_.ensure(size_t(N));
  cuda_check(cudaMemcpyAsync(hr, d_res, sizeof(NodeRes) * N, cudaMemcpyDeviceToHost, st_),
             "D2H res");
  pend_dres_ = d_res;
  pend_launches_ = launches;
  pend_hist_ = nh;
  pend_exact_ = exact.size();
}

void WaveRunner::collect(const WaveSpec& w, std::vector<NodeRes>& res) {
  const int N = pend_n_;
  res.assign(size_t(N), NodeRes{});
  if (N == 0) return;
  cuda_check(cudaStreamSynchronize(st_), "wave sync");
  std::memcpy(res.data(), h_res_.p, sizeof(NodeRes) * N);
  const size_t nh = pend_hist_;
  const int launches = pend_launches_;
  const bool timing = collect_stats;
  stats.waves++;
  stats.nodes += uint64_t(N);
  stats.hist_nodes += nh;
  stats.exact_nodes += pend_exact_;
  stats.launches += uint64_t(launches);
  if (nh) stats.hist_count_launches++;
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
}

std::vector<uint32_t> WaveRunner::fetch_row_terms(const WaveSpec& w, uint32_t node, uint32_t row) {
  const uint32_t R = w.R;
  uint32_t rp[2];
  cuda_check(cudaMemcpy(rp, last_rp_ + size_t(node) * (R + 1) + row, 8, cudaMemcpyDeviceToHost),
             "fetch row_ptr");
  std::vector<uint32_t> out(rp[1] - rp[0]);
  if (!out.empty())
    cuda_check(cudaMemcpy(out.data(), last_terms_ + w.nodes[node].term_off + rp[0], 4 * out.size(),
                          cudaMemcpyDeviceToHost),
               "fetch terms");
  return out;
}

}  // namespace sofg
