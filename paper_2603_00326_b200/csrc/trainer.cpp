#include "trainer.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "host_rng.hpp"
#include "kernels.hpp"

namespace sofg {

// ------------------------------------------------------------------------------ thread pool
ThreadPool::ThreadPool(int n) {
  if (n < 1) n = 1;
  for (int i = 0; i < n - 1; ++i) workers_.emplace_back([this] { worker(); });
}

ThreadPool::~ThreadPool() {
  {
    std::lock_guard<std::mutex> g(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  for (auto& t : workers_) t.join();
}

void ThreadPool::worker() {
  uint64_t seen = 0;
  for (;;) {
    const std::function<void(size_t)>* job;
    size_t n;
    {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      job = job_;
      n = job_n_;
      ++active_;
    }
    if (job) {
      const size_t g = std::max<size_t>(1, n / (size_t(workers_.size() + 1) * 16));
      for (size_t i0 = next_.fetch_add(g); i0 < n; i0 = next_.fetch_add(g))
        for (size_t i = i0; i < std::min(n, i0 + g); ++i) (*job)(i);
    }
    {
      std::lock_guard<std::mutex> g(mu_);
      if (--active_ == 0) done_cv_.notify_all();
    }
  }
}

void ThreadPool::parallel_for(size_t n, const std::function<void(size_t)>& f) {
  if (n == 0) return;
  if (workers_.empty() || n < 2) {
    for (size_t i = 0; i < n; ++i) f(i);
    return;
  }
  {
    std::lock_guard<std::mutex> g(mu_);
    job_ = &f;
    job_n_ = n;
    next_.store(0);
    ++gen_;
  }
  cv_.notify_all();
  {
    const size_t g = std::max<size_t>(1, n / (size_t(workers_.size() + 1) * 16));
    for (size_t i0 = next_.fetch_add(g); i0 < n; i0 = next_.fetch_add(g))
      for (size_t i = i0; i < std::min(n, i0 + g); ++i) f(i);
  }
  std::unique_lock<std::mutex> lk(mu_);
  done_cv_.wait(lk, [&] { return active_ == 0 && next_.load() >= n; });
  job_ = nullptr;
}

std::vector<size_t> ThreadPool::chunks(size_t n, size_t grain,
                                       const std::function<void(size_t, size_t, size_t)>& f) {
  size_t c = std::max<size_t>(1, std::min<size_t>(size_t(size()) * 4, (n + grain - 1) / std::max<size_t>(grain, 1)));
  std::vector<size_t> b(c + 1);
  for (size_t i = 0; i <= c; ++i) b[i] = n * i / c;
  parallel_for(c, [&](size_t i) { f(i, b[i], b[i + 1]); });
  return b;
}

namespace {
std::mutex g_recycle_mu;
std::vector<FlatForest> g_recycled;
}  // namespace

void recycle_forest(FlatForest&& f) {
  std::lock_guard<std::mutex> g(g_recycle_mu);
  if (g_recycled.size() < 2) g_recycled.push_back(std::move(f));
}

// Swaps recycled storage (capacity, no contents) into an empty forest.
void adopt_recycled(FlatForest& out) {
  if (!out.left.empty()) return;  // appending to a non-empty forest: keep its arrays
  std::lock_guard<std::mutex> g(g_recycle_mu);
  if (g_recycled.empty()) return;
  FlatForest& r = g_recycled.back();
  auto take = [](auto& dst, auto& src) {
    src.clear();
    dst.swap(src);
  };
  take(out.left, r.left);
  take(out.right, r.right);
  take(out.pred, r.pred);
  take(out.thr, r.thr);
  take(out.feat, r.feat);
  take(out.weight, r.weight);
  r.tree_off.resize(out.tree_off.size());
  std::copy(out.tree_off.begin(), out.tree_off.end(), r.tree_off.begin());
  out.tree_off.swap(r.tree_off);
  r.term_off.resize(out.term_off.size());
  std::copy(out.term_off.begin(), out.term_off.end(), r.term_off.begin());
  out.term_off.swap(r.term_off);
  g_recycled.pop_back();
}

// ------------------------------------------------------------------------------ scheduler
namespace {

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t).count();
}

struct BNode {
  int32_t left = -1, right = -1, pred = -1;
  float thr = 0.f;
  uint32_t term_off = 0, term_len = 0;  // into the tree's term pool
};

// Class counts carried inline in Open (more classes: per-tree side arrays, see grow_trees).
constexpr int kOpenClasses = 4;

constexpr uint32_t kNoSpec = 0xffffffffu;  // spec_pos of a child whose binomial was not drawn ahead

struct Open {  // 64 bytes: the per-level frontier is rewritten twice per node (post, prep)
  uint64_t seed;
  uint32_t tree;
  int32_t bnode;
  uint32_t begin, n, depth, attempt;
  uint32_t pos;   // engine outputs consumed before this attempt's binomial draw
  uint32_t z;     // binomial draw for this attempt (valid when has_z)
  uint32_t zpos;  // stream position after it
  uint32_t has_z;
  uint32_t counts[kOpenClasses];
};
static_assert(sizeof(Open) == 64, "Open layout");

// Host structures of grow_trees kept across calls (per calling thread): their capacity is
// reused, so a training step does not fault in hundreds of MB of fresh pages.
struct GrowScratch {
  std::vector<std::vector<BNode>> trees;
  std::vector<std::vector<uint32_t>> pools;
  std::vector<std::vector<Open>> fr, sp, nx, rt, dn;
  std::vector<std::vector<uint32_t>> wide;  // class counts per tree node (k > kMaxClasses)
  std::vector<uint32_t> spec_z, spec_pos;
  std::vector<NodeIn> nodes;
};

int32_t argmax_first(const uint32_t* c, int k) {  // std::max_element: first maximum
  int32_t b = 0;
  for (int i = 1; i < k; ++i)
    if (c[i] > c[b]) b = i;
  return b;
}

}  // namespace

void grow_trees(WaveRunner& eng, const TrainParams& P0, ThreadPool& pool,
                const std::vector<std::vector<uint32_t>>& roots,
                const std::vector<uint64_t>& root_seeds, uint32_t root_depth, FlatForest& out,
                HostTimes& times) {
  const auto t_start = Clock::now();
  TrainParams P = P0;  // local copy: idle_work is dropped once it reports no more work
  cuda_check(cudaSetDevice(eng.device()), "cudaSetDevice");
  DeviceData& D = eng.data();
  const int k = D.k;
  const size_t B = roots.size();
  if (B == 0) return;
  const uint64_t cells = uint64_t(P.R) * D.d;
  if (cells >= (1ull << 32)) throw std::invalid_argument("projection matrix has >= 2^32 cells");
  host::BinomialDraw binom(cells, P.density);

  // ---- root segments: tree b occupies [off[b], off[b+1]) of the level buffers -------------
  auto t0 = Clock::now();
  std::vector<uint64_t> off(B + 1, 0);
  for (size_t b = 0; b < B; ++b) off[b + 1] = off[b] + roots[b].size();
  const uint64_t total = off[B];
  if (total >= (1ull << 32)) throw std::invalid_argument("batch exceeds 2^32 samples");
  DevBuf<uint32_t>* idx = eng.lvl_idx;
  DevBuf<uint8_t>* lab = eng.lvl_lab;
  for (int i = 0; i < 2; ++i) {
    idx[i].ensure(total);
    lab[i].ensure(total);
  }
  // Root segments: sample ids to the device; labels and class counts gathered there. Strictly
  // increasing root lists (bootstrap samples: sorted sets) travel as one bit per dataset row and
  // are expanded on the device (n/8 bytes per tree instead of 4 bytes per sample, ~20x fewer).
  uint64_t maxn = 0;
  for (size_t b = 0; b < B; ++b) maxn = std::max<uint64_t>(maxn, roots[b].size());
  DevBuf<uint64_t>& d_off = eng.tree_off;
  d_off.ensure(B + 1);
  std::vector<uint32_t> root_counts(B * size_t(k));
  std::vector<unsigned char> increasing(B, 1);
  {
    const uint64_t W = (D.n + 31) / 32;  // bitmap words per tree
    const size_t tail = 8 * (B + 1) + 4 * size_t(k) * B;
    // one pass per tree: its bitmap, and whether its list is strictly increasing
    unsigned char* stg = eng.staging.ensure(4 * W * B + tail);
    pool.parallel_for(B, [&](size_t b) {
      uint32_t* bw = reinterpret_cast<uint32_t*>(stg) + b * W;
      std::memset(bw, 0, 4 * W);
      int64_t prev = -1;
      bool inc = true;
      for (const uint32_t s : roots[b]) {
        inc &= int64_t(s) > prev;
        prev = int64_t(s);
        bw[s >> 5] |= 1u << (s & 31);
      }
      increasing[b] = inc ? 1 : 0;
    });
  }
  bool bitmap = true;
  for (unsigned char x : increasing) bitmap = bitmap && x;
  {
    const uint64_t W = (D.n + 31) / 32;  // bitmap words per tree
    const size_t id_bytes = bitmap ? 4 * W * B : 4 * total;
    unsigned char* stg = eng.staging.ensure(id_bytes + 8 * (B + 1) + 4 * size_t(k) * B);
    uint32_t* hi = reinterpret_cast<uint32_t*>(stg);
    uint64_t* ho = reinterpret_cast<uint64_t*>(stg + id_bytes);
    uint32_t* hc = reinterpret_cast<uint32_t*>(stg + id_bytes + 8 * (B + 1));
    if (!bitmap)  // some list is not a sorted set: the ids themselves
      pool.parallel_for(B, [&](size_t b) { std::memcpy(hi + off[b], roots[b].data(), 4 * roots[b].size()); });
    std::memcpy(ho, off.data(), 8 * (B + 1));
    DevBuf<uint32_t>& d_cnt = eng.root_counts;
    d_cnt.ensure(size_t(k) * B);
    cuda_check(cudaMemcpyAsync(d_off.p, ho, 8 * (B + 1), cudaMemcpyHostToDevice, eng.stream()), "H2D off");
    if (bitmap) {
      DevBuf<uint32_t>& d_bits = eng.root_bits;
      d_bits.ensure(W * B);
      cuda_check(cudaMemcpyAsync(d_bits.p, hi, 4 * W * B, cudaMemcpyHostToDevice, eng.stream()), "H2D root bits");
      cuda_check(launch_bits_to_ids(d_bits.p, W, uint32_t(B), d_off.p, idx[0].p, eng.stream()), "bits_to_ids");
    } else {
      cuda_check(cudaMemcpyAsync(idx[0].p, hi, 4 * total, cudaMemcpyHostToDevice, eng.stream()), "H2D idx");
    }
    cuda_check(launch_root_labels(idx[0].p, d_off.p, uint32_t(B), maxn, D.lab.p, lab[0].p, k, d_cnt.p,
                                  eng.stream()),
               "root_labels");
    cuda_check(cudaMemcpyAsync(hc, d_cnt.p, 4 * size_t(k) * B, cudaMemcpyDeviceToHost, eng.stream()),
               "D2H root counts");
    cuda_check(cudaStreamSynchronize(eng.stream()), "root sync");
    std::memcpy(root_counts.data(), hc, 4 * size_t(k) * B);
  }
  // Inverse map for the projection sweep (sweep.cu): needs each tree's samples to be distinct
  // (bootstrap_sample returns a sorted set; explicit active sets are checked).
  DevBuf<uint32_t>& inv = eng.inv;
  bool use_inv = D.XR.p != nullptr;
  if (use_inv) {
    std::vector<unsigned char> distinct(B, 1);
    pool.parallel_for(B, [&](size_t b) {
      const std::vector<uint32_t>& r = roots[b];
      if (!increasing[b]) {
        std::vector<uint32_t> c(r);
        std::sort(c.begin(), c.end());
        distinct[b] = std::adjacent_find(c.begin(), c.end()) == c.end();
      }
    });
    for (unsigned char x : distinct) use_inv = use_inv && x;
  }
  if (use_inv) {
    inv.ensure(D.n * B);
    cuda_check(launch_inv_init(idx[0].p, d_off.p, uint32_t(B), D.n, maxn, inv.p, eng.stream()),
               "inv_init");
  }

  static thread_local GrowScratch S;
  std::vector<std::vector<BNode>>& trees = S.trees;
  std::vector<std::vector<uint32_t>>& pools = S.pools;
  // More than kOpenClasses classes: class counts live in per-tree side arrays (node v of tree b at
  // wc[b][v * k, v * k + k)) instead of Open::counts.
  const bool wide = k > kOpenClasses;
  std::vector<std::vector<uint32_t>>& wc = S.wide;
  if (trees.size() < B) {
    trees.resize(B);
    pools.resize(B);
  }
  if (wide && wc.size() < B) wc.resize(B);
  auto counts_of = [&](const Open& o) -> const uint32_t* {
    return wide ? wc[o.tree].data() + size_t(o.bnode) * size_t(k) : o.counts;
  };
  // The frontier is kept in P parts; part p owns trees [B*p/P, B*(p+1)/P), so parts are processed
  // in parallel without sharing a tree and never need to be concatenated.
  const size_t NP = std::max<size_t>(1, std::min<size_t>(B, size_t(pool.size()) * 4));
  std::vector<std::vector<Open>>&fr = S.fr, &sp = S.sp, &nx = S.nx, &rt = S.rt;
  std::vector<std::vector<Open>>& dn = S.dn;  // the last posted wave's nodes (deferred bookkeeping)
  for (auto* v : {&fr, &sp, &nx, &rt, &dn}) {
    if (v->size() < NP) v->resize(NP);
    for (size_t p = 0; p < NP; ++p) (*v)[p].clear();
  }
  pool.parallel_for(NP, [&](size_t p) {
    for (size_t b = B * p / NP; b < B * (p + 1) / NP; ++b) {
      trees[b].clear();
      pools[b].clear();
      trees[b].reserve(1024);
      trees[b].emplace_back();
      Open o{};
      o.tree = uint32_t(b);
      o.bnode = 0;
      o.begin = uint32_t(off[b]);
      o.n = uint32_t(roots[b].size());
      o.depth = root_depth;
      o.seed = root_seeds[b];
      if (wide)
        wc[b].assign(root_counts.begin() + ptrdiff_t(b * size_t(k)), root_counts.begin() + ptrdiff_t((b + 1) * size_t(k)));
      else
        for (int c = 0; c < k; ++c) o.counts[c] = root_counts[b * size_t(k) + size_t(c)];
      fr[p].push_back(o);
    }
  });
  times.ms_roots += ms_since(t0);
  DepthProfile* prof = P.profile;
  if (prof) prof->add(root_depth, 0.0, B, total);
  std::vector<uint64_t> part_splits(prof ? NP : 0), part_split_n(prof ? NP : 0);

  int cur = 0;
  double prev_wave_ms = 0.0, idle_chunk_ms = 1.0;
  static const bool level_log = std::getenv("SOFG_LEVEL_LOG") != nullptr;
  std::vector<uint32_t>&spec_z = S.spec_z, &spec_pos = S.spec_pos;
  std::vector<size_t> poff(NP + 1);
  WaveSpec w;
  w.nodes.swap(S.nodes);  // returned below: the node array's capacity persists
  w.R = P.R;
  w.d = uint32_t(D.d);
  w.bins = uint32_t(P.bins);
  w.two_level = P.two_level;
  w.k = k;
  w.inv = use_inv ? inv.p : nullptr;
  w.B = uint32_t(B);
  w.total = total;
  if (const char* e = std::getenv("SOFG_PROJECT_MODE")) w.force_mode = std::atoi(e);
  if (const char* e = std::getenv("SOFG_HIST_CHUNK")) w.chunk_cap = std::max(256, std::atoi(e));
  eng.set_pool(&pool);

  auto count_open = [](const std::vector<std::vector<Open>>& v) {
    size_t t = 0;
    for (const auto& x : v) t += x.size();
    return t;
  };

  // forest.hpp:178-179: a node is split iff it is impure, large enough and above max_depth
  auto can_split_c = [&](const uint32_t* counts, uint32_t n, uint32_t depth) {
    uint32_t top = 0;
    for (int cc = 0; cc < k; ++cc) top = std::max(top, counts[cc]);
    return top < n && n >= P.min_samples_split && n >= 2 && (!P.max_depth || depth < *P.max_depth);
  };
  auto can_split = [&](const Open& o) { return can_split_c(counts_of(o), o.n, o.depth); };
  // The roots are filtered here; children are filtered when they are created (post below), so
  // every later level's frontier is already the list of nodes to split.
  pool.parallel_for(NP, [&](size_t p) {
    std::vector<Open> keep;
    for (const Open& o : fr[p]) {
      if (can_split(o))
        keep.push_back(o);
      else
        trees[o.tree][size_t(o.bnode)].pred = argmax_first(counts_of(o), k);  // forest.hpp:233-236
    }
    fr[p].swap(keep);
  });

  // Tree records of the last posted wave (its nodes in dn, results in dres; the engine keeps a
  // wave's results and long-row terms readable until the next collect).
  struct alignas(64) Counter {  // one cache line per tree: parts update their trees concurrently
    uint32_t v;
  };
  std::vector<Counter> tsize(B);
  for (size_t b = 0; b < B; ++b) tsize[b].v = uint32_t(trees[b].size());
  const NodeRes* dres = nullptr;
  const uint32_t* dcl = nullptr;  // its left class counts [node][k]
  std::vector<size_t> dpoff(NP + 1, 0);
  bool pending = false;
  auto bookkeep = [&]() {
    if (!pending) return;
    pool.parallel_for(NP, [&](size_t p) {
      for (size_t j = 0; j < dn[p].size(); ++j) {
        const size_t i = dpoff[p] + j;
        const Open& o = dn[p][j];
        const NodeRes& r = dres[i];
        std::vector<BNode>& tr = trees[o.tree];
        if (r.row >= 0 && r.n_left > 0 && r.n_left < o.n) {
          std::vector<uint32_t>& tp = pools[o.tree];
          const int32_t L = int32_t(tr.size());
          BNode& pn = tr[size_t(o.bnode)];
          pn.thr = r.threshold;
          pn.left = L;
          pn.right = L + 1;
          pn.term_off = uint32_t(tp.size());
          pn.term_len = r.n_terms;
          if (r.n_terms <= uint32_t(kWinTermsMax)) {
            tp.insert(tp.end(), r.terms, r.terms + r.n_terms);
          } else {
            const uint32_t* t = eng.fetch_row_terms(w, uint32_t(i), uint32_t(r.row));
            tp.insert(tp.end(), t, t + r.n_terms);
          }
          tr.emplace_back();
          tr.emplace_back();
          uint32_t lcb[kMaxClasses] = {}, rcb[kMaxClasses] = {};
          const uint32_t* lc = lcb;
          const uint32_t* rc = rcb;
          if (wide) {  // written by the critical pass (post) at the children's node ids
            lc = wc[o.tree].data() + size_t(L) * size_t(k);
            rc = lc + k;
          } else {
            const uint32_t* cl = dcl + i * size_t(k);
            for (int c = 0; c < k; ++c) {
              lcb[c] = cl[c];
              rcb[c] = o.counts[c] - cl[c];
            }
          }
          if (!can_split_c(lc, r.n_left, o.depth + 1)) tr[size_t(L)].pred = argmax_first(lc, k);
          if (!can_split_c(rc, o.n - r.n_left, o.depth + 1)) tr[size_t(L) + 1].pred = argmax_first(rc, k);
        } else if (o.attempt >= P.max_split_retries) {
          tr[size_t(o.bnode)].pred = argmax_first(counts_of(o), k);
        }
      }
    });
    pending = false;
  };

  while (count_open(fr) > 0) {
    times.levels++;
    t0 = Clock::now();
    pool.parallel_for(NP, [&](size_t p) {
      sp[p].swap(fr[p]);
      fr[p].clear();
      nx[p].clear();
    });
    times.ms_prep += ms_since(t0);
    while (count_open(sp) > 0) {
      t0 = Clock::now();
      poff[0] = 0;
      for (size_t p = 0; p < NP; ++p) poff[p + 1] = poff[p] + sp[p].size();
      const size_t N = poff[NP];
      w.nodes.resize(N);
      // binomial draws not done speculatively (roots, retries), parent entropies, node records
      const auto tb = Clock::now();
      pool.parallel_for(NP, [&](size_t p) {
        {  // fresh engines (roots, children not drawn ahead): batched, their seedings primed together
          constexpr size_t kB = 256;
          uint64_t seeds[kB];
          uint32_t zs[kB], us[kB];
          size_t at[kB], c = 0;
          auto flush = [&]() {
            binom.batch(seeds, c, zs, us);
            for (size_t q = 0; q < c; ++q) {
              Open& o = sp[p][at[q]];
              o.z = zs[q];
              o.zpos = us[q];
              o.has_z = 1;
            }
            c = 0;
          };
          for (size_t j = 0; j < sp[p].size(); ++j) {
            const Open& o = sp[p][j];
            if (o.has_z || o.pos != 0) continue;
            seeds[c] = o.seed;
            at[c++] = j;
            if (c == kB) flush();
          }
          if (c) flush();
        }
        for (size_t j = 0; j < sp[p].size(); ++j) {
          Open& o = sp[p][j];
          if (!o.has_z) {  // retries: the stream continues after the previous attempt
            uint64_t used;
            o.z = uint32_t(binom(o.seed, o.pos, &used));
            o.zpos = uint32_t(used);
            o.has_z = 1;
          }
          NodeIn& nd = w.nodes[poff[p] + j];
          nd.parent = host::entropy(counts_of(o), k);
          nd.seed = o.seed;
          nd.begin = o.begin;
          nd.n = o.n;
          nd.z = o.z;
          nd.pos = o.zpos;
          const bool hist = P.mode == 1 || (P.mode == 2 && o.n > P.breakeven);  // split.hpp:46-48
          nd.flags = hist ? kNodeHist : 0u;
          nd.hist_slot = 0;
          nd.tree = o.tree;
        }
      });
      times.ms_binomial += ms_since(tb);
      // term offsets: per-part sums, then a parallel fill
      std::vector<uint64_t> pz(NP + 1, 0);
      pool.parallel_for(NP, [&](size_t p) {
        uint64_t z = 0;
        for (size_t j = 0; j < sp[p].size(); ++j) z += w.nodes[poff[p] + j].z;
        pz[p + 1] = z;
      });
      for (size_t p = 0; p < NP; ++p) pz[p + 1] += pz[p];
      if (pz[NP] >= (1ull << 32)) throw std::runtime_error("wave term count overflow");
      pool.parallel_for(NP, [&](size_t p) {
        uint64_t t = pz[p];
        for (size_t j = 0; j < sp[p].size(); ++j) {
          w.nodes[poff[p] + j].term_off = uint32_t(t);
          t += w.nodes[poff[p] + j].z;
        }
      });
      w.idx_in = idx[cur].p;
      w.lab_in = lab[cur].p;
      w.idx_out = idx[cur ^ 1].p;
      w.lab_out = lab[cur ^ 1].p;
      const double lv_prep = ms_since(t0);
      times.ms_prep += lv_prep;
      t0 = Clock::now();
      const auto t_submit = t0;
      eng.submit(w);
      const double lv_submit = ms_since(t0);
      times.ms_submit += lv_submit;
      t0 = Clock::now();
      bookkeep();  // the previous wave's tree records, while this wave runs
      times.ms_book += ms_since(t0);

      // While the GPU searches this wave: draw the children's attempt-0 binomials. They depend
      // only on the child seeds derive_seed(seed, 1|2) (forest.hpp:226-228), known already. Drawn
      // in chunks until the wave is done: a child whose draw was not reached by then gets it in
      // the next prep, and only if it is split at all (about half of all children are leaves).
      // With few host threads per GPU the draws outlast the waves of the widest levels.
      t0 = Clock::now();
      spec_z.resize(2 * N);
      spec_pos.resize(2 * N);
      {
        std::atomic<bool> stop{false};
        std::atomic<int64_t> next_poll{0};
        auto wave_over = [&]() {  // one thread queries the wave's event at a time, every >= 50 us
          if (stop.load(std::memory_order_relaxed)) return true;
          const int64_t now = std::chrono::duration_cast<std::chrono::microseconds>(
                                  Clock::now().time_since_epoch()).count();
          int64_t due = next_poll.load(std::memory_order_relaxed);
          if (now < due || !next_poll.compare_exchange_strong(due, now + 50)) return false;
          if (eng.wave_done()) stop.store(true, std::memory_order_relaxed);
          return stop.load(std::memory_order_relaxed);
        };
        pool.parallel_for(NP, [&](size_t p) {
          constexpr size_t kChunk = 128;  // parents per chunk
          const size_t m = sp[p].size();
          uint64_t seeds[2 * kChunk];
          for (size_t j0 = 0; j0 < m; j0 += kChunk) {
            if (wave_over()) {
              std::fill(spec_pos.begin() + std::ptrdiff_t(2 * (poff[p] + j0)),
                        spec_pos.begin() + std::ptrdiff_t(2 * (poff[p] + m)), kNoSpec);
              return;
            }
            const size_t c = std::min(kChunk, m - j0);
            for (size_t j = 0; j < c; ++j) {
              const uint64_t seed = sp[p][j0 + j].seed;
              seeds[2 * j] = host::derive_seed(seed, 1);
              seeds[2 * j + 1] = host::derive_seed(seed, 2);
            }
            binom.batch(seeds, 2 * c, spec_z.data() + 2 * (poff[p] + j0), spec_pos.data() + 2 * (poff[p] + j0));
          }
        });
      }
      const double lv_spec = ms_since(t0);
      times.ms_spec += lv_spec;
      t0 = Clock::now();
      double lv_sync = 0.0;
      if (level_log) {
        eng.wait_wave();
        lv_sync = ms_since(t0);
      }
      if (P.idle_work && prev_wave_ms > 0.0) {
        // only chunks expected to end before the wave does (this level's wave is at least as
        // long as the last one while the frontier grows; later levels stop the work)
        bool more = true;
        while (more && !eng.wave_done() && ms_since(t_submit) + idle_chunk_ms < prev_wave_ms) {
          const auto tc = Clock::now();
          more = P.idle_work();
          idle_chunk_ms = std::max(idle_chunk_ms, ms_since(tc));
        }
        if (!more) P.idle_work = nullptr;
      }
      const NodeRes* res = eng.collect_view(w);
      const uint32_t* wcl = eng.class_counts_view();  // the partition's left class counts [node][k]
      prev_wave_ms = ms_since(t_submit);
      const double lv_wait = ms_since(t0);
      if (std::getenv("SOFG_WAVE_HASH")) {  // debugging aid: per-wave result digest
        uint64_t hsh = 1469598103934665603ull;
        for (size_t i = 0; i < N; ++i) {
          const uint64_t v = (uint64_t(uint32_t(res[i].row)) << 32) ^ res[i].n_left ^
                             (uint64_t(__builtin_bit_cast(uint32_t, res[i].threshold)) << 16);
          hsh = (hsh ^ v) * 1099511628211ull;
        }
        std::fprintf(stderr, "[wave] level %llu nodes %zu sweep %d hash %016llx\n",
                     (unsigned long long)times.levels, N, int(eng.last_was_sweep()),
                     (unsigned long long)hsh);
        if (const char* dump = std::getenv("SOFG_WAVE_DUMP")) {  // node records + results
          if (FILE* fh = std::fopen(dump, "ab")) {
            const uint64_t nn = N;
            std::fwrite(&nn, 8, 1, fh);
            std::fwrite(w.nodes.data(), sizeof(NodeIn), N, fh);
            for (size_t i = 0; i < N; ++i) {
              const uint32_t rec[4] = {uint32_t(res[i].row), __builtin_bit_cast(uint32_t, res[i].threshold),
                                       res[i].n_left, res[i].n_left_search};
              std::fwrite(rec, 4, 4, fh);
            }
            std::fclose(fh);
          }
        }
      }
      times.ms_wait += lv_wait;

      if (prof) {
        uint32_t depth = 0;
        for (size_t p = 0; p < NP; ++p)
          if (!sp[p].empty()) {
            depth = sp[p][0].depth;
            break;
          }
        const float* ph = eng.last_phase_ms();
        const int bk = DepthProfile::bucket(depth);
        prof->add(depth, 1e-3 * double(eng.last_wave_ms()), 0, 0);
        for (int i = 0; i < 4; ++i) {
          prof->phases[bk][i] += 1e-3 * double(ph[i]);
          prof->split_seconds += 1e-3 * double(ph[i]);
        }
      }

      t0 = Clock::now();
      // Critical pass: the children (the next wave's input) and retries. The tree records of this
      // wave (thresholds, terms, links, leaf predictions) are filled by bookkeep() after the next
      // wave is submitted, overlapping its kernels.
      pool.parallel_for(NP, [&](size_t p) {
        rt[p].clear();
        uint64_t n_splits = 0, n_split_samples = 0;
        for (size_t j = 0; j < sp[p].size(); ++j) {
          const size_t i = poff[p] + j;
          const Open& o = sp[p][j];
          const NodeRes& r = res[i];
          if (r.row >= 0 && r.n_left > 0 && r.n_left < o.n) {
            const int32_t L = int32_t(tsize[o.tree].v);
            tsize[o.tree].v += 2;
            Open l{}, rr{};
            l.tree = rr.tree = o.tree;
            l.bnode = L;
            rr.bnode = L + 1;
            l.depth = rr.depth = o.depth + 1;
            l.begin = o.begin;
            l.n = r.n_left;
            rr.begin = o.begin + r.n_left;
            rr.n = o.n - r.n_left;
            l.seed = host::derive_seed(o.seed, 1);  // forest.hpp:226-228
            rr.seed = host::derive_seed(o.seed, 2);
            l.z = spec_z[2 * i];
            l.zpos = spec_pos[2 * i];
            rr.z = spec_z[2 * i + 1];
            rr.zpos = spec_pos[2 * i + 1];
            l.has_z = l.zpos != kNoSpec;  // else drawn in the next prep (if the child is split)
            rr.has_z = rr.zpos != kNoSpec;
            if (wide) {  // children's counts at node ids L, L + 1 of the tree's side array
              std::vector<uint32_t>& v = wc[o.tree];
              if (v.size() < size_t(L + 2) * size_t(k)) v.resize(std::max(v.size() * 2, size_t(L + 2) * size_t(k)));
              const uint32_t* pc = v.data() + size_t(o.bnode) * size_t(k);
              const uint32_t* cl = wcl + i * size_t(k);
              uint32_t* lc = v.data() + size_t(L) * size_t(k);
              for (int c = 0; c < k; ++c) {
                lc[c] = cl[c];
                lc[k + c] = pc[c] - cl[c];
              }
            } else {
              const uint32_t* cl = wcl + i * size_t(k);
              for (int c = 0; c < k; ++c) {
                l.counts[c] = cl[c];
                rr.counts[c] = o.counts[c] - cl[c];
              }
            }
            if (can_split(l)) nx[p].push_back(l);
            if (can_split(rr)) nx[p].push_back(rr);
            ++n_splits;
            n_split_samples += o.n;
          } else if (o.attempt < P.max_split_retries) {  // forest.hpp:187,211: next attempt
            Open a = o;
            a.attempt++;
            a.pos = r.pos_after;
            a.has_z = 0;
            rt[p].push_back(a);
          }
        }
        if (prof) {
          part_splits[p] = n_splits;
          part_split_n[p] = n_split_samples;
        }
        dn[p].swap(sp[p]);
        sp[p].swap(rt[p]);
      });
      if (prof) {  // children of this wave's splits: two nodes each at depth + 1
        uint64_t ns = 0, nn = 0;
        for (size_t p = 0; p < NP; ++p) {
          ns += part_splits[p];
          nn += part_split_n[p];
        }
        uint32_t depth = 0;
        for (size_t p = 0; p < NP; ++p)
          if (!dn[p].empty()) {
            depth = dn[p][0].depth;
            break;
          }
        if (ns) prof->add(size_t(depth) + 1, 0.0, 2 * ns, nn);
      }
      dres = res;
      dcl = wcl;
      dpoff = poff;
      pending = true;
      times.ms_post += ms_since(t0);
      if (level_log) {
        std::fprintf(stderr, "[level %llu] nodes %zu gpu %.2f prep %.2f submit %.2f spec %.2f sync %.2f collect %.2f post %.2f ms\n",
                     (unsigned long long)times.levels, N, double(eng.last_wave_ms()), lv_prep, lv_submit, lv_spec,
                     lv_sync, lv_wait - lv_sync, ms_since(t0));
      }
    }
    cur ^= 1;
    fr.swap(nx);
  }

  bookkeep();
  S.nodes.swap(w.nodes);

  // ---- reference node order: ids assigned at split time in depth-first order (H4) ------------
  t0 = Clock::now();
  std::vector<uint64_t> node_base(B + 1, 0), term_base(B + 1, 0);
  for (size_t b = 0; b < B; ++b) {
    node_base[b + 1] = node_base[b] + trees[b].size();
    term_base[b + 1] = term_base[b] + pools[b].size();
  }
  const size_t N0 = out.left.size(), Q0 = out.feat.size(), T0 = out.tree_off.size();
  adopt_recycled(out);
  out.left.resize(N0 + node_base[B]);
  out.right.resize(N0 + node_base[B]);
  out.pred.resize(N0 + node_base[B]);
  out.thr.resize(N0 + node_base[B]);
  out.term_off.resize(N0 + node_base[B] + 1);
  out.feat.resize(Q0 + term_base[B]);
  out.weight.resize(Q0 + term_base[B]);
  out.tree_off.resize(T0 + B);
  out.term_off[N0] = int64_t(Q0);
  // Node ids without a depth-first walk: the reference numbers the two children of a node when it
  // splits, visiting nodes depth-first, left first (forest.hpp:214-229), so the left child of an
  // internal node v gets id 1 + 2 * (internal nodes before v in preorder). Children are created
  // after their parent (level order), so one reverse pass counts each subtree's internal nodes,
  // one forward pass gives every node's id, and the output is written in id order by scattered
  // stores while tr and the term pool are read sequentially.
  pool.parallel_for(B, [&](size_t b) {
    const std::vector<BNode>& tr = trees[b];
    const std::vector<uint32_t>& tp = pools[b];
    const size_t nn = tr.size();
    std::vector<uint32_t> cnt(nn), id(nn);  // internal nodes in the subtree, then preorder rank
    for (size_t v = nn; v-- > 0;) {
      const BNode& nv = tr[v];
      cnt[v] = nv.left >= 0 ? 1u + cnt[size_t(nv.left)] + cnt[size_t(nv.right)] : 0u;
    }
    std::vector<uint32_t> pre(nn);  // internal nodes before v in preorder
    pre[0] = 0;
    id[0] = 0;
    std::vector<uint64_t> toff(nn + 1, 0);  // term_len by id, then exclusive prefix
    for (size_t v = 0; v < nn; ++v) {
      const BNode& nv = tr[v];
      if (nv.left >= 0) {
        const size_t L = size_t(nv.left), Rn = size_t(nv.right);
        pre[L] = pre[v] + 1;
        pre[Rn] = pre[v] + 1 + cnt[L];
        id[L] = 1 + 2 * pre[v];
        id[Rn] = id[L] + 1;
      }
      toff[id[v] + 1] = nv.term_len;
    }
    for (size_t u = 0; u < nn; ++u) toff[u + 1] += toff[u];
    const size_t q0 = N0 + node_base[b];
    const uint64_t tq0 = Q0 + term_base[b];
    for (size_t v = 0; v < nn; ++v) {
      const BNode& nv = tr[v];
      const size_t q = q0 + id[v];
      out.left[q] = nv.left >= 0 ? int32_t(id[size_t(nv.left)]) : -1;
      out.right[q] = nv.right >= 0 ? int32_t(id[size_t(nv.right)]) : -1;
      out.pred[q] = nv.pred;
      out.thr[q] = nv.left >= 0 ? nv.thr : 0.f;
      uint64_t tq = tq0 + toff[id[v]];
      for (uint32_t t = 0; t < nv.term_len; ++t, ++tq) {
        const uint32_t e = tp[nv.term_off + t];
        out.feat[tq] = e >> 1;
        out.weight[tq] = (e & 1u) ? -1.f : 1.f;
      }
      out.term_off[q + 1] = int64_t(tq0 + toff[id[v] + 1]);
    }
    out.tree_off[T0 + b] = int64_t(N0 + node_base[b + 1]);
  });
  times.ms_final += ms_since(t0);
  times.ms_total += ms_since(t_start);
}

}  // namespace sofg
