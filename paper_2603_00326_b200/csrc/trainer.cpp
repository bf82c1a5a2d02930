#include "trainer.hpp"

#include <algorithm>
#include <chrono>
#include <cstring>

#include "host_rng.hpp"

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
    if (job)
      for (size_t i = next_.fetch_add(1); i < n; i = next_.fetch_add(1)) (*job)(i);
    {
      std::lock_guard<std::mutex> g(mu_);
      if (--active_ == 0) done_cv_.notify_all();
    }
  }
}

void ThreadPool::parallel_for(size_t n, const std::function<void(size_t)>& f) {
  if (n == 0) return;
  if (workers_.empty() || n < 64) {
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
  for (size_t i = next_.fetch_add(1); i < n; i = next_.fetch_add(1)) f(i);
  std::unique_lock<std::mutex> lk(mu_);
  done_cv_.wait(lk, [&] { return active_ == 0 && next_.load() >= n; });
  job_ = nullptr;
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
  std::vector<uint32_t> terms;  // feature << 1 | negative
};

struct Open {
  uint32_t tree;
  int32_t bnode;
  uint32_t begin, n, depth, attempt;
  uint64_t seed;
  uint64_t pos;  // engine outputs consumed before this attempt's binomial draw
  uint32_t counts[kMaxClasses];
};

int32_t argmax_first(const uint32_t* c, int k) {  // std::max_element: first maximum
  int32_t b = 0;
  for (int i = 1; i < k; ++i)
    if (c[i] > c[b]) b = i;
  return b;
}

}  // namespace

void grow_trees(WaveRunner& eng, const TrainParams& P, ThreadPool& pool,
                const std::vector<std::vector<uint32_t>>& roots,
                const std::vector<uint64_t>& root_seeds, uint32_t root_depth, FlatForest& out,
                HostTimes& times) {
  const auto t_start = Clock::now();
  DeviceData& D = eng.data();
  const int k = D.k;
  const size_t B = roots.size();
  if (B == 0) return;
  const uint64_t cells = uint64_t(P.R) * D.d;
  if (cells >= (1ull << 32)) throw std::invalid_argument("projection matrix has >= 2^32 cells");
  host::BinomialDraw binom(cells, P.density);

  // ---- root segments: tree b occupies [off[b], off[b+1]) of the level buffers -------------
  std::vector<uint64_t> off(B + 1, 0);
  for (size_t b = 0; b < B; ++b) off[b + 1] = off[b] + roots[b].size();
  const uint64_t total = off[B];
  if (total >= (1ull << 32)) throw std::invalid_argument("batch exceeds 2^32 samples");
  DevBuf<uint32_t> idx[2];
  DevBuf<uint8_t> lab[2];
  for (int i = 0; i < 2; ++i) {
    idx[i].exact(total);
    lab[i].exact(total);
  }
  {
    PinnedBuf<uint32_t> hidx;
    PinnedBuf<uint8_t> hlab;
    uint32_t* hi = hidx.ensure(total);
    uint8_t* hl = hlab.ensure(total);
    for (size_t b = 0; b < B; ++b) {
      std::memcpy(hi + off[b], roots[b].data(), 4 * roots[b].size());
      for (size_t j = 0; j < roots[b].size(); ++j) hl[off[b] + j] = uint8_t(D.labels_host[roots[b][j]]);
    }
    cuda_check(cudaMemcpyAsync(idx[0].p, hi, 4 * total, cudaMemcpyHostToDevice, eng.stream()), "H2D idx");
    cuda_check(cudaMemcpyAsync(lab[0].p, hl, total, cudaMemcpyHostToDevice, eng.stream()), "H2D lab");
    cuda_check(cudaStreamSynchronize(eng.stream()), "sync roots");
  }

  std::vector<std::vector<BNode>> trees(B);
  std::vector<Open> frontier;
  frontier.reserve(B);
  for (size_t b = 0; b < B; ++b) {
    trees[b].emplace_back();
    Open o{};
    o.tree = uint32_t(b);
    o.bnode = 0;
    o.begin = uint32_t(off[b]);
    o.n = uint32_t(roots[b].size());
    o.depth = root_depth;
    o.seed = root_seeds[b];
    for (uint32_t s : roots[b]) o.counts[D.labels_host[s]]++;
    frontier.push_back(o);
  }

  int cur = 0;
  std::vector<Open> split_list, retry, next;
  std::vector<uint64_t> zs, poss;
  std::vector<double> parents;
  std::vector<NodeRes> res;
  WaveSpec w;
  w.R = P.R;
  w.d = uint32_t(D.d);
  w.bins = uint32_t(P.bins);
  w.k = k;

  while (!frontier.empty()) {
    times.levels++;
    split_list.clear();
    next.clear();
    for (const Open& o : frontier) {
      uint32_t top = 0;
      for (int c = 0; c < k; ++c) top = std::max(top, o.counts[c]);
      const bool can = top < o.n && o.n >= P.min_samples_split && o.n >= 2 &&
                       (!P.max_depth || o.depth < *P.max_depth);  // forest.hpp:178-179
      if (can)
        split_list.push_back(o);
      else
        trees[o.tree][size_t(o.bnode)].pred = argmax_first(o.counts, k);
    }
    while (!split_list.empty()) {
      const size_t N = split_list.size();
      zs.resize(N);
      poss.resize(N);
      parents.resize(N);
      const auto tb = Clock::now();
      pool.parallel_for(N, [&](size_t i) {
        const Open& o = split_list[i];
        uint64_t used;
        zs[i] = binom(o.seed, o.pos, &used);
        poss[i] = used;
        parents[i] = host::entropy(o.counts, k);
      });
      times.ms_binomial += ms_since(tb);
      w.nodes.resize(N);
      uint64_t term_off = 0;
      for (size_t i = 0; i < N; ++i) {
        const Open& o = split_list[i];
        NodeIn& nd = w.nodes[i];
        nd.seed = o.seed;
        nd.begin = o.begin;
        nd.n = o.n;
        nd.z = uint32_t(zs[i]);
        nd.pos = uint32_t(poss[i]);
        const bool hist = P.mode == 1 || (P.mode == 2 && o.n > P.breakeven);  // split.hpp:46-48
        nd.flags = hist ? kNodeHist : 0u;
        nd.term_off = uint32_t(term_off);
        nd.hist_slot = 0;
        nd.tree = o.tree;
        nd.parent = parents[i];
        term_off += zs[i];
      }
      if (term_off >= (1ull << 32)) throw std::runtime_error("wave term count overflow");
      w.idx_in = idx[cur].p;
      w.lab_in = lab[cur].p;
      w.idx_out = idx[cur ^ 1].p;
      w.lab_out = lab[cur ^ 1].p;
      eng.run(w, res);

      retry.clear();
      for (size_t i = 0; i < N; ++i) {
        Open& o = split_list[i];
        const NodeRes& r = res[i];
        if (r.row >= 0 && r.n_left > 0 && r.n_left < o.n) {
          std::vector<BNode>& tr = trees[o.tree];
          const int32_t L = int32_t(tr.size());
          {
            BNode& p = tr[size_t(o.bnode)];
            p.thr = r.threshold;
            p.left = L;
            p.right = L + 1;
            if (r.n_terms <= uint32_t(kWinTermsMax))
              p.terms.assign(r.terms, r.terms + r.n_terms);
            else
              p.terms = eng.fetch_row_terms(w, uint32_t(i), uint32_t(r.row));
          }
          tr.emplace_back();
          tr.emplace_back();
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
          for (int c = 0; c < k; ++c) {
            l.counts[c] = r.left_counts[c];
            rr.counts[c] = o.counts[c] - r.left_counts[c];
          }
          next.push_back(l);
          next.push_back(rr);
        } else if (o.attempt < P.max_split_retries) {  // forest.hpp:187,211: next attempt
          o.attempt++;
          o.pos = r.pos_after;
          retry.push_back(o);
        } else {
          trees[o.tree][size_t(o.bnode)].pred = argmax_first(o.counts, k);
        }
      }
      split_list.swap(retry);
    }
    cur ^= 1;
    frontier.swap(next);
  }

  // ---- reference node order: ids assigned at split time in depth-first order (H4) ------------
  for (size_t b = 0; b < B; ++b) {
    const std::vector<BNode>& tr = trees[b];
    std::vector<int32_t> id(tr.size(), -1), order;
    order.reserve(tr.size());
    std::vector<int32_t> stack{0};
    id[0] = 0;
    int32_t next_id = 1;
    while (!stack.empty()) {
      const int32_t v = stack.back();
      stack.pop_back();
      order.push_back(v);
      const BNode& nv = tr[size_t(v)];
      if (nv.left >= 0) {
        id[size_t(nv.left)] = next_id;
        id[size_t(nv.right)] = next_id + 1;
        next_id += 2;
        stack.push_back(nv.right);
        stack.push_back(nv.left);
      }
    }
    std::vector<int32_t> by_id(tr.size());
    for (size_t v = 0; v < tr.size(); ++v) by_id[size_t(id[v])] = int32_t(v);
    for (size_t q = 0; q < tr.size(); ++q) {
      const BNode& nv = tr[size_t(by_id[q])];
      out.left.push_back(nv.left >= 0 ? id[size_t(nv.left)] : -1);
      out.right.push_back(nv.right >= 0 ? id[size_t(nv.right)] : -1);
      out.pred.push_back(nv.pred);
      out.thr.push_back(nv.left >= 0 ? nv.thr : 0.f);
      for (uint32_t t : nv.terms) {
        out.feat.push_back(t >> 1);
        out.weight.push_back((t & 1u) ? -1.f : 1.f);
      }
      out.term_off.push_back(int64_t(out.feat.size()));
    }
    out.tree_off.push_back(int64_t(out.left.size()));
  }
  times.ms_total += ms_since(t_start);
}

}  // namespace sofg
