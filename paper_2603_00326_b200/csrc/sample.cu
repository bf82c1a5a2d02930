// Per-node random structure regenerated on the device from (seed, stream position):
//
//  k_sample_projection  — sample_projection_matrix (reference projection.hpp:57-82) after the
//                         host's binomial draw: Floyd over R*d cells (random.hpp:31-45), ascending
//                         cell order, one coin per cell. Output: CSR per node.
//  k_hist_draws         — the Floyd position draws of sample_boundaries for every row of a
//                         histogram node (histogram.hpp:47-53), consumed in row order from the
//                         same engine (split.hpp:272-276), with Lemire rejections handled inline.
//  k_hist_boundaries    — resolves each row's Floyd set, gathers the picked projected values,
//                         sorts them and emits midpoint_down of distinct neighbours
//                         (histogram.hpp:56-60).
#include <cuda_runtime.h>

#include "common.hpp"
#include "dev_util.cuh"
#include "kernels.hpp"

#ifndef SOFG_DRAW_THREADS
#define SOFG_DRAW_THREADS 128  // threads per histogram node of k_hist_draws (64: 32.7, 128: 32.9, 256: 38.7, 512: 49.6 ms per step)
#endif
#ifndef SOFG_BND_MINB_SMALL
#define SOFG_BND_MINB_SMALL 10  // min CTAs per SM (register cap) of k_hist_boundaries for <= 256 picks (none: 86.2, 10: 82.5, 12: 123 ms per step)
#endif
#define SOFG_BND_MINB(EPL) ((EPL) <= 8 ? SOFG_BND_MINB_SMALL : 0)
#ifndef SOFG_BND_WARPS
#define SOFG_BND_WARPS 4  // (node, row) warps per CTA of k_hist_boundaries
#endif
#ifndef SOFG_SAMPLE_WARPS
#define SOFG_SAMPLE_WARPS 4  // warps (nodes) per CTA of k_sample_projection (8: 54.6, 4: 47.8, 2: 45.1 ms per step with per-warp seeding; seeded by one warp for the CTA: 8: 45.0, 4: 38.6, 2: 44.7)
#endif
#include "mt64.cuh"

namespace sofg {
namespace dev {

// ------------------------------------------------------------------------------------------
// Projection sampler: one warp per node.
// smem per warp: 624 u64 (two engine blocks) + 2 * zpad u32 (sorted set, draw order).
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(32 * SOFG_SAMPLE_WARPS) k_sample_projection(
    const NodeIn* __restrict__ nodes, int n_nodes, uint32_t d, uint32_t R, int zpad,
    uint32_t* __restrict__ terms, uint32_t* __restrict__ row_ptr, uint32_t* __restrict__ pos_after,
    uint32_t* __restrict__ gkeys, uint32_t* __restrict__ gaux) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int node = blockIdx.x * (blockDim.x >> 5) + wib;
  // dense matrices (large z): the cell sets live in global scratch instead of shared memory
  const size_t per_warp = size_t(2 * kMtN) * 8 + (gkeys ? 0 : size_t(2 * zpad) * 4);
  // The engines' sequential seeding (311 dependent steps each) for all of the CTA's nodes at once,
  // lane j of warp 0 for node j: one warp instruction advances every node's recurrence, where a
  // lane-0-per-warp seeding spent the same instruction count on each node alone.
  if (wib == 0 && lane < int(blockDim.x >> 5)) {
    const int nj = int(blockIdx.x * (blockDim.x >> 5)) + lane;
    if (nj < n_nodes && !(nodes[nj].flags & kNodeGivenCsr))
      mt_seed_lane(reinterpret_cast<uint64_t*>(smem_raw + per_warp * size_t(lane)) + kMtN,
                   split_mix64(nodes[nj].seed));
  }
  __syncthreads();
  if (node >= n_nodes) return;
  unsigned char* base = smem_raw + per_warp * wib;
  uint64_t* blk = reinterpret_cast<uint64_t*>(base);
  uint32_t* keys = gkeys ? gkeys + size_t(node) * 2 * zpad
                         : reinterpret_cast<uint32_t*>(base + size_t(2 * kMtN) * 8);
  uint32_t* draws = keys + zpad;

  const NodeIn nd = nodes[node];
  uint32_t* rp = row_ptr + size_t(node) * (R + 1);
  if (nd.flags & kNodeGivenCsr) return;  // host supplied the matrix and pos_after

  const uint32_t z = nd.z;
  int zp = 32;  // this node's sort width (the shared arrays are sized for the wave's largest z)
  while (zp < int(z)) zp <<= 1;
  const uint64_t cells = uint64_t(R) * d;
  WarpStream s;
  s.init_preseeded(blk, lane);
  s.skip(nd.pos, lane);
  uint64_t used = nd.pos;

  // Floyd draws t_q = uniform(0, cells - z + q), q = 0..z-1, in stream order.
  uint32_t q = 0;
  while (q < z) {
    const uint32_t cnt = min(32u, z - q);
    uint64_t t = 0;
    bool ok = true;
    const uint64_t x = s.window32(lane, lane);  // collective: every lane calls it
    if (lane < int(cnt)) ok = lemire_accept(x, cells - z + q + lane + 1, &t);
    const unsigned bad = __ballot_sync(0xffffffffu, !ok);
    const uint32_t take = bad ? uint32_t(__ffs(bad) - 1) : cnt;
    if (lane < int(take)) draws[q + lane] = uint32_t(t);
    s.advance(int(take), lane);
    used += take;
    q += take;
    if (bad) {  // output rejected: it is consumed, the same draw retries on the next output
      s.advance(1, lane);
      used += 1;
    }
  }
  __syncwarp();

  // Set = {t_q} unless some t collides (prob ~ z^2 / 2 cells); sort and test neighbours.
  if (gaux) {
    // large matrices: warp LSD radix sort (8-bit digits over the bits of cells - 1), stable
    // scatter by in-order 32-key chunks; ping-pong through the node's scratch
    uint32_t* tmp = gaux + size_t(node) * 2 * zpad;  // [zpad]
    uint32_t* cnt = tmp + zpad;                       // [256] digit offsets
    int bits = 0;
    while (bits < 32 && ((cells - 1) >> bits) != 0) bits += 8;
    const uint32_t* src = draws;
    uint32_t* dst = (bits / 8) % 2 ? keys : tmp;  // the last pass lands in keys
    if (bits == 0) dst = keys;
    for (int sh = 0; sh < bits; sh += 8) {
      for (int b = lane; b < 256; b += 32) cnt[b] = 0;
      __syncwarp();
      for (uint32_t i = lane; i < z; i += 32) atomicAdd(cnt + ((src[i] >> sh) & 255u), 1u);
      __syncwarp();
      {  // exclusive scan of the 256 counts (8 per lane)
        uint32_t c8[8], loc = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          c8[e] = cnt[lane * 8 + e];
          loc += c8[e];
        }
        uint32_t tot;
        uint32_t run = warp_excl_scan_u32(loc, lane, &tot);
        __syncwarp();
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          cnt[lane * 8 + e] = run;
          run += c8[e];
        }
      }
      __syncwarp();
      for (uint32_t b = 0; b < z; b += 32) {
        const uint32_t i = b + uint32_t(lane);
        const uint32_t key = i < z ? src[i] : 0u;
        const uint32_t dg = i < z ? ((key >> sh) & 255u) : 256u;
        const unsigned peers = __match_any_sync(0xffffffffu, dg);
        const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
        const uint32_t base = dg < 256u ? cnt[dg] : 0u;
        if (i < z) dst[base + rank] = key;
        __syncwarp();
        if (dg < 256u && rank == 0) cnt[dg] = base + __popc(peers);
        __syncwarp();
      }
      src = dst;
      dst = dst == keys ? tmp : keys;
    }
    if (bits == 0)
      for (uint32_t i = lane; i < z; i += 32) keys[i] = draws[i];
    for (int i = int(z) + lane; i < zpad; i += 32) keys[i] = 0xffffffffu;
    __syncwarp();
  } else {
    for (int i = lane; i < zp; i += 32) keys[i] = i < int(z) ? draws[i] : 0xffffffffu;
    __syncwarp();
    if (gkeys) warp_bitonic_sort(keys, zp, lane); else warp_sort_via_regs(keys, zp, lane);
  }
  bool dup = false;
  for (int i = lane + 1; i < int(z); i += 32) dup |= keys[i] == keys[i - 1];
  if (__any_sync(0xffffffffu, dup) && gaux) {
    // Exact Floyd resolution (random.hpp:36-44) without the serial scan: draw i collides when its
    // value appeared at an earlier index (C1, from the smallest index per sorted value), or when
    // it equals J0 + j for an earlier colliding draw j (Floyd inserts J0 + j instead); the flags
    // are a monotone fixpoint. The set is then {t_i : no collision} u {J0 + i : collision}.
    const uint32_t J0 = uint32_t(cells - z);
    uint32_t* minidx = gaux + size_t(node) * 2 * zpad;
    uint32_t* flag = minidx + zpad;
    auto lower = [&](uint32_t t) {
      uint32_t lo = 0, hi = z;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (keys[mid] < t) lo = mid + 1; else hi = mid;
      }
      return lo;
    };
    for (uint32_t i = lane; i < z; i += 32) minidx[i] = 0xffffffffu;
    __syncwarp();
    for (uint32_t i = lane; i < z; i += 32) atomicMin(minidx + lower(draws[i]), i);
    __syncwarp();
    for (uint32_t i = lane; i < z; i += 32) flag[i] = minidx[lower(draws[i])] != i ? 1u : 0u;
    __syncwarp();
    for (;;) {
      bool ch = false;
      for (uint32_t i = lane; i < z; i += 32) {
        if (flag[i]) continue;
        const uint32_t t = draws[i];
        if (t >= J0 && t - J0 < i && flag[t - J0]) {
          flag[i] = 1u;
          ch = true;
        }
      }
      __syncwarp();
      if (!__any_sync(0xffffffffu, ch)) break;
    }
    // The set is distinct(all t) u {J0 + i : collision} (every drawn value ends up in the set),
    // both sides already sorted: merge them instead of sorting again.
    uint32_t* uq = minidx;  // distinct sorted draw values (minidx is no longer needed)
    uint32_t u = 0;
    for (uint32_t b = 0; b < z; b += 32) {
      const uint32_t p = b + uint32_t(lane);
      const bool keep = p < z && (p == 0 || keys[p] != keys[p - 1]);
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (keep) uq[u + __popc(m & ((1u << lane) - 1u))] = keys[p];
      u += __popc(m);
    }
    __syncwarp();
    auto in_uq = [&](uint32_t v) {  // binary search in uq[0..u)
      uint32_t lo = 0, hi = u;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (uq[mid] < v) lo = mid + 1; else hi = mid;
      }
      return lo;
    };
    // replacement values J0 + i (increasing in i) not already drawn, compacted in place into
    // draws[] (entries are only read at indices >= the write index)
    uint32_t c = 0;
    for (uint32_t b = 0; b < z; b += 32) {
      const uint32_t i = b + uint32_t(lane);
      bool add = false;
      uint32_t v = 0;
      if (i < z && flag[i]) {
        v = J0 + i;
        const uint32_t at = in_uq(v);
        add = !(at < u && uq[at] == v);
      }
      const unsigned m = __ballot_sync(0xffffffffu, add);
      __syncwarp();
      if (add) draws[c + __popc(m & ((1u << lane) - 1u))] = v;
      c += __popc(m);
      __syncwarp();
    }
    // merge: final rank = own index + number of smaller elements of the other list
    for (uint32_t p = lane; p < u; p += 32) {
      const uint32_t v = uq[p];
      uint32_t lo = 0, hi = c;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (draws[mid] < v) lo = mid + 1; else hi = mid;
      }
      keys[p + lo] = v;
    }
    for (uint32_t q = lane; q < c; q += 32) keys[q + in_uq(draws[q])] = draws[q];
    __syncwarp();
  } else if (__any_sync(0xffffffffu, dup)) {
    // Exact Floyd resolution in draw order (random.hpp:36-44): a collision inserts j instead.
    for (uint32_t i = 0; i < z; ++i) {
      const uint32_t t = draws[i];
      bool hit = false;
      for (uint32_t p = lane; p < i; p += 32) hit |= keys[p] == t;
      hit = __any_sync(0xffffffffu, hit);
      __syncwarp();
      if (lane == 0) keys[i] = hit ? uint32_t(cells - z + i) : t;
      __syncwarp();
    }
    for (int i = lane; i < zp; i += 32)
      if (i >= int(z)) keys[i] = 0xffffffffu;
    __syncwarp();
    if (gkeys) warp_bitonic_sort(keys, zp, lane); else warp_sort_via_regs(keys, zp, lane);
  }

  // Coins: cell i (ascending) gets the top bit of the next output (uniform_int<int>(0,1)).
  uint32_t* out = terms + nd.term_off;
  for (uint32_t b = 0; b < z; b += 32) {
    const uint64_t x = s.window32(lane, lane);
    const uint32_t i = b + lane;
    if (i < z) {
      const uint32_t cell = keys[i];
      const bool plus = (x >> 63) != 0;
      out[i] = encode_term(cell % d, !plus);
    }
    const uint32_t c = min(32u, z - b);
    s.advance(int(c), lane);
    used += c;
  }
  // row_ptr[r] = #cells < r*d
  for (uint32_t r = lane; r <= R; r += 32) {
    const uint64_t lim = uint64_t(r) * d;
    uint32_t lo = 0, hi = z;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (uint64_t(keys[mid]) < lim) lo = mid + 1; else hi = mid;
    }
    rp[r] = lo;
  }
  if (lane == 0) pos_after[node] = uint32_t(used);
}

// ------------------------------------------------------------------------------------------
// Histogram boundary draws: one CTA (256 threads) per histogram node. Generates the R*m Lemire
// draws of the R consecutive sample_boundaries calls. Output: draws[slot][R*m] (u32),
// pos_split[node] = stream position after the picks.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(SOFG_DRAW_THREADS) k_hist_draws(
    const NodeIn* __restrict__ nodes, const uint32_t* __restrict__ hist_nodes, int n_hist,
    uint32_t R, uint32_t bins, const uint32_t* __restrict__ pos_after_proj,
    uint32_t* __restrict__ draws, uint32_t* __restrict__ pos_split) {
  __shared__ uint64_t A[kMtN], B[kMtN];
  __shared__ int s_first_bad;
  const int h = blockIdx.x;
  if (h >= n_hist) return;
  const uint32_t node = hist_nodes[h];
  const NodeIn nd = nodes[node];
  const uint32_t n = nd.n;
  const uint32_t start_pos = pos_after_proj[node];
  const uint32_t m = min(bins, n);
  const int tid = threadIdx.x;
  if (n < 2 || bins < 2 || m == n) {  // histogram.hpp:42-49: no draws
    if (tid == 0) pos_split[node] = start_pos;
    return;
  }
  // seed + first twist
  if (tid == 0) mt_seed_lane(B, split_mix64(nd.seed));
  __syncthreads();
  mt_twist_block(B, A, tid, blockDim.x);
  uint64_t* cur_blk = A;
  uint64_t* nxt_blk = B;
  uint64_t pos = start_pos;
  while (pos >= uint64_t(kMtN)) {
    mt_twist_block(cur_blk, nxt_blk, tid, blockDim.x);
    uint64_t* t = cur_blk;
    cur_blk = nxt_blk;
    nxt_blk = t;
    pos -= kMtN;
  }
  int cur = int(pos);
  uint64_t used = start_pos;
  const uint64_t total = uint64_t(R) * m;
  uint32_t* out = draws + size_t(h) * R * bins;  // fixed stride R*bins per histogram node
  uint64_t q = 0;
  while (q < total) {
    const int avail = kMtN - cur;
    const uint64_t want = min(uint64_t(avail), total - q);
    if (tid == 0) s_first_bad = 0x7fffffff;
    __syncthreads();
    // One pass over [cur, cur+want): every draw is written as if no earlier output in the window
    // were rejected, and the first rejection is found. Draws at or after it are shifted by that
    // rejected output; they are rewritten by the next windows, which start right after it and
    // write every later position again in order (rejections are rare: range <= n << 2^64).
    for (int o = tid; o < int(want); o += blockDim.x) {
      const uint64_t x = mt_temper(cur_blk[cur + o]);
      const uint64_t qq = q + uint64_t(o);
      const uint32_t i = uint32_t(qq % m);
      uint64_t t;
      if (!lemire_accept(x, uint64_t(n - m + i) + 1, &t)) atomicMin(&s_first_bad, o);
      out[qq] = uint32_t(t);
    }
    __syncthreads();
    const int fb = s_first_bad;
    const int take = fb == 0x7fffffff ? int(want) : fb;
    q += uint64_t(take);
    cur += take + (fb == 0x7fffffff ? 0 : 1);
    used += uint64_t(take) + (fb == 0x7fffffff ? 0 : 1);
    if (cur >= kMtN) {
      __syncthreads();
      mt_twist_block(cur_blk, nxt_blk, tid, blockDim.x);
      uint64_t* t = cur_blk;
      cur_blk = nxt_blk;
      nxt_blk = t;
      cur -= kMtN;
    }
    __syncthreads();
  }
  if (tid == 0) pos_split[node] = uint32_t(used);
}

// ------------------------------------------------------------------------------------------
// Boundaries (reference sample_boundaries, histogram.hpp:42-80): one warp per (histogram node,
// row), EPL = mpad/32 draws per lane held in registers (blocked layout: lane l owns draw indices
// [l*EPL, (l+1)*EPL)). smem per warp: a 2*mpad-slot hash table (u64) + mpad collision flags.
//   1. C1_i: draw t_i equals an earlier draw (hash table of draw values + smallest index).
//   2. D_i = C1_i or (t_i - J0 < i and D_{t_i - J0}) (Floyd's replacement J0 + i is itself picked
//      later): monotone fixpoint over the flags.
//   3. gather the picked values (EPL independent loads per lane), register bitonic sort,
//      midpoints of consecutive distinct values, compacted in order.
// ------------------------------------------------------------------------------------------
template <int EPL>
__global__ void __launch_bounds__(32 * SOFG_BND_WARPS, SOFG_BND_MINB(EPL)) k_hist_boundaries(
    const NodeIn* __restrict__ nodes, const uint32_t* __restrict__ hist_nodes, int n_hist,
    uint32_t R, uint32_t bins, const uint32_t* __restrict__ draws,
    const uint64_t* __restrict__ gbase, const float* __restrict__ G,
    float* __restrict__ bnd, uint32_t* __restrict__ nb_out) {
  constexpr int MP = 32 * EPL;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const uint64_t item = uint64_t(blockIdx.x) * (blockDim.x >> 5) + wib;
  if (item >= uint64_t(n_hist) * R) return;
  const uint32_t h = uint32_t(item / R);
  const uint32_t r = uint32_t(item % R);
  unsigned char* base = smem_raw + size_t(MP) * 17 * wib;
  uint64_t* ht = reinterpret_cast<uint64_t*>(base);                   // [2*MP]
  uint8_t* col = reinterpret_cast<uint8_t*>(base + size_t(MP) * 16);  // [MP]

  const uint32_t node = hist_nodes[h];
  const NodeIn nd = nodes[node];
  const uint32_t n = nd.n;
  float* out = bnd + (size_t(h) * R + r) * (bins - 1);
  if (n < 2 || bins < 2) {
    if (lane == 0) nb_out[size_t(h) * R + r] = 0;
    return;
  }
  const uint32_t m = min(bins, n);
  const uint32_t J0 = n - m;
  const uint32_t Rp = vpitch(R);
  const float* Vn = G + gbase[node] + r;  // row r of the node's V block (sweep.cu)
  const uint32_t i0 = uint32_t(lane * EPL);
  uint32_t key[EPL];

  if (m < n) {
    const uint32_t* t = draws + size_t(h) * R * bins + size_t(r) * m;
    uint32_t tv[EPL];
#pragma unroll
    for (int e = 0; e < EPL; ++e) tv[e] = i0 + e < m ? __ldg(t + i0 + e) : 0u;
    constexpr uint32_t TS = 2u * MP;  // load <= 1/2
    constexpr int TB = 31 - __builtin_clz(TS);
    uint32_t* hk = reinterpret_cast<uint32_t*>(ht);  // [TS] draw values (~0 = empty)
    uint32_t* hi = hk + TS;                          // [TS] smallest index holding the value
#pragma unroll
    for (int e = 0; e < 2 * EPL; ++e) {
      hk[e * 32 + lane] = ~0u;
      hi[e * 32 + lane] = ~0u;
    }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      const uint32_t i = i0 + uint32_t(e);
      if (i < m) {
        uint32_t sl = (tv[e] * 0x9E3779B1u) >> (32 - TB);
        for (;;) {
          const uint32_t old = atomicCAS(hk + sl, ~0u, tv[e]);
          if (old == ~0u || old == tv[e]) {
            atomicMin(hi + sl, i);
            break;
          }
          sl = (sl + 1) & (TS - 1);
        }
      }
    }
    __syncwarp();
    uint32_t done = 0;  // bit e: flag of draw i0+e known set (C1 first: all lookups, then the stores)
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      const uint32_t i = i0 + uint32_t(e);
      if (i < m) {
        uint32_t sl = (tv[e] * 0x9E3779B1u) >> (32 - TB);
        while (hk[sl] != tv[e]) sl = (sl + 1) & (TS - 1);
        done |= (hi[sl] != i ? 1u : 0u) << e;
      }
    }
#pragma unroll
    for (int e = 0; e < EPL; ++e) col[i0 + uint32_t(e)] = uint8_t(done >> e & 1u);
    __syncwarp();
    for (;;) {  // each pass reads every flag, then writes the new ones (no read/write overlap)
      uint32_t add = 0;
#pragma unroll
      for (int e = 0; e < EPL; ++e) {
        const uint32_t i = i0 + uint32_t(e);
        if (!(done >> e & 1u) && i < m && tv[e] >= J0 && tv[e] - J0 < i && col[tv[e] - J0]) add |= 1u << e;
      }
      __syncwarp();
#pragma unroll
      for (int e = 0; e < EPL; ++e)
        if (add >> e & 1u) col[i0 + uint32_t(e)] = 1;
      done |= add;
      __syncwarp();
      if (!__any_sync(0xffffffffu, add != 0)) break;
    }
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      const uint32_t i = i0 + uint32_t(e);
      const uint32_t pidx = (done >> e & 1u) ? J0 + i : tv[e];
      key[e] = i < m ? order_key(__ldg(Vn + uint64_t(pidx) * Rp)) : 0xffffffffu;
    }
  } else {
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      const uint32_t i = i0 + uint32_t(e);
      key[e] = i < m ? order_key(__ldg(Vn + uint64_t(i) * Rp)) : 0xffffffffu;
    }
  }
  reg_bitonic_sort_k<EPL, uint32_t, (EPL >= 16)>(key, lane);
  // midpoints of consecutive distinct values (float comparison: -0 == +0), in order
  const uint32_t prev_last = __shfl_up_sync(0xffffffffu, key[EPL - 1], 1);
  uint32_t emit = 0;
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    const uint32_t i = i0 + uint32_t(e);
    const uint32_t pk = e == 0 ? prev_last : key[e > 0 ? e - 1 : 0];
    if (i >= 1 && i < m && order_key_inv(pk) < order_key_inv(key[e])) emit |= 1u << e;
  }
  uint32_t total;
  uint32_t pos = warp_excl_scan_u32(uint32_t(__popc(emit)), lane, &total);
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    if (emit >> e & 1u) {
      const uint32_t pk = e == 0 ? prev_last : key[e > 0 ? e - 1 : 0];
      out[pos++] = midpoint_down(order_key_inv(pk), order_key_inv(key[e]));
    }
  }
  if (lane == 0) nb_out[size_t(h) * R + r] = total;
}

// Boundaries for more than 1024 bins (sample_boundaries with m = min(bins, n) up to kMaxBins picks,
// histogram.hpp:42-61): one CTA of 256 threads per (node, row), thread t owning draws
// [t EPT, (t + 1) EPT); the same three steps as k_hist_boundaries (hash of first indices, the
// D-fixpoint, gather) with the picked keys bitonic-sorted in shared memory and the midpoints
// compacted by a block scan. Shared memory: 2 * MP hash slots (value, index) + MP keys + MP flags.
constexpr int kBndCtaThreads = 256;
template <int MP>
__global__ void __launch_bounds__(kBndCtaThreads) k_hist_boundaries_cta(
    const NodeIn* __restrict__ nodes, const uint32_t* __restrict__ hist_nodes, int n_hist, uint32_t R,
    uint32_t bins, const uint32_t* __restrict__ draws, const uint64_t* __restrict__ gbase,
    const float* __restrict__ G, float* __restrict__ bnd, uint32_t* __restrict__ nb_out) {
  constexpr int EPT = MP / kBndCtaThreads;
  constexpr uint32_t TS = 2u * MP;
  constexpr int TB = 31 - __builtin_clz(TS);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* hk = reinterpret_cast<uint32_t*>(smem_raw);  // [TS] draw values (~0 = empty)
  uint32_t* hi = hk + TS;                                // [TS] smallest index holding the value
  uint32_t* keys = hi + TS;                              // [MP]
  uint8_t* col = reinterpret_cast<uint8_t*>(keys + MP);  // [MP]
  __shared__ uint32_t s_warp[kBndCtaThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t h = uint32_t(blockIdx.x / R), r = uint32_t(blockIdx.x % R);
  if (h >= uint32_t(n_hist)) return;
  const uint32_t node = hist_nodes[h];
  const uint32_t n = nodes[node].n;
  float* out = bnd + (size_t(h) * R + r) * (bins - 1);
  if (n < 2 || bins < 2) {
    if (tid == 0) nb_out[size_t(h) * R + r] = 0;
    return;
  }
  const uint32_t m = min(bins, n), J0 = n - m, Rp = vpitch(R);
  const float* Vn = G + gbase[node] + r;
  const uint32_t i0 = uint32_t(tid * EPT);
  if (m < n) {
    const uint32_t* t = draws + size_t(h) * R * bins + size_t(r) * m;
    uint32_t tv[EPT];
#pragma unroll
    for (int e = 0; e < EPT; ++e) tv[e] = i0 + e < m ? __ldg(t + i0 + e) : 0u;
    for (uint32_t i = tid; i < TS; i += kBndCtaThreads) {
      hk[i] = ~0u;
      hi[i] = ~0u;
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const uint32_t i = i0 + uint32_t(e);
      if (i < m) {
        uint32_t sl = (tv[e] * 0x9E3779B1u) >> (32 - TB);
        for (;;) {
          const uint32_t old = atomicCAS(hk + sl, ~0u, tv[e]);
          if (old == ~0u || old == tv[e]) {
            atomicMin(hi + sl, i);
            break;
          }
          sl = (sl + 1) & (TS - 1);
        }
      }
    }
    __syncthreads();
    uint32_t c1 = 0;  // C1: an earlier draw has the same value (all lookups, then the stores)
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const uint32_t i = i0 + uint32_t(e);
      if (i < m) {
        uint32_t sl = (tv[e] * 0x9E3779B1u) >> (32 - TB);
        while (hk[sl] != tv[e]) sl = (sl + 1) & (TS - 1);
        c1 |= (hi[sl] != i ? 1u : 0u) << e;
      }
    }
#pragma unroll
    for (int e = 0; e < EPT; ++e) col[i0 + uint32_t(e)] = uint8_t(c1 >> e & 1u);
    __syncthreads();
    uint32_t done = c1;  // this thread's flags, also kept in registers
    for (;;) {  // D_i = C1_i or (J0 <= t_i < J0 + i and D_{t_i - J0}): monotone fixpoint
      uint32_t add = 0;  // read every flag, then write the new ones
#pragma unroll
      for (int e = 0; e < EPT; ++e) {
        const uint32_t i = i0 + uint32_t(e);
        if (!(done >> e & 1u) && i < m && tv[e] >= J0 && tv[e] - J0 < i && col[tv[e] - J0]) add |= 1u << e;
      }
      __syncthreads();
#pragma unroll
      for (int e = 0; e < EPT; ++e)
        if (add >> e & 1u) col[i0 + uint32_t(e)] = 1;
      done |= add;
      if (__syncthreads_or(add != 0) == 0) break;
    }
    uint32_t kv[EPT];  // all gathers in flight before the stores
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const uint32_t i = i0 + uint32_t(e);
      kv[e] = i < m ? order_key(__ldg(Vn + uint64_t((done >> e & 1u) ? J0 + i : tv[e]) * Rp)) : 0xffffffffu;
    }
#pragma unroll
    for (int e = 0; e < EPT; ++e) keys[i0 + uint32_t(e)] = kv[e];
  } else {
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const uint32_t i = i0 + uint32_t(e);
      keys[i] = i < m ? order_key(__ldg(Vn + uint64_t(i) * Rp)) : 0xffffffffu;
    }
  }
  __syncthreads();
  for (uint32_t sz = 2; sz <= uint32_t(MP); sz <<= 1)  // bitonic sort, ascending
    for (uint32_t st = sz >> 1; st > 0; st >>= 1) {
      for (uint32_t i = tid; i < uint32_t(MP); i += kBndCtaThreads) {
        const uint32_t j = i ^ st;
        if (j > i) {
          const uint32_t a = keys[i], b = keys[j];
          if ((a > b) == ((i & sz) == 0)) {
            keys[i] = b;
            keys[j] = a;
          }
        }
      }
      __syncthreads();
    }
  // midpoints of consecutive distinct values (float comparison: -0 == +0), compacted in order
  uint32_t cnt = 0;
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    const uint32_t i = i0 + uint32_t(e);
    cnt += (i >= 1 && i < m && order_key_inv(keys[i - 1]) < order_key_inv(keys[i])) ? 1u : 0u;
  }
  uint32_t wt;
  const uint32_t wex = warp_excl_scan_u32(cnt, lane, &wt);
  if (lane == 0) s_warp[w] = wt;
  __syncthreads();
  uint32_t pos = wex, total = 0;
  for (int ww = 0; ww < kBndCtaThreads / 32; ++ww) {
    if (ww < w) pos += s_warp[ww];
    total += s_warp[ww];
  }
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    const uint32_t i = i0 + uint32_t(e);
    if (i >= 1 && i < m && order_key_inv(keys[i - 1]) < order_key_inv(keys[i]))
      out[pos++] = midpoint_down(order_key_inv(keys[i - 1]), order_key_inv(keys[i]));
  }
  if (tid == 0) nb_out[size_t(h) * R + r] = total;
}

}  // namespace dev

// ---------------------------------------------------------------------------- launchers
static int next_pow2(int x) {
  int p = 32;
  while (p < x) p <<= 1;
  return p;
}

cudaError_t launch_sample_projection(const NodeIn* nodes, int n_nodes, uint32_t d, uint32_t R,
                                     uint32_t zmax, uint32_t* terms, uint32_t* row_ptr,
                                     uint32_t* pos_after, Scratch& scratch, cudaStream_t st) {
  if (n_nodes == 0) return cudaSuccess;
  const int zpad = next_pow2(int(zmax));
  const bool global_sets = size_t(2 * dev::kMtN) * 8 + size_t(2 * zpad) * 4 > 96 * 1024;
  const size_t per_warp = size_t(2 * dev::kMtN) * 8 + (global_sets ? 0 : size_t(2 * zpad) * 4);
  int warps = SOFG_SAMPLE_WARPS;
  while (warps > 1 && per_warp * warps > 96 * 1024) warps >>= 1;
  const size_t smem = per_warp * warps;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(dev::k_sample_projection, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kSmemOptin);
  // global scratch for very dense matrices (owned by the caller's WaveRunner)
  uint32_t* gkeys = nullptr;
  if (global_sets) {
    gkeys = static_cast<uint32_t*>(scratch.get(Scratch::kSampleKeys, size_t(n_nodes) * 2 * size_t(zpad) * 4, st));
    if (!gkeys) return cudaErrorMemoryAllocation;
  }
  // collision resolution scratch for large matrices (the serial draw-order scan is O(z^2))
  uint32_t* gaux = nullptr;
  if (zpad >= 1024) {
    gaux = static_cast<uint32_t*>(scratch.get(Scratch::kSampleAux, size_t(n_nodes) * 2 * size_t(zpad) * 4, st));
    if (!gaux) return cudaErrorMemoryAllocation;
  }
  const int grid = (n_nodes + warps - 1) / warps;
  dev::k_sample_projection<<<grid, warps * 32, smem, st>>>(nodes, n_nodes, d, R, zpad, terms,
                                                           row_ptr, pos_after, gkeys, gaux);
  return cudaGetLastError();
}

cudaError_t launch_hist_draws(const NodeIn* nodes, const uint32_t* hist_nodes, int n_hist,
                              uint32_t R, uint32_t bins, const uint32_t* pos_after_proj,
                              uint32_t* draws, uint32_t* pos_split, cudaStream_t st) {
  if (n_hist == 0) return cudaSuccess;
  dev::k_hist_draws<<<n_hist, SOFG_DRAW_THREADS, 0, st>>>(nodes, hist_nodes, n_hist, R, bins, pos_after_proj,
                                            draws, pos_split);
  return cudaGetLastError();
}

cudaError_t launch_hist_boundaries(const NodeIn* nodes, const uint32_t* hist_nodes, int n_hist,
                                   uint32_t R, uint32_t bins, const uint32_t* draws,
                                   const uint32_t* terms, const uint32_t* row_ptr,
                                   const uint64_t* gbase, const float* G, float* bnd,
                                   uint32_t* nb, cudaStream_t st) {
  (void)terms;
  (void)row_ptr;
  if (n_hist == 0) return cudaSuccess;
  const int mpad = next_pow2(int(bins));
  const size_t smem = size_t(mpad) * 17 * SOFG_BND_WARPS;  // per warp: hash table + flags
  const uint64_t items = uint64_t(n_hist) * R;
  const unsigned grid = unsigned((items + SOFG_BND_WARPS - 1) / SOFG_BND_WARPS);
  auto go = [&](auto kern) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptin);
    kern<<<grid, 32 * SOFG_BND_WARPS, smem, st>>>(nodes, hist_nodes, n_hist, R, bins, draws, gbase, G, bnd, nb);
    return cudaGetLastError();
  };
  switch (mpad) {
    case 32: return go(dev::k_hist_boundaries<1>);
    case 64: return go(dev::k_hist_boundaries<2>);
    case 128: return go(dev::k_hist_boundaries<4>);
    case 256: return go(dev::k_hist_boundaries<8>);
    case 512: return go(dev::k_hist_boundaries<16>);
    case 1024: return go(dev::k_hist_boundaries<32>);
    default: break;
  }
  auto go_cta = [&](auto kern) {  // more than 1024 bins: one CTA per (node, row)
    const size_t smem_cta = size_t(mpad) * 21;  // hash 2 x 2 MP words, keys MP words, flags MP bytes
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptin);
    kern<<<unsigned(uint64_t(n_hist) * R), dev::kBndCtaThreads, smem_cta, st>>>(nodes, hist_nodes, n_hist, R, bins, draws,
                                                                               gbase, G, bnd, nb);
    return cudaGetLastError();
  };
  switch (mpad) {
    case 2048: return go_cta(dev::k_hist_boundaries_cta<2048>);
    case 4096: return go_cta(dev::k_hist_boundaries_cta<4096>);
    case 8192: return go_cta(dev::k_hist_boundaries_cta<8192>);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace sofg
