// Device-side std::mt19937_64 and libstdc++'s Lemire downscale, warp-cooperative.
//
// The reference draws every random decision from one engine per tree node,
// make_rng(seed) = std::mt19937_64(split_mix64(seed)) (reference random.hpp:26, forest.hpp:183).
// Integer-only consumers of that stream — Floyd cell picks and ±1 coins in
// sample_projection_matrix (projection.hpp:72-80) and the boundary picks in sample_boundaries
// (histogram.hpp:47-53, random.hpp:31-45) — are regenerated here bit-exactly, so the host only
// ships (seed, stream position). The binomial draw (libm-dependent) stays on the host.
//
// Engine: 312 x u64 state, twist in two dependency-free phases (156 + 156 words), tempering.
// uniform_int_distribution<u64>(0, j) on a 64-bit engine is Lemire's nearly-divisionless method
// (libstdc++ bits/uniform_int_dist.h:257-281 with _Wp = unsigned __int128):
//   p = x * (j+1); if lo(p) < j+1 and lo(p) < (2^64 - (j+1)) % (j+1): redraw; result hi(p).
#pragma once
#include <cstdint>

namespace sofg {
namespace dev {

constexpr int kMtN = 312;
constexpr int kMtM = 156;
constexpr uint64_t kMtA = 0xB5026F5AA96619E9ull;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull;
constexpr uint64_t kLower = 0x7FFFFFFFull;

__host__ __device__ __forceinline__ uint64_t split_mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= (y >> 43);
  return y;
}

__device__ __forceinline__ uint64_t mt_mix(uint64_t cur, uint64_t next, uint64_t far) {
  const uint64_t y = (cur & kUpper) | (next & kLower);
  return far ^ (y >> 1) ^ ((y & 1ull) ? kMtA : 0ull);
}

// Sequential seeding (std::mersenne_twister_engine::seed): one lane writes all 312 words.
__device__ __forceinline__ void mt_seed_lane(uint64_t* st, uint64_t s) {
  st[0] = s;
#pragma unroll 4
  for (int i = 1; i < kMtN; ++i) {
    s = 6364136223846793005ull * (s ^ (s >> 62)) + uint64_t(i);
    st[i] = s;
  }
}

// Out-of-place twist of block `a` into `b` (b = next 312 raw words), warp-cooperative.
// Phase 1: b[i] = mix(a[i], a[i+1], a[i+156]) for i < 156 (reads only a).
// Phase 2: b[i] = mix(a[i], a[i+1] | b[0], b[i-156]) for i >= 156.
__device__ __forceinline__ void mt_twist_warp(const uint64_t* a, uint64_t* b, int lane) {
  for (int i = lane; i < kMtN - kMtM; i += 32) b[i] = mt_mix(a[i], a[i + 1], a[i + kMtM]);
  __syncwarp();
  for (int i = kMtN - kMtM + lane; i < kMtN; i += 32) {
    const uint64_t nxt = (i + 1 < kMtN) ? a[i + 1] : b[0];
    b[i] = mt_mix(a[i], nxt, b[i - (kMtN - kMtM)]);
  }
  __syncwarp();
}

// Same, block-cooperative (nthreads threads, caller syncs before and after).
__device__ __forceinline__ void mt_twist_block(const uint64_t* a, uint64_t* b, int tid, int nthr) {
  for (int i = tid; i < kMtN - kMtM; i += nthr) b[i] = mt_mix(a[i], a[i + 1], a[i + kMtM]);
  __syncthreads();
  for (int i = kMtN - kMtM + tid; i < kMtN; i += nthr) {
    const uint64_t nxt = (i + 1 < kMtN) ? a[i + 1] : b[0];
    b[i] = mt_mix(a[i], nxt, b[i - (kMtN - kMtM)]);
  }
  __syncthreads();
}

// Lemire accept test for range r = j+1 (r >= 1): returns true and sets *t when x is accepted.
__device__ __forceinline__ bool lemire_accept(uint64_t x, uint64_t r, uint64_t* t) {
  const uint64_t lo = x * r;
  *t = __umul64hi(x, r);
  if (lo < r) {
    const uint64_t thr = (0ull - r) % r;
    if (lo < thr) return false;
  }
  return true;
}

// Warp-wide view of one engine's output stream held in two shared-memory blocks.
// Raw (untempered) words live in blk[0..312) (current) and blk[312..624) (next). `cur` is the
// index of the next output within the current block. All lanes hold identical copies of the
// bookkeeping; calls are warp-collective.
struct WarpStream {
  uint64_t* cur_blk;
  uint64_t* nxt_blk;
  int cur;
  bool nxt_ready;

  __device__ __forceinline__ void init_seeded(uint64_t* storage, uint64_t seed, int lane) {
    cur_blk = storage;
    nxt_blk = storage + kMtN;
    if (lane == 0) mt_seed_lane(nxt_blk, split_mix64(seed));
    __syncwarp();
    // first output triggers a twist of the seeded state
    mt_twist_warp(nxt_blk, cur_blk, lane);
    cur = 0;
    nxt_ready = false;
  }

  // Same, for a state whose seeded words the caller already wrote to storage[312..624).
  __device__ __forceinline__ void init_preseeded(uint64_t* storage, int lane) {
    cur_blk = storage;
    nxt_blk = storage + kMtN;
    __syncwarp();
    mt_twist_warp(nxt_blk, cur_blk, lane);
    cur = 0;
    nxt_ready = false;
  }

  __device__ __forceinline__ void ensure_next(int lane) {
    if (!nxt_ready) {
      mt_twist_warp(cur_blk, nxt_blk, lane);
      nxt_ready = true;
    }
  }

  // Raw word at offset k (0 <= k < 312 + 312 - cur) from the cursor; needs ensure_next when the
  // window crosses the block.
  __device__ __forceinline__ uint64_t peek(int k) const {
    const int i = cur + k;
    return i < kMtN ? cur_blk[i] : nxt_blk[i - kMtN];
  }

  __device__ __forceinline__ void advance(int k, int lane) {
    cur += k;
    while (cur >= kMtN) {  // k <= 312 in practice, loop only for skip()
      ensure_next(lane);   // the window may end exactly on the block boundary
      uint64_t* t = cur_blk;
      cur_blk = nxt_blk;
      nxt_blk = t;
      cur -= kMtN;
      nxt_ready = false;
      __syncwarp();
    }
  }

  // Discard `count` outputs (warp-collective).
  __device__ __forceinline__ void skip(uint64_t count, int lane) {
    while (count > 0) {
      const uint64_t room = uint64_t(kMtN - cur);
      if (count < room) {
        cur += int(count);
        return;
      }
      count -= room;
      ensure_next(lane);
      advance(int(room), lane);
    }
  }

  // Tempered output at offset k (k < 32) from the cursor; makes sure the window is valid.
  __device__ __forceinline__ uint64_t window32(int k, int lane) {
    if (cur + 32 > kMtN) ensure_next(lane);
    return mt_temper(peek(k));
  }
};

}  // namespace dev
}  // namespace sofg
