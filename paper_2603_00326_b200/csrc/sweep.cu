// Projection stage of a wave: every open node's projected rows (reference apply_projection,
// projection.hpp:86-108, called per row by find_node_split, split.hpp:247-250) written to the
// wave's value block V. Node i owns V[vbase[i] .. + n_i * Rp): sample j of the node (its j-th
// active sample) has its R projected values contiguous at V[vbase[i] + j*Rp + r] (Rp = R rounded
// up to 8, one 32-byte sector per 8 rows). Downstream kernels read rows with vector loads.
//
// Two producers write the same V:
//
//  k_row_sweep       sample-major sweep over the row-major copy of the table (XR). Each CTA takes
//                    one sample s at a time: it looks up, through the batch's inverse map
//                    inv[s][tree] (position of s in the tree's level buffer) and pos_node, every
//                    open node of the wave that contains s, streams the sample's 16 KB row into
//                    shared memory once, and computes all R rows of every such node from shared
//                    memory. One coalesced read of the table row serves the ~60 trees that hold the
//                    sample, instead of ~60 x 192 scattered 4-byte gathers from the column-major
//                    table (each a 32-byte L2 sector); V is written with coalesced 128-byte stores.
//  k_project_gather  node-major gathers from the column-major table (used for waves that cover
//                    few samples — retries, deep levels — and for primitive entry points whose
//                    active sets need not be distinct).
//
// Terms of a row are combined exactly as the reference does: ascending feature order, the first
// term assigns, later terms add, all in double, one rounding to float; an empty row is 0.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.hpp"
#include "dev_util.cuh"
#include "kernels.hpp"
#include "sweep_common.cuh"

namespace sofg {
namespace dev {

// Column-major X[f*ld + s] -> row-major XR[s*ldr + f] (32x32 smem tiles).
__global__ void __launch_bounds__(256) k_transpose_rows(const float* __restrict__ X, uint64_t ld,
                                                        uint64_t n, uint64_t d,
                                                        float* __restrict__ XR, uint64_t ldr) {
  __shared__ float tile[32][33];
  const uint64_t s0 = uint64_t(blockIdx.x) * 32, f0 = uint64_t(blockIdx.y) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int i = ty; i < 32; i += 8) {
    const uint64_t f = f0 + i, s = s0 + tx;
    tile[i][tx] = (f < d && s < n) ? X[f * ld + s] : 0.f;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const uint64_t s = s0 + i, f = f0 + tx;
    if (s < n && f < ldr) XR[s * ldr + f] = tile[tx][i];
  }
}

// inv[s*B + tree(p)] = p for every position p of the root level buffer (tree b owns
// [off[b], off[b+1])). inv is pre-filled with ~0.
__global__ void k_inv_init(const uint32_t* __restrict__ idx, const uint64_t* __restrict__ off,
                           uint32_t B, uint32_t* __restrict__ inv) {
  const uint32_t b = blockIdx.y;
  const uint64_t p0 = off[b], p1 = off[b + 1];
  for (uint64_t p = p0 + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < p1;
       p += uint64_t(gridDim.x) * blockDim.x)
    inv[uint64_t(idx[p]) * B + b] = uint32_t(p);
}

// pos_node[p] = wave node owning level position p (pre-filled with ~0 for closed nodes).
__global__ void __launch_bounds__(256) k_pos_fill(const NodeIn* __restrict__ nodes,
                                                  const Tile* __restrict__ tiles,
                                                  uint32_t* __restrict__ pos_node) {
  const Tile tl = tiles[blockIdx.x];
  const uint32_t begin = nodes[tl.node].begin + tl.start;
  for (uint32_t l = threadIdx.x; l < tl.len; l += blockDim.x) pos_node[begin + l] = tl.node;
}

// +-x of term t (bit 0 = negative weight) as a double; negation is exact, so this equals the
// reference's weight * double(x) for weights +-1.
__device__ __forceinline__ double signed_term(const float* xs, uint32_t t) {
  return double(__uint_as_float(__float_as_uint(xs[t >> 1]) ^ (t << 31)));
}

// Combine the terms [q0, q1) of one row for a sample whose features are in `xs` (shared memory).
__device__ __forceinline__ float project_from(const float* xs, const uint32_t* tm, uint32_t q0,
                                              uint32_t q1) {
  if (q1 <= q0) return 0.f;
  double acc = signed_term(xs, tm[q0]);
  for (uint32_t q = q0 + 1; q < q1; ++q) acc = __dadd_rn(acc, signed_term(xs, tm[q]));
  return __double2float_rn(acc);
}

template <typename E>
__global__ void __launch_bounds__(128) k_aug_build(const NodeIn* __restrict__ nodes, int n_nodes,
                                                   const uint32_t* __restrict__ terms,
                                                   const uint32_t* __restrict__ row_ptr, uint32_t R,
                                                   uint32_t d, E* __restrict__ aug,
                                                   uint16_t* __restrict__ qsplit,
                                                   const uint64_t* __restrict__ vbase,
                                                   uint32_t* __restrict__ pnode) {
  constexpr uint32_t A = 16 / sizeof(E);
  extern __shared__ uint32_t s_empty_pre[];  // [4 warps][R + 1]: empty rows before row r
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int node = int(blockIdx.x) * 4 + w;
  if (node >= n_nodes) return;
  uint32_t* epre = s_empty_pre + size_t(w) * (R + 1);
  const NodeIn nd = nodes[node];
  const uint32_t* rp = row_ptr + size_t(node) * (R + 1);
  const uint32_t* tm = terms + nd.term_off;
  E* out = aug + aug_off<E>(nd.term_off, uint32_t(node), R);
  uint32_t carry = 0;
  for (uint32_t r0 = 0; r0 < R; r0 += 32) {
    const uint32_t r = r0 + uint32_t(lane);
    const bool empty = r < R && __ldg(rp + r + 1) == __ldg(rp + r);
    const unsigned m = __ballot_sync(0xffffffffu, empty);
    if (r < R) epre[r] = carry + __popc(m & ((1u << lane) - 1u));
    carry += __popc(m);
  }
  if (lane == 0) epre[R] = carry;
  __syncwarp();
  // Quarter boundaries balanced by entry count: entries before row r are
  // E(r) = (rp[r] - rp[0]) + epre[r] (strictly increasing: every row has >= 1 entry); quarter c
  // starts at the first row with E(r) >= c * T / kQ.
  const uint32_t rp0 = __ldg(rp);
  const uint32_t T = (__ldg(rp + R) - rp0) + carry;
  uint32_t qs[kQ + 1];
  qs[0] = 0;
  qs[kQ] = R;
#pragma unroll
  for (int c = 1; c < kQ; ++c) {
    const uint32_t target = (uint32_t(c) * T + kQ / 2) / kQ;
    uint32_t below = 0;
    for (uint32_t r0 = 0; r0 <= R; r0 += 32) {
      const uint32_t r = r0 + uint32_t(lane);
      const bool lt = r <= R && (__ldg(rp + r) - rp0) + epre[r] < target;
      below += __popc(__ballot_sync(0xffffffffu, lt));
    }
    qs[c] = min(below, R);
  }
  if (lane < kQ) qsplit[size_t(node) * kQ + lane] = uint16_t(lane + 1 < kQ ? qs[lane + 1] : R);
  static_assert(kQ == 4, "pnode packs four quarter boundaries");
  if (pnode && lane == 0) {  // pair record of level position p: x + p * Rp / 8, y, z, w
    const uint32_t Rp8 = vpitch(R) / 8;
    uint4 pn;
    pn.x = uint32_t(__ldg(vbase + node) >> 3) - nd.begin * Rp8;  // mod 2^32: the records fit 32 bits
    pn.y = uint32_t(aug_off<E>(nd.term_off, uint32_t(node), R));
    pn.z = qs[1] | (qs[2] << 16);
    pn.w = qs[3] | (R << 16);
    reinterpret_cast<uint4*>(pnode)[node] = pn;
  }
  // element e of list c -> entry ((e / A) * kQ + c) * A + e % A of the node block
  auto at = [&](uint32_t c, uint32_t e) { return ((e / A) * kQ + c) * A + (e % A); };
  for (uint32_t r = uint32_t(lane); r < R; r += 32) {
    uint32_t c = 0;
#pragma unroll
    for (int cc = 1; cc < kQ; ++cc) c += r >= qs[cc] ? 1u : 0u;
    const uint32_t ra = qs[c];
    const uint32_t q0 = __ldg(rp + r), q1 = __ldg(rp + r + 1);
    const uint32_t e0 = (q0 - __ldg(rp + ra)) + (epre[r] - epre[ra]);
    if (q1 == q0) {
      out[at(c, e0)] = E((d << 2) | 2u);
    } else {
      for (uint32_t q = q0; q < q1; ++q) {
        const uint32_t t = __ldg(tm + q);
        out[at(c, e0 + (q - q0))] = E(((t >> 1) << 2) | (q + 1 == q1 ? 2u : 0u) | (t & 1u));
      }
    }
  }
  // neutral entries up to the end of each list's last chunk
#pragma unroll
  for (int c = 0; c < kQ; ++c) {
    const uint32_t ra = qs[c], rb = qs[c + 1];
    const uint32_t len = (__ldg(rp + rb) - __ldg(rp + ra)) + (epre[rb] - epre[ra]);
    for (uint32_t e = len + uint32_t(lane); e < (len + A - 1) / A * A; e += 32) out[at(uint32_t(c), e)] = E(d << 2);
  }
}

// ------------------------------------------------------------------------------------------
// Sample-major sweep. A CTA takes K consecutive samples at a time: their rows stream into shared
// memory (cp.async; one coalesced read of each row per level) and the inverse map lists every
// open node of the wave that holds one of them. Then kQ lanes per (node, sample) pair each walk
// one sub-list in order — 16-byte loads with four in flight, the entries' feature reads as
// independent shared-memory loads, one double accumulator per row — and park their rows in a
// per-lane staging slot, written to V at the end with vector stores.
// ------------------------------------------------------------------------------------------
constexpr int kSweepThreadsMax = 256;  // CTA size: 256 for ~60+ trees per wave, 128 below

struct Pair {
  uint32_t node, j, k, pad;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = uint32_t(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// smem: xs[K][ldr] | pairs[K*B] | out[NT][pitch]
template <typename E, int NT>
__global__ void __launch_bounds__(NT) k_row_sweep(
    const float* __restrict__ XR, uint64_t ldr, uint32_t N, uint32_t K,
    const uint32_t* __restrict__ inv, uint32_t B, const uint32_t* __restrict__ pos_node,
    const NodeIn* __restrict__ nodes, const uint64_t* __restrict__ vbase,
    const E* __restrict__ aug, const uint16_t* __restrict__ qsplit, uint32_t R, float* __restrict__ V) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* xs = reinterpret_cast<float*>(smem_raw);
  Pair* pairs = reinterpret_cast<Pair*>(smem_raw + size_t(K) * ldr * 4);
  const uint32_t pitch = stage_pitch(R);
  constexpr uint32_t P = 32u / kQ;
  const int lane = threadIdx.x & 31;
  float* wstage = reinterpret_cast<float*>(pairs + size_t(K) * B) + size_t(threadIdx.x >> 5) * P * pitch;
  __shared__ uint32_t s_cnt;
  const uint32_t Rp = vpitch(R);
  const uint32_t nvec = uint32_t(ldr / 4);
  const uint32_t KB = K * B;
  const uint32_t c = threadIdx.x % kQ;  // my sub-list
  constexpr uint32_t kPairsPerRound = NT / kQ;
  for (uint32_t i = uint32_t(lane); i < P * (Rp - R); i += 32)  // pad rows of the staging stay zero
    wstage[(i / (Rp - R)) * pitch + R + i % (Rp - R)] = 0.f;

  for (uint32_t s0 = blockIdx.x * K; s0 < N; s0 += gridDim.x * K) {
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    // ---- rows of the K samples -> shared memory (asynchronous)
    const uint32_t ks = min(K, N - s0);
    {
      const float4* src = reinterpret_cast<const float4*>(XR + uint64_t(s0) * ldr);
      float4* dst = reinterpret_cast<float4*>(xs);
      for (uint32_t v = threadIdx.x; v < ks * nvec; v += NT) cp_async16(dst + v, src + v);
    }
    // ---- (node, j) pairs of the K samples: inv -> level position -> wave node
    for (uint32_t e0 = 0; e0 < KB; e0 += NT) {
      const uint32_t e = e0 + threadIdx.x;
      const uint32_t k = e / B;
      uint32_t node = ~0u, p = ~0u;
      if (e < KB && k < ks) {
        p = __ldcs(inv + uint64_t(s0) * B + e);
        if (p != ~0u) node = __ldg(pos_node + p);
      }
      const bool act = node != ~0u;
      const unsigned m = __ballot_sync(0xffffffffu, act);
      uint32_t base = 0;
      if (lane == 0 && m) base = atomicAdd(&s_cnt, uint32_t(__popc(m)));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (act) pairs[base + __popc(m & ((1u << lane) - 1u))] = Pair{node, p - __ldg(&nodes[node].begin), k, 0u};
    }
    cp_async_wait_all();
    __syncthreads();
    const uint32_t cnt = s_cnt;
    const uint32_t rounds = (cnt + kPairsPerRound - 1) / kPairsPerRound;  // uniform
    for (uint32_t rd = 0; rd < rounds; ++rd) {
      const uint32_t pi = rd * kPairsPerRound + threadIdx.x / kQ;
      uint32_t ra = 0, rb = 0;  // this lane's rows (none when the slot is empty)
      const uint4* a4 = reinterpret_cast<const uint4*>(aug);
      const char* xb = reinterpret_cast<const char*>(xs);
      uint64_t vout = 0;
      if (pi < cnt) {
        const Pair pr = pairs[pi];
        a4 = reinterpret_cast<const uint4*>(aug + aug_off<E>(__ldg(&nodes[pr.node].term_off), pr.node, R)) + c;
        xb = reinterpret_cast<const char*>(xs + size_t(pr.k) * ldr);
        vout = __ldg(vbase + pr.node) + uint64_t(pr.j) * Rp;
        quarter_rows(qsplit + size_t(pr.node) * kQ, c, R, ra, rb);
      }
      const uint32_t out_base = uint32_t(__cvta_generic_to_shared(wstage + (uint32_t(lane) / kQ) * pitch));
      walk_rows<E>(a4, xb, ra, rb, out_base);
      __syncwarp();
      const uint32_t p_warp = rd * kPairsPerRound + (threadIdx.x & ~31u) / kQ;  // the warp's first pair
      const uint32_t np = cnt > p_warp ? min(P, cnt - p_warp) : 0u;
      write_pairs(wstage, pitch, Rp, np, V, vout, lane);
      __syncwarp();
    }
    __syncthreads();
  }
}

// Gather producer: a CTA takes one partition tile (<= kTileElems samples of one node); each warp
// handles 32 samples at a time, lane = sample. The node's CSR is staged in shared memory; each
// lane walks the terms in order with 8 independent gathers in flight and closes rows at their
// row_ptr boundaries (uniform across the warp). Rows are staged per warp as [32][Rp] and written
// out with coalesced stores.
constexpr int kGatherWarps = 8;
__global__ void __launch_bounds__(256) k_project_gather(
    const NodeIn* __restrict__ nodes, const Tile* __restrict__ tiles,
    const uint64_t* __restrict__ vbase, const uint32_t* __restrict__ terms,
    const uint32_t* __restrict__ row_ptr, uint32_t R, const uint32_t* __restrict__ idx,
    const float* __restrict__ X, uint64_t ld, float* __restrict__ V, bool stage_terms) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t Rp = vpitch(R);
  const Tile tl = tiles[blockIdx.x];
  const NodeIn nd = nodes[tl.node];
  const uint32_t* rpg = row_ptr + size_t(tl.node) * (R + 1);
  const uint32_t z = __ldg(rpg + R) - __ldg(rpg);
  float* stg = reinterpret_cast<float*>(smem_raw) + size_t(w) * 32 * Rp;
  uint32_t* s_rp = reinterpret_cast<uint32_t*>(smem_raw + size_t(kGatherWarps) * 32 * Rp * 4);
  const uint32_t* s_tm;  // the node's terms: shared memory, or global (L1) for dense matrices
  if (stage_terms) {
    uint32_t* st_tm = s_rp + R + 1;
    for (uint32_t q = threadIdx.x; q < z; q += blockDim.x) st_tm[q] = __ldg(terms + nd.term_off + q);
    s_tm = st_tm;
  } else {
    s_tm = terms + nd.term_off;
  }
  for (uint32_t r = threadIdx.x; r <= R; r += blockDim.x) s_rp[r] = __ldg(rpg + r);
  __syncthreads();
  float* Vn = V + vbase[tl.node];
  for (uint32_t c0 = uint32_t(w) * 32; c0 < tl.len; c0 += 32 * kGatherWarps) {
    const uint32_t jl = c0 + uint32_t(lane);
    const bool ok = jl < tl.len;
    const float* xcol = X + (ok ? idx[nd.begin + tl.start + jl] : idx[nd.begin + tl.start]);
    uint32_t r = 0;
    while (r < R && s_rp[r + 1] == s_rp[r]) stg[size_t(lane) * Rp + r++] = 0.f;  // leading empty rows
    uint32_t rend = r < R ? s_rp[r + 1] : ~0u;
    double acc = 0.0;
    bool first = true;
    for (uint32_t q0 = 0; q0 < z; q0 += 8) {
      float x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t q = q0 + uint32_t(u);
        x[u] = q < z ? gather(xcol + uint64_t(s_tm[q] >> 1) * ld) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t q = q0 + uint32_t(u);
        if (q < z) {
          const double dx = double(__uint_as_float(__float_as_uint(x[u]) ^ (s_tm[q] << 31)));
          acc = first ? dx : __dadd_rn(acc, dx);
          first = false;
          if (q + 1 == rend) {  // row r complete; following empty rows are zero
            stg[size_t(lane) * Rp + r] = __double2float_rn(acc);
            first = true;
            ++r;
            while (r < R && s_rp[r + 1] == s_rp[r]) stg[size_t(lane) * Rp + r++] = 0.f;
            rend = r < R ? s_rp[r + 1] : ~0u;
          }
        }
      }
    }
    for (; r < R; ++r) stg[size_t(lane) * Rp + r] = 0.f;  // (only when z == 0)
    __syncwarp();
    const uint32_t cnt = min(32u, tl.len - c0);
    float* dstv = Vn + uint64_t(tl.start + c0) * Rp;
    for (uint32_t i = uint32_t(lane); i < cnt * Rp; i += 32) dstv[i] = stg[i];
    __syncwarp();
  }
}

}  // namespace dev

cudaError_t launch_transpose_rows(const float* X, uint64_t ld, uint64_t n, uint64_t d, float* XR,
                                  uint64_t ldr, cudaStream_t st) {
  const uint64_t gx = (n + 31) / 32, gy = (ldr + 31) / 32;
  if (gy > 65535) return cudaErrorInvalidValue;
  for (uint64_t x0 = 0; x0 < gx; x0 += 1u << 30) {
    const unsigned bx = unsigned(std::min<uint64_t>(gx - x0, 1u << 30));
    dev::k_transpose_rows<<<dim3(bx, unsigned(gy)), 256, 0, st>>>(X + x0 * 32, ld, n - x0 * 32, d,
                                                                   XR + x0 * 32 * ldr, ldr);
  }
  return cudaGetLastError();
}

cudaError_t launch_inv_init(const uint32_t* idx, const uint64_t* off, uint32_t B, uint64_t n_samples,
                            uint64_t max_per_tree, uint32_t* inv, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(inv, 0xff, 4 * n_samples * B, st);
  if (e != cudaSuccess || B == 0) return e;
  const unsigned gx = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((max_per_tree + 255) / 256, 1024)));
  dev::k_inv_init<<<dim3(gx, B), 256, 0, st>>>(idx, off, B, inv);
  return cudaGetLastError();
}

cudaError_t launch_pos_fill(const NodeIn* nodes, const Tile* tiles, int n_tiles, uint64_t total,
                            uint32_t* pos_node, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(pos_node, 0xff, 4 * total, st);
  if (e != cudaSuccess || n_tiles == 0) return e;
  dev::k_pos_fill<<<n_tiles, 256, 0, st>>>(nodes, tiles, pos_node);
  return cudaGetLastError();
}

bool aug_narrow(uint32_t d) { return d < 8192; }

size_t aug_bytes(uint64_t total_terms, uint32_t n_nodes, uint32_t R, uint32_t d) {
  const size_t es = aug_narrow(d) ? 2 : 4, A = 16 / es;
  // kQ interleaved lists per node (aug_off), plus one chunk row of alignment and the walk's
  // prefetch window (8 chunk rows) past the last block
  return (size_t(dev::kQ) * (size_t(total_terms) + size_t(n_nodes) * (R + 2 * A)) + 9 * dev::kQ * A) * es;
}

cudaError_t launch_aug_build(const NodeIn* nodes, int n_nodes, const uint32_t* terms,
                             const uint32_t* row_ptr, uint32_t R, uint32_t d, void* aug,
                             uint16_t* qsplit, const uint64_t* vbase, uint32_t* pnode, cudaStream_t st) {
  if (n_nodes == 0) return cudaSuccess;
  if (R > 65535) return cudaErrorInvalidValue;
  const size_t smem = size_t(4) * (R + 1) * 4;
  if (aug_narrow(d))
    dev::k_aug_build<uint16_t><<<(n_nodes + 3) / 4, 128, smem, st>>>(
        nodes, n_nodes, terms, row_ptr, R, d, static_cast<uint16_t*>(aug), qsplit, vbase, pnode);
  else
    dev::k_aug_build<uint32_t><<<(n_nodes + 3) / 4, 128, smem, st>>>(
        nodes, n_nodes, terms, row_ptr, R, d, static_cast<uint32_t*>(aug), qsplit, vbase, pnode);
  return cudaGetLastError();
}

static int sweep_threads(uint32_t B) {
  static const int force = std::getenv("SOFG_SWEEP_NT") ? std::atoi(std::getenv("SOFG_SWEEP_NT")) : 0;
  if (force) return force;
  return B * 5 / 8 > 40 ? 256 : 128;
}

static size_t sweep_smem_k(uint64_t ldr, uint32_t B, uint32_t R, uint32_t K) {
  return size_t(K) * ldr * 4 + size_t(K) * B * sizeof(dev::Pair) +
         size_t(sweep_threads(B) / 32) * (32 / dev::kQ) * dev::stage_pitch(R) * 4;
}

// Samples per CTA iteration: enough (node, sample) pairs to fill the CTA's lanes (a sample sits
// in ~63% of the batch's trees), within shared memory.
static uint32_t sweep_k(uint64_t ldr, uint32_t B, uint32_t R) {
  const uint32_t per = std::max<uint32_t>(1, B * 5 / 8);  // pairs per sample
  // about two rounds of pair slots per chunk: one round per sample leaves a mostly empty second
  // round whenever a sample sits in more trees than there are slots (measured at 100 trees:
  // K = 1 -> 496 ms, K = 2 -> 470 ms, K = 3 -> 533 ms of sweep per step)
  const uint32_t want = std::max<uint32_t>(1, (2 * uint32_t(sweep_threads(B)) / dev::kQ + per / 2) / per);
  static const int force_k = std::getenv("SOFG_SWEEP_K") ? std::atoi(std::getenv("SOFG_SWEEP_K")) : 0;
  uint32_t K = force_k ? uint32_t(force_k) : std::min<uint32_t>(want, 8);
  while (K > 1 && sweep_smem_k(ldr, B, R, K) > 112 * 1024) --K;
  return K;
}

void row_sweep_variant(uint32_t B, uint32_t d, uint32_t* cta_threads, uint32_t* entry_bytes) {
  *cta_threads = uint32_t(sweep_threads(B));
  *entry_bytes = aug_narrow(d) ? 2u : 4u;
}

size_t row_sweep_smem(uint64_t ldr, uint32_t B, uint32_t R) {
  return sweep_smem_k(ldr, B, R, sweep_k(ldr, B, R));
}

template <typename E, int NT>
static cudaError_t launch_sweep_t(const float* XR, uint64_t ldr, uint32_t N, const uint32_t* inv,
                                  uint32_t B, const uint32_t* pos_node, const NodeIn* nodes,
                                  const uint64_t* vbase, const void* aug, const uint16_t* qsplit,
                                  uint32_t R, float* V, int n_sm, cudaStream_t st) {
  const uint32_t K = sweep_k(ldr, B, R);
  const size_t smem = sweep_smem_k(ldr, B, R, K);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(dev::k_row_sweep<E, NT>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptin);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dev::k_row_sweep<E, NT>, NT, smem);
  const uint32_t groups = (N + K - 1) / K;
  const unsigned grid = unsigned(std::max(1, std::min<int>(int(groups), n_sm * std::max(per_sm, 1))));
  dev::k_row_sweep<E, NT><<<grid, NT, smem, st>>>(
      XR, ldr, N, K, inv, B, pos_node, nodes, vbase, static_cast<const E*>(aug), qsplit, R, V);
  return cudaGetLastError();
}

cudaError_t launch_row_sweep(const float* XR, uint64_t ldr, uint32_t N, const uint32_t* inv,
                             uint32_t B, const uint32_t* pos_node, const NodeIn* nodes,
                             const uint64_t* vbase, const void* aug, const uint16_t* qsplit, uint32_t R,
                             uint32_t d, float* V, int n_sm, cudaStream_t st) {
  const bool wide = sweep_threads(B) == 256;
  if (aug_narrow(d))
    return wide ? launch_sweep_t<uint16_t, 256>(XR, ldr, N, inv, B, pos_node, nodes, vbase, aug, qsplit, R, V, n_sm, st)
                : launch_sweep_t<uint16_t, 128>(XR, ldr, N, inv, B, pos_node, nodes, vbase, aug, qsplit, R, V, n_sm, st);
  return wide ? launch_sweep_t<uint32_t, 256>(XR, ldr, N, inv, B, pos_node, nodes, vbase, aug, qsplit, R, V, n_sm, st)
              : launch_sweep_t<uint32_t, 128>(XR, ldr, N, inv, B, pos_node, nodes, vbase, aug, qsplit, R, V, n_sm, st);
}

cudaError_t launch_project_gather(const NodeIn* nodes, const Tile* tiles, int n_tiles,
                                  const uint64_t* vbase, const uint32_t* terms,
                                  const uint32_t* row_ptr, uint32_t R, uint32_t zmax,
                                  const uint32_t* idx, const float* X, uint64_t ld, float* V,
                                  cudaStream_t st) {
  if (n_tiles == 0) return cudaSuccess;
  size_t smem = size_t(dev::kGatherWarps) * 32 * vpitch(R) * 4 + size_t(R + 1 + zmax) * 4;
  const bool stage_terms = smem <= size_t(kSmemOptin);
  if (!stage_terms) smem = size_t(dev::kGatherWarps) * 32 * vpitch(R) * 4 + size_t(R + 1) * 4;
  if (smem > size_t(kSmemOptin)) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(dev::k_project_gather,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptin);
  if (e != cudaSuccess) return e;
  dev::k_project_gather<<<n_tiles, 256, smem, st>>>(nodes, tiles, vbase, terms, row_ptr, R, idx, X,
                                                   ld, V, stage_terms);
  return cudaGetLastError();
}

}  // namespace sofg
