// Projection stage, pipelined sweep (the producer/consumer form of k_row_sweep, sweep.cu).
//
// Same computation — every open node's projected rows into the wave's value block V, one pass of
// the row-major table XR per level — organised as a persistent, warp-specialised kernel:
//
//  k_pair_build      one warp per sample s: the inverse map inv[s][tree] -> level position ->
//                    wave node, compacted into the sample's pair list: for every open node that
//                    holds s, a 16-byte record {V offset of the (node, s) rows, start of the
//                    node's term lists}. pcnt[s] = number of records.
//  k_row_sweep_pipe  one CTA per SM. Warp NCW (producer, one lane) walks the CTA's samples and,
//                    for each sample with pairs, waits for a free ring slot (empty mbarrier), arms
//                    the slot's full mbarrier with the byte count and issues two bulk async copies
//                    (cp.async.bulk, the TMA engine): the sample's table row and its pair list.
//                    It then publishes the sample's work as chunks of 32 / kQ pairs into a ticket
//                    queue in shared memory. The NCW consumer warps take tickets in order, wait
//                    on the slot's full barrier, walk their pairs' term lists against the staged
//                    row (walk_rows, sweep_common.cuh) and write V with vector stores; the warp
//                    that completes a sample's last chunk releases the slot (empty mbarrier).
//                    No CTA-wide barrier after setup: warps run decoupled, and a sample's chunks
//                    are spread over whichever warps are free.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.hpp"
#include "dev_util.cuh"
#include "kernels.hpp"
#include "sweep_common.cuh"

namespace sofg {
namespace dev {

struct PairRec {
  uint32_t vout8;         // float index of the pair's row block in V, / 8 (blocks are 32-byte aligned)
  uint32_t aug;           // entry index of the node's block of interleaved term lists
  uint16_t q[kQ];         // the node's quarter boundaries (qsplit, sweep_common.cuh)
};
static_assert(sizeof(PairRec) == 16, "PairRec layout");

#ifndef SOFG_PIPE_CONSUMERS
#define SOFG_PIPE_CONSUMERS 16
#endif
constexpr int kPipeConsumers = SOFG_PIPE_CONSUMERS;  // consumer warps per CTA
constexpr uint32_t kChunkPairs = 32u / kQ;          // pairs per consumer-warp ticket
constexpr uint32_t kEndStage = 0xffffffffu;

// ---- mbarrier / bulk-copy primitives (sm_90+ PTX) -------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return uint32_t(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
// global -> shared bulk copy completing on `bar` (bytes and both addresses multiples of 16)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---- pair lists ----------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_pair_build(const uint32_t* __restrict__ inv, uint32_t B,
                                                    uint32_t N, const uint32_t* __restrict__ pos_node,
                                                    const uint4* __restrict__ pnode, uint32_t R,
                                                    uint32_t PB, PairRec* __restrict__ recs,
                                                    uint32_t* __restrict__ pcnt) {
  const int lane = threadIdx.x & 31;
  const uint32_t Rp8 = vpitch(R) / 8;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  constexpr int C = 4;  // 32-tree chunks whose dependent load chains (inv -> pos_node -> pnode) overlap
  for (uint32_t s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); s < N; s += warps) {
    uint32_t cnt = 0;
    for (uint32_t b00 = 0; b00 < B; b00 += 32 * C) {
      uint32_t p[C], node[C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const uint32_t b = b00 + 32 * c + uint32_t(lane);
        p[c] = b < B ? __ldcs(inv + uint64_t(s) * B + b) : ~0u;
      }
#pragma unroll
      for (int c = 0; c < C; ++c) node[c] = p[c] != ~0u ? __ldg(pos_node + p[c]) : ~0u;
      uint4 pn[C];
#pragma unroll
      for (int c = 0; c < C; ++c)
        if (node[c] != ~0u) pn[c] = __ldg(pnode + node[c]);  // one 16-byte record per node (aug_build)
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const bool act = node[c] != ~0u;
        const unsigned m = __ballot_sync(0xffffffffu, act);
        if (act) {
          uint4 rec = pn[c];
          rec.x += p[c] * Rp8;  // (V block of position 0 + p * Rp) / 8, mod 2^32
          const uint32_t idx = cnt + __popc(m & ((1u << lane) - 1u));
          *reinterpret_cast<uint4*>(recs + uint64_t(s) * PB + idx) = rec;
        }
        cnt += __popc(m);
      }
    }
    if (lane == 0) pcnt[s] = cnt;
  }
}

// ---- the pipelined sweep -------------------------------------------------------------------
// smem: rows[S][ldr] | recs[S][PB] | full[S] | empty[S] | queue[QN] (uint4) | done[S] | ticket |
//       out staging [NCW * 32][pitch]
template <typename E>
__global__ void __launch_bounds__((kPipeConsumers + 1) * 32, 1) k_row_sweep_pipe(
    const float* __restrict__ XR, uint64_t ldr, uint32_t N, const PairRec* __restrict__ recs_g,
    const uint32_t* __restrict__ pcnt, uint32_t PB, const E* __restrict__ aug, uint32_t R,
    float* __restrict__ V, uint32_t S, uint32_t QN) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* rows = reinterpret_cast<float*>(smem_raw);
  PairRec* recs = reinterpret_cast<PairRec*>(rows + size_t(S) * ldr);
  uint64_t* full = reinterpret_cast<uint64_t*>(recs + size_t(S) * PB);
  uint64_t* empty = full + S;
  uint4* queue = reinterpret_cast<uint4*>(empty + S);
  uint32_t* done = reinterpret_cast<uint32_t*>(queue + QN);
  uint32_t* ticket = done + S;
  const uint32_t pitch = stage_pitch(R);
  constexpr uint32_t P = 32u / kQ;
  float* stage_out = reinterpret_cast<float*>(smem_raw) +
                     ((reinterpret_cast<unsigned char*>(ticket + 1) - smem_raw + 15) / 16) * 4;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t Rp = vpitch(R);

  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < S; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, 1);
      done[i] = 0;
    }
    *ticket = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  for (uint32_t i = threadIdx.x; i < QN; i += blockDim.x) queue[i] = make_uint4(~0u, 0, 0, 0);
  __syncthreads();

  volatile uint32_t* vq = reinterpret_cast<volatile uint32_t*>(queue);
  if (warp == kPipeConsumers) {  // ---------------------------------------------- producer
    if (lane != 0) return;
    uint32_t stage = 0, t = 0;
    const uint32_t row_bytes = uint32_t(ldr * 4);
    uint32_t s = blockIdx.x;
    uint32_t cnt_next = s < N ? __ldg(pcnt + s) : 0u;
    for (; s < N; s += gridDim.x) {
      const uint32_t cnt = cnt_next;
      if (s + gridDim.x < N) cnt_next = __ldg(pcnt + s + gridDim.x);
      if (cnt == 0) continue;
      const uint32_t slot = stage % S, k = stage / S;
      if (k > 0) mbar_wait(empty + slot, (k - 1) & 1u);  // stage - S has been released
      done[slot] = 0;
      mbar_arrive_expect_tx(full + slot, row_bytes + cnt * uint32_t(sizeof(PairRec)));
      bulk_g2s(rows + size_t(slot) * ldr, XR + uint64_t(s) * ldr, row_bytes, full + slot);
      bulk_g2s(recs + size_t(slot) * PB, recs_g + uint64_t(s) * PB, cnt * uint32_t(sizeof(PairRec)),
               full + slot);
      const uint32_t ticket_stage = slot | ((k & 1u) << 16);  // slot and full-barrier parity
      for (uint32_t p0 = 0; p0 < cnt; p0 += kChunkPairs, ++t) {
        volatile uint32_t* q = vq + 4 * (t % QN);
        q[1] = ticket_stage;
        q[2] = p0 | (min(kChunkPairs, cnt - p0) << 16);
        q[3] = cnt;
        __threadfence_block();
        q[0] = t;
      }
      ++stage;
    }
    for (int i = 0; i < kPipeConsumers; ++i, ++t) {
      volatile uint32_t* q = vq + 4 * (t % QN);
      q[1] = kEndStage;
      __threadfence_block();
      q[0] = t;
    }
    return;
  }

  // ------------------------------------------------------------------------------ consumers
  const uint32_t c = uint32_t(lane) % kQ;  // my sub-list
  float* wstage = stage_out + size_t(warp) * P * pitch;
  for (uint32_t i = uint32_t(lane); i < P * (Rp - R); i += 32)  // pad rows of the staging stay zero
    wstage[(i / (Rp - R)) * pitch + R + i % (Rp - R)] = 0.f;
  const uint32_t out_base = smem_u32(wstage + (uint32_t(lane) / kQ) * pitch);
  for (;;) {
    uint32_t T = 0;
    if (lane == 0) T = atomicAdd(ticket, 1u);
    T = __shfl_sync(0xffffffffu, T, 0);
    uint32_t stg = 0, pn = 0, cnt = 0;
    if (lane == 0) {
      volatile uint32_t* q = vq + 4 * (T % QN);
      while (q[0] != T) __nanosleep(32);
      __threadfence_block();
      stg = q[1];
      pn = q[2];
      cnt = q[3];
    }
    stg = __shfl_sync(0xffffffffu, stg, 0);
    if (stg == kEndStage) break;
    pn = __shfl_sync(0xffffffffu, pn, 0);
    cnt = __shfl_sync(0xffffffffu, cnt, 0);
    const uint32_t slot = stg & 0xffffu;
    mbar_wait(full + slot, stg >> 16);
    const uint32_t p0 = pn & 0xffffu, np = pn >> 16;
    const uint32_t pl = uint32_t(lane) / kQ;
    const bool act = pl < np;
    uint32_t ra = 0, rb = 0;
    const uint4* a4 = reinterpret_cast<const uint4*>(aug);
    uint64_t vout = 0;
    if (act) {
      const uint4 pr = *reinterpret_cast<const uint4*>(recs + size_t(slot) * PB + p0 + pl);
      a4 = reinterpret_cast<const uint4*>(aug + pr.y) + c;
      vout = uint64_t(pr.x) << 3;
      const uint64_t qv = uint64_t(pr.z) | (uint64_t(pr.w) << 32);  // qsplit: starts of quarters 1..3, R
      ra = c ? uint32_t(qv >> (16 * (c - 1))) & 0xffffu : 0u;
      rb = uint32_t(qv >> (16 * c)) & 0xffffu;
    }
    walk_rows<E>(a4, reinterpret_cast<const char*>(rows + size_t(slot) * ldr), ra, rb, out_base);
    __syncwarp();
    write_pairs(wstage, pitch, Rp, np, V, vout, lane);
    __syncwarp();
    if (lane == 0) {
      const uint32_t before = atomicAdd(done + slot, np);
      if (before + np == cnt) mbar_arrive(empty + slot);  // the sample's last chunk: slot free
    }
  }
}

}  // namespace dev

namespace {
size_t pipe_fixed_smem(uint32_t R, uint32_t QN) {
  return size_t(QN) * 16 + 256 + size_t(dev::kPipeConsumers) * (32 / dev::kQ) * dev::stage_pitch(R) * 4;
}
size_t pipe_stage_bytes(uint64_t ldr, uint32_t PB) { return size_t(ldr) * 4 + size_t(PB) * sizeof(dev::PairRec) + 16 + 4; }
uint32_t pipe_pb(uint32_t B) { return (B + 1u) & ~1u; }
uint32_t pipe_qn(uint32_t S, uint32_t PB) {
  uint32_t need = S * ((PB + dev::kChunkPairs - 1) / dev::kChunkPairs) + dev::kPipeConsumers + 8;
  uint32_t q = 64;
  while (q < need) q <<= 1;
  return q;
}
uint32_t pipe_stages(uint64_t ldr, uint32_t B, uint32_t R) {
  const uint32_t PB = pipe_pb(B);
  for (uint32_t S = 8; S >= 2; --S) {
    const size_t bytes = size_t(S) * pipe_stage_bytes(ldr, PB) + pipe_fixed_smem(R, pipe_qn(S, PB));
    if (bytes <= size_t(kSmemOptin)) return S;
  }
  return 0;
}
}  // namespace

bool row_sweep_pipe_fits(uint64_t ldr, uint32_t B, uint32_t R) { return pipe_stages(ldr, B, R) >= 2; }

size_t pair_rec_bytes() { return sizeof(dev::PairRec); }

cudaError_t launch_pair_build(const uint32_t* inv, uint32_t B, uint32_t N, const uint32_t* pos_node,
                              const uint32_t* pnode, uint32_t R, uint32_t d, void* recs, uint32_t* pcnt,
                              int n_sm, cudaStream_t st) {
  (void)d;
  const uint32_t PB = pipe_pb(B);
  const unsigned grid = unsigned(std::min<uint64_t>((uint64_t(N) + 7) / 8, uint64_t(n_sm) * 16));
  dev::k_pair_build<<<grid, 256, 0, st>>>(inv, B, N, pos_node, reinterpret_cast<const uint4*>(pnode), R, PB,
                                          static_cast<dev::PairRec*>(recs), pcnt);
  return cudaGetLastError();
}

cudaError_t launch_row_sweep_pipe(const float* XR, uint64_t ldr, uint32_t N, const void* recs,
                                  const uint32_t* pcnt, uint32_t B, const void* aug, uint32_t R,
                                  uint32_t d, float* V, int n_sm, cudaStream_t st) {
  const uint32_t S = pipe_stages(ldr, B, R);
  if (S < 2) return cudaErrorInvalidValue;
  const uint32_t PB = pipe_pb(B), QN = pipe_qn(S, PB);
  const size_t smem = size_t(S) * pipe_stage_bytes(ldr, PB) + pipe_fixed_smem(R, QN);
  const unsigned grid = unsigned(std::max(1, std::min<int>(n_sm, int(N))));
  const int threads = (dev::kPipeConsumers + 1) * 32;
  auto go = [&](auto kern, const auto* a) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemOptin);
    if (e != cudaSuccess) return e;
    kern<<<grid, threads, smem, st>>>(XR, ldr, N, static_cast<const dev::PairRec*>(recs), pcnt, PB, a, R, V,
                                      S, QN);
    return cudaGetLastError();
  };
  if (aug_narrow(d)) return go(dev::k_row_sweep_pipe<uint16_t>, static_cast<const uint16_t*>(aug));
  return go(dev::k_row_sweep_pipe<uint32_t>, static_cast<const uint32_t*>(aug));
}

}  // namespace sofg
