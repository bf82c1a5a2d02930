// Shared pieces of the two projection-sweep kernels (sweep.cu: k_row_sweep, sweep_pipe.cu:
// k_row_sweep_pipe): the augmented term-list layout and the per-lane term walk.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "common.hpp"

namespace sofg {
namespace dev {

// ------------------------------------------------------------------------------------------
// Augmented term lists for the sweep. A node's R rows are split into kQ contiguous row ranges
// ("quarters"; quarter c = rows [qs_c, qs_{c+1}) with qs_0 = 0, qs_kQ = R), each with its own list:
// the CSR terms of its rows in order, each entry feature << 2 | last << 1 | negative (so entry & ~3
// is the feature's byte offset in a row of XR), with one dummy entry (feature d: the zero pad
// column of XR) for every empty row, so walking a list completes its rows in order. The quarter
// boundaries are chosen per node (k_aug_build) so the kQ lists hold about the same number of
// entries — the kQ lanes of a (node, sample) pair then finish together. Entries are u16 when
// d < 8192, else u32. The kQ lists of a node are interleaved in 16-byte chunks — chunk i of list
// c at chunk index i * kQ + c of the node's block — so the kQ lanes that walk one (node, sample)
// pair read one contiguous 64-byte span per step. A list's last chunk is filled up with neutral
// entries (zero column, no row end); chunks past a list's end are never consumed.
// Node i's block starts at entry aug_off(term_off_i, i, R); its boundaries qs_1..qs_{kQ-1} are
// qsplit[i * kQ + 0 .. kQ - 2] (u16; qsplit[i * kQ + kQ - 1] = R).
// ------------------------------------------------------------------------------------------
constexpr int kQ = 4;

template <typename E>
__host__ __device__ __forceinline__ uint64_t aug_off(uint32_t term_off, uint32_t i, uint32_t R) {
  constexpr uint64_t A = 16 / sizeof(E), CH = kQ * A;
  return (kQ * (uint64_t(term_off) + uint64_t(i) * (R + 2 * A)) + CH - 1) / CH * CH;
}
// rows [ra, rb) of quarter c from the node's boundaries (qsplit layout above)
__device__ __forceinline__ void quarter_rows(const uint16_t* q, uint32_t c, uint32_t R, uint32_t& ra,
                                             uint32_t& rb) {
  ra = c == 0 ? 0u : uint32_t(q[c - 1]);
  rb = c + 1 == kQ ? R : uint32_t(q[c]);
}

template <typename E>
__device__ __forceinline__ void unpack16(const uint4& v, uint32_t (&e)[16 / sizeof(E)]) {
  if constexpr (sizeof(E) == 2) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      e[2 * i] = w[i] & 0xffffu;
      e[2 * i + 1] = w[i] >> 16;
    }
  } else {
    e[0] = v.x;
    e[1] = v.y;
    e[2] = v.z;
    e[3] = v.w;
  }
}

// Staging of completed rows, per (node, sample) pair: pair p of a warp at stage + p * pitch
// floats, row r at + r; rows [R, vpitch(R)) stay zero. pitch = 4 (mod 32) words spreads the 8 pairs
// of a warp over the banks.
__host__ __device__ __forceinline__ uint32_t stage_pitch(uint32_t R) { return (vpitch(R) + 31u) / 32u * 32u + 4u; }

// Warp write-out of the warp's np = 32 / kQ (or fewer) staged pairs to V: pair p's vpitch(R)
// floats go to V + vout_p (vout_p = the vout of lane p * kQ; 32-byte aligned) as float4 copies, so
// a warp store instruction covers whole 128-byte lines. The pair index of a float4 comes from a
// multiply-high by the reciprocal (exact for the f < 2^32 / R4 used here), not a division.
__device__ __forceinline__ void write_pairs(const float* stage, uint32_t pitch, uint32_t Rp, uint32_t np,
                                            float* V, uint64_t vout, int lane) {
  const uint32_t R4 = Rp / 4;
  const uint32_t magic = 0xffffffffu / R4 + 1u;
  constexpr uint32_t P = 32u / kQ;
  for (uint32_t f0 = 0; f0 < P * R4; f0 += 32) {  // uniform trip count (the shuffle needs all lanes)
    const uint32_t f = f0 + uint32_t(lane);
    const uint32_t p = __umulhi(f, magic);
    const uint64_t vo = __shfl_sync(0xffffffffu, vout, int(p * kQ) & 31);
    if (f >= P * R4 || p >= np) continue;
    const uint32_t r0 = 4 * (f - p * R4);
    *reinterpret_cast<float4*>(V + vo + r0) = *reinterpret_cast<const float4*>(stage + p * pitch + r0);
  }
}

// One lane's term walk: rows [r, rb) of a (node, sample) pair whose table row sits in shared memory
// at xb, entries read from `a4` (global; 16-byte vectors). Each completed row is rounded to float
// and stored to shared memory at byte address out_base + 4 * row. Terms combine exactly as the
// reference (projection.hpp:101-105): ascending feature order, the first term assigns, later
// terms add, in double, one rounding to float; empty rows come through as one zero-column entry.
// Warp-synchronous: all 32 lanes call it (a lane with nothing to do passes r == rb).
// Two register sets of four vectors ping-pong so the next four loads are in flight while the
// current four are consumed (sub-lists are followed by >= 128 readable bytes). A vector is
// consumed only while the lane still has rows to close: entries past its sub-list are neutral
// pads or another list's. `a4` points at the lane's first chunk; chunks of one list are kQ apart.
template <typename E>
__device__ __forceinline__ void walk_rows(const uint4* __restrict__ a4, const char* xb, uint32_t r,
                                          uint32_t rb, uint32_t out_base) {
  constexpr int EPV = 16 / sizeof(E);  // entries per 16-byte load
  double acc = 0.0;
  bool first = true;
  uint32_t oa = out_base + 4u * r;  // shared address of the next row to close
  const uint32_t oe = out_base + 4u * rb;
  auto consume = [&](const uint4& q) {
    if (oa >= oe) return;
    uint32_t e[EPV];
    unpack16<E>(q, e);
    uint32_t xv[EPV];
#pragma unroll
    for (int u = 0; u < EPV; ++u) xv[u] = *reinterpret_cast<const uint32_t*>(xb + (e[u] & ~3u));
#pragma unroll
    for (int u = 0; u < EPV; ++u) {
      const double dx = double(__uint_as_float(xv[u] ^ (e[u] << 31)));
      const double sum = __dadd_rn(acc, dx);
      acc = first ? dx : sum;
      first = (e[u] & 2u) != 0u;
      if (first) {
        const float v = __double2float_rn(acc);
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(oa), "f"(v) : "memory");
        oa += 4u;
      }
    }
  };
  uint4 A0 = make_uint4(0, 0, 0, 0), A1 = A0, A2 = A0, A3 = A0, B0 = A0, B1 = A0, B2 = A0, B3 = A0;
  if (oa < oe) {
    A0 = __ldg(a4);
    A1 = __ldg(a4 + kQ);
    A2 = __ldg(a4 + 2 * kQ);
    A3 = __ldg(a4 + 3 * kQ);
  }
  for (uint32_t it = 4 * kQ;; it += 8 * kQ) {
    if (!__any_sync(0xffffffffu, oa < oe)) break;
    if (oa < oe) {
      B0 = __ldg(a4 + it);
      B1 = __ldg(a4 + it + kQ);
      B2 = __ldg(a4 + it + 2 * kQ);
      B3 = __ldg(a4 + it + 3 * kQ);
    }
    consume(A0);
    consume(A1);
    consume(A2);
    consume(A3);
    if (!__any_sync(0xffffffffu, oa < oe)) break;
    if (oa < oe) {
      A0 = __ldg(a4 + it + 4 * kQ);
      A1 = __ldg(a4 + it + 5 * kQ);
      A2 = __ldg(a4 + it + 6 * kQ);
      A3 = __ldg(a4 + it + 7 * kQ);
    }
    consume(B0);
    consume(B1);
    consume(B2);
    consume(B3);
  }
}

}  // namespace dev
}  // namespace sofg
