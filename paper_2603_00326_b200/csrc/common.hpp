// Plain descriptors shared by the host frontier scheduler and the sm_100a kernels.
//
// A "wave" is one launch sequence over a set of open tree nodes (all open nodes of one depth
// across a batch of trees, or the retry attempts of that depth). The reference grows one node at
// a time (detail::TreeGrower::grow_from, reference forest.hpp:157-240); here every node of a
// depth is one entry of a NodeIn array and every kernel walks that array.
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define SOFG_HD __host__ __device__
#else
#define SOFG_HD
#endif

namespace sofg {

constexpr int kMaxClasses = 8;       // class counts carried inline (NodeRes, host frontier, register kernels)
constexpr int kMaxClassesWide = 64;  // class_count supported (above kMaxClasses: wide.cu, side arrays)
constexpr int kMaxBins = 8192;       // bin_count supported by the histogram splitter (> 1024: CTA boundaries, wide.cu counts)
constexpr int kExactSmemMax = 2048;  // largest node the shared-memory exact splitter sorts
constexpr int kTileElems = 1024;     // partition tile
constexpr int kWinTermsMax = 8;      // winning-row terms returned inline per node (longer rows: k_win_terms)
constexpr int kHistRowsPerCta = 8;   // rows (one per warp) per histogram CTA
constexpr uint64_t kFallbackBreakeven = 1024;  // reference calibrate.hpp:43

enum NodeFlags : uint32_t {
  kNodeHist = 1u,         // histogram method (else exact), split.hpp:46-48
  kNodeGivenCsr = 2u,     // projection matrix supplied by the host (primitive entry points)
};

// One open node of a wave (host-written, device-read).
struct NodeIn {
  uint64_t seed;       // node seed: engine = mt19937_64(split_mix64(seed))   (forest.hpp:183)
  uint32_t begin;      // first element of the node's segment in the idx/label arrays
  uint32_t n;          // active samples
  uint32_t z;          // total projection nonzeros (binomial draw, projection.hpp:66-67)
  uint32_t pos;        // engine outputs consumed before the Floyd cell draws
  uint32_t flags;      // NodeFlags
  uint32_t term_off;   // first term of this node's CSR in the wave's term array
  uint32_t hist_slot;  // index among the wave's histogram nodes (hist only)
  uint32_t tree;       // batch-local tree (diagnostics)
  double parent;       // entropy of the node's class counts (host, split.hpp:20-31)
};
static_assert(sizeof(NodeIn) == 48, "NodeIn layout");

// Per-node result of a wave (device-written).
struct NodeRes {
  double gain;           // best information gain (bits)
  int32_t row;           // winning projection row, -1 when no positive-gain split exists
  float threshold;       // split threshold (left iff value <= threshold, forest.hpp:205)
  uint32_t n_left_search;  // n_left reported by the split search (split.hpp:115,167)
  uint32_t n_left;       // left count of the partition (v <= thr)
  uint32_t pos_after;    // engine outputs consumed by this attempt (projection + picks)
  uint32_t n_terms;      // winning row term count
  uint32_t sectors;      // distinct 32 B sectors of the node's sample ids (stats only)
  uint32_t _pad;
  uint32_t terms[kWinTermsMax];  // winning row terms: feature << 1 | (weight < 0)
};
// The partition's left class counts travel in a separate [node][k] array (k_part_flags), so the
// per-wave device-to-host copy is 72 + 4 k bytes per node.
static_assert(sizeof(NodeRes) == 72, "NodeRes layout");

// Per-(histogram node, row) search result.
struct RowRes {
  double gain;
  float threshold;
  uint32_t n_left;
  int32_t valid;
  int32_t _pad;
};

// Histogram work item: one CTA counts `len` elements of node `node` for rows
// [row0, row0 + kHistRowsPerCta).
struct HistWork {
  uint32_t node;   // wave node index
  uint32_t row0;
  uint32_t start;  // offset inside the node segment
  uint32_t len;
  uint32_t chunk;  // chunk index within (node,row group)
  uint32_t n_chunks;
};

// Partition tile: elements [start, start+len) of node `node`'s segment.
struct Tile {
  uint32_t node;
  uint32_t start;
  uint32_t len;
  uint32_t tile_in_node;
};

// Row pitch of the wave's projected-value block V (sample j of node i at V[vbase[i] + j*Rp]):
// R rounded up to 8 rows so 8 consecutive rows of a sample are one aligned 32-byte sector.
SOFG_HD inline uint32_t vpitch(uint32_t R) { return (R + 7u) & ~7u; }

// Term encoding: feature index in the high 31 bits, sign in bit 0 (1 = weight -1).
SOFG_HD inline uint32_t encode_term(uint32_t feature, bool negative) {
  return (feature << 1) | (negative ? 1u : 0u);
}

}  // namespace sofg
