// rq_internal.cuh -- shared layout and device math of the B200 rigidq library.
//
// Layout summary:
//  * bodies are concatenated; body j owns beads [bead_off[j], bead_off[j+1])
//    and nodes [node_off[j], node_off[j+1]) with node_off[j] = 2*bead_off[j]-j;
//    node ids inside a body are the reference's postorder ids (tree.py:127-129).
//  * every internal node has a compact factor record (Householder vectors of
//    the LQ of factor.py:90-109 + taus; explicit 3x3 mixer for BEAD_BEAD).
//  * the apply path streams "chunks": forests of maximal subtrees ("tiles")
//    of <= tile_leaves beads, whose records are re-packed level-major and
//    struct-of-arrays into one contiguous, 16-byte aligned blob per chunk.
//    Nodes above the tiles form a small per-body "top tree".
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace rq {

enum NodeCase : int { LEAF = 0, BEAD_BEAD = 1, RIGID_BEAD = 2, GENERAL = 3 };

// flags byte of a node: bits 0-1 case, bit 2 swapped, bits 3-5 sign flips
// (1 = the row of omega is negated, i.e. s_i = -1; factor.py:104-108).
__host__ __device__ inline int flag_case(unsigned f) { return f & 3u; }
__host__ __device__ inline bool flag_swapped(unsigned f) { return (f >> 2) & 1u; }
__host__ __device__ inline unsigned flag_signs(unsigned f) { return (f >> 3) & 7u; }

// compact record sizes (doubles): BEAD_BEAD explicit 3x3 g; RIGID_BEAD /
// GENERAL Householder record (HH<6> / HH<9>) followed by the ratios a, b.
// Padded to an even count so records stay 16-byte aligned (LDS.128 / double2).
__host__ __device__ constexpr int rec_size(int c) {
  return c == BEAD_BEAD ? 10 : (c == RIGID_BEAD ? 18 : (c == GENERAL ? 26 : 0));
}
__host__ __device__ constexpr int res_rows(int c) {
  return c == RIGID_BEAD ? 3 : (c == GENERAL ? 6 : 0);
}

// ---- apply layout -------------------------------------------------------

struct LevelDesc {       // one height level of a chunk, 32 bytes
  int32_t slot_begin;    // first chunk-local slot of the level
  int32_t nG, nR, nB;    // nodes per case (slots ordered GEN, RB, BB)
  int32_t recG, recR, recB;  // double offsets of the per-case record groups (AoS, rec_size stride)
  int32_t pad;
};

struct NodeMeta {        // 8 bytes, one per in-chunk internal node (slot order)
  uint16_t x, y;         // formula-x/-y child: bit 15 set -> bead (local index), else slot
  uint16_t res;          // residue offset in the chunk staging buffer
  uint16_t flags;        // case | swapped | signs
};

// Chunk blob layout (16-byte aligned sections):
//   ChunkDesc (64 B) | TileDesc[n_tiles] | LevelDesc[n_levels] | NodeMeta[n_nodes] | perm[n_beads] | records
struct ChunkDesc {
  int64_t blob_off;      // byte offset of the blob (16-byte aligned)
  int32_t blob_bytes;    // multiple of 16
  int32_t n_nodes;
  int32_t n_beads;       // local bead window [bead_begin, bead_begin+n_beads) in tree order
  int32_t n_levels;
  int32_t n_tiles;
  int32_t body;
  int64_t bead_begin;    // global tree-order bead index of local bead 0
  int64_t tile_begin;    // first TileDesc
  int32_t off_meta;      // byte offsets inside the blob
  int32_t off_perm;
  int32_t off_rec;
  int32_t n_res;         // residue doubles staged
};

struct TileDesc {        // 32 bytes; copies live in the chunk blob after the ChunkDesc header
  int32_t root_slot;     // chunk-local slot of the tile root
  int32_t scratch;       // exchange slot with the top tree, -1 if the tile root is the body root
  int32_t res_q;         // body-relative complement (Q~) offset of the tile's first residue
  int32_t res_count;     // 3L - 6
  int32_t res_local;     // offset in the chunk staging buffer
  int32_t pad[3];
};

struct TopNode {         // node with more than tile_leaves beads
  int32_t x, y;          // >= 0: exchange slot; < 0: ~(global tree-order bead index)
  int32_t self_slot;     // exchange slot of this node
  int32_t res_q;         // body-relative Q~ offset of its residue rows (-1 if none)
  int32_t nx, ny;
  int32_t body;
  uint16_t flags;
  uint16_t is_root;
  int64_t rec_off;       // offset of its record in the compact record table
};

// perm entries in a chunk blob: body-local original bead index, or
// (PERM_FOREIGN | idx) for beads handled by the top tree (singleton tiles).
constexpr uint32_t PERM_FOREIGN = 0x80000000u;
constexpr uint16_t SRC_BEAD = 0x8000u;

// ---- device math --------------------------------------------------------

// Apply H_i = I - tau v v^T (v[i] = 1 implicit, v[j<i] = 0) to y (length K).
template <int K>
__host__ __device__ __forceinline__ void householder(double (&y)[K], const double* vi, double tau, int i) {
  double d = y[i];
#pragma unroll
  for (int j = i + 1; j < K; j++) d += vi[j - i - 1] * y[j];
  double td = tau * d;
  y[i] -= td;
#pragma unroll
  for (int j = i + 1; j < K; j++) y[j] -= td * vi[j - i - 1];
}

// Record layout for K in {6, 9}: v0 (K-1), v1 (K-2), v2 (K-3), tau0, tau1, tau2.
template <int K>
struct HH {
  static constexpr int O0 = 0, O1 = K - 1, O2 = 2 * K - 3, OT = 3 * K - 6, SIZE = 3 * K - 3;
  static constexpr int RA = SIZE, RB = SIZE + 1;  // ratios a = sqrt(n_x/n), b = sqrt(n_y/n)
};
// NodeFactor.ratios of a BEAD_BEAD node: sqrt(1/2) (factor.py:85-87)
constexpr double BB_RATIO = 0.70710678118654757;

}  // namespace rq
