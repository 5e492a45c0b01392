// rq_internal.cuh -- shared layout and device math of the B200 rigidq library.
//
// Layout summary:
//  * bodies are concatenated; body j owns beads [bead_off[j], bead_off[j+1])
//    and nodes [node_off[j], node_off[j+1]) with node_off[j] = 2*bead_off[j]-j;
//    node ids inside a body are the reference's postorder ids (tree.py:127-129).
//  * every internal node has a compact factor record (Householder vectors of
//    the LQ of factor.py:90-109 + taus; explicit 3x3 mixer for BEAD_BEAD).
//  * the apply path sweeps "tiles" (maximal subtrees of <= tile_leaves beads)
//    through wavefront streams of step blocks (rq_wave.cuh); the nodes above
//    the tiles form a small per-body "top tree" (TopNode / staged top blobs).
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

// Debug builds (make check -> librigidq_b200_check.so, -DRQ_DEBUG_CHECKS=1): device-side
// bounds / staging-phase asserts in the hot kernels (compute-sanitizer is unavailable on the
// GPU pool); a failed check prints its site and traps.
#ifndef RQ_DEBUG_CHECKS
#define RQ_DEBUG_CHECKS 0
#endif
#define RQ_CHECK(cond, what)                                                                        \
  do {                                                                                              \
    if (RQ_DEBUG_CHECKS && !(cond)) {                                                               \
      printf("rq check failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__,          \
             (int)blockIdx.x, (int)threadIdx.x);                                                    \
      __trap();                                                                                     \
    }                                                                                               \
  } while (0)

namespace rq {

enum NodeCase : int { LEAF = 0, BEAD_BEAD = 1, RIGID_BEAD = 2, GENERAL = 3 };

// flags byte of a node: bits 0-1 case, bit 2 swapped, bits 3-5 sign flips
// (1 = the row of omega is negated, i.e. s_i = -1; factor.py:104-108).
__host__ __device__ inline int flag_case(unsigned f) { return f & 3u; }
__host__ __device__ inline bool flag_swapped(unsigned f) { return (f >> 2) & 1u; }
__host__ __device__ inline unsigned flag_signs(unsigned f) { return (f >> 3) & 7u; }

// compact record sizes (doubles): BEAD_BEAD explicit 3x3 g; RIGID_BEAD /
// GENERAL compact-WY record (WY<6> / WY<9>) followed by the ratios a, b.
// Padded to an even count so records stay 16-byte aligned (LDS.128 / double2).
__host__ __device__ constexpr int rec_size(int c) {
  return c == BEAD_BEAD ? 10 : (c == RIGID_BEAD ? 20 : (c == GENERAL ? 30 : 0));
}
__host__ __device__ constexpr int res_rows(int c) {
  return c == RIGID_BEAD ? 3 : (c == GENERAL ? 6 : 0);
}

// ---- top trees (nodes with more than S beads) ----------------------------

struct TopNode {         // node with more than tile_leaves beads
  int32_t x, y;          // >= 0: exchange slot; < 0: ~(global tree-order bead index)
  int32_t self_slot;     // exchange slot of this node
  int32_t res_q;         // body-relative Q~ offset of its residue rows (-1 if none)
  int32_t x_top, y_top;  // 1 if the formula-x / -y child is itself a top-tree node
  int32_t body;
  uint16_t flags;
  uint16_t is_root;
  int64_t rec_off;       // offset of its record in the compact record table
};

// Per-body top-tree blob (one TMA bulk copy per body, swept in shared memory):
//   TopHdr | int32 level_begin[n_levels+1] | TopMeta[n_nodes] | int32 inputs[n_inputs] | records
struct TopHdr {          // 48 bytes
  int32_t n_nodes, n_levels, n_inputs, body;
  int32_t off_meta, off_in, off_rec, bytes;
  int32_t root_slot;     // piece blobs: exchange slot of the piece root (-1 otherwise)
  int32_t pad[3];
};
// A top tree too large for one blob is cut into PIECES (maximal subtrees of top nodes with at
// most X beads) and an APEX (its nodes with more than X beads); a piece root hands its vector
// to the apex (upward) / receives its RV-set from it (downward) through its exchange slot.
struct TopMeta {         // 16 bytes, nodes sorted by height
  int16_t x, y;          // >= 0: local top node; < 0: ~input index
  uint16_t flags;
  uint16_t is_root;      // 1: body root; 2: piece root (vector to / from the exchange slot)
  int32_t res_q;         // body-relative Q~ offset of its residue rows (-1 if none)
  int32_t rec;           // double offset of its record in the record area
};
// top-blob inputs: >= 0 exchange slot (a tile root), < 0 ~(body-local original bead index)

// Householder work layout for K in {3, 6, 9}: v0 (K-1), v1 (K-2), v2 (K-3), tau0, tau1, tau2.
template <int K>
struct HH {
  static constexpr int O0 = 0, O1 = K - 1, O2 = 2 * K - 3, OT = 3 * K - 6, SIZE = 3 * K - 3;
};

// Compact-WY record: Q = H0 H1 H2 = I - V T V^T (V unit lower trapezoidal, T
// upper triangular 3x3, LAPACK dlarft 'F','C').  omega = S Q^T.
//   V0 (K-1: rows 1..K-1) | V1 (K-2: rows 2..) | V2 (K-3: rows 3..) |
//   T00 T01 T02 T11 T12 T22 | a = sqrt(n_x/n) | b = sqrt(n_y/n)
template <int K>
struct WY {
  static constexpr int V0 = 0, V1 = K - 1, V2 = 2 * K - 3, T = 3 * K - 6;
  static constexpr int RA = 3 * K, RB = 3 * K + 1, SIZE = 3 * K + 2;
};
// NodeFactor.ratios of a BEAD_BEAD node: sqrt(1/2) (factor.py:85-87)
constexpr double BB_RATIO = 0.70710678118654757;


// ---- device math --------------------------------------------------------

// y <- (I - V T' V^T) y with T' = T (trans = false) or T^T (trans = true);
// record in the WY<K> layout, element e at rec[e * st].
template <int K, bool TRANS>
__host__ __device__ __forceinline__ void wy_apply(const double *rec, int st, double (&y)[K]) {
  using W = WY<K>;
  // w = V^T y (implicit unit diagonal), two accumulators per dot
  double w0a = y[0], w0b = 0.0, w1a = y[1], w1b = 0.0, w2a = y[2], w2b = 0.0;
#pragma unroll
  for (int j = 1; j < K; j++) {
    const double v = rec[(W::V0 + j - 1) * st];
    if (j & 1) w0b = fma(v, y[j], w0b); else w0a = fma(v, y[j], w0a);
  }
#pragma unroll
  for (int j = 2; j < K; j++) {
    const double v = rec[(W::V1 + j - 2) * st];
    if (j & 1) w1b = fma(v, y[j], w1b); else w1a = fma(v, y[j], w1a);
  }
#pragma unroll
  for (int j = 3; j < K; j++) {
    const double v = rec[(W::V2 + j - 3) * st];
    if (j & 1) w2b = fma(v, y[j], w2b); else w2a = fma(v, y[j], w2a);
  }
  const double w0 = w0a + w0b, w1 = w1a + w1b, w2 = w2a + w2b;
  const double T00 = rec[(W::T + 0) * st], T01 = rec[(W::T + 1) * st], T02 = rec[(W::T + 2) * st];
  const double T11 = rec[(W::T + 3) * st], T12 = rec[(W::T + 4) * st], T22 = rec[(W::T + 5) * st];
  double z0, z1, z2;
  if (TRANS) {  // T^T (lower)
    z0 = T00 * w0;
    z1 = fma(T01, w0, T11 * w1);
    z2 = fma(T02, w0, fma(T12, w1, T22 * w2));
  } else {      // T (upper)
    z0 = fma(T00, w0, fma(T01, w1, T02 * w2));
    z1 = fma(T11, w1, T12 * w2);
    z2 = T22 * w2;
  }
  y[0] -= z0;
  y[1] -= fma(rec[(W::V0 + 0) * st], z0, z1);
  y[2] -= fma(rec[(W::V0 + 1) * st], z0, fma(rec[(W::V1 + 0) * st], z1, z2));
#pragma unroll
  for (int j = 3; j < K; j++)
    y[j] -= fma(rec[(W::V0 + j - 1) * st], z0, fma(rec[(W::V1 + j - 2) * st], z1, rec[(W::V2 + j - 3) * st] * z2));
}

// y <- omega y = S Q^T y
template <int K>
__host__ __device__ __forceinline__ void omega_wy(const double *rec, int st, unsigned signs, double (&y)[K]) {
  wy_apply<K, true>(rec, st, y);
  if (signs & 1u) y[0] = -y[0];
  if (signs & 2u) y[1] = -y[1];
  if (signs & 4u) y[2] = -y[2];
}

// y <- omega^T y = Q S y
template <int K>
__host__ __device__ __forceinline__ void omega_t_wy(const double *rec, int st, unsigned signs, double (&y)[K]) {
  if (signs & 1u) y[0] = -y[0];
  if (signs & 2u) y[1] = -y[1];
  if (signs & 4u) y[2] = -y[2];
  wy_apply<K, false>(rec, st, y);
}

}  // namespace rq
