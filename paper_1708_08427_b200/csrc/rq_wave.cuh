// rq_wave.cuh -- layout of the wavefront apply streams (rq_wave.cu).
//
// The tile nodes of a plan (all internal nodes below the top trees) are split
// into G streams, one per persistent CTA.  Each stream is a sequence of STEPS:
// a step holds up to (CAP_G GENERAL, CAP_R RIGID_BEAD, CAP_B BEAD_BEAD) nodes
// whose children were all produced by earlier steps of the same stream (or are
// beads), so the CTA sweeps a stream with one barrier per step.  Tiles enter a
// stream staggered (a tile's height-h nodes go to step e_tile + h - 1, e_tile
// the earliest step at which all its levels fit), so the upper, sparse levels
// of one tile share steps with the dense lower levels of the next ones -- the
// steps are ~2.5x fuller than level-synchronous chunks.
//
// The upward sweep (upward_apply, matfree.py:95-121) runs the steps forward,
// the downward sweep (downward_apply, matfree.py:124-151) backward.  Every step
// is one contiguous block; each direction TMA-copies its own contiguous part:
//
//   HDR_D | DG[n_dg] | DM[n] | HDR_U | REC | UM[n] | UG[n_ug]
//   \______________ DOWN copy ______________/
//                           \_____________ UP copy ______________/
//
//   HDR    : a DirHdr (32 B) per direction: counts, section offsets within that
//            direction's copy, and where the block two steps further in that
//            direction lies (the producer issues its TMA from it: no global loads)
//   REC    : packed records, BB | RB | GEN groups (AoS, wave_rec_size doubles; GEN's odd size last)
//   UM / DM: per-node metadata of the upward / downward sweep (16 B each)
//   UG     : upward gather list of step s+2: global bead index per bead (4 B)
//   DG     : downward gather list of step s-2: residue rows / tile-root
//            RV-sets (8 B entries)
// Each stream starts and ends with two node-free steps that only carry gather
// lists, so gathers always run two steps ahead of their use.
#pragma once

#include <cstdint>

#include "rq_internal.cuh"

namespace rq {

struct StepDesc {     // 16 bytes (also the block header)
  uint32_t off16;     // block byte offset / 16 in the wave blob
  uint8_t nG, nR, nB;
  uint8_t pad0;
  uint16_t n_ug;      // upward gathers held by this block (beads of step s+2)
  uint16_t n_dg;      // downward gathers held by this block (nodes of step s-2)
  uint32_t pad1;
};

// upward metadata: x, y = M slots (internal children) or bead offsets (doubles) in the
// step's gather region (BEAD_BEAD: both, RIGID_BEAD: y); self = M slot of the
// output; row = first residue row (private residue layout, see Plan::res_base);
// aux = exchange slot (tile root) or body (body root)
struct WaveUpMeta {
  uint16_t x, y, self, flags;
  uint32_t row, aux;
};
// downward metadata: x, y = M slots (internal) or global original bead indices
// (BEAD_BEAD: both, RIGID_BEAD: y); self = M slot of the node's RV-set, or its
// offset in the gather region for tile roots; vres = offset of its residues
struct WaveDnMeta {
  uint32_t x, y;
  uint16_t self, flags, vres, pad;
};
// downward gather entry
struct WaveGather {
  uint32_t src;   // residue row / exchange slot / body
  uint16_t dst;   // double offset in the gather region (even: 16-byte copies)
  uint16_t kind;  // WG_*
};
// Gathers are 16-byte cp.async.cg copies (L2 only: the scattered rows do not pollute L1;
// two copies cover a bead instead of three).  A bead's 3 doubles sit in a 4-double window starting
// at the even row below 3b (offset b & 1); a residue run [row, row + rr) in the window
// [row & ~1, ...) of wv_pieces(row, rr) 16-byte pieces (offset row & 1).
__host__ __device__ inline int wv_pieces(int64_t row, int rr) { return (int)(((row & 1) + rr + 1) >> 1); }
enum : uint16_t { WG_RES3 = 0, WG_RES6 = 1, WG_SLOT = 2, WG_ROOT = 3 };
// meta flag bits above the node flags (bits 0-5: case | swapped | signs)
constexpr uint16_t WF_TILE_ROOT = 1u << 6;  // output to / input from an exchange slot
constexpr uint16_t WF_BODY_ROOT = 1u << 7;  // the body root (output to / input from `roots`)
constexpr uint16_t WF_BB_NEG = 1u << 8;     // BEAD_BEAD: g = -R(q) (det g = -1)
constexpr int WF_TAU_ZERO_SHIFT = 9;        // bits 9..11: reflector i of a WY record is the identity (tau_i = 0)

__host__ __device__ inline uint32_t al16u(uint32_t x) { return (x + 15u) & ~15u; }

// per-direction block header (the first 32 bytes of each direction's copy)
struct DirHdr {
  uint8_t nG, nR, nB, pad0;
  uint16_t n_list;      // gather entries (UP: beads of step s+2; DOWN: nodes of step s-2)
  uint16_t o_list;      // byte offsets inside this direction's copy
  uint16_t o_meta;
  uint16_t o_rec;
  uint16_t next_bytes;  // copy size of the block two steps further in this direction
  uint16_t pad1;
  uint32_t next_off16;  // its byte offset / 16 in the blob
  uint32_t step;        // global step index of this block (staging-phase checks)
  uint32_t round;       // round whose first tile starts at this step in this direction, ~0u if none
  uint32_t pad2;
};
static_assert(sizeof(DirHdr) == 32, "DirHdr is 32 bytes");

struct WaveSec {  // byte offsets inside a block
  uint32_t dg, dm, uhdr, rec, um, ug, end;
  // each direction's copy: [up0, end) upward, [0, dn_end) downward
  __host__ __device__ uint32_t up0() const { return uhdr; }
  __host__ __device__ uint32_t dn_end() const { return um; }
};
// Records in the step blocks are packed.  A GENERAL / RIGID_BEAD compact-WY record keeps V and
// the ratios a, b only: each reflector's tau is 2 / (v^T v) (H = I - tau v v^T is a reflection;
// dlarfg's tau = 0, H = I, is a flag bit in the node meta), and T's off-diagonal entries follow
// from V and the taus as in lq_factor (rq_lq.cuh) -- the sweep rebuilds them (~1 ulp).
// GENERAL 23 (vs 30; odd: stored after the other groups and read with 8-byte loads, whose
// 184-byte stride keeps a warp's lanes on distinct banks), RIGID_BEAD 14 (vs 20) doubles.  A BEAD_BEAD node's 3x3 g is orthogonal
// (the mixer of two beads is, factor.py:130-170), so the blocks carry it as a unit quaternion q
// (4 doubles vs 10) and a flag bit for det g = -1 (g = -R(q)); the sweep rebuilds g to ~1 ulp.
//   V0 (K-1) | V1 (K-2) | V2 (K-3) | a b [| pad]        q_w q_x q_y q_z
__host__ __device__ constexpr int wave_rec_size(int c) {
  return c == BEAD_BEAD ? 4 : (c == RIGID_BEAD ? 14 : (c == GENERAL ? 23 : 0));
}
// g (3x3 row-major, orthogonal) -> unit quaternion of s g with s = sign(det g) (Shepperd's
// method: the largest of the four squared components is taken from the diagonal)
__host__ __device__ inline bool wave_pack_bb(const double *g, double *q) {
  const double det = g[0] * (g[4] * g[8] - g[5] * g[7]) - g[1] * (g[3] * g[8] - g[5] * g[6]) +
                     g[2] * (g[3] * g[7] - g[4] * g[6]);
  const double sg = det < 0.0 ? -1.0 : 1.0;
  double M[9];
  for (int e = 0; e < 9; e++) M[e] = sg * g[e];
  const double tr = M[0] + M[4] + M[8];
  double w, x, y, z;
  if (tr > 0.0) {
    const double s = 2.0 * sqrt(tr + 1.0);
    w = 0.25 * s; x = (M[7] - M[5]) / s; y = (M[2] - M[6]) / s; z = (M[3] - M[1]) / s;
  } else if (M[0] > M[4] && M[0] > M[8]) {
    const double s = 2.0 * sqrt(1.0 + M[0] - M[4] - M[8]);
    w = (M[7] - M[5]) / s; x = 0.25 * s; y = (M[1] + M[3]) / s; z = (M[2] + M[6]) / s;
  } else if (M[4] > M[8]) {
    const double s = 2.0 * sqrt(1.0 + M[4] - M[0] - M[8]);
    w = (M[2] - M[6]) / s; x = (M[1] + M[3]) / s; y = 0.25 * s; z = (M[5] + M[7]) / s;
  } else {
    const double s = 2.0 * sqrt(1.0 + M[8] - M[0] - M[4]);
    w = (M[3] - M[1]) / s; x = (M[2] + M[6]) / s; y = (M[5] + M[7]) / s; z = 0.25 * s;
  }
  const double nrm = sqrt(w * w + x * x + y * y + z * z);
  q[0] = w / nrm; q[1] = x / nrm; q[2] = y / nrm; q[3] = z / nrm;
  return det < 0.0;
}
// unit quaternion -> rotation (row-major), negated when neg
__host__ __device__ inline void wave_unpack_bb(const double *q, bool neg, double *g) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  const double s = neg ? -2.0 : 2.0, one = neg ? -1.0 : 1.0;
  g[0] = one - s * (y * y + z * z); g[1] = s * (x * y - w * z);       g[2] = s * (x * z + w * y);
  g[3] = s * (x * y + w * z);       g[4] = one - s * (x * x + z * z); g[5] = s * (y * z - w * x);
  g[6] = s * (x * z - w * y);       g[7] = s * (y * z + w * x);       g[8] = one - s * (x * x + y * y);
}
__host__ __device__ inline uint32_t wave_rec_bytes(uint32_t nG, uint32_t nR, uint32_t nB) {
  // 16-byte multiple: the sections after it (and the TMA copy sizes) stay 16-byte aligned
  return al16u(8u * (wave_rec_size(GENERAL) * nG + wave_rec_size(RIGID_BEAD) * nR + wave_rec_size(BEAD_BEAD) * nB));
}
// compact-WY record (WY<K> layout, T upper part + ratios) -> packed wave record; returns the
// tau = 0 mask (bit i: reflector i is the identity)
template <int K>
__host__ __device__ inline unsigned wave_pack_wy(const double *src, double *dst) {
  using W = WY<K>;
  for (int e = 0; e < W::T; e++) dst[e] = src[e];  // V
  dst[W::T + 0] = src[W::RA];
  dst[W::T + 1] = src[W::RB];
  return (src[W::T + 0] == 0.0 ? 1u : 0u) | (src[W::T + 3] == 0.0 ? 2u : 0u) | (src[W::T + 5] == 0.0 ? 4u : 0u);
}
__host__ __device__ inline WaveSec wave_sections(uint32_t nG, uint32_t nR, uint32_t nB, uint32_t n_ug,
                                                 uint32_t n_dg) {
  const uint32_t n = nG + nR + nB;
  WaveSec s;
  s.dg = 32u;
  s.dm = s.dg + al16u(8u * n_dg);
  s.uhdr = s.dm + 16u * n;
  s.rec = s.uhdr + 32u;
  s.um = s.rec + wave_rec_bytes(nG, nR, nB);
  s.ug = s.um + 16u * n;
  s.end = s.ug + al16u(4u * n_ug);
  return s;
}
__host__ __device__ inline WaveSec wave_sections(const StepDesc &d) {
  return wave_sections(d.nG, d.nR, d.nB, d.n_ug, d.n_dg);
}

// per-step capacities (the scheduler never exceeds them; they size shared memory)
struct WaveCaps {
  int g = 48, r = 48, b = 64;   // nodes per case (swept on config 2)
  int rm = 12288;               // record + one-direction metadata bytes
  int beads = 128;              // upward gathers (beads) per step
  int vd = 512;                 // downward gather-region doubles per step
  int dg = 96;                  // downward gather entries per step
};

}  // namespace rq
