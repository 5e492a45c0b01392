// rq_wave.cu -- wavefront apply streams: layout builder and sweep kernel.
//
// Restates the tile part of upward_apply (Algorithm 2, matfree.py:95-121,
// merge_infosets matfree.py:41-62) and downward_apply (Algorithm 3,
// matfree.py:124-151, split_rvset matfree.py:65-83).  The nodes above the
// tiles (per-body top trees) stay with k_top2 / k_top_df (rq_apply.cu).
//
// Layout (rq_wave.cuh): the tiles (maximal subtrees with <= S beads, in body
// order) are split into G contiguous streams of about equal node count, one
// per persistent CTA.  Inside a stream the tiles are placed greedily: tile t
// enters at the earliest step e_t >= e_{t-1} at which every one of its height
// levels fits the per-step capacities (WaveCaps), and its height-h nodes run at
// step e_t + h - 1.  Every node's children therefore run at earlier steps.
// Each node's 6-vector (upward output / downward RV-set) lives in one of M
// shared-memory slots from its producer's step to its consumer's step; the
// slots are assigned per stream by interval colouring (lowest free slot),
// which is optimal for interval graphs, so M = the stream's peak live count.
//
// Kernel k_wave<UP> (128 threads, one CTA per stream): per step, one TMA bulk
// copy of the block (issued two steps ahead into a 2-stage ring; each block's
// header locates the block two steps further, so the producer never waits on a
// global load), gathers for step +2 (cp.async into a 3-region ring), the
// case-uniform node pass (GENERAL, RIGID_BEAD and BEAD_BEAD nodes each padded
// to whole warps), one CTA barrier.  Outputs go straight to global memory
// (residues upward, bead velocities downward); tile-root 6-vectors go to the
// exchange slots the top-tree kernels read.  No tensor cores: HBM-bound sweep
// of tiny fp64 orthogonal transforms.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "rq_nodeops.cuh"
#include "rq_plan.hpp"
#include "rq_wave.cuh"

namespace rq {
namespace {

constexpr int NT = 256;
inline size_t al128(size_t x) { return (x + 127) / 128 * 128; }
inline unsigned nblk(int64_t n, int t = NT) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

template <class In, class Out>
void ex_scan(const In *in, Out *out, int64_t n, cudaStream_t s) {
  if (n <= 0) return;
  size_t tb = 0;
  RQ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, s));
  DBuf tmp;
  tmp.alloc(tb);
  RQ_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, n, s));
}
template <class T>
void d2h(T *dst, const void *src, size_t count, cudaStream_t s) {
  RQ_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToHost, s));
  RQ_CUDA(cudaStreamSynchronize(s));
}
template <class T>
T d2h1(const void *src, cudaStream_t s) {
  T v;
  d2h(&v, src, 1, s);
  return v;
}

// ---- builder ---------------------------------------------------------------------

struct TLev {  // one height level of a tile (its requirements on a step)
  int16_t g, r, b, beads, vd, dg;
  int32_t rm;
};

struct NodeArrays {
  const int64_t *node_off, *bead_off, *rec_off, *res_base;
  const int32_t *node_body, *start, *stop, *left, *right, *parent, *height, *res_off, *perm, *slot_scan;
  const uint8_t *flags;
};

__device__ __forceinline__ int nodeL(const NodeArrays &A, int64_t g) { return A.stop[g] - A.start[g]; }

// per tile: internal node count and height (0 for singleton tiles)
__global__ void k_wv_tiles(const int64_t *tile_root, int64_t nt, NodeArrays A, int64_t *tnodes, int64_t *theight) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nt) return;
  const int64_t g = tile_root[t];
  const int L = nodeL(A, g);
  tnodes[t] = L >= 2 ? L - 1 : 0;
  theight[t] = L >= 2 ? A.height[g] : 0;
}

__device__ __forceinline__ int wv_rank(int cs) { return cs == GENERAL ? 0 : (cs == RIGID_BEAD ? 1 : 2); }
__device__ __forceinline__ int wv_beads(int cs) { return cs == BEAD_BEAD ? 2 : (cs == RIGID_BEAD ? 1 : 0); }

// node -> tile map (tile-internal nodes only)
__global__ void k_wv_node_tile(const int64_t *tile_root, int64_t nt, NodeArrays A, int32_t *node_tile) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nt) return;
  const int64_t g = tile_root[t];
  const int L = nodeL(A, g);
  if (L < 2) return;
  for (int64_t q = g - 2 * (int64_t)L + 2; q <= g; q++)
    if (nodeL(A, q) >= 2) node_tile[q] = (int32_t)t;
}

// Stream of each tile.  The tile list (body order) is cut into R rounds of equal node count
// and every round into G contiguous ranges; stream c takes range c of every round, round
// after round.  All CTAs therefore work inside the same round at any time, so the vector
// rows of the bodies in flight (gathers, scattered outputs) stay L2-resident while their
// 32-byte sectors are shared by neighbouring beads.
// tile -> (stream, round): rounds split the node scan evenly; within a round stream c takes
// range c -- evenly, or for rounds >= R0 by the cumulative weights W (G + 1 entries, W[0] = 0,
// W[G] = 1) of the second placement pass (build_wave's tail rebalancing)
__global__ void k_wv_tile_key(const int64_t *node_scan, int64_t nt, int64_t total, int64_t G, int64_t R,
                              const double *W, int64_t R0, uint64_t *key, int32_t *val) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nt) return;
  const double x = (double)node_scan[t] / (double)std::max<int64_t>(total, 1) * (double)R;  // in [0, R)
  const int64_t r = std::min<int64_t>(R - 1, (int64_t)x);
  int64_t c;
  if (W != nullptr && r >= R0) {
    const double f = x - (double)r;
    int64_t lo = 0, hi = G;  // last c with W[c] <= f
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (W[mid] <= f) lo = mid;
      else hi = mid;
    }
    c = lo;
  } else {
    c = std::min<int64_t>(G - 1, (int64_t)((x - (double)r) * (double)G));
  }
  key[t] = (uint64_t)(c * R + r);
  val[t] = (int32_t)t;
}
__global__ void k_wv_stream_first(const uint64_t *key, int64_t nt, int64_t R, int64_t *first) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nt) return;
  const int64_t c = (int64_t)(key[i] / R), cp = i == 0 ? -1 : (int64_t)(key[i - 1] / R);
  for (int64_t x = cp + 1; x <= c; x++) first[x] = i;  // streams (cp, c] start at sorted tile i
}
__global__ void k_wv_gather64(const int64_t *src, const int32_t *order, int64_t n, int64_t *dst) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[order[i]];
}

__device__ __forceinline__ bool wv_fits(const TLev &l, const TLev &v, const WaveCaps &c) {
  return l.g + v.g <= c.g && l.r + v.r <= c.r && l.b + v.b <= c.b && l.beads + v.beads <= c.beads &&
         l.vd + v.vd <= c.vd && l.dg + v.dg <= c.dg && l.rm + v.rm <= c.rm;
}

// Node-level list scheduling, one warp per stream: the stream's tiles in order, each tile's
// nodes in postorder; a node goes to the earliest step after its children's (and not before
// the floor = the first step of the previous tile) with room for it.  Any node shape fits (no
// rigid tile rows), so tiles can be large and the top trees small.  The step loads live in a
// shared-memory ring of WRING steps ahead of the floor.  The greedy choice is serial (lane
// 0), but the warp first stages each chunk of WV_CH tile nodes -- their step requirements
// and tile-local child indices -- in shared memory with coalesced loads, so the serial loop
// never waits on a global load (one dependent L2 round trip per node otherwise: 12 -> ~1 ms
// per pass on config 2).  A tile is a contiguous postorder range, so its children's steps
// sit in a tile-local array.
constexpr int WRING = 1024;
constexpr int WV_CH = 256;
constexpr int WV_MAXT = 2048;  // nodes of the largest tile (tile_leaves <= 1024)
__global__ void __launch_bounds__(32) k_wv_place_nodes(const int64_t *sfirst, int64_t G, const int32_t *order,
                                                      const int64_t *tile_root, NodeArrays A, WaveCaps caps,
                                                      int32_t *node_step, int64_t *n_steps, int32_t *tile_first,
                                                      int32_t *tile_last, const int32_t *tile_round, int R0,
                                                      int64_t *round_floor, int *bad, int mode, TLev *save_ring,
                                                      int32_t *save_state) {
  __shared__ TLev ring[WRING];
  __shared__ TLev cv[WV_CH];
  __shared__ int16_t clc[WV_CH], crc[WV_CH];  // tile-local children (-1: a bead; clc -2: node skipped)
  __shared__ int32_t lstep[WV_MAXT];
  const int64_t c = blockIdx.x;
  const int lane = threadIdx.x;
  if (c >= G) return;
  for (int i = lane; i < WRING; i += 32) ring[i] = TLev{};
  __syncwarp();
  int floor = 0, last = 0;  // uniform across the warp
  bool seen = false;
  // mode 1 saves the stream's state (step loads, floor, last) where it enters the tail rounds
  // (>= R0); mode 2 (the rebalancing pass: same tiles, same order and same steps before the
  // tail) restores it and places the tail tiles only
  auto save = [&]() {
    for (int k = lane; k < WRING; k += 32) save_ring[c * WRING + k] = ring[k];
    if (lane == 0) { save_state[2 * c] = floor; save_state[2 * c + 1] = last; }
  };
  if (mode == 2) {
    for (int k = lane; k < WRING; k += 32) ring[k] = save_ring[c * WRING + k];
    floor = save_state[2 * c];
    last = save_state[2 * c + 1];
    seen = true;
    __syncwarp();
  }
  for (int64_t i = sfirst[c]; i < sfirst[c + 1]; i++) {
    const int64_t t = order[i];
    const bool tail = tile_round[t] >= R0;
    if (mode == 2 && !tail) continue;
    if (!seen && tail) {  // where this stream enters the rebalanced tail rounds
      if (lane == 0) round_floor[c] = floor;
      if (mode == 1) save();
      seen = true;
    }
    const int64_t g = tile_root[t];
    const int L = nodeL(A, g);
    if (L < 2) continue;
    const int j = A.node_body[g];
    const int64_t nb = A.node_off[j];
    const int64_t rb = A.res_base[j];
    const int64_t q0 = g - 2 * (int64_t)L + 2;
    const int cnt = (int)(g - q0 + 1);
    if (cnt > WV_MAXT) {
      if (lane == 0) atomicExch(bad, 1);
      return;
    }
    int tmin = INT32_MAX, tmax = 0;
    for (int base = 0; base < cnt; base += WV_CH) {
      const int nch = min(WV_CH, cnt - base);
      for (int e = lane; e < nch; e += 32) {
        const int64_t q = q0 + base + e;
        if (nodeL(A, q) < 2) { clc[e] = -2; continue; }
        const int64_t lc = nb + A.left[q], rc = nb + A.right[q];
        clc[e] = nodeL(A, lc) >= 2 ? (int16_t)(lc - q0) : (int16_t)-1;
        crc[e] = nodeL(A, rc) >= 2 ? (int16_t)(rc - q0) : (int16_t)-1;
        const int cs = flag_case(A.flags[q]);
        const int root = q == g, rr = res_rows(cs);
        TLev v{};
        if (cs == GENERAL) v.g = 1;
        else if (cs == RIGID_BEAD) v.r = 1;
        else v.b = 1;
        v.beads = (int16_t)wv_beads(cs);
        v.vd = (int16_t)((rr ? 2 * wv_pieces(rb + A.res_off[q] - 6, rr) : 0) + 6 * root);
        v.dg = (int16_t)((rr > 0) + root);
        v.rm = 8 * wave_rec_size(cs) + 16;
        cv[e] = v;
      }
      __syncwarp();
      // every lane runs the (uniform) greedy loop; the step search tests 32 steps at once
      for (int e = 0; e < nch; e++) {
        if (clc[e] == -2) continue;
        int ready = floor;
        if (clc[e] >= 0) ready = max(ready, lstep[clc[e]] + 1);
        if (crc[e] >= 0) ready = max(ready, lstep[crc[e]] + 1);
        const TLev v = cv[e];
        int st = -1;
        for (int sb = ready;; sb += 32) {
          const int cand = sb + lane;
          const bool ok = cand - floor < WRING && wv_fits(ring[cand % WRING], v, caps);
          const unsigned m = __ballot_sync(0xffffffffu, ok);
          if (m) { st = sb + __ffs(m) - 1; break; }
          if (sb + 32 - floor >= WRING) break;  // the earliest step with room is out of the window
        }
        if (st < 0) {
          if (lane == 0) atomicExch(bad, 1);
          return;
        }
        if (lane == 0) {
          TLev &l = ring[st % WRING];
          l.g += v.g; l.r += v.r; l.b += v.b; l.beads += v.beads; l.vd += v.vd; l.dg += v.dg; l.rm += v.rm;
          lstep[base + e] = st;
        }
        tmin = min(tmin, st);
        tmax = max(tmax, st);
        last = max(last, st + 1);
        __syncwarp();
      }
      for (int e = lane; e < nch; e += 32)
        if (clc[e] != -2) node_step[q0 + base + e] = lstep[base + e];
      __syncwarp();
    }
    if (lane == 0) {
      tile_first[t] = tmin;
      tile_last[t] = tmax;
    }
    for (int f = floor + lane; f < tmin; f += 32) ring[f % WRING] = TLev{};  // steps no later tile can use
    floor = max(floor, tmin);
    __syncwarp();
  }
  if (!seen && mode == 1) save();
  if (lane == 0) {
    if (!seen) round_floor[c] = last;
    n_steps[c] = last + 4;  // two gather-only steps at each end
  }
}

// sort key of every tile node: (global step, case rank)
__global__ void k_wv_keys(int64_t NN, NodeArrays A, const int32_t *node_tile, const int32_t *node_step,
                          const int64_t *step_first, uint64_t *keys, int32_t *vals, const int32_t *tile_stream) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= NN) return;
  uint64_t key = ~0ull;
  const int32_t t = node_tile[g];
  if (t >= 0) {
    const int64_t c = tile_stream[t];
    const int64_t gs = step_first[c] + 2 + node_step[g];
    key = ((uint64_t)gs << 2) | (uint64_t)wv_rank(flag_case(A.flags[g]));
  }
  keys[g] = key;
  vals[g] = (int32_t)g;
}

__global__ void k_wv_tile_stream(const uint64_t *key, const int32_t *order, int64_t nt, int64_t R, int32_t *tile_stream,
                                 int32_t *tile_round) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nt) return;
  tile_stream[order[i]] = (int32_t)(key[i] / R);
  tile_round[order[i]] = (int32_t)(key[i] % R);
}

// per step and direction: the round of the tiles that start there (upward: entry row;
// downward: last row), for the run-time round window (k_wave throttles CTAs that run ahead)
__global__ void k_wv_round_marks(int64_t nt, const int64_t *tnodes, const int32_t *tile_stream, const int32_t *tile_round,
                                 const int32_t *tile_first, const int32_t *tile_last, const int64_t *step_first,
                                 int *up_mark, int *dn_mark) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nt || tnodes[t] == 0) return;
  const int64_t base = step_first[tile_stream[t]] + 2;
  atomicMax(&up_mark[base + tile_first[t]], tile_round[t]);
  atomicMin(&dn_mark[base + tile_last[t]], tile_round[t]);
}

struct StepCnt {
  int32_t g, r, b, ug, dg;
};

// per sorted node: step counts, list counts, step of the node, per-node list sizes
__global__ void k_wv_count(const uint64_t *keys, const int32_t *vals, int64_t n, NodeArrays A, StepCnt *sc,
                           int64_t *step_of, int64_t *sfirst_sorted, int32_t *nb, int32_t *vd, int32_t *nd,
                           const int32_t *node_tile, const int64_t *tile_root) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int64_t gs = (int64_t)(keys[p] >> 2);
  const int64_t g = vals[p];
  const int cs = flag_case(A.flags[g]);
  if (cs == GENERAL) atomicAdd(&sc[gs].g, 1);
  else if (cs == RIGID_BEAD) atomicAdd(&sc[gs].r, 1);
  else atomicAdd(&sc[gs].b, 1);
  const int root = tile_root[node_tile[g]] == g;
  const int beads = wv_beads(cs), dge = (res_rows(cs) > 0) + root;
  if (beads) atomicAdd(&sc[gs - 2].ug, beads);
  if (dge) atomicAdd(&sc[gs + 2].dg, dge);
  step_of[g] = gs;
  if (p == 0 || (int64_t)(keys[p - 1] >> 2) != gs) sfirst_sorted[gs] = p;
  nb[p] = beads;
  const int rr = res_rows(cs);
  vd[p] = (rr ? 2 * wv_pieces(A.res_base[A.node_body[g]] + A.res_off[g] - 6, rr) : 0) + 6 * root;
  nd[p] = dge;
}

__global__ void k_wv_step_bytes(const StepCnt *sc, int64_t ns, int64_t *bytes, unsigned long long *mx) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= ns) return;
  const StepCnt c = sc[s];
  const WaveSec S = wave_sections(c.g, c.r, c.b, c.ug, c.dg);
  bytes[s] = S.end;
  atomicMax(&mx[0], (unsigned long long)(S.end - S.uhdr));  // upward copy
  atomicMax(&mx[1], (unsigned long long)S.um);              // downward copy
}

__global__ void k_wv_descs(const StepCnt *sc, const int64_t *off, int64_t ns, StepDesc *d, uint8_t *blob) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= ns) return;
  const StepCnt c = sc[s];
  StepDesc D;
  D.off16 = (uint32_t)(off[s] >> 4);
  D.nG = (uint8_t)c.g; D.nR = (uint8_t)c.r; D.nB = (uint8_t)c.b;
  D.n_ug = (uint16_t)c.ug; D.n_dg = (uint16_t)c.dg;
  D.pad0 = 0;
  D.pad1 = 0;
  d[s] = D;
}

// the two direction headers of every block (after all descriptors exist)
__global__ void k_wv_headers(const StepDesc *d, int64_t ns, uint8_t *blob, const int *up_mark, const int *dn_mark) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= ns) return;
  const StepDesc D = d[s];
  const WaveSec S = wave_sections(D);
  uint8_t *B = blob + ((int64_t)D.off16 << 4);
  DirHdr u{}, w{};
  u.step = w.step = (uint32_t)s;
  u.round = up_mark[s] >= 0 ? (uint32_t)up_mark[s] : ~0u;
  w.round = dn_mark[s] != INT32_MAX ? (uint32_t)dn_mark[s] : ~0u;
  u.nG = w.nG = D.nG;
  u.nR = w.nR = D.nR;
  u.nB = w.nB = D.nB;
  // upward copy [uhdr, end): header | records | metadata | bead list
  u.n_list = D.n_ug;
  u.o_rec = (uint16_t)(S.rec - S.uhdr);
  u.o_meta = (uint16_t)(S.um - S.uhdr);
  u.o_list = (uint16_t)(S.ug - S.uhdr);
  u.next_off16 = 0xffffffffu;
  if (s + 2 < ns) {
    const WaveSec N = wave_sections(d[s + 2]);
    u.next_off16 = (uint32_t)(((((int64_t)d[s + 2].off16) << 4) + N.uhdr) >> 4);
    u.next_bytes = (uint16_t)(N.end - N.uhdr);
  }
  // downward copy [0, um): header | gather list | metadata | (upward header) | records
  w.n_list = D.n_dg;
  w.o_list = (uint16_t)S.dg;
  w.o_meta = (uint16_t)S.dm;
  w.o_rec = (uint16_t)S.rec;
  w.next_off16 = 0xffffffffu;
  if (s >= 2) {
    const WaveSec N = wave_sections(d[s - 2]);
    w.next_off16 = d[s - 2].off16;
    w.next_bytes = (uint16_t)N.um;
  }
  *reinterpret_cast<DirHdr *>(B) = w;
  *reinterpret_cast<DirHdr *>(B + S.uhdr) = u;
}

// one warp per stream: interval colouring of the node 6-vectors (lowest free slot; optimal
// for interval graphs, so the slot count is the stream's peak live count).  The free set is a
// 1024-bit mask, one 32-bit word per lane, so the lowest free slot is a ballot + ffs; a slot
// is released once the step of its consumer (the parent) has passed, checked by every lane
// over its word when the step advances.  The warp stages each chunk of WV_CH nodes' (step,
// release step) pairs first, so the loop never waits on the dependent global loads (node ->
// tile -> root, node -> body -> parent -> step) of a node.
constexpr int WV_MAX_SLOTS = 1024;
__global__ void __launch_bounds__(32) k_wv_slots(const int64_t *node_first, int64_t G, const int32_t *vals,
                                                NodeArrays A, const int64_t *step_of, const int32_t *node_tile,
                                                const int64_t *tile_root, int32_t *slot_of, int *max_slots,
                                                int *overflow) {
  const int64_t c = blockIdx.x;
  const int lane = threadIdx.x;
  if (c >= G) return;
  __shared__ int64_t rel[WV_MAX_SLOTS];            // release step of a busy slot
  __shared__ int64_t cstep[WV_CH], crel[WV_CH];  // crel < 0: tile root (no slot)
  __shared__ int32_t cslot[WV_CH];
  uint32_t freew = 0xffffffffu;  // slots 32 lane .. 32 lane + 31
  int64_t cur = -1;
  int next = 0;  // 1 + the highest slot used
  for (int64_t p0 = node_first[c]; p0 < node_first[c + 1]; p0 += WV_CH) {
    const int64_t rem = node_first[c + 1] - p0;
    const int nch = rem < WV_CH ? (int)rem : WV_CH;
    for (int e = lane; e < nch; e += 32) {
      const int64_t g = vals[p0 + e];
      if (tile_root[node_tile[g]] == g) {  // tile roots exchange through global memory
        crel[e] = -1;
        continue;
      }
      cstep[e] = step_of[g];
      crel[e] = step_of[A.node_off[A.node_body[g]] + A.parent[g]];
    }
    __syncwarp();
    for (int e = 0; e < nch; e++) {
      if (crel[e] < 0) continue;
      const int64_t gs = cstep[e];
      if (gs != cur) {  // release every busy slot whose consumer ran before step gs
        uint32_t busy = ~freew;
        while (busy) {
          const int bit = __ffs(busy) - 1;
          busy &= busy - 1;
          if (rel[32 * lane + bit] < gs) freew |= 1u << bit;
        }
        cur = gs;
      }
      const unsigned m = __ballot_sync(0xffffffffu, freew != 0);
      if (!m) {
        if (lane == 0) atomicExch(overflow, 1);
        return;
      }
      const int fl = __ffs(m) - 1;
      const uint32_t w = __shfl_sync(0xffffffffu, freew, fl);
      const int sl = 32 * fl + __ffs(w) - 1;
      if (lane == fl) freew &= ~(1u << (sl & 31));
      if (lane == 0) {
        rel[sl] = crel[e];
        cslot[e] = sl;
      }
      next = max(next, sl + 1);
      __syncwarp();
    }
    for (int e = lane; e < nch; e += 32)
      if (crel[e] >= 0) slot_of[vals[p0 + e]] = cslot[e];
    __syncwarp();
  }
  if (lane == 0) atomicMax(max_slots, next);
}

struct WriteIn {
  NodeArrays A;
  const uint64_t *keys;
  const int32_t *vals;
  const StepDesc *desc;
  const int64_t *sfirst_sorted;
  const int64_t *bscan, *vscan, *dscan;
  const int32_t *slot_of, *node_tile;
  const int64_t *tile_root;
  const double *rec;
  uint8_t *blob;
};

__global__ void k_wv_write(WriteIn w, int64_t n) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  const NodeArrays &A = w.A;
  const int64_t gs = (int64_t)(w.keys[p] >> 2);
  const int64_t g = w.vals[p];
  const StepDesc D = w.desc[gs];
  const WaveSec S = wave_sections(D);
  const int64_t pf = w.sfirst_sorted[gs];
  const int pos = (int)(p - pf);
  const unsigned f = A.flags[g];
  const int cs = flag_case(f);
  uint8_t *B = w.blob + ((int64_t)D.off16 << 4);
  // record
  int rq_off;
  // record groups BEAD_BEAD | RIGID_BEAD | GENERAL (GENERAL's odd size last, so the others stay
  // 16-byte aligned); meta / node positions keep the G | R | B order
  if (cs == BEAD_BEAD) rq_off = (pos - D.nG - D.nR) * wave_rec_size(BEAD_BEAD);
  else if (cs == RIGID_BEAD) rq_off = D.nB * wave_rec_size(BEAD_BEAD) + (pos - D.nG) * wave_rec_size(RIGID_BEAD);
  else rq_off = D.nB * wave_rec_size(BEAD_BEAD) + D.nR * wave_rec_size(RIGID_BEAD) + pos * wave_rec_size(GENERAL);
  double *R = reinterpret_cast<double *>(B + S.rec) + rq_off;
  const double *src = w.rec + A.rec_off[g];
  bool bb_neg = false;
  unsigned tau_zero = 0;
  if (cs == GENERAL) tau_zero = wave_pack_wy<9>(src, R);
  else if (cs == RIGID_BEAD) tau_zero = wave_pack_wy<6>(src, R);
  else bb_neg = wave_pack_bb(src, R);
  // children in formula order
  const int j = A.node_body[g];
  const int64_t nb0 = A.node_off[j], b0 = A.bead_off[j];
  int xi = A.left[g], yi = A.right[g];
  if (flag_swapped(f)) { const int t = xi; xi = yi; yi = t; }
  const int64_t tr = w.tile_root[w.node_tile[g]];
  const bool troot = tr == g;
  const bool broot = troot && A.parent[g] < 0;
  const uint16_t rf = (uint16_t)(troot ? (broot ? WF_BODY_ROOT : WF_TILE_ROOT) : 0);
  // bead positions (upward gather region of this step): x bead first, then y
  const int bpos = (int)(w.bscan[p] - w.bscan[pf]);
  const int vpos = (int)(w.vscan[p] - w.vscan[pf]);
  auto orig_bead = [&](int id) -> uint32_t { return (uint32_t)(b0 + A.perm[b0 + A.start[nb0 + id]]); };
  WaveUpMeta um;
  WaveDnMeta dm;
  um.flags = dm.flags = (uint16_t)((f & 0x3fu) | rf | (bb_neg ? WF_BB_NEG : 0) | (tau_zero << WF_TAU_ZERO_SHIFT));
  um.self = dm.self = 0;
  dm.pad = 0;
  um.row = 0;
  um.aux = 0;
  // a bead's 3 doubles: window of 4 at 4 * position, offset (bead & 1)
  auto boff = [&](int id, int k) -> uint16_t { return (uint16_t)(4 * (bpos + k) + (orig_bead(id) & 1u)); };
  if (cs == BEAD_BEAD) {
    um.x = boff(xi, 0); um.y = boff(yi, 1);
    dm.x = orig_bead(xi); dm.y = orig_bead(yi);
  } else if (cs == RIGID_BEAD) {
    um.x = (uint16_t)w.slot_of[nb0 + xi]; um.y = boff(yi, 0);
    dm.x = (uint32_t)w.slot_of[nb0 + xi]; dm.y = orig_bead(yi);
  } else {
    um.x = (uint16_t)w.slot_of[nb0 + xi]; um.y = (uint16_t)w.slot_of[nb0 + yi];
    dm.x = (uint32_t)w.slot_of[nb0 + xi]; dm.y = (uint32_t)w.slot_of[nb0 + yi];
  }
  const int rr = res_rows(cs);
  const int64_t row = A.res_base[j] + A.res_off[g] - 6;
  const int rwin = rr ? 2 * wv_pieces(row, rr) : 0;  // residue window (doubles, even)
  if (rr) um.row = (uint32_t)row;
  dm.vres = (uint16_t)(vpos + (row & 1));
  if (troot) {
    um.aux = broot ? (uint32_t)j : (uint32_t)A.slot_scan[g];
    dm.self = (uint16_t)(vpos + rwin);
  } else {
    um.self = (uint16_t)w.slot_of[g];
    dm.self = (uint16_t)w.slot_of[g];
  }
  reinterpret_cast<WaveUpMeta *>(B + S.um)[pos] = um;
  reinterpret_cast<WaveDnMeta *>(B + S.dm)[pos] = dm;
  // upward gathers of this node's beads: held by block gs - 2
  if (cs != GENERAL) {
    const StepDesc Du = w.desc[gs - 2];
    uint32_t *UG = reinterpret_cast<uint32_t *>(w.blob + ((int64_t)Du.off16 << 4) + wave_sections(Du).ug);
    if (cs == BEAD_BEAD) { UG[bpos] = orig_bead(xi); UG[bpos + 1] = orig_bead(yi); }
    else UG[bpos] = orig_bead(yi);
  }
  // downward gathers (residues, root RV-set): held by block gs + 2
  if (rr || troot) {
    const StepDesc Dd = w.desc[gs + 2];
    const int64_t pfd = w.sfirst_sorted[gs];
    int di = (int)(w.dscan[p] - w.dscan[pfd]);
    WaveGather *DG = reinterpret_cast<WaveGather *>(w.blob + ((int64_t)Dd.off16 << 4) + wave_sections(Dd).dg);
    if (rr) {
      WaveGather e;
      e.src = (uint32_t)row;
      e.dst = (uint16_t)vpos;
      e.kind = rr == 3 ? WG_RES3 : WG_RES6;
      DG[di++] = e;
    }
    if (troot) {
      WaveGather e;
      e.src = broot ? (uint32_t)j : (uint32_t)A.slot_scan[g];
      e.dst = (uint16_t)(vpos + rwin);
      e.kind = broot ? WG_ROOT : WG_SLOT;
      DG[di++] = e;
    }
  }
}

}  // namespace

// ---- builder driver ----------------------------------------------------------------

void build_wave(Plan &p, const WaveBuildIn &in, cudaStream_t s) {
  SetupTimer tm(s);
  p.wave_streams = 0;
  p.wave_steps = 0;
  const int64_t nt = in.n_tiles;
  if (nt == 0) return;
  WaveCaps caps;
  if (const char *e = getenv("RQ_WAVE_CAPS")) {  // g,r,b,rm
    int g = 0, r = 0, b = 0, rm = 0;
    if (sscanf(e, "%d,%d,%d,%d", &g, &r, &b, &rm) == 4) { caps.g = g; caps.r = r; caps.b = b; caps.rm = rm; }
  }
  p.wave_caps = caps;
  NodeArrays A{in.node_off, in.bead_off, in.rec_off, in.res_base, in.node_body, in.start, in.stop, in.left,
               in.right,    in.parent,   in.height,  in.res_off,  in.perm,      in.slot_scan, in.flags};
  const int64_t NN = p.NN;
  DBuf tnodes, theight, node_scan;
  tnodes.alloc(nt * 8);
  theight.alloc(nt * 8);
  node_scan.alloc((nt + 1) * 8);
  k_wv_tiles<<<nblk(nt), NT, 0, s>>>(in.tile_root, nt, A, tnodes.as<int64_t>(), theight.as<int64_t>());
  ex_scan(tnodes.as<int64_t>(), node_scan.as<int64_t>(), nt + 0, s);
  const int64_t total_nodes = d2h1<int64_t>(node_scan.as<int64_t>() + nt - 1, s) + d2h1<int64_t>(tnodes.as<int64_t>() + nt - 1, s);
  RQ_CUDA(cudaMemcpyAsync(node_scan.as<int64_t>() + nt, &total_nodes, 8, cudaMemcpyHostToDevice, s));
  if (total_nodes == 0) return;
  // streams: one per resident CTA
  int sms = 0;
  RQ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p.device));
  p.sms = sms;
  int per_sm = 4;
  if (const char *e = getenv("RQ_WAVE_CTAS_PER_SM")) per_sm = std::max(1, std::min(16, atoi(e)));
  int64_t G = (int64_t)sms * per_sm;
  G = std::max<int64_t>(1, std::min<int64_t>(G, (total_nodes + 15) / 16));
  DBuf node_tile, bad;
  node_tile.alloc(NN * 4);
  RQ_CUDA(cudaMemsetAsync(node_tile.p, 0xff, NN * 4, s));
  bad.alloc(4);
  RQ_CUDA(cudaMemsetAsync(bad.p, 0, 4, s));
  k_wv_node_tile<<<nblk(nt), NT, 0, s>>>(in.tile_root, nt, A, node_tile.as<int32_t>());
  // streams: range c of every round
  int64_t R = std::max<int64_t>(1, p.N / 170000);
  R = std::min<int64_t>(R, std::max<int64_t>(1, nt / G));  // at least a tile per stream and round
  if (const char *e = getenv("RQ_WAVE_ROUNDS")) R = std::max(1, atoi(e));
  p.wave_rounds = R;
  DBuf tkey, tval, tkey2, order, sfirst, tile_stream, tn_sorted, n_scan_s, tile_round;
  tkey.alloc(nt * 8);
  tval.alloc(nt * 4);
  tkey2.alloc(nt * 8);
  order.alloc(nt * 4);
  sfirst.alloc((G + 1) * 8);
  tile_stream.alloc(nt * 4);
  tn_sorted.alloc(nt * 8);
  n_scan_s.alloc((nt + 1) * 8);
  tile_round.alloc(nt * 4);
  DBuf node_step, n_steps, step_first, tile_first, tile_last, round_floor, Wd;
  node_step.alloc(NN * 4);
  n_steps.alloc(G * 8);
  step_first.alloc((G + 1) * 8);
  tile_first.alloc(nt * 4);
  tile_last.alloc(nt * 4);
  round_floor.alloc(G * 8);
  // Tail rebalancing: placement noise accumulates over the rounds (stream step counts spread
  // ~10% around the mean at S = 128), and the sweep lasts as long as the longest stream.  A
  // first pass places everything with even ranges; the second re-cuts the last quarter of the
  // rounds (rounds >= R0) so that every stream, starting from where pass 1 found it at round
  // R0, ends at the same step T (same node rate nu for all streams).
  const int64_t R0 = R - (R + 3) / 4;
  DBuf save_ring, save_state;
  save_ring.alloc((size_t)G * WRING * sizeof(TLev));
  save_state.alloc((size_t)G * 2 * 4);
  auto assign_place = [&](const double *W, int mode) {
    tm.mark("place (other)");
    k_wv_tile_key<<<nblk(nt), NT, 0, s>>>(node_scan.as<int64_t>(), nt, total_nodes, G, R, W, R0, tkey.as<uint64_t>(),
                                           tval.as<int32_t>());
    {
      size_t tb = 0;
      RQ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, tkey.as<uint64_t>(), tkey2.as<uint64_t>(), tval.as<int32_t>(),
                                              order.as<int32_t>(), (int)nt, 0, 64, s));
      DBuf tmp;
      tmp.alloc(tb);
      RQ_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, tkey.as<uint64_t>(), tkey2.as<uint64_t>(), tval.as<int32_t>(),
                                              order.as<int32_t>(), (int)nt, 0, 64, s));
    }
    {
      std::vector<int64_t> h(G + 1, -1);
      RQ_CUDA(cudaMemcpyAsync(sfirst.p, h.data(), (G + 1) * 8, cudaMemcpyHostToDevice, s));
      k_wv_stream_first<<<nblk(nt), NT, 0, s>>>(tkey2.as<uint64_t>(), nt, R, sfirst.as<int64_t>());
      d2h(h.data(), sfirst.p, G + 1, s);
      h[G] = nt;
      for (int64_t c = G - 1; c >= 0; c--)
        if (h[c] < 0) h[c] = h[c + 1];
      RQ_CUDA(cudaMemcpyAsync(sfirst.p, h.data(), (G + 1) * 8, cudaMemcpyHostToDevice, s));
    }
    k_wv_tile_stream<<<nblk(nt), NT, 0, s>>>(tkey2.as<uint64_t>(), order.as<int32_t>(), nt, R,
                                              tile_stream.as<int32_t>(), tile_round.as<int32_t>());
    // node-level placement
    k_wv_place_nodes<<<(unsigned)G, 32, 0, s>>>(sfirst.as<int64_t>(), G, order.as<int32_t>(), in.tile_root, A, caps,
                                                 node_step.as<int32_t>(), n_steps.as<int64_t>(),
                                                 tile_first.as<int32_t>(), tile_last.as<int32_t>(),
                                                 tile_round.as<int32_t>(), (int)R0, round_floor.as<int64_t>(),
                                                 bad.as<int>(), mode, save_ring.as<TLev>(), save_state.as<int32_t>());
    if (d2h1<int>(bad.p, s)) throw Error(RQ_ERR_VALUE, "wave layout: a node does not fit the step window");
    tm.mark("place pass");
  };
  assign_place(nullptr, 1);
  bool rebalance = G > 1 && R > 1;
  if (const char *e = getenv("RQ_WAVE_REBALANCE")) rebalance = rebalance && atoi(e) != 0;
  if (rebalance) {
    std::vector<int64_t> ns(G), fl(G);
    d2h(ns.data(), n_steps.p, G, s);
    d2h(fl.data(), round_floor.p, G, s);
    const int64_t max1 = *std::max_element(ns.begin(), ns.end());
    double span = 0;  // steps the tail rounds took in pass 1
    for (int64_t c = 0; c < G; c++) span += std::max<double>(1.0, (double)(ns[c] - 4 - fl[c]));
    // ends at T: sum_c max(0, T - F_c) = span (same node rate, same total tail work)
    double lo = (double)*std::min_element(fl.begin(), fl.end()), hi = lo + span + 1.0;
    for (int it = 0; it < 100; it++) {
      const double T = 0.5 * (lo + hi);
      double tot = 0;
      for (int64_t c = 0; c < G; c++) tot += std::max(0.0, T - (double)fl[c]);
      (tot < span ? lo : hi) = T;
    }
    std::vector<double> W(G + 1, 0.0);
    for (int64_t c = 0; c < G; c++) W[c + 1] = W[c] + std::max(0.0, hi - (double)fl[c]);
    for (int64_t c = 1; c <= G; c++) W[c] /= W[G];
    W[G] = 1.0 + 1e-12;
    Wd.alloc((G + 1) * 8);
    RQ_CUDA(cudaMemcpyAsync(Wd.p, W.data(), (G + 1) * 8, cudaMemcpyHostToDevice, s));
    RQ_CUDA(cudaStreamSynchronize(s));
    assign_place(Wd.as<double>(), 2);
    d2h(ns.data(), n_steps.p, G, s);
    const int64_t max2 = *std::max_element(ns.begin(), ns.end());
    if (getenv("RQ_VERBOSE")) fprintf(stderr, "[rq] wave rebalance R0=%lld: max steps %lld -> %lld\n", (long long)R0,
                                      (long long)max1, (long long)max2);
    if (max2 > max1) assign_place(nullptr, 0);  // pass 1 was better
  }
  k_wv_gather64<<<nblk(nt), NT, 0, s>>>(tnodes.as<int64_t>(), order.as<int32_t>(), nt, tn_sorted.as<int64_t>());
  ex_scan(tn_sorted.as<int64_t>(), n_scan_s.as<int64_t>(), nt, s);
  RQ_CUDA(cudaMemcpyAsync(n_scan_s.as<int64_t>() + nt, &total_nodes, 8, cudaMemcpyHostToDevice, s));
  ex_scan(n_steps.as<int64_t>(), step_first.as<int64_t>(), G, s);
  const int64_t NS = d2h1<int64_t>(step_first.as<int64_t>() + G - 1, s) + d2h1<int64_t>(n_steps.as<int64_t>() + G - 1, s);
  RQ_CUDA(cudaMemcpyAsync(step_first.as<int64_t>() + G, &NS, 8, cudaMemcpyHostToDevice, s));
  tm.mark("wave place");
  // node order: (global step, case)
  DBuf keys, vals, keys2, vals2;
  keys.alloc(NN * 8);
  vals.alloc(NN * 4);
  keys2.alloc(NN * 8);
  vals2.alloc(NN * 4);
  k_wv_keys<<<nblk(NN), NT, 0, s>>>(NN, A, node_tile.as<int32_t>(), node_step.as<int32_t>(), step_first.as<int64_t>(),
                                     keys.as<uint64_t>(), vals.as<int32_t>(), tile_stream.as<int32_t>());
  {
    int bits = 2;
    while ((int64_t(1) << (bits - 2)) <= NS) bits++;
    size_t tb = 0;
    RQ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.as<uint64_t>(), keys2.as<uint64_t>(),
                                            vals.as<int32_t>(), vals2.as<int32_t>(), (int)NN, 0, 64, s));
    DBuf tmp;
    tmp.alloc(tb);
    RQ_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.as<uint64_t>(), keys2.as<uint64_t>(),
                                            vals.as<int32_t>(), vals2.as<int32_t>(), (int)NN, 0, 64, s));
    (void)bits;
  }
  keys.reset();
  vals.reset();
  tm.mark("wave sort");
  // counts
  const int64_t n = total_nodes;
  DBuf sc, step_of, sfs, nb, vd, nd, bscan, vscan, dscan;
  sc.alloc(NS * sizeof(StepCnt));
  RQ_CUDA(cudaMemsetAsync(sc.p, 0, NS * sizeof(StepCnt), s));
  step_of.alloc(NN * 8);
  sfs.alloc(NS * 8);
  RQ_CUDA(cudaMemsetAsync(sfs.p, 0, NS * 8, s));
  nb.alloc(n * 4);
  vd.alloc(n * 4);
  nd.alloc(n * 4);
  bscan.alloc(n * 8);
  vscan.alloc(n * 8);
  dscan.alloc(n * 8);
  k_wv_count<<<nblk(n), NT, 0, s>>>(keys2.as<uint64_t>(), vals2.as<int32_t>(), n, A, sc.as<StepCnt>(),
                                     step_of.as<int64_t>(), sfs.as<int64_t>(), nb.as<int32_t>(), vd.as<int32_t>(),
                                     nd.as<int32_t>(), node_tile.as<int32_t>(), in.tile_root);
  ex_scan(nb.as<int32_t>(), bscan.as<int64_t>(), n, s);
  ex_scan(vd.as<int32_t>(), vscan.as<int64_t>(), n, s);
  ex_scan(nd.as<int32_t>(), dscan.as<int64_t>(), n, s);
  // block offsets
  DBuf bytes, off, mx;
  bytes.alloc(NS * 8);
  off.alloc((NS + 1) * 8);
  mx.alloc(16);
  RQ_CUDA(cudaMemsetAsync(mx.p, 0, 16, s));
  k_wv_step_bytes<<<nblk(NS), NT, 0, s>>>(sc.as<StepCnt>(), NS, bytes.as<int64_t>(), mx.as<unsigned long long>());
  ex_scan(bytes.as<int64_t>(), off.as<int64_t>(), NS, s);
  const int64_t blob_bytes = d2h1<int64_t>(off.as<int64_t>() + NS - 1, s) + d2h1<int64_t>(bytes.as<int64_t>() + NS - 1, s);
  if (blob_bytes >= (int64_t(1) << 36)) throw Error(RQ_ERR_VALUE, "wave layout exceeds 64 GB");
  {
    unsigned long long h[2];
    d2h(h, mx.p, 2, s);
    p.wave_stage_bytes = (int64_t)al128((size_t)std::max(h[0], h[1]));
  }
  p.wave_blob.alloc(blob_bytes);
  RQ_CUDA(cudaMemsetAsync(p.wave_blob.p, 0, blob_bytes, s));
  p.wave_desc.alloc(NS * sizeof(StepDesc));
  k_wv_descs<<<nblk(NS), NT, 0, s>>>(sc.as<StepCnt>(), off.as<int64_t>(), NS, p.wave_desc.as<StepDesc>(),
                                      p.wave_blob.as<uint8_t>());
  {
    DBuf marks;
    marks.alloc(NS * 8);
    std::vector<int> init(2 * NS);
    for (int64_t i = 0; i < NS; i++) { init[i] = -1; init[NS + i] = INT32_MAX; }
    RQ_CUDA(cudaMemcpyAsync(marks.p, init.data(), NS * 8, cudaMemcpyHostToDevice, s));
    k_wv_round_marks<<<nblk(nt), NT, 0, s>>>(nt, tnodes.as<int64_t>(), tile_stream.as<int32_t>(),
                                              tile_round.as<int32_t>(), tile_first.as<int32_t>(), tile_last.as<int32_t>(),
                                              step_first.as<int64_t>(), marks.as<int>(), marks.as<int>() + NS);
    k_wv_headers<<<nblk(NS), NT, 0, s>>>(p.wave_desc.as<StepDesc>(), NS, p.wave_blob.as<uint8_t>(), marks.as<int>(),
                                          marks.as<int>() + NS);
    RQ_CUDA(cudaStreamSynchronize(s));
  }
  // run-time round window: CTAs more than `window` rounds ahead of the slowest wait (a
  // performance hint only: bounded waits, never a data dependency)
  {
    // (long runs only: over a few dozen rounds the streams do not drift apart; config 2 with 24
    // rounds runs 1% faster without it, config 4's 1261 rounds 26% faster with it)
    const double round_bytes = 48.0 * (double)p.N / (double)R;
    p.wave_window = R < 64 ? 0 : (int)std::max<int64_t>(8, std::min<int64_t>(R, (int64_t)(40e6 / std::max(round_bytes, 1.0))));
    if (const char *e = getenv("RQ_WAVE_WINDOW")) p.wave_window = std::max(0, atoi(e));
  }
  tm.mark("wave counts");
  // slots
  DBuf slot_of, node_first, msl;
  slot_of.alloc(NN * 4);
  RQ_CUDA(cudaMemsetAsync(slot_of.p, 0, NN * 4, s));
  node_first.alloc((G + 1) * 8);
  {
    // a stream's nodes are contiguous in the sorted order: node_first[c] = nodes of earlier streams
    std::vector<int64_t> hs(G + 1), hn(nt + 1);
    d2h(hs.data(), sfirst.p, G + 1, s);
    d2h(hn.data(), n_scan_s.p, nt + 1, s);
    std::vector<int64_t> nf(G + 1);
    for (int64_t c = 0; c <= G; c++) nf[c] = hn[hs[c]];
    RQ_CUDA(cudaMemcpyAsync(node_first.p, nf.data(), (G + 1) * 8, cudaMemcpyHostToDevice, s));
  }
  msl.alloc(8);
  RQ_CUDA(cudaMemsetAsync(msl.p, 0, 8, s));
  k_wv_slots<<<(unsigned)G, 32, 0, s>>>(node_first.as<int64_t>(), G, vals2.as<int32_t>(), A, step_of.as<int64_t>(),
                                         node_tile.as<int32_t>(), in.tile_root, slot_of.as<int32_t>(), msl.as<int>(),
                                         msl.as<int>() + 1);
  {
    int h[2];
    d2h(h, msl.p, 2, s);
    if (h[1]) throw Error(RQ_ERR_VALUE, "wave layout: more than 1024 live node vectors in a stream");
    p.wave_mslots = std::max(1, h[0]);
  }
  tm.mark("wave slots");
  WriteIn w{A,
            keys2.as<uint64_t>(),
            vals2.as<int32_t>(),
            p.wave_desc.as<StepDesc>(),
            sfs.as<int64_t>(),
            bscan.as<int64_t>(),
            vscan.as<int64_t>(),
            dscan.as<int64_t>(),
            slot_of.as<int32_t>(),
            node_tile.as<int32_t>(),
            in.tile_root,
            in.rec,
            p.wave_blob.as<uint8_t>()};
  k_wv_write<<<nblk(n), NT, 0, s>>>(w, n);
  RQ_CUDA(cudaGetLastError());
  tm.mark("wave write");
  if (getenv("RQ_LAYOUT_HASH")) {  // layout identity checks across builder versions (tools)
    std::vector<uint8_t> hb((size_t)blob_bytes);
    RQ_CUDA(cudaStreamSynchronize(s));
    RQ_CUDA(cudaMemcpy(hb.data(), p.wave_blob.p, (size_t)blob_bytes, cudaMemcpyDeviceToHost));
    uint64_t h = 1469598103934665603ull;
    for (uint8_t x : hb) h = (h ^ x) * 1099511628211ull;
    fprintf(stderr, "[rq] wave layout: %lld steps, %lld bytes, %d slots, fnv %016llx\n", (long long)NS,
            (long long)blob_bytes, p.wave_mslots, (unsigned long long)h);
  }
  p.wave_stream_first.alloc((G + 1) * 8);
  RQ_CUDA(cudaMemcpyAsync(p.wave_stream_first.p, step_first.p, (G + 1) * 8, cudaMemcpyDeviceToDevice, s));
  // per-direction bytes streamed per application (algorithmic bytes of the sweep)
  {
    std::vector<StepDesc> hd(NS);
    d2h(hd.data(), p.wave_desc.p, NS, s);
    int64_t up = 0, dn = 0;
    for (const auto &d : hd) {
      const WaveSec S = wave_sections(d);
      up += S.end - S.uhdr;
      dn += S.um;
    }
    p.wave_up_bytes = up;
    p.wave_down_bytes = dn;
  }
  RQ_CUDA(cudaStreamSynchronize(s));
  p.wave_streams = G;
  p.wave_steps = NS;
  p.wave_blob_bytes = blob_bytes;
  p.wave_nodes = n;
  if (getenv("RQ_VERBOSE")) {
    std::vector<int64_t> sf(G + 1);
    d2h(sf.data(), p.wave_stream_first.p, G + 1, s);
    int64_t mx = 0;
    for (int64_t c = 0; c < G; c++) mx = std::max(mx, sf[c + 1] - sf[c]);
    fprintf(stderr, "[rq] wave: %lld streams x %lld rounds, %lld steps (%.1f per stream, max %lld, %.1f nodes per step), "
                    "blob %.1f MB (up %.1f, down %.1f), M slots %d, stage %lld B, window %d\n",
            (long long)G, (long long)R, (long long)NS, (double)NS / G, (long long)mx,
            (double)n / std::max<int64_t>(1, NS - 4 * G), blob_bytes / 1e6, p.wave_up_bytes / 1e6,
            p.wave_down_bytes / 1e6, p.wave_mslots, (long long)p.wave_stage_bytes, p.wave_window);
  }
}

// ---- sweep kernel ------------------------------------------------------------------

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void *ptr) { return (uint32_t)__cvta_generic_to_shared(ptr); }
__device__ __forceinline__ void mbar_init(uint32_t bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, unsigned bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t addr, unsigned parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void cp8(uint32_t dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp16(uint32_t dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// packed wave record -> compact-WY record in registers: tau_i = 2 / (v_i^T v_i) (0 when the
// node's flag says so) and T's off-diagonal entries as lq_factor forms them (rq_lq.cuh)
template <int K>
__device__ __forceinline__ void unpack_wy(const double *P, unsigned flags,
                                          double (&R)[rec_size(K == 9 ? GENERAL : RIGID_BEAD)]) {
  using W = WY<K>;
  constexpr int NQ = wave_rec_size(K == 9 ? GENERAL : RIGID_BEAD);
  double Q[NQ];
  if constexpr (NQ % 2 == 0) {
    const double2 *p2 = reinterpret_cast<const double2 *>(P);
#pragma unroll
    for (int i = 0; i < NQ / 2; i++) {
      const double2 v = p2[i];
      Q[2 * i] = v.x;
      Q[2 * i + 1] = v.y;
    }
  } else {  // odd size: 8-byte loads
#pragma unroll
    for (int i = 0; i < NQ; i++) Q[i] = P[i];
  }
#pragma unroll
  for (int e = 0; e < W::T; e++) R[e] = Q[e];
  // v_i (v_i[i] = 1, v_i[r < i] = 0, v_i[r > i] = V_i[r - i - 1])
  auto Vv = [&](int i, int r) -> double { return Q[(i == 0 ? W::V0 : (i == 1 ? W::V1 : W::V2)) + r - i - 1]; };
  auto vdot = [&](int i, int j) {  // v_i^T v_j, i < j
    double d = Vv(i, j);
#pragma unroll
    for (int r = j + 1; r < K; r++) d = fma(Vv(i, r), Vv(j, r), d);
    return d;
  };
  auto vnorm2 = [&](int i) {
    double d = 1.0;
#pragma unroll
    for (int r = i + 1; r < K; r++) d = fma(Vv(i, r), Vv(i, r), d);
    return d;
  };
  // the three taus from one division: tau_i = 2 / s_i
  const double s0 = vnorm2(0), s1 = vnorm2(1), s2 = vnorm2(2);
  const double s01 = s0 * s1, r = 2.0 / (s01 * s2);
  const unsigned tz = flags >> WF_TAU_ZERO_SHIFT;
  const double T00 = (tz & 1u) ? 0.0 : r * (s1 * s2);
  const double T11 = (tz & 2u) ? 0.0 : r * (s0 * s2);
  const double T22 = (tz & 4u) ? 0.0 : r * s01;
  const double T01 = -T11 * T00 * vdot(0, 1);
  const double t0 = vdot(0, 2), t1 = vdot(1, 2);
  const double T02 = -T22 * (T00 * t0 + T01 * t1);
  const double T12 = -T22 * (T11 * t1);
  R[W::T + 0] = T00;
  R[W::T + 1] = T01;
  R[W::T + 2] = T02;
  R[W::T + 3] = T11;
  R[W::T + 4] = T12;
  R[W::T + 5] = T22;
  R[W::RA] = Q[W::T + 0];
  R[W::RB] = Q[W::T + 1];
}

template <int CS>
__device__ __forceinline__ void ld_rec(const double *rec, unsigned flags, double (&R)[rec_size(CS)]) {
  if constexpr (CS == GENERAL) {
    unpack_wy<9>(rec, flags, R);
  } else if constexpr (CS == RIGID_BEAD) {
    unpack_wy<6>(rec, flags, R);
  } else {  // BEAD_BEAD: the sign of g is applied by bb_sign (meta flag WF_BB_NEG)
    const double2 *r2 = reinterpret_cast<const double2 *>(rec);
    const double2 q01 = r2[0], q23 = r2[1];
    const double q[4] = {q01.x, q01.y, q23.x, q23.y};
    wave_unpack_bb(q, false, R);
  }
}
// BEAD_BEAD with det g = -1: g = -R(q)
template <int CS>
__device__ __forceinline__ void bb_sign(unsigned flags, double (&R)[rec_size(CS)]) {
  if constexpr (CS == BEAD_BEAD) {
    if (flags & WF_BB_NEG) {
#pragma unroll
      for (int e = 0; e < 9; e++) R[e] = -R[e];
    }
  }
}
__device__ __forceinline__ void ld6(const double *q, double (&v)[6]) {
  const double2 *q2 = reinterpret_cast<const double2 *>(q);
#pragma unroll
  for (int i = 0; i < 3; i++) {
    const double2 w = q2[i];
    v[2 * i] = w.x;
    v[2 * i + 1] = w.y;
  }
}
__device__ __forceinline__ void st6(double *q, const double (&v)[6]) {
  double2 *q2 = reinterpret_cast<double2 *>(q);
#pragma unroll
  for (int i = 0; i < 3; i++) q2[i] = make_double2(v[2 * i], v[2 * i + 1]);
}

// one node of the upward sweep (merge_infosets, matfree.py:41-62)
template <int CS>
__device__ __forceinline__ void wv_up(const double *rec, const WaveUpMeta *UMp, double *M, const double *V,
                                      double *out, double *scratch, double *roots) {
  double R[rec_size(CS)];
  const WaveUpMeta md = *UMp;
  ld_rec<CS>(rec, md.flags, R);
  bb_sign<CS>(md.flags, R);
  double mx[6], my[6];
  if (CS == BEAD_BEAD) {
    const double *f = V + md.x;
    mx[0] = f[0]; mx[1] = f[1]; mx[2] = f[2]; mx[3] = 0.0; mx[4] = 0.0; mx[5] = 0.0;
  } else {
    ld6(M + 6 * md.x, mx);
  }
  if (CS != GENERAL) {
    const double *f = V + md.y;
    my[0] = f[0]; my[1] = f[1]; my[2] = f[2]; my[3] = 0.0; my[4] = 0.0; my[5] = 0.0;
  } else {
    ld6(M + 6 * md.y, my);
  }
  double aa, bb, mp[6], res[6];
  rec_ratios(CS, R, 1, aa, bb);
  merge(CS, R, 1, flag_signs(md.flags), aa, bb, mx, my, mp, res);
  if (CS != BEAD_BEAD) {
    double *o = out + md.row;
#pragma unroll
    for (int r = 0; r < res_rows(CS); r++) o[r] = res[r];
  }
  if (md.flags & (WF_TILE_ROOT | WF_BODY_ROOT)) {
    double *dst = (md.flags & WF_TILE_ROOT) ? scratch + 6 * (int64_t)md.aux : (roots ? roots + 6 * (int64_t)md.aux : nullptr);
    if (dst) {
#pragma unroll
      for (int r = 0; r < 6; r++) dst[r] = mp[r];
    }
  } else {
    st6(M + 6 * md.self, mp);
  }
}

// one node of the downward sweep (split_rvset, matfree.py:65-83)
template <int CS>
__device__ __forceinline__ void wv_down(const double *rec, const WaveDnMeta *DMp, double *M, const double *V,
                                        double *out) {
  double R[rec_size(CS)];
  const WaveDnMeta md = *DMp;
  ld_rec<CS>(rec, md.flags, R);
  bb_sign<CS>(md.flags, R);
  double lp[6], res[6] = {0, 0, 0, 0, 0, 0}, lx[6], ly[6];
  if (md.flags & (WF_TILE_ROOT | WF_BODY_ROOT)) {
    const double *q = V + md.self;
#pragma unroll
    for (int r = 0; r < 6; r++) lp[r] = q[r];
  } else {
    ld6(M + 6 * md.self, lp);
  }
#pragma unroll
  for (int r = 0; r < res_rows(CS); r++) res[r] = V[md.vres + r];
  double aa, bb;
  rec_ratios(CS, R, 1, aa, bb);
  split(CS, R, 1, flag_signs(md.flags), aa, bb, lp, res, lx, ly);
  if (CS == BEAD_BEAD) {
    double *o = out + 3 * (int64_t)md.x;
    o[0] = lx[0]; o[1] = lx[1]; o[2] = lx[2];
  } else {
    st6(M + 6 * md.x, lx);
  }
  if (CS != GENERAL) {
    double *o = out + 3 * (int64_t)md.y;
    o[0] = ly[0]; o[1] = ly[1]; o[2] = ly[2];
  } else {
    st6(M + 6 * md.y, ly);
  }
}

struct WaveCtx {
  const StepDesc *steps;
  const int64_t *stream_first;
  const uint8_t *blob;
  const double *in;
  double *out;
  double *scratch;
  double *roots;
  uint32_t stage_bytes, o_m, o_v, vreg;  // shared memory: NST stages | M | 3 gather regions (vreg doubles each)
  int64_t in_len;                        // doubles in `in` (16-byte windows never read past it)
  int mslots;                            // node-vector slots (debug checks)
  // run-time round window (nullptr: off): per-round arrival counters of this direction
  uint32_t *round_ctr;
  uint32_t round_target;                 // arrivals per round when every CTA has passed it
  uint32_t *abandon;                     // == epoch: a window wait timed out in this launch
  uint32_t epoch;
  int rounds, window;
};

#ifndef RQ_WAVE_MIN_BLOCKS
#define RQ_WAVE_MIN_BLOCKS 4
#endif

template <bool UP, int NST>
__global__ void __launch_bounds__(128, RQ_WAVE_MIN_BLOCKS) k_wave(WaveCtx a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[NST];
  const int tid = threadIdx.x;
  constexpr int PROD = 96;  // lane 0 of warp 3 (a BEAD_BEAD warp: the cheapest node path)
  const int64_t s0 = a.stream_first[blockIdx.x], s1 = a.stream_first[blockIdx.x + 1];
  const int n = (int)(s1 - s0);
  const uint32_t sm_u = smem_u32(smem), bar_u = smem_u32(bar);
  double *M = reinterpret_cast<double *>(smem + a.o_m);
  double *Vb = reinterpret_cast<double *>(smem + a.o_v);
  const uint32_t vb_u = sm_u + a.o_v;
  auto blk = [&](int t) -> int64_t { return UP ? s0 + t : s1 - 1 - t; };
  auto span = [&](const StepDesc &d, uint32_t &off, uint32_t &bytes) {
    const WaveSec S = wave_sections(d);
    if (UP) { off = S.uhdr; bytes = S.end - S.uhdr; }
    else { off = 0; bytes = S.um; }
  };
  if (tid == PROD) {
    for (int i = 0; i < NST; i++) mbar_init(bar_u + 8 * i, 1);
    fence_mbar_init();
    for (int t = 0; t < NST && t < n; t++) {  // the first blocks; later ones come from the headers
      const StepDesc d = a.steps[blk(t)];
      uint32_t off, bytes;
      span(d, off, bytes);
      mbar_expect_tx(bar_u + 8 * t, bytes);
      bulk_g2s(sm_u + t * a.stage_bytes, a.blob + ((int64_t)d.off16 << 4) + off, bytes, bar_u + 8 * t);
    }
  }
  __syncthreads();
  pdl_wait();  // vectors and exchange slots may come from the previous kernel
  unsigned phase = 0;
  int st = 0;
  int cur_round = UP ? -1 : a.rounds;  // rounds this CTA has entered (arrivals counted)
  for (int t = 0; t < n; t++, st = (st == NST - 1) ? 0 : st + 1) {
    mbar_wait(bar_u + 8 * st, (phase >> st) & 1u);
    phase ^= 1u << st;
    const unsigned char *B = smem + st * a.stage_bytes;
    const DirHdr h = *reinterpret_cast<const DirHdr *>(B);
    // round window: entering round r, wait (bounded) until every CTA has entered round r -/+ window,
    // so the vector rows in flight stay within a few L2-resident rounds; the other threads run on
    // and the step's closing barrier holds the CTA
    if (a.round_ctr && h.round != ~0u && (UP ? (int)h.round > cur_round : (int)h.round < cur_round)) {
      const int r = (int)h.round;
      if (tid == 0) {
        if (UP) for (int q = cur_round + 1; q <= r; q++) atomicAdd(a.round_ctr + q, 1u);
        else for (int q = cur_round - 1; q >= r; q--) atomicAdd(a.round_ctr + q, 1u);
        const int lag = UP ? r - a.window : r + a.window;
        if (lag >= 0 && lag < a.rounds) {
          const long long t0 = clock64();
          // a wait that times out means the grid is not all resident (e.g. another application's
          // sweep shares the GPU): the window is then abandoned for the rest of this launch
          while ((int32_t)(*(volatile uint32_t *)(a.round_ctr + lag) - a.round_target) < 0 &&
                 *(volatile uint32_t *)a.abandon != a.epoch) {
            if (clock64() - t0 > 200000) {
              atomicExch(a.abandon, a.epoch);
              break;
            }
            __nanosleep(128);
          }
        }
      }
      cur_round = r;
    }
    RQ_CHECK(h.step == (uint32_t)blk(t), "staged block is the expected step (TMA landed, phase right)");
    RQ_CHECK(h.o_list <= a.stage_bytes && h.o_meta <= a.stage_bytes && h.o_rec <= a.stage_bytes, "sections");
    // gathers for step t + 2 (into region (t + 2) % 3): 16-byte L2 copies (cp.async.cg)
    {
      const int rg = (t + 2) % 3;
      const uint32_t vg = vb_u + 8u * (uint32_t)(rg * a.vreg);
      if (UP) {
        const uint32_t *ug = reinterpret_cast<const uint32_t *>(B + h.o_list);
        for (int i = tid; i < h.n_list; i += 128) {
          const int64_t b = ug[i];
          const int64_t w0 = 3 * b - (b & 1);  // even: 16-byte aligned window of 4 doubles
          RQ_CHECK(4 * i + 4 <= (int)a.vreg && 3 * b + 3 <= a.in_len, "upward gather bounds");
          const uint32_t dst = vg + 32u * (uint32_t)i;
          if (w0 + 4 <= a.in_len) {
            cp16(dst, a.in + w0);
            cp16(dst + 16, a.in + w0 + 2);
          } else {  // the vector's last bead: no read past the end
            const uint32_t d1 = dst + 8u * (uint32_t)(b & 1);
            cp8(d1, a.in + 3 * b);
            cp8(d1 + 8, a.in + 3 * b + 1);
            cp8(d1 + 16, a.in + 3 * b + 2);
          }
        }
      } else {
        const WaveGather *dg = reinterpret_cast<const WaveGather *>(B + h.o_list);
        for (int i = tid; i < h.n_list; i += 128) {
          const WaveGather e = dg[i];
          const uint32_t dst = vg + 8u * e.dst;
          RQ_CHECK((e.dst & 1) == 0 && e.dst + 8 <= a.vreg, "downward gather bounds");
          if (e.kind == WG_RES3 || e.kind == WG_RES6) {
            const int64_t row = e.src;
            const int rr = e.kind == WG_RES3 ? 3 : 6;
            const int np = wv_pieces(row, rr);
            const int64_t w0 = row & ~(int64_t)1;
            if (w0 + 2 * np <= a.in_len) {
              for (int k = 0; k < np; k++) cp16(dst + 16u * k, a.in + w0 + 2 * k);
            } else {
              const uint32_t d1 = dst + 8u * (uint32_t)(row & 1);
              for (int r = 0; r < rr; r++) cp8(d1 + 8u * r, a.in + row + r);
            }
          } else if (e.kind == WG_SLOT) {
            const double *src = a.scratch + 6 * (int64_t)e.src;
            for (int k = 0; k < 3; k++) cp16(dst + 16u * k, src + 2 * k);
          } else if (a.roots) {
            const double *src = a.roots + 6 * (int64_t)e.src;
            for (int k = 0; k < 3; k++) cp16(dst + 16u * k, src + 2 * k);
          } else {
            double *z = Vb + rg * a.vreg + e.dst;
            for (int r = 0; r < 6; r++) z[r] = 0.0;  // Q~^T: zero root RV-set (matfree.py:167-168)
          }
        }
      }
      cp_commit();
    }
    // nodes of step t (gather region t % 3)
    {
      const double *V = Vb + (t % 3) * a.vreg;
      const int nG = h.nG, nR = h.nR, nB = h.nB;
      const int gG = (nG + 31) & ~31, gR = (nR + 31) & ~31;
      const int tot = gG + gR + nB;
      const double *R = reinterpret_cast<const double *>(B + h.o_rec);
      const int oB = 0, oR = wave_rec_size(BEAD_BEAD) * nB, oG = oR + wave_rec_size(RIGID_BEAD) * nR;
      if (UP) {
        const WaveUpMeta *UM = reinterpret_cast<const WaveUpMeta *>(B + h.o_meta);
        if (RQ_DEBUG_CHECKS)
          for (int q = tid; q < nG + nR + nB; q += 128) {
            const WaveUpMeta md = UM[q];
            const int cs = q < nG ? GENERAL : (q < nG + nR ? RIGID_BEAD : BEAD_BEAD);
            RQ_CHECK(flag_case(md.flags) == cs, "upward meta case");
            RQ_CHECK(cs == BEAD_BEAD ? md.x + 3 <= (int)a.vreg : md.x < a.mslots, "upward x source");
            RQ_CHECK(cs != GENERAL ? md.y + 3 <= (int)a.vreg : md.y < a.mslots, "upward y source");
            RQ_CHECK((md.flags & (WF_TILE_ROOT | WF_BODY_ROOT)) || md.self < a.mslots, "upward output slot");
          }
        for (int q = tid; q < tot; q += 128) {
          if (q < gG) {
            if (q < nG) wv_up<GENERAL>(R + oG + q * wave_rec_size(GENERAL), UM + q, M, V, a.out, a.scratch, a.roots);
          } else if (q < gG + gR) {
            const int qq = q - gG;
            if (qq < nR)
              wv_up<RIGID_BEAD>(R + oR + qq * wave_rec_size(RIGID_BEAD), UM + nG + qq, M, V, a.out, a.scratch, a.roots);
          } else {
            const int qq = q - gG - gR;
            wv_up<BEAD_BEAD>(R + oB + qq * wave_rec_size(BEAD_BEAD), UM + nG + nR + qq, M, V, a.out, a.scratch, a.roots);
          }
        }
      } else {
        const WaveDnMeta *DM = reinterpret_cast<const WaveDnMeta *>(B + h.o_meta);
        if (RQ_DEBUG_CHECKS)
          for (int q = tid; q < nG + nR + nB; q += 128) {
            const WaveDnMeta md = DM[q];
            const int cs = q < nG ? GENERAL : (q < nG + nR ? RIGID_BEAD : BEAD_BEAD);
            RQ_CHECK(flag_case(md.flags) == cs, "downward meta case");
            RQ_CHECK(cs == BEAD_BEAD || md.x < (uint32_t)a.mslots, "downward x slot");
            RQ_CHECK(cs != GENERAL || md.y < (uint32_t)a.mslots, "downward y slot");
            RQ_CHECK((md.flags & (WF_TILE_ROOT | WF_BODY_ROOT)) ? md.self + 6 <= a.vreg : md.self < a.mslots,
                     "downward input");
            RQ_CHECK(md.vres + 6 <= a.vreg, "downward residues");
          }
        for (int q = tid; q < tot; q += 128) {
          if (q < gG) {
            if (q < nG) wv_down<GENERAL>(R + oG + q * wave_rec_size(GENERAL), DM + q, M, V, a.out);
          } else if (q < gG + gR) {
            const int qq = q - gG;
            if (qq < nR) wv_down<RIGID_BEAD>(R + oR + qq * wave_rec_size(RIGID_BEAD), DM + nG + qq, M, V, a.out);
          } else {
            const int qq = q - gG - gR;
            wv_down<BEAD_BEAD>(R + oB + qq * wave_rec_size(BEAD_BEAD), DM + nG + nR + qq, M, V, a.out);
          }
        }
      }
    }
    cp_wait<1>();  // this thread's gathers for step t + 1
    __syncthreads();
    if (tid == PROD && t + NST < n) {  // stage st is free: block t + NST (located by this block's header)
      RQ_CHECK(h.next_off16 != 0xffffffffu && h.next_bytes <= a.stage_bytes, "next block location");
      mbar_expect_tx(bar_u + 8 * st, h.next_bytes);
      bulk_g2s(sm_u + st * a.stage_bytes, a.blob + ((int64_t)h.next_off16 << 4), h.next_bytes, bar_u + 8 * st);
    }
  }
  if (a.round_ctr && tid == 0) {  // arrivals for the rounds this stream has no tile in
    if (UP) for (int q = cur_round + 1; q < a.rounds; q++) atomicAdd(a.round_ctr + q, 1u);
    else for (int q = cur_round - 1; q >= 0; q--) atomicAdd(a.round_ctr + q, 1u);
  }
}

}  // namespace

size_t wave_smem(const Plan &p, uint32_t *o_m, uint32_t *o_v, uint32_t *vreg) {
  const uint32_t st = (uint32_t)p.wave_stage_bytes;
  const uint32_t vr = (uint32_t)std::max(4 * p.wave_caps.beads, p.wave_caps.vd);
  const uint32_t om = (uint32_t)p.wave_nst * st;
  const uint32_t ov = om + (uint32_t)al128(48 * (size_t)p.wave_mslots);
  if (o_m) *o_m = om;
  if (o_v) *o_v = ov;
  if (vreg) *vreg = vr;
  return ov + 3 * 8 * (size_t)vr;
}

void wave_prepare(const Plan &p) {
  if (p.wave_ready || !p.wave_streams) return;
  const size_t sm = wave_smem(p, nullptr, nullptr, nullptr);
  for (const void *f : {(const void *)k_wave<true, 2>, (const void *)k_wave<false, 2>})
    ensure_smem_attr(f, sm);
  int occ = 0;
  RQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void *)k_wave<true, 2>, 128, sm));
  p.wave_ctas_per_sm = occ;
  if (occ < 1) throw Error(RQ_ERR_CUDA, "wave kernel does not fit on an SM (smem " + std::to_string(sm) + ")");
  p.wave_ready = true;
}

void run_wave(const Plan &p, bool up, const double *in, double *out, double *scratch, double *roots, cudaStream_t s,
              uint32_t *round_ctr, uint32_t epoch, uint32_t *abandon) {
  if (!p.wave_streams) return;
  if (reinterpret_cast<uintptr_t>(in) & 15) throw Error(RQ_ERR_VALUE, "wave sweep input must be 16-byte aligned");
  wave_prepare(p);
  WaveCtx a{};
  a.steps = p.wave_desc.as<StepDesc>();
  a.stream_first = p.wave_stream_first.as<int64_t>();
  a.blob = p.wave_blob.as<uint8_t>();
  a.in = in;
  a.out = out;
  a.scratch = scratch;
  a.roots = roots;
  a.stage_bytes = (uint32_t)p.wave_stage_bytes;
  const size_t sm = wave_smem(p, &a.o_m, &a.o_v, &a.vreg);
  a.in_len = up ? 3 * p.N : p.res_base[p.m];
  a.mslots = p.wave_mslots;
  a.rounds = (int)p.wave_rounds;
  a.window = p.wave_window;
  // the window waits assume every CTA of the grid is resident (bounded anyway)
  if (round_ctr && p.wave_window > 0 && p.wave_window < p.wave_rounds &&
      (int64_t)p.wave_ctas_per_sm * p.sms >= p.wave_streams) {
    a.round_ctr = round_ctr;
    a.round_target = (uint32_t)((int64_t)epoch * p.wave_streams);
    a.abandon = abandon;
    a.epoch = epoch;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p.wave_streams);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (up) RQ_CUDA(cudaLaunchKernelEx(&cfg, k_wave<true, 2>, a));
  else RQ_CUDA(cudaLaunchKernelEx(&cfg, k_wave<false, 2>, a));
}

}  // namespace rq
