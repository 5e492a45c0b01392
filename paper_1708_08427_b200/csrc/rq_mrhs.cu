// rq_mrhs.cu -- multi-right-hand-side application (k >= RQ_MRHS_MIN columns):
// Q V, Q^T W, Q~ V, Q~^T G for (rows, k) row-major blocks (matfree.py:86-92:
// a 2-D v applies the operator column by column; the reference does it as
// one gemm per node, matfree.py:55-60).
//
// Design (tiles): every warp runs a "stack machine" over one unit (a tile =
// maximal subtree of <= mrhs_tile beads) for 32
// columns at once: lane = column, so all lanes share one node, its record is
// a broadcast load, and every vector access is one coalesced 256-byte row
// segment of the (rows, k) block.  Nodes are visited in heavy-child-first
// postorder, so the stack of pending information vectors never holds more than
// floor(log2(leaves)) + 1 entries (the lighter child always has at most half
// the leaves); it lives in shared memory, [depth][6][32] doubles per warp.
// Bead inputs/outputs are read/written straight from/to the vector blocks;
// tile roots exchange their 6-vectors with the top units through a scratch
// block [slot][6][k].  Units are independent, warps never synchronise.
//
// Unit program: entries at a fixed 256-byte stride (forward for Q, backward
// for Q^T), each = SEntry header (16 B) + the node's compact record.
//
// Design (top trees, the nodes above the tiles): level-parallel.  The top nodes
// of all bodies are sorted by height; one launch per height level runs a warp
// per (node, group of 32 columns), lane = column: children from the tile
// exchange rows, the top exchange rows [top node][6][k] or the bead rows, so a
// single large body (config 3) is swept with the whole GPU instead of one warp.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cub/cub.cuh>

#include "rq_nodeops.cuh"
#include "rq_plan.hpp"

namespace rq {

namespace {

constexpr int ENTRY_BYTES = 256;
constexpr int MRHS_NT = 128;  // 4 independent warps per block


// ---- program builder ------------------------------------------------------------------

struct BuildCtx {
  int S;
  int64_t big;  // bodies with more beads sweep their top tree level-parallel (k_mrhs_top)
  int64_t NN, m;
  const int64_t *bead_off, *node_off, *rec_off;
  const int32_t *start, *stop, *left, *right, *parent, *res_off, *perm;
  const uint8_t *flags;
  const double *rec;
};

__device__ __forceinline__ int64_t body_of_node(const BuildCtx &c, int64_t g) {
  int64_t lo = 0, hi = c.m;  // node_off[lo] <= g < node_off[hi]
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) / 2;
    if (c.node_off[mid] <= g) lo = mid; else hi = mid;
  }
  return lo;
}

// unit roots: tile roots (2 <= L <= S, parent absent or > S) and big-body roots (L > S)
__global__ void k_unit_flags(BuildCtx c, int32_t *is_tile_unit, int32_t *is_top_unit, int32_t *tile_nodes,
                             int32_t *top_count) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= c.NN) return;
  const int64_t j = body_of_node(c, g);
  const int L = c.stop[g] - c.start[g];
  const int nj = (int)(c.bead_off[j + 1] - c.bead_off[j]);
  const bool root = (g - c.node_off[j]) == 2 * (int64_t)nj - 2;
  const int Lp = root ? 0 : c.stop[c.node_off[j] + c.parent[g]] - c.start[c.node_off[j] + c.parent[g]];
  const bool tile = L >= 2 && L <= c.S && (root || Lp > c.S);
  is_tile_unit[g] = tile;
  tile_nodes[g] = tile ? L - 1 : 0;
  // top trees of bodies up to c.big beads: one stack-machine unit per body (the warp keeps
  // the top vectors in shared memory); larger ones run level-parallel (k_mrhs_top)
  const bool small_body = nj <= c.big;
  is_top_unit[g] = root && L > c.S && small_body;
  if (L > c.S && small_body) atomicAdd(&top_count[j], 1);
}

struct UnitDesc {  // 32 bytes
  int64_t entry0;  // first entry (index of ENTRY_BYTES blocks)
  int32_t n;       // entries (internal nodes of the unit)
  int32_t body;
  int32_t out_slot;  // tile unit: its scratch slot, -1 if its root is the body root; top unit: -1
  int32_t depth;     // stack entries needed
  int64_t root;      // global node id of the unit root
};

struct SEntry {    // 16 bytes; the record (rec_size doubles) follows
  int32_t x, y;    // formula-x / -y child: >= 0 body-local original bead; -1 stack; <= -2 scratch slot (-2 - v)
  int32_t res;     // body-relative Q~ row of the residues (res_off - 6), -1 for BEAD_BEAD
  uint8_t flags;   // case | swapped | signs
  uint8_t x_first; // both children on the stack: 1 if x finished first (y on top)
  uint16_t pad;
};

__global__ void k_unit_list(BuildCtx c, const int32_t *is_tile_unit, const int32_t *tile_scan,
                            const int64_t *tile_entry_scan, const int32_t *is_top_unit, const int32_t *top_scan,
                            const int64_t *top_entry_base, const int32_t *top_count, int64_t n_tile_units,
                            UnitDesc *units, int32_t *tile_slot_of) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= c.NN) return;
  const int64_t j = body_of_node(c, g);
  if (is_tile_unit[g]) {
    const int64_t u = tile_scan[g];
    UnitDesc d;
    d.entry0 = tile_entry_scan[g];
    d.n = c.stop[g] - c.start[g] - 1;
    d.body = (int32_t)j;
    const int nj = (int)(c.bead_off[j + 1] - c.bead_off[j]);
    const bool root = (g - c.node_off[j]) == 2 * (int64_t)nj - 2;
    d.out_slot = root ? -1 : (int32_t)u;
    d.depth = 0;
    d.root = g;
    units[u] = d;
    tile_slot_of[g] = (int32_t)u;
  }
  if (is_top_unit[g]) {
    const int64_t u = n_tile_units + top_scan[g];
    UnitDesc d;
    d.entry0 = top_entry_base[top_scan[g]];
    d.n = top_count[j];
    d.body = (int32_t)j;
    d.out_slot = -1;
    d.depth = 0;
    d.root = g;
    units[u] = d;
  }
}

// one thread per unit: heavy-first postorder, entries written in visiting order
__global__ void k_unit_program(BuildCtx c, UnitDesc *units, int64_t n_units, const int32_t *tile_slot_of,
                               uint8_t *prog, int32_t *max_depth_tile, int32_t *max_depth_top,
                               int64_t n_tile_units, unsigned long long *bytes) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= n_units) return;
  UnitDesc d = units[u];
  const int64_t j = d.body, no = c.node_off[j], bo = c.bead_off[j];
  const bool top = u >= n_tile_units;
  auto Lof = [&](int64_t g) { return c.stop[g] - c.start[g]; };
  auto in_unit = [&](int64_t g) { return Lof(g) >= 2 && (!top || Lof(g) > c.S); };
  // explicit DFS stack: (node, state) with state 0 = enter, 1 = first child done, 2 = both done
  constexpr int MAXS = 128;
  int64_t st_node[MAXS];
  int8_t st_state[MAXS];
  int sp = 0;
  st_node[sp] = d.root;
  st_state[sp] = 0;
  sp++;
  int64_t e = 0, used = 0;
  int depth = 0, maxdepth = 1;
  while (sp > 0) {
    const int64_t g = st_node[sp - 1];
    const int8_t s = st_state[sp - 1];
    const int64_t lc = no + c.left[g], rc = no + c.right[g];
    const bool heavy_left = Lof(lc) >= Lof(rc);
    const int64_t first = heavy_left ? lc : rc, second = heavy_left ? rc : lc;
    if (s == 0) {
      st_state[sp - 1] = 1;
      if (in_unit(first)) { st_node[sp] = first; st_state[sp] = 0; sp++; }
      continue;
    }
    if (s == 1) {
      st_state[sp - 1] = 2;
      if (in_unit(second)) { st_node[sp] = second; st_state[sp] = 0; sp++; }
      continue;
    }
    sp--;
    // emit g
    const unsigned f = c.flags[g];
    const int cs = flag_case(f);
    const int64_t xc = flag_swapped(f) ? rc : lc, yc = flag_swapped(f) ? lc : rc;
    auto src = [&](int64_t ch) -> int32_t {
      if (Lof(ch) == 1) return c.perm[bo + c.start[ch]];
      if (in_unit(ch)) return -1;
      return -2 - tile_slot_of[ch];
    };
    SEntry h;
    h.x = src(xc);
    h.y = src(yc);
    h.res = cs == BEAD_BEAD ? -1 : c.res_off[g] - 6;
    h.flags = (uint8_t)f;
    h.x_first = (uint8_t)(xc == first);
    h.pad = 0;
    uint8_t *dst = prog + (d.entry0 + e) * ENTRY_BYTES;
    *reinterpret_cast<SEntry *>(dst) = h;
    const double *r = c.rec + c.rec_off[g];
    double *rd = reinterpret_cast<double *>(dst + sizeof(SEntry));
    for (int i = 0; i < rec_size(cs); i++) rd[i] = r[i];
    used += sizeof(SEntry) + 8 * rec_size(cs);
    e++;
    // simulated information-vector stack: pop the stack children, push g
    maxdepth = max(maxdepth, depth);  // stack children resident before the pops
    depth += 1 - (h.x == -1) - (h.y == -1);
    maxdepth = max(maxdepth, depth);
  }
  units[u].depth = maxdepth;
  atomicMax(top ? max_depth_top : max_depth_tile, maxdepth);
  atomicAdd(&bytes[top ? 1 : 0], (unsigned long long)used);
}

// level-parallel top trees: one entry per top node (L > S), sorted by height
struct MTop {       // 32 bytes
  int32_t x, y;     // formula-x / -y child: >= 0 top index; <= -2 tile exchange slot (-2 - v); bead: BEAD_REF | orig
  int32_t res;      // body-relative Q~ row of the residues (res_off - 6), -1 for BEAD_BEAD
  int32_t body;
  int32_t flags;    // node flags | (is_root << 8)
  int32_t pad;
  int64_t rec_off;  // record in the plan's compact record table
};
constexpr int32_t BEAD_REF = 0x40000000;

__global__ void k_mtop_keys(BuildCtx c, const int32_t *height, uint64_t *key, int32_t *val, int32_t *is_top) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= c.NN) return;
  const int64_t j = body_of_node(c, g);
  const bool top = c.stop[g] - c.start[g] > c.S && c.bead_off[j + 1] - c.bead_off[j] > c.big;
  is_top[g] = top;
  key[g] = top ? ((uint64_t)height[g] << 40) | (uint64_t)g : ~0ull;
  val[g] = (int32_t)g;
}
__global__ void k_mtop_index(const int32_t *order, int64_t n, int32_t *tidx) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q < n) tidx[order[q]] = (int32_t)q;
}
__global__ void k_mtop_fill(BuildCtx c, const int32_t *order, int64_t n, const int32_t *tidx, const int32_t *tile_slot_of,
                            MTop *out) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int64_t g = order[q];
  const int64_t j = body_of_node(c, g), no = c.node_off[j], bo = c.bead_off[j];
  const unsigned f = c.flags[g];
  const int64_t lc = no + c.left[g], rc = no + c.right[g];
  const int64_t xc = flag_swapped(f) ? rc : lc, yc = flag_swapped(f) ? lc : rc;
  auto ref = [&](int64_t ch) -> int32_t {
    const int L = c.stop[ch] - c.start[ch];
    if (L == 1) return BEAD_REF | c.perm[bo + c.start[ch]];
    if (L > c.S) return tidx[ch];
    return -2 - tile_slot_of[ch];
  };
  MTop t;
  t.x = ref(xc);
  t.y = ref(yc);
  const int cs = flag_case(f);
  t.res = cs == BEAD_BEAD ? -1 : c.res_off[g] - 6;
  t.body = (int32_t)j;
  const int nj = (int)(c.bead_off[j + 1] - c.bead_off[j]);
  t.flags = (int32_t)f | (((g - no) == 2 * (int64_t)nj - 2) ? 256 : 0);
  t.pad = 0;
  t.rec_off = c.rec_off[g];
  out[q] = t;
}

// ---- kernels ----------------------------------------------------------------------------

struct MrhsCtx {
  const UnitDesc *units;
  int64_t n_units;  // units of this launch
  int64_t n_cg;     // column groups of 32
  const uint8_t *prog;
  const int64_t *bead_off;
  const double *in;
  double *out;
  double *scratch;  // [slot][6][K]
  int64_t K;
  int op;
  int depth;        // stack entries per warp
  long long *dbg;   // per-warp phase timers, only with -DRQ_TIMING
};
#ifndef RQ_TIMING
#define RQ_TIMING 0
#endif

// stack entry d, component r, this lane
#define STK(d, r) stk[((d) * 6 + (r)) * 32 + lane]

__device__ __forceinline__ uint32_t smem_u32m(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async16m(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32m(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit_m() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait_m() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void prefetch_l2m(const void *p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p) : "memory");
}

constexpr int RING = 8;      // unit entries staged per warp (cp.async, RING-1 ahead)
constexpr int PD = 4;        // gathered inputs of node t+PD are prefetched into L2 at node t
constexpr int L2_AHEAD = 12; // entries prefetched into L2 ahead of the ring

template <int CS>
__device__ __forceinline__ void lds_rec(const uint8_t *e, double (&R)[rec_size(GENERAL)]) {
  const double2 *r2 = reinterpret_cast<const double2 *>(e + sizeof(SEntry));
#pragma unroll
  for (int i = 0; i < rec_size(CS) / 2; i++) {
    const double2 v = r2[i];
    R[2 * i] = v.x;
    R[2 * i + 1] = v.y;
  }
}


// Per-lane views used by the node bodies: S = stack base + lane (entry d,
// component r at S[(6d + r) * 32]; every lane touches only its own column, so
// the stack needs no synchronisation); column-relative row pointers of the body.
// KS = k when specialised at compile time (row strides become immediates), else 0.
template <int KS>
struct LaneIO {
  double *S;
  const double *inB, *inR;  // bead rows / residue rows of the body (input)
  double *outB, *outR;      // bead rows / residue rows of the body (output)
  double *scr;              // exchange rows of tile roots
  int Kr;                   // runtime k (KS == 0)
  __device__ __forceinline__ int ki() const { return KS ? KS : Kr; }
};

template <bool ACT, int KS>
__device__ __forceinline__ void st_rows(double *p, const LaneIO<KS> &io, const double *v, int n, bool act) {
  if (ACT || act) {
#pragma unroll
    for (int r = 0; r < 6; r++)
      if (r < n) p[r * io.ki()] = v[r];
  }
}

// merge_infosets (matfree.py:41-62) for one node of a unit, 32 columns
template <int CS, bool ACT, int KS>
__device__ __forceinline__ void up_m(const int4 &hw, const double (&R)[rec_size(GENERAL)], const double (&gin)[6],
                                     const LaneIO<KS> &io, int &sp, bool act) {
  double mx[6], my[6];
  if (CS == BEAD_BEAD) {
#pragma unroll
    for (int r = 0; r < 3; r++) { mx[r] = gin[r]; my[r] = gin[3 + r]; mx[3 + r] = 0.0; my[3 + r] = 0.0; }
  } else {
    const bool xs = hw.x == -1, ys = CS == GENERAL && hw.y == -1;
    int dx = sp - 1, dy = sp - 1;
    if (xs && ys) {
      if (hw.w >> 8) dx = sp - 2; else dy = sp - 2;  // x finished first: y on top
    }
    if (xs) {
#pragma unroll
      for (int r = 0; r < 6; r++) mx[r] = io.S[(dx * 6 + r) * 32];
    } else {
      const double *px = io.scr + (-2 - hw.x) * 6 * io.ki();
#pragma unroll
      for (int r = 0; r < 6; r++) mx[r] = px[r * io.ki()];
    }
    if (CS == GENERAL) {
      if (ys) {
#pragma unroll
        for (int r = 0; r < 6; r++) my[r] = io.S[(dy * 6 + r) * 32];
      } else {
        const double *py = io.scr + (-2 - hw.y) * 6 * io.ki();
#pragma unroll
        for (int r = 0; r < 6; r++) my[r] = py[r * io.ki()];
      }
    } else {
#pragma unroll
      for (int r = 0; r < 3; r++) { my[r] = gin[3 + r]; my[3 + r] = 0.0; }
    }
    sp -= (int)xs + (int)ys;
  }
  double aa, bb, mp[6], res[6];
  rec_ratios(CS, R, 1, aa, bb);
  merge(CS, R, 1, flag_signs(hw.w & 0xff), aa, bb, mx, my, mp, res);
  if (CS != BEAD_BEAD) st_rows<ACT>(io.outR + hw.z * io.ki(), io, res, res_rows(CS), act);
#pragma unroll
  for (int r = 0; r < 6; r++) io.S[(sp * 6 + r) * 32] = mp[r];
  sp++;
}

// split_rvset (matfree.py:65-83) for one node of a unit, 32 columns
template <int CS, bool ACT, int KS>
__device__ __forceinline__ void down_m(const int4 &hw, const double (&R)[rec_size(GENERAL)],
                                       const double (&gin)[6], const LaneIO<KS> &io, int &sp, bool act) {
  double lp[6], lx[6], ly[6];
  sp--;
#pragma unroll
  for (int r = 0; r < 6; r++) lp[r] = io.S[(sp * 6 + r) * 32];
  double aa, bb;
  rec_ratios(CS, R, 1, aa, bb);
  split(CS, R, 1, flag_signs(hw.w & 0xff), aa, bb, lp, gin, lx, ly);
  // child outputs: beads -> velocity rows; tile roots -> exchange rows; others -> stack,
  // pushed so that the child finished LAST upward (visited next here) ends on top
  auto emit = [&](int32_t src, const double (&l)[6], bool bead) {
    if (bead) {
      st_rows<ACT>(io.outB + 3 * src * io.ki(), io, l, 3, act);
    } else if (src == -1) {
#pragma unroll
      for (int r = 0; r < 6; r++) io.S[(sp * 6 + r) * 32] = l[r];
      sp++;
    } else {
      st_rows<ACT>(io.scr + (-2 - src) * 6 * io.ki(), io, l, 6, act);
    }
  };
  if (CS == BEAD_BEAD) {
    emit(hw.x, lx, true);
    emit(hw.y, ly, true);
  } else if (CS == RIGID_BEAD) {
    emit(hw.x, lx, false);
    emit(hw.y, ly, true);
  } else if (hw.x == -1 && hw.y == -1 && !(hw.w >> 8)) {
    emit(hw.y, ly, false);
    emit(hw.x, lx, false);
  } else {
    emit(hw.x, lx, false);
    emit(hw.y, ly, false);
  }
}

// gathered inputs of a node (issued one node ahead): UP: bead rows of the bead
// children (BEAD_BEAD: x and y, RIGID_BEAD: y); DOWN: the node's residue rows
template <bool UP, int KS>
__device__ __forceinline__ void fetch_m(const int4 &hw, const LaneIO<KS> &io, double (&g)[6]) {
  const int cs = flag_case(hw.w & 0xff);
  const int k = io.ki();
  if (UP) {
    if (cs == BEAD_BEAD) {
      const double *px = io.inB + 3 * hw.x * k, *py = io.inB + 3 * hw.y * k;
      g[0] = __ldg(px); g[1] = __ldg(px + k); g[2] = __ldg(px + 2 * k);
      g[3] = __ldg(py); g[4] = __ldg(py + k); g[5] = __ldg(py + 2 * k);
    } else if (cs == RIGID_BEAD) {
      const double *py = io.inB + 3 * hw.y * k;
      g[3] = __ldg(py); g[4] = __ldg(py + k); g[5] = __ldg(py + 2 * k);
    }
  } else {
    const double *pr = io.inR + hw.z * k;
    if (cs == GENERAL) {
#pragma unroll
      for (int r = 0; r < 6; r++) g[r] = __ldg(pr + r * k);
    } else if (cs == RIGID_BEAD) {
      g[0] = __ldg(pr); g[1] = __ldg(pr + k); g[2] = __ldg(pr + 2 * k);
    }
  }
}

template <bool UP, bool ACT, int KS>
__device__ __forceinline__ void run_unit(const MrhsCtx &a, const UnitDesc &U, double *stk, uint8_t *ring, int lane,
                                         int64_t col) {
  const int64_t K = a.K;
  const bool act = ACT || col < K;
  const int64_t cc = act ? col : 0;  // clamped column: inactive lanes read valid memory, never store
  const bool full = (a.op == RQ_OP_QV || a.op == RQ_OP_QTV);
  const int64_t bead0 = a.bead_off[U.body];
  const int64_t sbase = full ? 3 * bead0 + 6 : 3 * bead0 - 6 * (int64_t)U.body;
  const uint8_t *E = a.prog + U.entry0 * ENTRY_BYTES;
  const int n = U.n;
  LaneIO<KS> io;
  io.S = stk + lane;
  io.Kr = (int)K;  // body-relative 32-bit row offsets (host guarantees rows * k < 2^31)
  io.inB = a.in + 3 * bead0 * K + cc;
  io.outB = a.out + 3 * bead0 * K + cc;
  io.inR = a.in + sbase * K + cc;
  io.outR = a.out + sbase * K + cc;
  io.scr = a.scratch + cc;
  // entry t (visiting order) lives at E + idx(t); the downward sweep visits backwards
  auto idx = [&](int t) -> int64_t { return (int64_t)(UP ? t : n - 1 - t) * ENTRY_BYTES; };
  auto issue = [&](int t) {
    if (t < n && lane < ENTRY_BYTES / 16) cp_async16m(ring + (t % RING) * ENTRY_BYTES + 16 * lane, E + idx(t) + 16 * lane);
    cp_commit_m();
  };
  auto slot = [&](int t) -> const uint8_t * { return ring + (t % RING) * ENTRY_BYTES; };
  for (int t = 0; t < L2_AHEAD && t < n; t++)
    if (lane < 2) prefetch_l2m(E + idx(t) + 128 * lane);
  for (int t = 0; t < RING - 1; t++) issue(t);
  cp_wait_m<RING - 1 - PD>();  // entries <= PD-1 resident
  __syncwarp();
  // L2 prefetch of the gathered rows of node t (bead rows / residue rows), one line per lane
  const int64_t col0 = col - lane;
  const double *pfB = a.in + 3 * bead0 * K + col0, *pfR = a.in + sbase * K + col0;
  auto prefetch_inputs = [&](int t) {
    if (t >= n || lane >= 12) return;
    const int4 hw = *reinterpret_cast<const int4 *>(slot(t));
    const int half = lane & 1;
    if (UP) {
      const int b = lane < 6 ? hw.x : hw.y, r = (lane % 6) >> 1;
      if (b >= 0) prefetch_l2m(pfB + (3 * (int64_t)b + r) * K + 16 * half);
    } else {
      const int r = lane >> 1;
      if (hw.z >= 0 && r < res_rows(flag_case(hw.w & 0xff))) prefetch_l2m(pfR + (int64_t)(hw.z + r) * K + 16 * half);
    }
  };
  for (int t = 0; t < PD; t++) prefetch_inputs(t);
  double gA[6], gB[6];
  if (n > 0) fetch_m<UP>(*reinterpret_cast<const int4 *>(slot(0)), io, gA);
  int sp = 0;
  if (!UP) {  // root RV-set of the unit
#pragma unroll
    for (int r = 0; r < 6; r++) {
      double v = 0.0;  // Q~^T: zero root RV-set (matfree.py:167-168)
      if (U.out_slot >= 0) v = io.scr[(U.out_slot * 6 + r) * io.ki()];
      else if (a.op == RQ_OP_QTV) v = io.inB[r * io.ki()];
      io.S[r * 32] = v;
    }
    sp = 1;
  }
  // one node: entries <= t+PD resident after the wait; the refill of ring slot
  // t-1 is issued after the __syncwarp that ends every lane's reads of it
  auto step = [&](int t, const double (&gin)[6], double (&gnx)[6]) {
    cp_wait_m<RING - 2 - PD>();
    __syncwarp();
    issue(t + RING - 1);
    if (lane < 2 && t + L2_AHEAD < n) prefetch_l2m(E + idx(t + L2_AHEAD) + 128 * lane);
    prefetch_inputs(t + PD);
    const uint8_t *e = slot(t);
    const int4 hw = *reinterpret_cast<const int4 *>(e);
    const int cs = flag_case(hw.w & 0xff);
    if (t + 1 < n) fetch_m<UP>(*reinterpret_cast<const int4 *>(slot(t + 1)), io, gnx);
    double R[rec_size(GENERAL)];
    if (cs == GENERAL) {
      lds_rec<GENERAL>(e, R);
      if (UP) up_m<GENERAL, ACT>(hw, R, gin, io, sp, act); else down_m<GENERAL, ACT>(hw, R, gin, io, sp, act);
    } else if (cs == RIGID_BEAD) {
      lds_rec<RIGID_BEAD>(e, R);
      if (UP) up_m<RIGID_BEAD, ACT>(hw, R, gin, io, sp, act); else down_m<RIGID_BEAD, ACT>(hw, R, gin, io, sp, act);
    } else {
      lds_rec<BEAD_BEAD>(e, R);
      if (UP) up_m<BEAD_BEAD, ACT>(hw, R, gin, io, sp, act); else down_m<BEAD_BEAD, ACT>(hw, R, gin, io, sp, act);
    }
  };
  for (int t = 0; t < n; t += 2) {  // ping-pong input registers (no copies)
    step(t, gA, gB);
    RQ_CHECK(sp >= 0 && sp <= a.depth, "multi-RHS stack depth");
    if (t + 1 < n) step(t + 1, gB, gA);
    RQ_CHECK(sp >= 0 && sp <= a.depth, "multi-RHS stack depth");
  }
  cp_wait_m<0>();
  if (UP && (ACT || act)) {  // unit root
    if (U.out_slot >= 0) {
#pragma unroll
      for (int r = 0; r < 6; r++) io.scr[(U.out_slot * 6 + r) * io.ki()] = io.S[((sp - 1) * 6 + r) * 32];
    } else if (a.op == RQ_OP_QV) {
#pragma unroll
      for (int r = 0; r < 6; r++) io.outB[r * io.ki()] = io.S[((sp - 1) * 6 + r) * 32];
    }
  }
  __syncwarp();
}

// MODE (a template parameter, so each column layout gets its own register allocation):
// 0: K == 32, 1: K a multiple of 32, 2: any K (inactive lanes in the last column group)
// MINB: CTAs per SM the registers are bounded for.  Upward tile units run best at 3 (no
// spills; 4 spilled ~90 bytes), the few top units and every downward launch at 4
// (measured on config 5).
template <bool UP, int MODE, int MINB>
__global__ void __launch_bounds__(MRHS_NT, MINB) k_mrhs(MrhsCtx a) {
  extern __shared__ __align__(16) double smem_m[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const size_t warp_doubles = (size_t)a.depth * 6 * 32 + RING * ENTRY_BYTES / 8;
  double *stk = smem_m + (size_t)wib * warp_doubles;
  uint8_t *ring = reinterpret_cast<uint8_t *>(stk + (size_t)a.depth * 6 * 32);
  const int64_t GW = (int64_t)gridDim.x * (MRHS_NT / 32);
  for (int64_t item = (int64_t)blockIdx.x * (MRHS_NT / 32) + wib; item < a.n_units * a.n_cg; item += GW) {
    const UnitDesc U = a.units[item / a.n_cg];
    const int64_t col = (item % a.n_cg) * 32 + lane;
    if (MODE == 0) run_unit<UP, true, 32>(a, U, stk, ring, lane, col);
    else if (MODE == 1) run_unit<UP, true, 0>(a, U, stk, ring, lane, col);
    else run_unit<UP, false, 0>(a, U, stk, ring, lane, col);
  }
}
#undef STK

__global__ void k_small_m(const int32_t *bodies, int64_t n, const int64_t *bead_off, const double *in,
                          double *out, int64_t K) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= 3 * n * K) return;
  const int64_t b = t / (3 * K), rc = t % (3 * K);
  const int64_t i = 3 * bead_off[bodies[b]] * K + rc;
  out[i] = in[i];
}

struct MTopCtx {
  const MTop *top;
  int64_t q0, n;      // this level's top nodes [q0, q0 + n)
  int64_t n_cg;       // column groups of 32
  const double *rec;
  const int64_t *bead_off;
  const double *in;
  double *out;
  double *tx;         // top exchange [top][6][K]
  double *scr;        // tile exchange [slot][6][K]
  int64_t K;
  int op;
};

// one warp per (top node, column group): merge (UP) / split (DOWN), lane = column
template <bool UP>
__global__ void __launch_bounds__(128) k_mrhs_top(MTopCtx a) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= a.n * a.n_cg) return;
  const int64_t q = a.q0 + w / a.n_cg;
  const int64_t col = (w % a.n_cg) * 32 + lane;
  const bool act = col < a.K;
  const int64_t K = a.K, c = act ? col : 0;
  const MTop T = a.top[q];
  const int cs = flag_case(T.flags & 0xff);
  double R[rec_size(GENERAL)];
  {
    const double2 *r2 = reinterpret_cast<const double2 *>(a.rec + T.rec_off);
#pragma unroll
    for (int i = 0; i < rec_size(GENERAL) / 2; i++) {
      double2 v = make_double2(0.0, 0.0);
      if (2 * i < rec_size(cs)) v = __ldg(r2 + i);
      R[2 * i] = v.x;
      R[2 * i + 1] = v.y;
    }
  }
  const bool full = (a.op == RQ_OP_QV || a.op == RQ_OP_QTV);
  const int64_t bead0 = a.bead_off[T.body];
  const int64_t sbase = full ? 3 * bead0 + 6 : 3 * bead0 - 6 * (int64_t)T.body;
  auto vec = [&](int32_t ref) -> double * {  // 6-vector rows of a top node / tile root (column c)
    return ref >= 0 ? a.tx + (int64_t)ref * 6 * K + c : a.scr + (int64_t)(-2 - ref) * 6 * K + c;
  };
  double aa, bb;
  rec_ratios(cs, R, 1, aa, bb);
  if (UP) {
    double mx[6], my[6], mp[6], res[6];
    auto load = [&](int32_t ref, double (&m)[6]) {
      if (ref & BEAD_REF && ref > 0) {
        const double *p = a.in + (3 * (bead0 + (ref & ~BEAD_REF))) * K + c;
        m[0] = __ldg(p); m[1] = __ldg(p + K); m[2] = __ldg(p + 2 * K); m[3] = m[4] = m[5] = 0.0;
      } else {
        const double *p = vec(ref);
#pragma unroll
        for (int r = 0; r < 6; r++) m[r] = __ldcg(p + r * K);
      }
    };
    load(T.x, mx);
    load(T.y, my);
    merge(cs, R, 1, flag_signs(T.flags & 0xff), aa, bb, mx, my, mp, res);
    if (!act) return;
    for (int r = 0; r < res_rows(cs); r++) a.out[(sbase + T.res + r) * K + c] = res[r];
    if (T.flags & 256) {
      if (a.op == RQ_OP_QV)
        for (int r = 0; r < 6; r++) a.out[(3 * bead0 + r) * K + c] = mp[r];
    } else {
      double *p = a.tx + q * 6 * K + c;
#pragma unroll
      for (int r = 0; r < 6; r++) __stcg(p + r * K, mp[r]);
    }
  } else {
    double lp[6], res[6] = {0, 0, 0, 0, 0, 0}, lx[6], ly[6];
    if (T.flags & 256) {
#pragma unroll
      for (int r = 0; r < 6; r++) lp[r] = a.op == RQ_OP_QTV ? a.in[(3 * bead0 + r) * K + c] : 0.0;
    } else {
      const double *p = a.tx + q * 6 * K + c;
#pragma unroll
      for (int r = 0; r < 6; r++) lp[r] = __ldcg(p + r * K);
    }
    for (int r = 0; r < res_rows(cs); r++) res[r] = a.in[(sbase + T.res + r) * K + c];
    split(cs, R, 1, flag_signs(T.flags & 0xff), aa, bb, lp, res, lx, ly);
    if (!act) return;
    auto store = [&](int32_t ref, const double (&l)[6]) {
      if (ref & BEAD_REF && ref > 0) {
        double *p = a.out + (3 * (bead0 + (ref & ~BEAD_REF))) * K + c;
        p[0] = l[0]; p[K] = l[1]; p[2 * K] = l[2];
      } else {
        double *p = vec(ref);
#pragma unroll
        for (int r = 0; r < 6; r++) __stcg(p + r * K, l[r]);
      }
    };
    store(T.x, lx);
    store(T.y, ly);
  }
}

template <class T>
T d2h1m(const void *src, cudaStream_t s) {
  T v;
  RQ_CUDA(cudaMemcpyAsync(&v, src, sizeof(T), cudaMemcpyDeviceToHost, s));
  RQ_CUDA(cudaStreamSynchronize(s));
  return v;
}

}  // namespace

void build_mrhs(const Plan &p, cudaStream_t s) {
  std::lock_guard<std::mutex> lock(p.mrhs_mu);
  if (p.mrhs_built) return;
  const int64_t NN = p.NN, m = p.m;
  BuildCtx c;
  c.S = p.mrhs_tile;  // unit size of the column-parallel programs (independent of the wave tiles)
  c.big = 65536;
  if (const char *e = getenv("RQ_MRHS_TOP_LEVELS")) c.big = std::max<int64_t>(0, atoll(e));
  c.NN = NN;
  c.m = m;
  c.bead_off = p.bead_off_d.as<int64_t>();
  c.node_off = p.node_off_d.as<int64_t>();
  c.rec_off = p.rec_off.as<int64_t>();
  c.start = p.start.as<int32_t>();
  c.stop = p.stop.as<int32_t>();
  c.left = p.left.as<int32_t>();
  c.right = p.right.as<int32_t>();
  c.parent = p.parent.as<int32_t>();
  c.res_off = p.res_off.as<int32_t>();
  c.perm = p.perm.as<int32_t>();
  c.flags = p.flags.as<uint8_t>();
  c.rec = p.rec.as<double>();
  auto nb = [](int64_t n) { return (unsigned)std::max<int64_t>(1, (n + 255) / 256); };
  DBuf is_tile, is_top, tile_nodes, top_count, tile_scan, top_scan, tile_entry_scan, slot_of, dmax, dbytes;
  const int64_t NNa = std::max<int64_t>(NN, 1);
  is_tile.alloc(NNa * 4);
  is_top.alloc(NNa * 4);
  tile_nodes.alloc(NNa * 4);
  top_count.alloc(std::max<int64_t>(m, 1) * 4);
  tile_scan.alloc(NNa * 4);
  top_scan.alloc(NNa * 4);
  tile_entry_scan.alloc(NNa * 8);
  slot_of.alloc(NNa * 4);
  dmax.alloc(8);
  RQ_CUDA(cudaMemsetAsync(top_count.p, 0, std::max<int64_t>(m, 1) * 4, s));
  RQ_CUDA(cudaMemsetAsync(slot_of.p, 0xff, NNa * 4, s));
  RQ_CUDA(cudaMemsetAsync(dmax.p, 0, 8, s));
  dbytes.alloc(16);
  RQ_CUDA(cudaMemsetAsync(dbytes.p, 0, 16, s));
  if (NN > 0) k_unit_flags<<<nb(NN), 256, 0, s>>>(c, is_tile.as<int32_t>(), is_top.as<int32_t>(),
                                                  tile_nodes.as<int32_t>(), top_count.as<int32_t>());
  // scans on the host side of the device (small, one-time): copy flags back
  std::vector<int32_t> h_tile(NN), h_top(NN), h_tn(NN), h_tc(m);
  if (NN) {
    RQ_CUDA(cudaMemcpyAsync(h_tile.data(), is_tile.p, NN * 4, cudaMemcpyDeviceToHost, s));
    RQ_CUDA(cudaMemcpyAsync(h_top.data(), is_top.p, NN * 4, cudaMemcpyDeviceToHost, s));
    RQ_CUDA(cudaMemcpyAsync(h_tn.data(), tile_nodes.p, NN * 4, cudaMemcpyDeviceToHost, s));
  }
  if (m) RQ_CUDA(cudaMemcpyAsync(h_tc.data(), top_count.p, m * 4, cudaMemcpyDeviceToHost, s));
  RQ_CUDA(cudaStreamSynchronize(s));
  std::vector<int32_t> h_tscan(NN), h_pscan(NN);
  std::vector<int64_t> h_escan(NN);
  int64_t nt = 0, np = 0, ne = 0;
  std::vector<int64_t> top_entry_base;
  std::vector<int64_t> h_body_of_top;
  for (int64_t g = 0; g < NN; g++) {
    h_tscan[g] = (int32_t)nt;
    h_escan[g] = ne;
    h_pscan[g] = (int32_t)np;
    if (h_tile[g]) { nt++; ne += h_tn[g]; }
    if (h_top[g]) np++;
  }
  // top-unit entries follow all tile-unit entries, in body order
  {
    int64_t e = ne;
    for (int64_t j = 0; j < m; j++) {
      if (h_tc[j] > 0) { top_entry_base.push_back(e); e += h_tc[j]; }
    }
    p.mrhs_entries = e;
  }
  p.n_tile_units = nt;
  p.n_top_units = np;
  RQ_CUDA(cudaMemcpyAsync(tile_scan.p, h_tscan.data(), NN * 4, cudaMemcpyHostToDevice, s));
  RQ_CUDA(cudaMemcpyAsync(top_scan.p, h_pscan.data(), NN * 4, cudaMemcpyHostToDevice, s));
  RQ_CUDA(cudaMemcpyAsync(tile_entry_scan.p, h_escan.data(), NN * 8, cudaMemcpyHostToDevice, s));
  DBuf teb;
  teb.alloc(std::max<size_t>(top_entry_base.size(), 1) * 8);
  if (!top_entry_base.empty())
    RQ_CUDA(cudaMemcpyAsync(teb.p, top_entry_base.data(), top_entry_base.size() * 8, cudaMemcpyHostToDevice, s));
  const int64_t nu = nt + np;
  p.mrhs_units.alloc(std::max<int64_t>(nu, 1) * sizeof(UnitDesc));
  p.mrhs_prog.alloc(std::max<int64_t>(p.mrhs_entries, 1) * ENTRY_BYTES);
  RQ_CUDA(cudaMemsetAsync(p.mrhs_prog.p, 0, std::max<int64_t>(p.mrhs_entries, 1) * ENTRY_BYTES, s));
  if (NN > 0)
    k_unit_list<<<nb(NN), 256, 0, s>>>(c, is_tile.as<int32_t>(), tile_scan.as<int32_t>(),
                                       tile_entry_scan.as<int64_t>(), is_top.as<int32_t>(), top_scan.as<int32_t>(),
                                       teb.as<int64_t>(), top_count.as<int32_t>(), nt,
                                       p.mrhs_units.as<UnitDesc>(), slot_of.as<int32_t>());
  if (nu > 0)
    k_unit_program<<<nb(nu), 256, 0, s>>>(c, p.mrhs_units.as<UnitDesc>(), nu, slot_of.as<int32_t>(),
                                          p.mrhs_prog.as<uint8_t>(), dmax.as<int32_t>(), dmax.as<int32_t>() + 1, nt,
                                          dbytes.as<unsigned long long>());
  RQ_CUDA(cudaGetLastError());
  int32_t hd[2] = {0, 0};
  RQ_CUDA(cudaMemcpyAsync(hd, dmax.p, 8, cudaMemcpyDeviceToHost, s));
  RQ_CUDA(cudaStreamSynchronize(s));
  unsigned long long hb[2] = {0, 0};
  RQ_CUDA(cudaMemcpy(hb, dbytes.p, 16, cudaMemcpyDeviceToHost));
  p.mrhs_tile_bytes = (int64_t)hb[0];
  p.mrhs_top_bytes = (int64_t)hb[1];
  p.mrhs_depth_tile = std::max(1, hd[0]);
  p.mrhs_depth_top = std::max(1, hd[1]);
  // level-parallel top trees: top nodes sorted by (height, id)
  {
    DBuf key, val, key2, val2, istop, tidx;
    key.alloc(NNa * 8);
    val.alloc(NNa * 4);
    key2.alloc(NNa * 8);
    val2.alloc(NNa * 4);
    istop.alloc(NNa * 4);
    tidx.alloc(NNa * 4);
    if (NN > 0) k_mtop_keys<<<nb(NN), 256, 0, s>>>(c, p.height.as<int32_t>(), key.as<uint64_t>(), val.as<int32_t>(),
                                                   istop.as<int32_t>());
    size_t tb = 0;
    RQ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.as<uint64_t>(), key2.as<uint64_t>(), val.as<int32_t>(),
                                            val2.as<int32_t>(), (int)NN, 0, 64, s));
    DBuf tmp;
    tmp.alloc(tb);
    RQ_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, key.as<uint64_t>(), key2.as<uint64_t>(), val.as<int32_t>(),
                                            val2.as<int32_t>(), (int)NN, 0, 64, s));
    std::vector<uint64_t> hk(NN);
    if (NN) RQ_CUDA(cudaMemcpyAsync(hk.data(), key2.p, NN * 8, cudaMemcpyDeviceToHost, s));
    RQ_CUDA(cudaStreamSynchronize(s));
    int64_t ntop = 0;
    while (ntop < NN && hk[ntop] != ~0ull) ntop++;
    p.n_mtop = ntop;
    p.h_mtop_level.clear();
    for (int64_t q = 0; q < ntop; q++)
      if (q == 0 || (hk[q] >> 40) != (hk[q - 1] >> 40)) p.h_mtop_level.push_back(q);
    p.h_mtop_level.push_back(ntop);
    p.mtop.alloc(std::max<int64_t>(ntop, 1) * sizeof(MTop));
    if (ntop) {
      k_mtop_index<<<nb(ntop), 256, 0, s>>>(val2.as<int32_t>(), ntop, tidx.as<int32_t>());
      k_mtop_fill<<<nb(ntop), 256, 0, s>>>(c, val2.as<int32_t>(), ntop, tidx.as<int32_t>(), slot_of.as<int32_t>(),
                                           p.mtop.as<MTop>());
    }
    RQ_CUDA(cudaStreamSynchronize(s));
  }
  // body -> unit ranges (host), for body-segmented applications
  std::vector<UnitDesc> hu(nu);
  if (nu) RQ_CUDA(cudaMemcpy(hu.data(), p.mrhs_units.p, nu * sizeof(UnitDesc), cudaMemcpyDeviceToHost));
  p.h_tile_unit_first.assign(m + 1, nt);
  p.h_top_unit_first.assign(m + 1, np);
  for (int64_t u = nt - 1; u >= 0; u--) p.h_tile_unit_first[hu[u].body] = u;
  for (int64_t u = np - 1; u >= 0; u--) p.h_top_unit_first[hu[nt + u].body] = u;
  for (int64_t j = m - 1; j >= 0; j--) {
    p.h_tile_unit_first[j] = std::min(p.h_tile_unit_first[j], p.h_tile_unit_first[j + 1]);
    p.h_top_unit_first[j] = std::min(p.h_top_unit_first[j], p.h_top_unit_first[j + 1]);
  }
  p.mrhs_built = true;
}

bool use_mrhs(const Plan &p, int64_t k) {
  if (k < p.mrhs_min) return false;
  int64_t max_n = 0;
  for (int64_t j = 0; j < p.m; j++) max_n = std::max(max_n, p.bead_off[j + 1] - p.bead_off[j]);
  // the kernels use 32-bit body-relative row offsets
  const int64_t lim32 = int64_t(1) << 31;
  if (!(3 * max_n * k < lim32 && 6 * std::max<int64_t>(p.n_slots, 1) * k < lim32)) return false;
  const char *pol = getenv("RQ_MRHS");  // "always" / "never" override the cost model (tests, tuning)
  if (pol && !strcmp(pol, "always")) return true;
  if (pol && !strcmp(pol, "never")) return false;
  // The column-parallel kernels beat the column loop from mrhs_min columns on (measured):
  // their top trees run level-parallel, so single large bodies no longer need the loop.
  return true;
}

void run_apply_mrhs(const Plan &p, int op, const double *in, double *out, int64_t k, cudaStream_t s,
                    unsigned phases, BodyRange range) {
  build_mrhs(p, s);
  const bool up = (op == RQ_OP_QV || op == RQ_OP_QTILDE_V);
  const bool all = range.j1 < 0;
  const int64_t j0 = all ? 0 : range.j0, j1 = all ? p.m : range.j1;
  const int64_t t0 = p.h_tile_unit_first[j0], t1 = p.h_tile_unit_first[j1];
  const int64_t q0 = p.h_top_unit_first[j0], q1 = p.h_top_unit_first[j1];
  const size_t scratch_bytes = (size_t)std::max<int64_t>(p.n_tile_units, 1) * 6 * k * 8;
  const size_t tx_bytes = (size_t)std::max<int64_t>(p.n_mtop, 1) * 6 * k * 8;
  Plan::StreamState &ss = p.state_for(s);
  if (ss.mrhs_scratch.bytes < scratch_bytes) ss.mrhs_scratch.alloc(scratch_bytes);
  if (ss.mrhs_tx.bytes < tx_bytes) ss.mrhs_tx.alloc(tx_bytes);
  if (!p.sms) RQ_CUDA(cudaDeviceGetAttribute(&p.sms, cudaDevAttrMultiProcessorCount, p.device));
  const int sms = p.sms;
  MrhsCtx a{};
  a.prog = p.mrhs_prog.as<uint8_t>();
  a.bead_off = p.bead_off_d.as<int64_t>();
  a.in = in;
  a.out = out;
  a.scratch = ss.mrhs_scratch.as<double>();
  a.K = k;
  a.op = op;
  a.n_cg = (k + 31) / 32;
  auto launch = [&](int64_t u0, int64_t u1, int depth, bool tiles) {
    if (u1 <= u0) return;
    a.units = p.mrhs_units.as<UnitDesc>() + u0;
    a.n_units = u1 - u0;
    a.depth = depth;
    const size_t smem = (size_t)(MRHS_NT / 32) * ((size_t)depth * 6 * 32 * 8 + RING * ENTRY_BYTES);
    const int mode = k == 32 ? 0 : ((k % 32) == 0 ? 1 : 2);
    void (*fn)(MrhsCtx) = nullptr;
    if (up && tiles) fn = mode == 0 ? k_mrhs<true, 0, 3> : (mode == 1 ? k_mrhs<true, 1, 3> : k_mrhs<true, 2, 3>);
    else if (up) fn = mode == 0 ? k_mrhs<true, 0, 4> : (mode == 1 ? k_mrhs<true, 1, 4> : k_mrhs<true, 2, 4>);
    else fn = mode == 0 ? k_mrhs<false, 0, 4> : (mode == 1 ? k_mrhs<false, 1, 4> : k_mrhs<false, 2, 4>);
    ensure_smem_attr((const void *)fn, smem);
    const int occ = occupancy_cached((const void *)fn, MRHS_NT, smem);
    if (occ < 1) throw Error(RQ_ERR_CUDA, "multi-RHS kernel does not fit on an SM");
    const int64_t items = a.n_units * a.n_cg;
    const int64_t blocks = std::min<int64_t>((items + MRHS_NT / 32 - 1) / (MRHS_NT / 32), (int64_t)sms * occ);
    fn<<<(unsigned)blocks, MRHS_NT, smem, s>>>(a);
  };
  static const bool timing = RQ_TIMING && getenv("RQ_TIMING") != nullptr;
  DBuf dbg;
  if (timing) {
    const size_t bytes = (size_t)sms * 32 * 4 * 64;
    dbg.alloc(bytes);
    RQ_CUDA(cudaMemsetAsync(dbg.p, 0, bytes, s));
    a.dbg = dbg.as<long long>();
  }
  const bool do_tiles = phases & 1u, do_top = phases & 2u;
  // top trees: one launch per height level (upward: leaves first; downward: root level first)
  auto top_levels = [&]() {
    if (!all) throw Error(RQ_ERR_VALUE, "body ranges are not supported by the multi-RHS top sweep");
    MTopCtx tc{};
    tc.top = p.mtop.as<MTop>();
    tc.n_cg = (k + 31) / 32;
    tc.rec = p.rec.as<double>();
    tc.bead_off = p.bead_off_d.as<int64_t>();
    tc.in = in;
    tc.out = out;
    tc.tx = ss.mrhs_tx.as<double>();
    tc.scr = ss.mrhs_scratch.as<double>();
    tc.K = k;
    tc.op = op;
    const int64_t nl = (int64_t)p.h_mtop_level.size() - 1;
    for (int64_t i = 0; i < nl; i++) {
      const int64_t l = up ? i : nl - 1 - i;
      tc.q0 = p.h_mtop_level[l];
      tc.n = p.h_mtop_level[l + 1] - tc.q0;
      const int64_t threads = tc.n * tc.n_cg * 32;
      if (up) k_mrhs_top<true><<<(unsigned)((threads + 127) / 128), 128, 0, s>>>(tc);
      else k_mrhs_top<false><<<(unsigned)((threads + 127) / 128), 128, 0, s>>>(tc);
    }
  };
  const int64_t nt = p.n_tile_units;
  if (up) {
    if (do_tiles) launch(t0, t1, p.mrhs_depth_tile, true);
    if (do_top) launch(nt + q0, nt + q1, p.mrhs_depth_top, false);
    if (do_top && p.n_mtop) top_levels();
  } else {
    if (do_top && p.n_mtop) top_levels();
    if (do_top) launch(nt + q0, nt + q1, p.mrhs_depth_top, false);
    if (do_tiles) launch(t0, t1, p.mrhs_depth_tile, true);
  }
  if (timing) {
    std::vector<long long> h((size_t)sms * 32 * 4 * 8);
    RQ_CUDA(cudaMemcpyAsync(h.data(), dbg.p, h.size() * 8, cudaMemcpyDeviceToHost, s));
    RQ_CUDA(cudaStreamSynchronize(s));
    double acc[8] = {0};
    for (size_t w = 0; w < h.size() / 8; w++) for (int i = 0; i < 8; i++) acc[i] += (double)h[8 * w + i];
    fprintf(stderr, "[rq timing] mrhs op %d: per node: ring wait %.0f, node %.0f, input-wait+sync %.0f (nodes %.0f)\n", op,
            acc[0] / acc[3], acc[1] / acc[3], acc[2] / acc[3], acc[3]);
  }
  const int64_t sm0 = all ? 0 : p.h_small_first[j0], sm1 = all ? p.n_small : p.h_small_first[j1];
  if ((phases & 4u) && sm1 > sm0 && op <= 1)
    k_small_m<<<(unsigned)((3 * (sm1 - sm0) * k + 255) / 256), 256, 0, s>>>(
        p.small_bodies.as<int32_t>() + sm0, sm1 - sm0, p.bead_off_d.as<int64_t>(), in, out, k);
  RQ_CUDA(cudaGetLastError());
}

}  // namespace rq
