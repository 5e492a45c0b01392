// rq_setup.cu -- batched per-body setup on the GPU: tree (tree.py:73-134),
// factors (factor.py:213-244) and the chunked apply layout.
//
// Pipeline (all bodies at once, no per-body host loop):
//   1. per-body bounding cube (tree.py:78-81)
//   2. per-bead ghost key: the bead's own midpoint-bisection walk z,y,x
//      (tree.py:96-114); bit d = (pos > mid_d).  The reference tree is the
//      binary radix tree of these keys (empty halves pruned = levels where a
//      node's keys agree).
//   3. radix sort of (body, key) -> perm (tree.py:368)
//   4. Karras radix-tree topology; reference postorder ids from
//        id(X) = start + C(start) + 2L - 2,  C(s) = #internal nodes with stop <= s
//   5. bottom-up factor pass, one launch per ghost-depth level (deepest first,
//      nodes case-sorted): centroids (tree.py:126), the three node cases
//      (factor.py:224-243), compact LQ records
//   6. apply layout: tiles (maximal subtrees with <= S beads, height-sorted per
//      body), chunks (greedy byte-budget packing of a body's tiles), level-major
//      AoS blobs, and the top tree above the tiles (staged blobs / dataflow).
// Compiled with --fmad=false (see rq_lq.cuh).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <tuple>
#include <string>
#include <thread>
#include <vector>

#include "rq_lq.cuh"
#include "rq_plan.hpp"

namespace rq {
namespace {

constexpr int NT = 256;
__constant__ int c_axis_cycle[3] = {2, 1, 0};  // tree.py:27

inline int nblk(int64_t n, int t = NT) { return (int)std::max<int64_t>(1, (n + t - 1) / t); }

__device__ __forceinline__ int find_body(const int64_t *off, int64_t m, int64_t i) {
  int64_t lo = 0, hi = m;  // off[lo] <= i < off[hi]
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (off[mid] <= i) lo = mid; else hi = mid;
  }
  return (int)lo;
}

__device__ __forceinline__ unsigned long long ord_key(double x) {
  unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double unord_key(unsigned long long u) {
  return __longlong_as_double((long long)((u >> 63) ? (u & 0x7fffffffffffffffull) : ~u));
}

struct Key128 {
  uint64_t hi, lo;
};
struct KeyDec {
  __host__ __device__ ::cuda::std::tuple<uint64_t &, uint64_t &> operator()(Key128 &k) const {
    return {k.hi, k.lo};
  }
};

// ---- 1. bodies, bounding cube ------------------------------------------------

__global__ void k_body_of(const int64_t *off, int64_t m, int64_t N, int32_t *body_of) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < N) body_of[i] = find_body(off, m, i);
}

__global__ void k_bbox(const double *pos, const int32_t *body_of, int64_t N,
                       unsigned long long *bmin, unsigned long long *bmax, long long *err) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  bool valid = i < N;
  int j = valid ? body_of[i] : -1;
  unsigned long long kmin[3], kmax[3];
  for (int a = 0; a < 3; a++) {
    double x = valid ? pos[i * 3 + a] : 0.0;
    if (valid && !isfinite(x)) atomicExch((unsigned long long *)&err[1], 1ull);
    kmin[a] = valid ? ord_key(x) : ~0ull;
    kmax[a] = valid ? ord_key(x) : 0ull;
  }
  unsigned full = 0xffffffffu;
  int j0 = __shfl_sync(full, j, 0);
  bool uniform = __all_sync(full, j == j0) && j0 >= 0;
  if (uniform) {
    for (int a = 0; a < 3; a++)
      for (int o = 16; o; o >>= 1) {
        unsigned long long vmin = __shfl_xor_sync(full, kmin[a], o);
        unsigned long long vmax = __shfl_xor_sync(full, kmax[a], o);
        kmin[a] = vmin < kmin[a] ? vmin : kmin[a];
        kmax[a] = vmax > kmax[a] ? vmax : kmax[a];
      }
    if ((threadIdx.x & 31) == 0)
      for (int a = 0; a < 3; a++) {
        atomicMin(&bmin[j0 * 3 + a], kmin[a]);
        atomicMax(&bmax[j0 * 3 + a], kmax[a]);
      }
  } else if (valid) {
    for (int a = 0; a < 3; a++) {
      atomicMin(&bmin[j * 3 + a], kmin[a]);
      atomicMax(&bmax[j * 3 + a], kmax[a]);
    }
  }
}

// tree.py:78-81: center = (lo+hi)/2; half = max(hi-lo) * (1+1e-9) / 2
__global__ void k_root_box(const unsigned long long *bmin, const unsigned long long *bmax,
                           int64_t m, double *box) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  double lo[3], hi[3];
  for (int a = 0; a < 3; a++) { lo[a] = unord_key(bmin[j * 3 + a]); hi[a] = unord_key(bmax[j * 3 + a]); }
  double ext = hi[0] - lo[0];
  for (int a = 1; a < 3; a++) { double e = hi[a] - lo[a]; if (e > ext) ext = e; }
  double half = ext * (1.0 + 1e-9) / 2.0;
  for (int a = 0; a < 3; a++) {
    double c = (lo[a] + hi[a]) / 2.0;
    box[j * 6 + a] = c - half;
    box[j * 6 + 3 + a] = c + half;
  }
}

// ---- 2. ghost keys -------------------------------------------------------------

__global__ void k_keys(const double *pos, const int32_t *body_of, const double *box, int64_t N,
                       int max_depth, int body_shift, Key128 *keys, int32_t *vals) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  int j = body_of[i];
  double p[3], cl[3], ch[3];
  for (int a = 0; a < 3; a++) {
    p[a] = pos[i * 3 + a];
    cl[a] = box[j * 6 + a];
    ch[a] = box[j * 6 + 3 + a];
  }
  uint64_t hi = 0, lo = 0;
  for (int d = 0; d < max_depth; d++) {
    int a = c_axis_cycle[d % 3];
    double mid = 0.5 * (cl[a] + ch[a]);
    unsigned bit = p[a] > mid;  // ties go to the lower half (tree.py:106)
    if (bit) cl[a] = mid; else ch[a] = mid;
    hi = (hi << 1) | (lo >> 63);
    lo = (lo << 1) | bit;
  }
  // body id above the key bits (bits [max_depth, max_depth + body_bits))
  if (body_shift >= 64) hi |= (uint64_t)j << (body_shift - 64);
  else {
    hi |= body_shift > 0 ? ((uint64_t)j >> (64 - body_shift)) : 0;
    lo |= (uint64_t)j << body_shift;
  }
  keys[i] = {hi, lo};
  vals[i] = (int32_t)i;
}

__device__ __forceinline__ int prefix_len(const Key128 &a, const Key128 &b, int max_depth) {
  uint64_t xh = a.hi ^ b.hi, xl = a.lo ^ b.lo;
  int clz = xh ? __clzll((long long)xh) : 64 + (xl ? __clzll((long long)xl) : 64);
  return clz - (128 - max_depth);
}

// ---- 3. after the sort: perm, tree-order positions, gaps -----------------------

__global__ void k_post_sort(const Key128 *keys, const int32_t *vals, const double *pos,
                            const int64_t *bead_off, const int32_t *body_of, int64_t N,
                            int max_depth, int32_t *perm, double *pos_tree, int16_t *gap,
                            long long *err) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  int j = body_of[i];
  int64_t src = vals[i];
  perm[i] = (int32_t)(src - bead_off[j]);
  for (int a = 0; a < 3; a++) pos_tree[i * 3 + a] = pos[src * 3 + a];
  int16_t g = -1;
  if (i + 1 < bead_off[j + 1]) {
    Key128 a = keys[i], b = keys[i + 1];
    if (a.hi == b.hi && a.lo == b.lo) {
      // tree.py:99-103: split depth exceeded without separating beads
      atomicMin((unsigned long long *)&err[0], (unsigned long long)j);
      g = 0;
    } else {
      g = (int16_t)prefix_len(a, b, max_depth);
    }
  }
  gap[i] = g;
}

// ---- 4. Karras radix tree ------------------------------------------------------

struct KarrasCtx {
  const Key128 *k;  // body base
  int n, max_depth;
  __device__ int delta(int i, int j) const {
    if (j < 0 || j >= n) return -1;
    return prefix_len(k[i], k[j], max_depth);
  }
};

__global__ void k_karras(const Key128 *keys, const int64_t *bead_off, int64_t m, int max_depth,
                         int64_t n_internal, int32_t *kfirst, int32_t *klast, int32_t *kgamma,
                         int32_t *cnt_stop) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n_internal) return;
  // body: largest j with bead_off[j] - j <= q
  int64_t lo = 0, hi = m;
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (bead_off[mid] - mid <= q) lo = mid; else hi = mid;
  }
  int j = (int)lo;
  int64_t base = bead_off[j];
  int n = (int)(bead_off[j + 1] - base);
  int i = (int)(q - (base - j));
  KarrasCtx c{keys + base, n, max_depth};
  int d = (c.delta(i, i + 1) - c.delta(i, i - 1)) > 0 ? 1 : -1;
  int dmin = c.delta(i, i - d);
  int lmax = 2;
  while (c.delta(i, i + lmax * d) > dmin) lmax <<= 1;
  int l = 0;
  for (int t = lmax >> 1; t >= 1; t >>= 1)
    if (c.delta(i, i + (l + t) * d) > dmin) l += t;
  int jj = i + l * d;
  int dnode = c.delta(i, jj);
  int s = 0;
  for (int div = 2;; div <<= 1) {
    int t = (l + div - 1) / div;
    if (c.delta(i, i + (s + t) * d) > dnode) s += t;
    if (t <= 1) break;
  }
  int gamma = i + s * d + (d < 0 ? -1 : 0);
  int first = min(i, jj), last = max(i, jj);
  kfirst[q] = first;
  klast[q] = last;
  kgamma[q] = gamma;
  atomicAdd(&cnt_stop[base + last], 1);  // internal node with stop = last + 1
}

struct TopoCtx {
  const int64_t *bead_off;
  const int32_t *cscan;  // inclusive scan of cnt_stop over all beads
  const int16_t *gap;
  __device__ int C(int j, int64_t base, int s) const {  // #internal nodes with stop <= s
    return s == 0 ? 0 : (int)(cscan[base + s - 1] - (base - j));
  }
  __device__ int g(int64_t base, int n, int k) const { return (k < 0 || k >= n - 1) ? -1 : gap[base + k]; }
};

__device__ __forceinline__ int16_t node_depth(const TopoCtx &t, int64_t base, int n, int s, int e) {
  int gl = t.g(base, n, s - 1), gr = t.g(base, n, e - 1);
  if (gl < 0 && gr < 0) return 0;  // root
  bool right = s > 0 && gl > gr;
  return (int16_t)((right ? gl : gr) + 1);
}

__global__ void k_topo_internal(TopoCtx t, const int64_t *node_off, int64_t m, const int32_t *kfirst,
                                const int32_t *klast, const int32_t *kgamma, int64_t n_internal,
                                int32_t *start, int32_t *stop, int32_t *left, int32_t *right,
                                int32_t *parent, int16_t *depth, int8_t *axis, uint8_t *flags) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= n_internal) return;
  int64_t lo = 0, hi = m;
  while (hi - lo > 1) {
    int64_t mid = (lo + hi) >> 1;
    if (t.bead_off[mid] - mid <= q) lo = mid; else hi = mid;
  }
  int j = (int)lo;
  int64_t base = t.bead_off[j];
  int n = (int)(t.bead_off[j + 1] - base);
  int first = kfirst[q], last = klast[q], gm = kgamma[q];
  int s = first, e = last + 1, L = e - s;
  int id = s + t.C(j, base, s) + 2 * L - 2;
  int Ll = gm - first + 1, Lr = last - gm;
  int idl = first + t.C(j, base, first) + 2 * Ll - 2;
  int idr = (gm + 1) + t.C(j, base, gm + 1) + 2 * Lr - 2;
  int64_t nb = node_off[j];
  start[nb + id] = s;
  stop[nb + id] = e;
  left[nb + id] = idl;
  right[nb + id] = idr;
  parent[nb + idl] = id;
  parent[nb + idr] = id;
  int lvl = t.g(base, n, gm);
  axis[nb + id] = (int8_t)c_axis_cycle[lvl % 3];
  depth[nb + id] = node_depth(t, base, n, s, e);
  int c = (Ll == 1 && Lr == 1) ? BEAD_BEAD : ((Ll == 1 || Lr == 1) ? RIGID_BEAD : GENERAL);
  flags[nb + id] = (uint8_t)(c | ((c == RIGID_BEAD && Ll == 1) ? 4 : 0));
}

__global__ void k_topo_leaf(TopoCtx t, const int64_t *node_off, const int32_t *body_of, int64_t N,
                            const double *pos_tree, int32_t *start, int32_t *stop, int32_t *left,
                            int32_t *right, int16_t *depth, int8_t *axis, uint8_t *flags,
                            double *centroid, int32_t *leaf_id) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  int j = body_of[i];
  int64_t base = t.bead_off[j];
  int n = (int)(t.bead_off[j + 1] - base);
  int li = (int)(i - base);
  int id = li + t.C(j, base, li);
  int64_t g = node_off[j] + id;
  start[g] = li;
  stop[g] = li + 1;
  left[g] = -1;
  right[g] = -1;
  axis[g] = -1;
  flags[g] = LEAF;
  depth[g] = n == 1 ? 0 : node_depth(t, base, n, li, li + 1);
  for (int a = 0; a < 3; a++) centroid[g * 3 + a] = pos_tree[i * 3 + a];
  leaf_id[i] = id;
}

// node -> body (binary search on node_off)
__global__ void k_node_sizes(const int64_t *node_off, int64_t m, int64_t NN, const uint8_t *flags,
                             int64_t *recsz, int32_t *rr, int32_t *node_body) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= NN) return;
  int c = flag_case(flags[g]);
  recsz[g] = rec_size(c);
  rr[g] = res_rows(c);
  node_body[g] = find_body(node_off, m, g);
}

__global__ void k_res_off(const int64_t *node_off, const int64_t *bead_off, const int32_t *node_body,
                          const int32_t *rr_scan, int64_t NN, int32_t *res_off) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= NN) return;
  int j = node_body[g];
  int64_t n = bead_off[j + 1] - bead_off[j];
  res_off[g] = rr_scan[g] - rr_scan[node_off[j]] + (n >= 2 ? 6 : 3);  // factor.py:198-204
}

// ---- 5. bottom-up factor pass (last arriver) --------------------------------------

struct FactorCtx {
  const int64_t *bead_off, *node_off;
  const int32_t *body_of, *leaf_id, *start, *stop, *left, *right, *parent;
  const double *pos_tree;
  const int64_t *rec_off;
  int32_t *counter, *height;
  uint8_t *flags;
  double *centroid, *t22, *rec;
};

__device__ inline void load_child(const FactorCtx &c, int64_t nb, int64_t base, int id, double cen[3],
                                  double t[9], int &L, int &h) {
  int64_t g = nb + id;
  L = c.stop[g] - c.start[g];
  if (L == 1) {
    for (int a = 0; a < 3; a++) cen[a] = c.pos_tree[(base + c.start[g]) * 3 + a];
    for (int a = 0; a < 9; a++) t[a] = 0.0;
    h = 0;
    return;
  }
  for (int a = 0; a < 3; a++) cen[a] = __ldcg(&c.centroid[g * 3 + a]);
  double p[6];
  for (int a = 0; a < 6; a++) p[a] = __ldcg(&c.t22[g * 6 + a]);
  t[0] = p[0]; t[1] = 0.0;  t[2] = 0.0;
  t[3] = p[1]; t[4] = p[2]; t[5] = 0.0;
  t[6] = p[3]; t[7] = p[4]; t[8] = p[5];
  h = __ldcg(&c.height[g]);
}

// One internal node (factor_all's per-node dispatch, factor.py:217-243); its children are done.
__device__ __forceinline__ void factor_node(const FactorCtx &c, int64_t base, int64_t nb, int64_t g) {
  int l = c.left[g], r = c.right[g];
  double cl[3], cr[3], tl[9], tr[9];
  int nl, nr, hl, hr;
  load_child(c, nb, base, l, cl, tl, nl, hl);
  load_child(c, nb, base, r, cr, tr, nr, hr);
  int n = nl + nr;
  double cp[3];
  for (int a = 0; a < 3; a++)  // tree.py:126
    cp[a] = ((double)nl * cl[a] + (double)nr * cr[a]) / (double)n;
  double t6[6];
  unsigned signs = 0;
  int cs = flag_case(c.flags[g]);
  double *rec = c.rec + c.rec_off[g];
  if (cs == BEAD_BEAD) {  // factor.py:224-225
    double d[3];
    for (int a = 0; a < 3; a++) d[a] = c.pos_tree[(base + c.start[nb + l]) * 3 + a] - cp[a];
    double gm[9];
    factor_bead_bead(d, t6, gm);
    for (int a = 0; a < 9; a++) rec[a] = gm[a];
  } else if (cs == RIGID_BEAD) {  // factor.py:226-236, 171-178
    bool sw = nl == 1;
    const double *cg = sw ? cr : cl;
    const double *tg = sw ? tr : tl;
    int nx = sw ? nr : nl;
    double dr[3], R[9];
    for (int a = 0; a < 3; a++) dr[a] = cg[a] - cp[a];
    skew3(dr, R);
    double sc = sqrt((double)((int64_t)nx * n));
    double cpl[18];
    for (int a = 0; a < 3; a++)
      for (int b = 0; b < 3; b++) {
        cpl[a * 6 + b] = tg[a * 3 + b];
        cpl[a * 6 + 3 + b] = sc * R[a * 3 + b];
      }
    double wy[WY<6>::SIZE];
    lq_factor<6>(cpl, t6, wy, signs);
    for (int a = 0; a < WY<6>::RA; a++) rec[a] = wy[a];
    rec[WY<6>::RA] = sqrt((double)nx / (double)n);  // NodeFactor.ratios (factor.py:85-87)
    rec[WY<6>::RB] = sqrt(1.0 / (double)n);
  } else {  // factor.py:237-243, 181-188
    double dr[3], R[9];
    for (int a = 0; a < 3; a++) dr[a] = cl[a] - cp[a];
    skew3(dr, R);
    double sc = sqrt((double)((int64_t)nl * n) / (double)nr);
    double cpl[27];
    for (int a = 0; a < 3; a++)
      for (int b = 0; b < 3; b++) {
        cpl[a * 9 + b] = tl[a * 3 + b];
        cpl[a * 9 + 3 + b] = tr[a * 3 + b];
        cpl[a * 9 + 6 + b] = sc * R[a * 3 + b];
      }
    double wy[WY<9>::SIZE];
    lq_factor<9>(cpl, t6, wy, signs);
    for (int a = 0; a < WY<9>::RA; a++) rec[a] = wy[a];
    rec[WY<9>::RA] = sqrt((double)nl / (double)n);
    rec[WY<9>::RB] = sqrt((double)nr / (double)n);
  }
  for (int a = 0; a < 3; a++) c.centroid[g * 3 + a] = cp[a];
  for (int a = 0; a < 6; a++) c.t22[g * 6 + a] = t6[a];
  c.height[g] = max(hl, hr) + 1;
  c.flags[g] = (uint8_t)((c.flags[g] & 7u) | (signs << 3));
}

// Internal nodes are factored level by level, deepest ghost depth first (a child's depth
// always exceeds its parent's, tree.py:116-123), each level's nodes ordered by case so the
// warps run one LQ shape (GEN 3x9, RB 3x6, BB closed form) without divergence.
// Sort key: (1023 - depth) << 2 | case rank; leaves get level 1024 (sorted last, skipped).
__global__ void k_factor_keys(const uint8_t *flags, const int32_t *start, const int32_t *stop,
                              const int16_t *depth, int64_t NN, uint32_t *key, int32_t *val) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= NN) return;
  uint32_t k = 1024u << 2;
  if (stop[g] - start[g] >= 2) {
    const int cs = flag_case(flags[g]);
    const uint32_t rank = cs == GENERAL ? 0u : (cs == RIGID_BEAD ? 1u : 2u);
    k = ((uint32_t)(1023 - min(1023, (int)depth[g])) << 2) | rank;
  }
  key[g] = k;
  val[g] = (int32_t)g;
}

// first sorted position of every depth-level key (bnd[L] for L = key >> 2; bnd sized 1025)
__global__ void k_level_bounds(const uint32_t *key, int64_t n, int32_t *bnd) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t L = key[i] >> 2;
  if (L > 1023u) return;
  if (i == 0 || (key[i - 1] >> 2) != L) bnd[L] = (int32_t)i;
}

__global__ void k_factor_level(FactorCtx c, const int32_t *order, const int32_t *node_body, int64_t b, int64_t e) {
  const int64_t i = b + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= e) return;
  const int64_t g = order[i];
  const int j = node_body[g];
  factor_node(c, c.bead_off[j], c.node_off[j], g);
}

// ---- 6. apply layout ------------------------------------------------------------

struct LayoutCtx {
  int S;
  int Hc;  // tile height cut (0: none): tiles are maximal subtrees with <= S leaves and height <= Hc
  const int64_t *bead_off, *node_off;
  const int32_t *node_body, *start, *stop, *parent, *height, *res_off;
  const int64_t *rec_off;
  const uint8_t *flags;
};

__device__ __forceinline__ int nodeL(const LayoutCtx &c, int64_t g) { return c.stop[g] - c.start[g]; }

// tile roots / top nodes / exchange slots
__global__ void k_classify(LayoutCtx c, int64_t NN, int32_t *is_tile, int32_t *is_slot, int32_t *is_top) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= NN) return;
  int j = c.node_body[g];
  int64_t nb = c.node_off[j];
  int L = nodeL(c, g);
  int p = c.parent[g];
  auto is_top_node = [&](int64_t q) { return nodeL(c, q) > c.S || (c.Hc > 0 && c.height[q] > c.Hc); };
  bool top = is_top_node(g);
  bool tile = !top && (p < 0 || is_top_node(nb + p));
  is_top[g] = top;
  is_tile[g] = tile;
  is_slot[g] = top || (tile && L >= 2);
}

struct TileTmp {
  int64_t root;      // global node id
  int32_t body, L, start, height;
};

__global__ void k_tiles(LayoutCtx c, int64_t NN, const int32_t *is_tile, const int32_t *tile_scan,
                        TileTmp *tiles, int32_t *marker) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= NN || !is_tile[g]) return;
  int t = tile_scan[g];  // exclusive
  int L = nodeL(c, g);
  int64_t first = g - 2 * L + 2;
  TileTmp T;
  T.root = g;
  T.body = c.node_body[g];
  T.L = L;
  T.start = c.start[g];
  T.height = c.height[g];
  tiles[t] = T;
  marker[first] = t;
}

__global__ void k_root_is_top(const int32_t *is_top, const int64_t *bead_off, const int64_t *node_off, int64_t m,
                              int32_t *out) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  const int64_t n = bead_off[j + 1] - bead_off[j];
  out[j] = is_top[node_off[j] + 2 * n - 2];
}

// tile renumbering after the per-body height sort
__global__ void k_tile_keys(const TileTmp *tiles, int64_t n, bool desc, uint64_t *key, int32_t *val) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  const uint32_t h = (uint32_t)min(tiles[t].height, 0xffff);
  key[t] = ((uint64_t)tiles[t].body << 16) | (desc ? 0xffffu - h : h);
  val[t] = (int32_t)t;
}

__global__ void k_tile_roots(const TileTmp *tiles, int64_t n, int64_t *roots) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) roots[t] = tiles[t].root;
}

__global__ void k_tile_permute(const TileTmp *tiles, const int32_t *order, int64_t n, TileTmp *sorted, int32_t *inv) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int32_t t = order[k];
  sorted[k] = tiles[t];
  inv[t] = (int32_t)k;
}

__global__ void k_count_big(const TileTmp *tiles, int64_t n, unsigned long long *cnt) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n && tiles[t].L >= 2) atomicAdd(cnt, 1ull);
}

__global__ void k_remap_tiles(int32_t *tile_of, int64_t NN, const int32_t *inv) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g < NN && tile_of[g] >= 0) tile_of[g] = inv[tile_of[g]];
}

// Sort key of a top node: (unit, height).  The unit is named by a node id: the body root for a
// whole top tree and for the apex of a split one (split_x[j] > 0: nodes with more than
// split_x[j] beads), else the root of the node's piece -- its highest ancestor with at most
// split_x[j] beads.
__global__ void k_top_fill(LayoutCtx c, int64_t NN, const int32_t *is_top, const int32_t *top_scan,
                           const int32_t *slot_scan, const int32_t *left, const int32_t *right,
                           const int64_t *split_x, TopNode *top, uint64_t *keys, int32_t *vals) {
  int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= NN || !is_top[g]) return;
  int t = top_scan[g];
  int j = c.node_body[g];
  int64_t nb = c.node_off[j];
  unsigned f = c.flags[g];
  int l = left[g], r = right[g];
  int xi = l, yi = r;
  if (flag_swapped(f)) { xi = r; yi = l; }
  auto ref = [&](int id) -> int32_t {
    int64_t cg = nb + id;
    int L = c.stop[cg] - c.start[cg];
    if (L == 1) return ~(int32_t)(c.bead_off[j] + c.start[cg]);
    return slot_scan[cg];
  };
  TopNode T;
  T.x = ref(xi);
  T.y = ref(yi);
  T.self_slot = slot_scan[g];
  int cs = flag_case(f);
  T.res_q = res_rows(cs) ? c.res_off[g] - 6 : -1;
  T.x_top = is_top[nb + xi];
  T.y_top = is_top[nb + yi];
  T.body = j;
  T.flags = (uint16_t)f;
  T.is_root = c.parent[g] < 0;
  T.rec_off = c.rec_off[g];
  top[t] = T;
  const int64_t root = nb + 2 * (c.bead_off[j + 1] - c.bead_off[j]) - 2;
  int64_t unit = root;
  const int64_t X = split_x[j];
  if (X > 0 && c.stop[g] - c.start[g] <= X) {
    unit = g;
    for (int64_t a = g; c.parent[a] >= 0;) {
      const int64_t pa = nb + c.parent[a];
      if (c.stop[pa] - c.start[pa] > X) break;
      unit = a = pa;
    }
  }
  keys[t] = ((uint64_t)unit << 32) | (uint64_t)c.height[g];
  vals[t] = t;
}

__global__ void k_top_gather(const TopNode *src, const int32_t *order, const uint64_t *keys_sorted,
                             int64_t n, TopNode *dst, int32_t *lvl_start_flag) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  dst[p] = src[order[p]];
  lvl_start_flag[p] = (p == 0 || keys_sorted[p] != keys_sorted[p - 1]) ? 1 : 0;
}

__global__ void k_top_unitflag(const uint64_t *keys_sorted, int64_t n, int32_t *uflag) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p < n) uflag[p] = (p == 0 || (keys_sorted[p] >> 32) != (keys_sorted[p - 1] >> 32)) ? 1 : 0;
}
// exclusive scan of the unit-start flags -> unit index of every node (inclusive scan - 1)
__global__ void k_top_unitfix(const int32_t *uflag, int64_t n, int32_t *tunit) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p < n) tunit[p] += uflag[p] - 1;
}

// level starts; per unit (at its first node): first level, body and kind (0 whole top tree,
// 1 piece, 2 apex)
__global__ void k_top_levels(const uint64_t *keys_sorted, const int32_t *flag, const int32_t *lvl_scan,
                             const int32_t *uflag, const int32_t *tunit, const TopNode *top, const int64_t *split_x,
                             const int64_t *bead_off, const int64_t *node_off, int64_t n, int32_t *toplvl,
                             int32_t *unit_lvl, int32_t *unit_body, int32_t *unit_kind) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n || !flag[p]) return;
  int lv = lvl_scan[p];
  toplvl[lv] = (int32_t)p;
  if (uflag[p]) {
    const int u = tunit[p];
    const int j = top[p].body;
    unit_lvl[u] = lv;
    unit_body[u] = j;
    const int64_t root = node_off[j] + 2 * (bead_off[j + 1] - bead_off[j]) - 2;
    unit_kind[u] = split_x[j] == 0 ? 0 : ((int64_t)(keys_sorted[p] >> 32) == root ? 2 : 1);
  }
}


// ---- staged top-tree blobs ------------------------------------------------------------

// top trees too large for shared memory (k_top_df): parent links and start nodes
__global__ void k_top_slot2top(const TopNode *top, int64_t nt, int32_t *slot2top) {
  int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q < nt) slot2top[top[q].self_slot] = (int32_t)q;
}
__global__ void k_top_links(const TopNode *top, int64_t q0, int64_t q1, const int32_t *slot2top, int32_t *parent,
                            int32_t *is_start, int32_t *need) {
  int64_t q = q0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= q1) return;
  const TopNode T = top[q];
  const int32_t cx = T.x >= 0 ? slot2top[T.x] : -1, cy = T.y >= 0 ? slot2top[T.y] : -1;
  if (cx >= 0) parent[cx] = (int32_t)q;
  if (cy >= 0) parent[cy] = (int32_t)q;
  is_start[q] = cx < 0 && cy < 0;
  need[q] = (cx >= 0) + (cy >= 0);  // arrivals before the node can be merged
}

__global__ void k_top_path_len(const int32_t *parent, const int32_t *starts, int64_t n, int64_t *len) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t l = 1;
  for (int q = starts[i]; parent[q] >= 0; q = parent[q]) l++;
  len[i] = l;
}
__global__ void k_top_path_write(const int32_t *parent, const int32_t *starts, int64_t n, const int64_t *off,
                                 int32_t *paths) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t w = off[i + 1] - 1;  // start node last, root first
  for (int q = starts[i];; q = parent[q]) {
    paths[w--] = q;
    if (parent[q] < 0) break;
  }
}

__global__ void k_top_slotmap(const TopNode *top, int64_t nt, const int32_t *tunit, const int32_t *unit_lvl,
                              const int32_t *toplvl, int32_t *slot_to_local, int32_t *slot_unit, int64_t *recsz) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nt) return;
  const TopNode T = top[p];
  const int u = tunit[p];
  const int first = toplvl[unit_lvl[u]];
  slot_to_local[T.self_slot] = (int32_t)(p - first);
  slot_unit[T.self_slot] = u;
  recsz[p] = rec_size(flag_case(T.flags));
}

// children outside the node's unit (tile roots, beads, piece roots under an apex) are inputs
__global__ void k_top_inputs(const TopNode *top, int64_t nt, const int32_t *slot_unit, const int32_t *tunit,
                             int32_t *nin) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nt) return;
  const TopNode T = top[p];
  const int u = tunit[p];
  int c = 0;
  if (T.x < 0 || slot_unit[T.x] != u) c++;
  if (T.y < 0 || slot_unit[T.y] != u) c++;
  nin[p] = c;
}

__host__ __device__ inline int64_t topblob_bytes(int n_nodes, int n_levels, int n_inputs, int64_t rec) {
  int64_t b = sizeof(TopHdr);
  b += ((int64_t)(n_levels + 1) * 4 + 15) / 16 * 16;
  b += (int64_t)n_nodes * sizeof(TopMeta);
  b += ((int64_t)n_inputs * 4 + 15) / 16 * 16;
  b += rec * 8;
  return (b + 15) / 16 * 16;
}

// one thread per top node: writes its meta, inputs and record; the body's first
// node also writes the header and level table
__global__ void k_top_blob(const TopNode *top, int64_t nt, const int32_t *tunit, const int32_t *unit_lvl,
                           const int32_t *unit_kind, const int32_t *toplvl, const int32_t *slot_to_local,
                           const int32_t *slot_unit, const int32_t *in_scan, const int64_t *rec_scan,
                           const int64_t *blob_off_of_tb, const double *rec, const int32_t *perm,
                           const int64_t *bead_off, uint8_t *blob) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= nt) return;
  const TopNode T = top[p];
  const int bi = tunit[p];
  const int lv0 = unit_lvl[bi], lv1 = unit_lvl[bi + 1];
  const int first = toplvl[lv0], last = toplvl[lv1];
  const int n_nodes = last - first, n_levels = lv1 - lv0;
  const int n_inputs = in_scan[last] - in_scan[first];
  const int64_t n_rec = rec_scan[last] - rec_scan[first];
  uint8_t *B = blob + blob_off_of_tb[bi];
  TopHdr h;
  h.n_nodes = n_nodes;
  h.n_levels = n_levels;
  h.n_inputs = n_inputs;
  h.body = T.body;
  h.off_meta = (int32_t)(sizeof(TopHdr) + ((int64_t)(n_levels + 1) * 4 + 15) / 16 * 16);
  h.off_in = h.off_meta + n_nodes * (int32_t)sizeof(TopMeta);
  h.off_rec = h.off_in + (int32_t)(((int64_t)n_inputs * 4 + 15) / 16 * 16);
  h.bytes = (int32_t)topblob_bytes(n_nodes, n_levels, n_inputs, n_rec);
  const bool piece = unit_kind[bi] == 1;
  h.root_slot = piece ? top[last - 1].self_slot : -1;  // nodes by height: the unit root is last
  h.pad[0] = h.pad[1] = h.pad[2] = 0;
  const int local = (int)(p - first);
  if (local == 0) {
    *reinterpret_cast<TopHdr *>(B) = h;
    int32_t *lv = reinterpret_cast<int32_t *>(B + sizeof(TopHdr));
    for (int l = 0; l <= n_levels; l++) lv[l] = toplvl[lv0 + l] - first;
  }
  int32_t *IN = reinterpret_cast<int32_t *>(B + h.off_in);
  int in_i = in_scan[p] - in_scan[first];
  auto ref = [&](int32_t c) -> int16_t {
    if (c >= 0 && slot_unit[c] == bi) return (int16_t)slot_to_local[c];
    IN[in_i] = c >= 0 ? c : ~perm[~(int64_t)c];  // slot, or ~(body-local original bead index)
    return (int16_t)~in_i++;
  };
  TopMeta md;
  md.x = ref(T.x);
  md.y = ref(T.y);
  md.flags = T.flags;
  md.is_root = T.is_root ? 1 : ((piece && local == n_nodes - 1) ? 2 : 0);
  md.res_q = T.res_q;
  md.rec = (int32_t)(rec_scan[p] - rec_scan[first]);
  reinterpret_cast<TopMeta *>(B + h.off_meta)[local] = md;
  double *R = reinterpret_cast<double *>(B + h.off_rec) + md.rec;
  const int rs = rec_size(flag_case(T.flags));
  for (int e = 0; e < rs; e++) R[e] = rec[T.rec_off + e];
  (void)bead_off;
}

// ---- helpers ------------------------------------------------------------------------

// node count per case (flags & 3), grid-stride with a shared-memory histogram
__global__ void k_case_count(const uint8_t *flags, int64_t NN, unsigned long long *cnt) {
  __shared__ unsigned int h[4];
  if (threadIdx.x < 4) h[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < NN; g += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&h[flags[g] & 3], 1u);
  __syncthreads();
  if (threadIdx.x < 4) atomicAdd(&cnt[threadIdx.x], (unsigned long long)h[threadIdx.x]);
}

// Host -> device copy of a (possibly pageable) host array.  Pageable cudaMemcpyAsync runs
// at ~8 GB/s on the B200 hosts; here RQ_H2D_THREADS host threads (8) copy 4 MiB pieces into
// their own pair of pinned slots and queue the DMA of each piece on the stream, so host
// copies and PCIe transfers overlap.  Pinned (page-locked / registered) sources and small
// arrays take the plain path.  The slots are allocated once per process.
void h2d_host(void *dst, const void *src, size_t bytes, cudaStream_t s) {
  constexpr size_t C = size_t(4) << 20;
  cudaPointerAttributes at{};
  const bool pinned = cudaPointerGetAttributes(&at, src) == cudaSuccess && at.type == cudaMemoryTypeHost;
  cudaGetLastError();  // clear a possible error from the attribute query on plain malloc'd memory
  int T = (int)std::min(8u, std::max(1u, std::thread::hardware_concurrency()));
  if (const char *e = getenv("RQ_H2D_THREADS")) T = std::max(0, std::min(16, atoi(e)));
  if (pinned || bytes < 4 * C || T == 0) {
    RQ_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
    return;
  }
  static std::mutex mu;
  static std::vector<void *> slot;
  static std::vector<cudaEvent_t> ev;
  std::lock_guard<std::mutex> lock(mu);
  while ((int)slot.size() < 2 * T) {
    void *h = nullptr;
    cudaEvent_t e;
    RQ_CUDA(cudaHostAlloc(&h, C, cudaHostAllocPortable));
    RQ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    RQ_CUDA(cudaEventRecord(e, s));
    slot.push_back(h);
    ev.push_back(e);
  }
  const size_t pieces = (bytes + C - 1) / C;
  std::vector<std::thread> th;
  std::vector<int> fail(T, 0);
  for (int t = 0; t < T; t++) {
    th.emplace_back([&, t]() {
      int use = 0;  // thread t owns slots 2t and 2t+1
      for (size_t i = (size_t)t; i < pieces; i += (size_t)T, use ^= 1) {
        const int sl = 2 * t + use;
        const size_t off = i * C, len = std::min(C, bytes - off);
        if (cudaEventSynchronize(ev[sl]) != cudaSuccess) { fail[t] = 1; return; }
        stage_copy(slot[sl], (const char *)src + off, len);
        if (cudaMemcpyAsync((char *)dst + off, slot[sl], len, cudaMemcpyHostToDevice, s) != cudaSuccess ||
            cudaEventRecord(ev[sl], s) != cudaSuccess) { fail[t] = 1; return; }
      }
    });
  }
  for (auto &x : th) x.join();
  for (int t = 0; t < T; t++)
    if (fail[t]) throw Error(RQ_ERR_CUDA, "staged host-to-device copy failed");
  // the slots are reused by the next call only after their events complete
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

template <class In, class Out>
void exclusive_scan(const In *in, Out *out, int64_t n, cudaStream_t s) {
  size_t tb = 0;
  RQ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, s));
  DBuf tmp;
  tmp.alloc(tb);
  RQ_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, n, s));
}

template <class In, class Out>
void inclusive_scan(const In *in, Out *out, int64_t n, cudaStream_t s) {
  size_t tb = 0;
  RQ_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, in, out, n, s));
  DBuf tmp;
  tmp.alloc(tb);
  RQ_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, tb, in, out, n, s));
}

struct MaxOp {
  __device__ int32_t operator()(int32_t a, int32_t b) const { return a > b ? a : b; }
};


// ---- duplicate-bead check (model.py:65-78) ----------------------------------------
// Hash grid with cell h = 64 * tol: a pair within tol lies in cells that the
// probe box [p - tol, p + tol] touches (<= 2 per axis, usually 1).

struct DupCtx {
  const double *pos;
  const int32_t *body_of;
  const int64_t *bead_off;
  const unsigned long long *bmin, *bmax;
  int32_t *table;
  uint64_t mask;
  unsigned long long *hit;  // per body: (i << 32) | j, min
  long long *err;
};

__device__ __forceinline__ void dup_params(const DupCtx &c, int j, double &tol, double lo[3]) {
  double d2 = 0.0;
  for (int a = 0; a < 3; a++) {
    lo[a] = unord_key(c.bmin[j * 3 + a]);
    double e = unord_key(c.bmax[j * 3 + a]) - lo[a];
    d2 += e * e;
  }
  tol = 1e-12 * sqrt(d2);
}

__device__ __forceinline__ uint64_t cell_hash(int j, long long x, long long y, long long z) {
  uint64_t h = (uint64_t)j * 0x9E3779B97F4A7C15ull;
  h ^= (uint64_t)x * 0xC2B2AE3D27D4EB4Full; h = (h << 31) | (h >> 33);
  h ^= (uint64_t)y * 0x165667B19E3779F9ull; h = (h << 29) | (h >> 35);
  h ^= (uint64_t)z * 0x27D4EB2F165667C5ull;
  h ^= h >> 33; h *= 0xff51afd7ed558ccdull; h ^= h >> 33;
  return h;
}

__device__ __forceinline__ long long cell_of(double x, double lo, double h) { return (long long)floor((x - lo) / h); }

__global__ void k_dup_insert(DupCtx c, int64_t N) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  int j = c.body_of[i];
  int64_t n = c.bead_off[j + 1] - c.bead_off[j];
  if (n < 2) return;
  double tol, lo[3];
  dup_params(c, j, tol, lo);
  if (tol == 0.0) { atomicMin((unsigned long long *)&c.err[2], (unsigned long long)j); return; }
  double h = 64.0 * tol;
  long long q[3];
  for (int a = 0; a < 3; a++) q[a] = cell_of(c.pos[i * 3 + a], lo[a], h);
  uint64_t s = cell_hash(j, q[0], q[1], q[2]) & c.mask;
  while (atomicCAS(&c.table[s], -1, (int32_t)i) != -1) s = (s + 1) & c.mask;
}

__global__ void k_dup_query(DupCtx c, int64_t N) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  int j = c.body_of[i];
  int64_t base = c.bead_off[j];
  int64_t n = c.bead_off[j + 1] - base;
  if (n < 2) return;
  double tol, lo[3];
  dup_params(c, j, tol, lo);
  if (tol == 0.0) return;
  double h = 64.0 * tol;
  double p[3];
  long long qlo[3], qhi[3];
  for (int a = 0; a < 3; a++) {
    p[a] = c.pos[i * 3 + a];
    qlo[a] = cell_of(p[a] - tol, lo[a], h);
    qhi[a] = cell_of(p[a] + tol, lo[a], h);
  }
  for (long long x = qlo[0]; x <= qhi[0]; x++)
    for (long long y = qlo[1]; y <= qhi[1]; y++)
      for (long long z = qlo[2]; z <= qhi[2]; z++) {
        uint64_t s = cell_hash(j, x, y, z) & c.mask;
        for (;;) {
          int32_t e = c.table[s];
          if (e < 0) break;
          if (e != i && c.body_of[e] == j) {
            double d2 = 0.0, q[3];
            bool same = true;
            for (int a = 0; a < 3; a++) {
              q[a] = c.pos[(int64_t)e * 3 + a];
              double dd = q[a] - p[a];
              d2 += dd * dd;
            }
            same = cell_of(q[0], lo[0], h) == x && cell_of(q[1], lo[1], h) == y && cell_of(q[2], lo[2], h) == z;
            if (same && sqrt(d2) <= tol) {
              unsigned long long a0 = (unsigned long long)(min((int64_t)e, i) - base);
              unsigned long long b0 = (unsigned long long)(max((int64_t)e, i) - base);
              atomicMin(&c.hit[j], (a0 << 32) | b0);
            }
          }
          s = (s + 1) & c.mask;
        }
      }
}

}  // namespace

int64_t Plan::device_bytes() const {
  const DBuf *bufs[] = {&bead_off_d, &node_off_d, &body_centroid, &root_box, &perm, &pos_tree,
                        &pos_orig, &body_of, &start, &stop, &left, &right, &parent, &depth, &axis,
                        &flags, &height, &centroid, &t22, &rec_off, &res_off, &rec, &top, &topbody, &topbody_lvl, &toplvl, &small_bodies, &err, &seg_body, &seg_begin, &body_seg, &topblob, &topblob_off, &topblob_body, &topblob_class, &topblob_order, &topbig, &top_parent, &top_need, &top_start, &top_paths, &top_path_off, &mrhs_units, &mrhs_prog,
                        &res_base_d, &wave_desc, &wave_stream_first, &wave_blob};
  int64_t s = 0;
  for (auto b : bufs) s += (int64_t)b->bytes;
  return s;
}

void compute_body_centroids(Plan &p, cudaStream_t s);  // rq_z.cu


void build_plan(Plan &p, const double *pos_in, const int64_t *offsets, int64_t m, int max_depth,
                bool host_input, cudaStream_t s) {
  SetupTimer tm(s);
  if (m < 1) throw Error(RQ_ERR_VALUE, "need at least one body");
  if (offsets[0] != 0) throw Error(RQ_ERR_VALUE, "offsets[0] must be 0");
  for (int64_t j = 0; j < m; j++)
    if (offsets[j + 1] <= offsets[j])
      throw Error(RQ_ERR_VALUE, "positions must be (n, 3) with n >= 1 for every body");
  const int64_t N = offsets[m];
  if (N >= (int64_t(1) << 30)) throw Error(RQ_ERR_VALUE, "too many beads for one plan (>= 2^30)");
  int body_bits = 0;
  while ((int64_t(1) << body_bits) < m) body_bits++;
  if (max_depth < 1 || max_depth + body_bits > 128)
    throw Error(RQ_ERR_VALUE, "max_depth must be in [1, 128 - ceil(log2 m)]");
  if (const char *e = getenv("RQ_TILE_LEAVES")) p.tile_leaves = std::min(1024, std::max(2, atoi(e)));
  if (const char *e = getenv("RQ_TILE_HEIGHT")) p.tile_height = std::max(0, atoi(e));
  if (const char *e = getenv("RQ_MRHS_MIN")) p.mrhs_min = std::max(2, atoi(e));
  if (const char *e = getenv("RQ_MRHS_TILE")) p.mrhs_tile = std::max(2, std::min(4096, atoi(e)));
  p.m = m;
  p.N = N;
  p.NN = 2 * N - m;
  p.max_depth = max_depth;
  p.bead_off.assign(offsets, offsets + m + 1);
  const int64_t NN = p.NN;
  std::vector<int64_t> node_off(m + 1);
  p.min_n = N;
  for (int64_t j = 0; j <= m; j++) node_off[j] = 2 * offsets[j] - j;
  for (int64_t j = 0; j < m; j++) p.min_n = std::min<int64_t>(p.min_n, offsets[j + 1] - offsets[j]);

  p.bead_off_d.alloc((m + 1) * 8);
  p.node_off_d.alloc((m + 1) * 8);
  p.res_base.assign(m + 1, 0);
  for (int64_t j = 0; j < m; j++) p.res_base[j + 1] = p.res_base[j] + std::max<int64_t>(0, 3 * (offsets[j + 1] - offsets[j]) - 6);
  p.res_base_d.alloc((m + 1) * 8);
  RQ_CUDA(cudaMemcpyAsync(p.res_base_d.p, p.res_base.data(), (m + 1) * 8, cudaMemcpyHostToDevice, s));
  RQ_CUDA(cudaMemcpyAsync(p.bead_off_d.p, offsets, (m + 1) * 8, cudaMemcpyHostToDevice, s));
  RQ_CUDA(cudaMemcpyAsync(p.node_off_d.p, node_off.data(), (m + 1) * 8, cudaMemcpyHostToDevice, s));
  p.pos_orig.alloc(N * 24);
  if (host_input) h2d_host(p.pos_orig.p, pos_in, N * 24, s);
  else RQ_CUDA(cudaMemcpyAsync(p.pos_orig.p, pos_in, N * 24, cudaMemcpyDeviceToDevice, s));
  p.err.alloc(8 * 8);
  {
    long long init[8] = {0x7fffffffffffffffLL, 0, 0, 0, 0, 0, 0, 0};
    RQ_CUDA(cudaMemcpyAsync(p.err.p, init, sizeof(init), cudaMemcpyHostToDevice, s));
  }
  const int64_t *boff = p.bead_off_d.as<int64_t>();
  const int64_t *noff = p.node_off_d.as<int64_t>();
  long long *err = p.err.as<long long>();
  const double *pos = p.pos_orig.as<double>();

  // 1. bodies + bounding cube
  p.body_of.alloc(N * 4);
  k_body_of<<<nblk(N), NT, 0, s>>>(boff, m, N, p.body_of.as<int32_t>());
  DBuf bmin, bmax;
  bmin.alloc(m * 24);
  bmax.alloc(m * 24);
  RQ_CUDA(cudaMemsetAsync(bmin.p, 0xff, m * 24, s));
  RQ_CUDA(cudaMemsetAsync(bmax.p, 0x00, m * 24, s));
  k_bbox<<<nblk(N), NT, 0, s>>>(pos, p.body_of.as<int32_t>(), N, bmin.as<unsigned long long>(),
                                 bmax.as<unsigned long long>(), err);
  p.root_box.alloc(m * 48);
  k_root_box<<<nblk(m), NT, 0, s>>>(bmin.as<unsigned long long>(), bmax.as<unsigned long long>(), m,
                                     p.root_box.as<double>());
  {
    long long e[2];
    d2h(e, err, 2, s);
    if (e[1]) throw Error(RQ_ERR_VALUE, "positions must be finite");
  }
  compute_body_centroids(p, s);

  tm.mark("bbox");
  // 2-3. keys + sort
  {
    DBuf keys, vals, keys2, vals2;
    keys.alloc(N * 16);
    vals.alloc(N * 4);
    keys2.alloc(N * 16);
    vals2.alloc(N * 4);
    k_keys<<<nblk(N), NT, 0, s>>>(pos, p.body_of.as<int32_t>(), p.root_box.as<double>(), N, max_depth,
                                   max_depth, keys.as<Key128>(), vals.as<int32_t>());
    int end_bit = max_depth + body_bits;
    size_t tb = 0;
    RQ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.as<Key128>(), keys2.as<Key128>(),
                                            vals.as<int32_t>(), vals2.as<int32_t>(), (int)N, KeyDec{},
                                            0, end_bit, s));
    DBuf tmp;
    tmp.alloc(tb);
    RQ_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, keys.as<Key128>(), keys2.as<Key128>(),
                                            vals.as<int32_t>(), vals2.as<int32_t>(), (int)N, KeyDec{},
                                            0, end_bit, s));
    tmp.reset();
    keys.reset();
    vals.reset();
    p.perm.alloc(N * 4);
    p.pos_tree.alloc(N * 24);
    DBuf gap;
    gap.alloc(N * 2);
    k_post_sort<<<nblk(N), NT, 0, s>>>(keys2.as<Key128>(), vals2.as<int32_t>(), pos, boff,
                                        p.body_of.as<int32_t>(), N, max_depth, p.perm.as<int32_t>(),
                                        p.pos_tree.as<double>(), gap.as<int16_t>(), err);
    long long dup = d2h1<long long>(err, s);
    if (dup != 0x7fffffffffffffffLL)
      throw Error(RQ_ERR_DUPLICATE, "body " + std::to_string(dup) +
                                        ": split depth " + std::to_string(max_depth) +
                                        " exceeded without separating beads (near-coincident input)");

    tm.mark("keys+sort");
    // 4. topology
    const int64_t n_internal = N - m;
    p.start.alloc(NN * 4);
    p.stop.alloc(NN * 4);
    p.left.alloc(NN * 4);
    p.right.alloc(NN * 4);
    p.parent.alloc(NN * 4);
    p.depth.alloc(NN * 2);
    p.axis.alloc(NN);
    p.flags.alloc(NN);
    p.centroid.alloc(NN * 24);
    RQ_CUDA(cudaMemsetAsync(p.parent.p, 0xff, NN * 4, s));
    DBuf cnt, cscan, leaf_id;
    cnt.alloc(N * 4);
    cscan.alloc(N * 4);
    leaf_id.alloc(N * 4);
    RQ_CUDA(cudaMemsetAsync(cnt.p, 0, N * 4, s));
    DBuf kfirst, klast, kgamma;
    kfirst.alloc(std::max<int64_t>(n_internal, 1) * 4);
    klast.alloc(std::max<int64_t>(n_internal, 1) * 4);
    kgamma.alloc(std::max<int64_t>(n_internal, 1) * 4);
    if (n_internal > 0)
      k_karras<<<nblk(n_internal), NT, 0, s>>>(keys2.as<Key128>(), boff, m, max_depth, n_internal,
                                                kfirst.as<int32_t>(), klast.as<int32_t>(),
                                                kgamma.as<int32_t>(), cnt.as<int32_t>());
    inclusive_scan(cnt.as<int32_t>(), cscan.as<int32_t>(), N, s);
    TopoCtx tc{boff, cscan.as<int32_t>(), gap.as<int16_t>()};
    if (n_internal > 0)
      k_topo_internal<<<nblk(n_internal), NT, 0, s>>>(
          tc, noff, m, kfirst.as<int32_t>(), klast.as<int32_t>(), kgamma.as<int32_t>(), n_internal,
          p.start.as<int32_t>(), p.stop.as<int32_t>(), p.left.as<int32_t>(), p.right.as<int32_t>(),
          p.parent.as<int32_t>(), p.depth.as<int16_t>(), p.axis.as<int8_t>(), p.flags.as<uint8_t>());
    k_topo_leaf<<<nblk(N), NT, 0, s>>>(tc, noff, p.body_of.as<int32_t>(), N, p.pos_tree.as<double>(),
                                        p.start.as<int32_t>(), p.stop.as<int32_t>(), p.left.as<int32_t>(),
                                        p.right.as<int32_t>(), p.depth.as<int16_t>(), p.axis.as<int8_t>(),
                                        p.flags.as<uint8_t>(), p.centroid.as<double>(),
                                        leaf_id.as<int32_t>());
    keys2.reset();
    vals2.reset();

    tm.mark("topology");
    // sizes, residue and record offsets
    DBuf recsz, rr, rr_scan, node_body;
    recsz.alloc(NN * 8);
    rr.alloc(NN * 4);
    rr_scan.alloc(NN * 4);
    node_body.alloc(NN * 4);
    k_node_sizes<<<nblk(NN), NT, 0, s>>>(noff, m, NN, p.flags.as<uint8_t>(), recsz.as<int64_t>(),
                                          rr.as<int32_t>(), node_body.as<int32_t>());
    p.rec_off.alloc((NN + 1) * 8);
    exclusive_scan(recsz.as<int64_t>(), p.rec_off.as<int64_t>(), NN, s);
    exclusive_scan(rr.as<int32_t>(), rr_scan.as<int32_t>(), NN, s);
    p.res_off.alloc(NN * 4);
    k_res_off<<<nblk(NN), NT, 0, s>>>(noff, boff, node_body.as<int32_t>(), rr_scan.as<int32_t>(), NN,
                                       p.res_off.as<int32_t>());
    {
      int64_t last_off = d2h1<int64_t>(p.rec_off.as<int64_t>() + NN - 1, s);
      int64_t last_sz = d2h1<int64_t>(recsz.as<int64_t>() + NN - 1, s);
      p.rec_doubles = last_off + last_sz;
    }
    RQ_CUDA(cudaMemcpyAsync(p.rec_off.as<int64_t>() + NN, &p.rec_doubles, 8, cudaMemcpyHostToDevice, s));
    recsz.reset();
    rr.reset();
    rr_scan.reset();

    tm.mark("offsets");
    // 5. factors
    p.t22.alloc(NN * 48);
    p.rec.alloc(std::max<int64_t>(p.rec_doubles, 1) * 8);
    RQ_CUDA(cudaMemsetAsync(p.rec.p, 0, std::max<int64_t>(p.rec_doubles, 1) * 8, s));
    p.height.alloc(NN * 4);
    RQ_CUDA(cudaMemsetAsync(p.height.p, 0, NN * 4, s));
    RQ_CUDA(cudaMemsetAsync(p.t22.p, 0, NN * 48, s));
    {
      DBuf counter;
      FactorCtx fc{boff,
                   noff,
                   p.body_of.as<int32_t>(),
                   leaf_id.as<int32_t>(),
                   p.start.as<int32_t>(),
                   p.stop.as<int32_t>(),
                   p.left.as<int32_t>(),
                   p.right.as<int32_t>(),
                   p.parent.as<int32_t>(),
                   p.pos_tree.as<double>(),
                   p.rec_off.as<int64_t>(),
                   counter.as<int32_t>(),
                   p.height.as<int32_t>(),
                   p.flags.as<uint8_t>(),
                   p.centroid.as<double>(),
                   p.t22.as<double>(),
                   p.rec.as<double>()};
      // level order: sort internal nodes by (deepest first, case), one launch per level
      DBuf fkey, fval, fkey2, fval2, bnd;
      fkey.alloc(NN * 4);
      fval.alloc(NN * 4);
      fkey2.alloc(NN * 4);
      fval2.alloc(NN * 4);
      bnd.alloc(1025 * 4);
      k_factor_keys<<<nblk(NN), NT, 0, s>>>(p.flags.as<uint8_t>(), p.start.as<int32_t>(), p.stop.as<int32_t>(),
                                             p.depth.as<int16_t>(), NN, fkey.as<uint32_t>(), fval.as<int32_t>());
      size_t tb = 0;
      RQ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, fkey.as<uint32_t>(), fkey2.as<uint32_t>(),
                                              fval.as<int32_t>(), fval2.as<int32_t>(), (int)NN, 0, 13, s));
      DBuf tmp;
      tmp.alloc(tb);
      RQ_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, fkey.as<uint32_t>(), fkey2.as<uint32_t>(),
                                              fval.as<int32_t>(), fval2.as<int32_t>(), (int)NN, 0, 13, s));
      RQ_CUDA(cudaMemsetAsync(bnd.p, 0xff, 1025 * 4, s));
      k_level_bounds<<<nblk(NN), NT, 0, s>>>(fkey2.as<uint32_t>(), NN, bnd.as<int32_t>());
      std::vector<int32_t> hb(1024);
      d2h(hb.data(), bnd.as<int32_t>(), 1024, s);
      std::vector<int64_t> lv;
      for (int L = 0; L < 1024; L++)
        if (hb[L] >= 0) lv.push_back(hb[L]);
      lv.push_back(n_internal);
      for (size_t i = 0; i + 1 < lv.size(); i++)
        k_factor_level<<<nblk(lv[i + 1] - lv[i], 128), 128, 0, s>>>(fc, fval2.as<int32_t>(), node_body.as<int32_t>(),
                                                                    lv[i], lv[i + 1]);
      RQ_CUDA(cudaGetLastError());
      RQ_CUDA(cudaStreamSynchronize(s));
    }

    tm.mark("factors");
    // 6. apply layout
    const int S = p.tile_leaves;
    LayoutCtx lc{S,
                 p.tile_height,
                 boff,
                 noff,
                 node_body.as<int32_t>(),
                 p.start.as<int32_t>(),
                 p.stop.as<int32_t>(),
                 p.parent.as<int32_t>(),
                 p.height.as<int32_t>(),
                 p.res_off.as<int32_t>(),
                 p.rec_off.as<int64_t>(),
                 p.flags.as<uint8_t>()};
    DBuf is_tile, is_slot, is_top, tile_scan, slot_scan, top_scan;
    is_tile.alloc(NN * 4);
    is_slot.alloc(NN * 4);
    is_top.alloc(NN * 4);
    tile_scan.alloc(NN * 4);
    slot_scan.alloc(NN * 4);
    top_scan.alloc(NN * 4);
    k_classify<<<nblk(NN), NT, 0, s>>>(lc, NN, is_tile.as<int32_t>(), is_slot.as<int32_t>(),
                                        is_top.as<int32_t>());
    exclusive_scan(is_tile.as<int32_t>(), tile_scan.as<int32_t>(), NN, s);
    exclusive_scan(is_slot.as<int32_t>(), slot_scan.as<int32_t>(), NN, s);
    exclusive_scan(is_top.as<int32_t>(), top_scan.as<int32_t>(), NN, s);
    auto count_of = [&](DBuf &flag, DBuf &scan) {
      return (int64_t)d2h1<int32_t>(scan.as<int32_t>() + NN - 1, s) +
             d2h1<int32_t>(flag.as<int32_t>() + NN - 1, s);
    };
    const int64_t n_tiles_all = count_of(is_tile, tile_scan);
    p.n_slots = count_of(is_slot, slot_scan);
    p.n_top = count_of(is_top, top_scan);

    DBuf tiles_tmp, marker, tile_of;
    tiles_tmp.alloc(n_tiles_all * sizeof(TileTmp));
    marker.alloc(NN * 4);
    tile_of.alloc(NN * 4);
    RQ_CUDA(cudaMemsetAsync(marker.p, 0xff, NN * 4, s));
    k_tiles<<<nblk(NN), NT, 0, s>>>(lc, NN, is_tile.as<int32_t>(), tile_scan.as<int32_t>(),
                                     tiles_tmp.as<TileTmp>(), marker.as<int32_t>());
    {
      size_t tb = 0;
      RQ_CUDA(cub::DeviceScan::InclusiveScan(nullptr, tb, marker.as<int32_t>(), tile_of.as<int32_t>(),
                                             MaxOp{}, NN, s));
      DBuf tmp;
      tmp.alloc(tb);
      RQ_CUDA(cub::DeviceScan::InclusiveScan(tmp.p, tb, marker.as<int32_t>(), tile_of.as<int32_t>(),
                                             MaxOp{}, NN, s));
    }
    tm.mark("tiles");
    // Tiles in body order; inside a body optionally ordered by height (stable radix sort on
    // (body, height), RQ_TILE_SORT=1; =2 descending).  The wave placement fills the steps
    // either way; the default keeps postorder.
    {
      const char *es = getenv("RQ_TILE_SORT");
      const int mode = es ? atoi(es) : 0;
      if (mode != 0 && n_tiles_all > 1) {
        DBuf tkey, tval, tkey2, tval2, sorted, inv;
        tkey.alloc(n_tiles_all * 8);
        tval.alloc(n_tiles_all * 4);
        tkey2.alloc(n_tiles_all * 8);
        tval2.alloc(n_tiles_all * 4);
        sorted.alloc(n_tiles_all * sizeof(TileTmp));
        inv.alloc(n_tiles_all * 4);
        k_tile_keys<<<nblk(n_tiles_all), NT, 0, s>>>(tiles_tmp.as<TileTmp>(), n_tiles_all, mode == 2,
                                                     tkey.as<uint64_t>(), tval.as<int32_t>());
        int end_bit = 16 + body_bits + 1;
        size_t tb = 0;
        RQ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, tkey.as<uint64_t>(), tkey2.as<uint64_t>(),
                                                tval.as<int32_t>(), tval2.as<int32_t>(), (int)n_tiles_all, 0,
                                                end_bit, s));
        DBuf tmp;
        tmp.alloc(tb);
        RQ_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, tkey.as<uint64_t>(), tkey2.as<uint64_t>(),
                                                tval.as<int32_t>(), tval2.as<int32_t>(), (int)n_tiles_all, 0,
                                                end_bit, s));
        k_tile_permute<<<nblk(n_tiles_all), NT, 0, s>>>(tiles_tmp.as<TileTmp>(), tval2.as<int32_t>(), n_tiles_all,
                                                        sorted.as<TileTmp>(), inv.as<int32_t>());
        RQ_CUDA(cudaMemcpyAsync(tiles_tmp.p, sorted.p, n_tiles_all * sizeof(TileTmp), cudaMemcpyDeviceToDevice, s));
        k_remap_tiles<<<nblk(NN), NT, 0, s>>>(tile_of.as<int32_t>(), NN, inv.as<int32_t>());
      }
      DBuf cb;
      cb.alloc(8);
      RQ_CUDA(cudaMemsetAsync(cb.p, 0, 8, s));
      if (n_tiles_all) k_count_big<<<nblk(n_tiles_all), NT, 0, s>>>(tiles_tmp.as<TileTmp>(), n_tiles_all, cb.as<unsigned long long>());
      p.n_tiles = (int64_t)d2h1<unsigned long long>(cb.p, s);
    }

    // wavefront streams over the same tiles
    {
      DBuf troots;
      troots.alloc(std::max<int64_t>(n_tiles_all, 1) * 8);
      if (n_tiles_all) k_tile_roots<<<nblk(n_tiles_all), NT, 0, s>>>(tiles_tmp.as<TileTmp>(), n_tiles_all, troots.as<int64_t>());
      WaveBuildIn wi{n_tiles_all,           troots.as<int64_t>(),      noff,
                     boff,                  p.rec_off.as<int64_t>(),   p.res_base_d.as<int64_t>(),
                     node_body.as<int32_t>(), p.start.as<int32_t>(),   p.stop.as<int32_t>(),
                     p.left.as<int32_t>(),  p.right.as<int32_t>(),     p.parent.as<int32_t>(),
                     p.height.as<int32_t>(), p.res_off.as<int32_t>(),  p.perm.as<int32_t>(),
                     slot_scan.as<int32_t>(), p.flags.as<uint8_t>(),   p.rec.as<double>()};
      build_wave(p, wi, s);
    }
    tm.mark("wave");
    // top tree
    {
      std::vector<int64_t> topbodies;
      std::vector<int32_t> smalls;
      // bodies with a top tree: their root is a top node (more than S beads, or taller
      // than the tile height cut)
      std::vector<int32_t> root_top(m, 0);
      {
        DBuf rt;
        rt.alloc(m * 4);
        k_root_is_top<<<nblk(m), NT, 0, s>>>(is_top.as<int32_t>(), boff, noff, m, rt.as<int32_t>());
        d2h(root_top.data(), rt.p, m, s);
      }
      for (int64_t j = 0; j < m; j++) {
        int64_t n = offsets[j + 1] - offsets[j];
        if (root_top[j]) topbodies.push_back(j);
        if (n == 1) smalls.push_back((int32_t)j);
      }
      p.n_topbodies = (int64_t)topbodies.size();
      p.n_small = (int64_t)smalls.size();
      p.h_small_first.assign(m + 1, p.n_small);
      for (int64_t i = p.n_small - 1; i >= 0; i--) p.h_small_first[smalls[i]] = i;
      for (int64_t j = m - 1; j >= 0; j--) p.h_small_first[j] = std::min(p.h_small_first[j], p.h_small_first[j + 1]);
      p.small_bodies.alloc(std::max<int64_t>(p.n_small, 1) * 4);
      if (p.n_small)
        RQ_CUDA(cudaMemcpyAsync(p.small_bodies.p, smalls.data(), p.n_small * 4, cudaMemcpyHostToDevice, s));
      const int64_t nt = p.n_top;
      p.top.alloc(std::max<int64_t>(nt, 1) * sizeof(TopNode));
      std::vector<int32_t> hb(topbodies.begin(), topbodies.end());
      p.topbody.alloc(std::max<int64_t>(p.n_topbodies, 1) * 4);
      if (p.n_topbodies)
        RQ_CUDA(cudaMemcpyAsync(p.topbody.p, hb.data(), p.n_topbodies * 4, cudaMemcpyHostToDevice, s));
      // top trees of bodies above split_min beads are cut into pieces (<= X beads) + an apex, so
      // every blob stays small (shared memory per CTA -> residency) and no tree needs the slow
      // dataflow sweep; X >= n/512 keeps the apex at ~2 x 512 nodes.  X = 8192: config 3 top pass
      // 45.7 -> 20.2 us (up), config 4 552 -> 460 us (X = 2048 / 4096 / 16384 measured worse)
      int64_t split_min = 16384;
      if (const char *e = getenv("RQ_TOP_SPLIT")) split_min = std::max<int64_t>(0, atoll(e));
      std::vector<int64_t> split_x(m, 0);
      for (int64_t j = 0; j < m; j++) {
        const int64_t n = offsets[j + 1] - offsets[j];
        if (split_min > 0 && root_top[j] && n > split_min) {
          static const int64_t x0 = [] {
            const char *e = getenv("RQ_TOP_SPLIT_X");
            return e ? std::max<int64_t>(256, atoll(e)) : int64_t(8192);  // measured: configs 3 and 4
          }();
          int64_t X = x0;
          while (X < n / 512) X *= 2;
          split_x[j] = X;
        }
      }
      DBuf d_split;
      d_split.alloc(std::max<int64_t>(m, 1) * 8);
      RQ_CUDA(cudaMemcpyAsync(d_split.p, split_x.data(), m * 8, cudaMemcpyHostToDevice, s));
      if (nt > 0) {
        DBuf tmp_top, tkeys, tvals, tkeys2, tvals2, lflag, lscan;
        tmp_top.alloc(nt * sizeof(TopNode));
        tkeys.alloc(nt * 8);
        tvals.alloc(nt * 4);
        tkeys2.alloc(nt * 8);
        tvals2.alloc(nt * 4);
        lflag.alloc(nt * 4);
        lscan.alloc(nt * 4);
        k_top_fill<<<nblk(NN), NT, 0, s>>>(lc, NN, is_top.as<int32_t>(), top_scan.as<int32_t>(),
                                            slot_scan.as<int32_t>(), p.left.as<int32_t>(), p.right.as<int32_t>(),
                                            d_split.as<int64_t>(), tmp_top.as<TopNode>(), tkeys.as<uint64_t>(),
                                            tvals.as<int32_t>());
        size_t tb = 0;
        RQ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, tkeys.as<uint64_t>(), tkeys2.as<uint64_t>(),
                                                tvals.as<int32_t>(), tvals2.as<int32_t>(), (int)nt, 0, 64, s));
        DBuf tmp;
        tmp.alloc(tb);
        RQ_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, tkeys.as<uint64_t>(), tkeys2.as<uint64_t>(),
                                                tvals.as<int32_t>(), tvals2.as<int32_t>(), (int)nt, 0, 64, s));
        k_top_gather<<<nblk(nt), NT, 0, s>>>(tmp_top.as<TopNode>(), tvals2.as<int32_t>(), tkeys2.as<uint64_t>(),
                                              nt, p.top.as<TopNode>(), lflag.as<int32_t>());
        exclusive_scan(lflag.as<int32_t>(), lscan.as<int32_t>(), nt, s);
        p.n_toplevels = d2h1<int32_t>(lscan.as<int32_t>() + nt - 1, s) + d2h1<int32_t>(lflag.as<int32_t>() + nt - 1, s);
        // blob units (whole top trees, pieces, apexes): unit index of every top node
        DBuf uflag, tunit;
        uflag.alloc(nt * 4);
        tunit.alloc(nt * 4);
        k_top_unitflag<<<nblk(nt), NT, 0, s>>>(tkeys2.as<uint64_t>(), nt, uflag.as<int32_t>());
        exclusive_scan(uflag.as<int32_t>(), tunit.as<int32_t>(), nt, s);
        const int64_t U = d2h1<int32_t>(tunit.as<int32_t>() + nt - 1, s) + d2h1<int32_t>(uflag.as<int32_t>() + nt - 1, s);
        k_top_unitfix<<<nblk(nt), NT, 0, s>>>(uflag.as<int32_t>(), nt, tunit.as<int32_t>());
        p.n_topunits = U;
        p.topbody_lvl.alloc((U + 1) * 4);
        DBuf unit_body, unit_kind;
        unit_body.alloc(U * 4);
        unit_kind.alloc(U * 4);
        p.toplvl.alloc((p.n_toplevels + 1) * 4);
        k_top_levels<<<nblk(nt), NT, 0, s>>>(tkeys2.as<uint64_t>(), lflag.as<int32_t>(), lscan.as<int32_t>(),
                                              uflag.as<int32_t>(), tunit.as<int32_t>(), p.top.as<TopNode>(),
                                              d_split.as<int64_t>(), boff, noff, nt, p.toplvl.as<int32_t>(),
                                              p.topbody_lvl.as<int32_t>(), unit_body.as<int32_t>(),
                                              unit_kind.as<int32_t>());
        int32_t endv[2] = {(int32_t)nt, (int32_t)p.n_toplevels};
        RQ_CUDA(cudaMemcpyAsync(p.toplvl.as<int32_t>() + p.n_toplevels, &endv[0], 4, cudaMemcpyHostToDevice, s));
        RQ_CUDA(cudaMemcpyAsync(p.topbody_lvl.as<int32_t>() + U, &endv[1], 4, cudaMemcpyHostToDevice, s));
        std::vector<int32_t> unit_body_h(U), unit_kind_h(U);
        d2h(unit_body_h.data(), unit_body.p, U, s);
        d2h(unit_kind_h.data(), unit_kind.p, U, s);
        // staged per-body top blobs
        DBuf slot2loc, slot2unit, nin, in_scan, recsz, rec_scan;
        slot2loc.alloc(std::max<int64_t>(p.n_slots, 1) * 4);
        RQ_CUDA(cudaMemsetAsync(slot2loc.p, 0xff, std::max<int64_t>(p.n_slots, 1) * 4, s));
        slot2unit.alloc(std::max<int64_t>(p.n_slots, 1) * 4);
        RQ_CUDA(cudaMemsetAsync(slot2unit.p, 0xff, std::max<int64_t>(p.n_slots, 1) * 4, s));
        nin.alloc((nt + 1) * 4);
        in_scan.alloc((nt + 1) * 4);
        recsz.alloc((nt + 1) * 8);
        rec_scan.alloc((nt + 1) * 8);
        RQ_CUDA(cudaMemsetAsync(nin.p, 0, (nt + 1) * 4, s));
        RQ_CUDA(cudaMemsetAsync(recsz.p, 0, (nt + 1) * 8, s));
        k_top_slotmap<<<nblk(nt), NT, 0, s>>>(p.top.as<TopNode>(), nt, tunit.as<int32_t>(), p.topbody_lvl.as<int32_t>(),
                                               p.toplvl.as<int32_t>(), slot2loc.as<int32_t>(), slot2unit.as<int32_t>(),
                                               recsz.as<int64_t>());
        k_top_inputs<<<nblk(nt), NT, 0, s>>>(p.top.as<TopNode>(), nt, slot2unit.as<int32_t>(), tunit.as<int32_t>(),
                                              nin.as<int32_t>());
        exclusive_scan(nin.as<int32_t>(), in_scan.as<int32_t>(), nt + 1, s);
        exclusive_scan(recsz.as<int64_t>(), rec_scan.as<int64_t>(), nt + 1, s);
        std::vector<int32_t> h_lvl(U + 1), h_toplvl(p.n_toplevels + 1), h_in(nt + 1);
        std::vector<int64_t> h_rec(nt + 1);
        d2h(h_lvl.data(), p.topbody_lvl.p, U + 1, s);
        d2h(h_toplvl.data(), p.toplvl.p, p.n_toplevels + 1, s);
        d2h(h_in.data(), in_scan.p, nt + 1, s);
        d2h(h_rec.data(), rec_scan.p, nt + 1, s);
        int64_t smem_cap = 112 * 1024;  // larger top trees go to the dataflow kernels (measured on config 4)
        if (const char *e = getenv("RQ_TOP_SMEM_KB")) smem_cap = std::max(0, atoi(e)) * 1024;
        std::vector<int64_t> blob_off(U, -1), small_off;
        std::vector<int32_t> small_tb, big_tb;
        std::vector<uint8_t> small_cls, small_phase;
        int64_t total = 0;
        p.max_topblob_smem = 0;
        for (int c = 0; c < Plan::N_TOPCLASS; c++) p.topclass_smem[c] = p.topclass_count[c] = 0;
        // shared-memory footprints per unit: header part (levels, meta, inputs) + vectors, and with
        // the records
        std::vector<int64_t> fp(U), fp_rec(U);
        std::vector<uint8_t> fits(U);
        std::vector<uint8_t> body_big(m, 0);  // a split tree with a unit that does not fit: all dataflow
        int64_t rec_all = 0;  // largest whole-blob footprint up to 48 KB
        for (int64_t bi = 0; bi < U; bi++) {
          const int first = h_toplvl[h_lvl[bi]], last = h_toplvl[h_lvl[bi + 1]];
          const int nn = last - first, ni = h_in[last] - h_in[first];
          const int64_t bytes = topblob_bytes(nn, h_lvl[bi + 1] - h_lvl[bi], ni, h_rec[last] - h_rec[first]);
          const int64_t hdr_bytes = bytes - 8 * (h_rec[last] - h_rec[first]);
          const int64_t vec_bytes = 48 * (int64_t)(std::max(ni, nn) + nn) + 128;
          fp[bi] = (hdr_bytes + 127) / 128 * 128 + vec_bytes;
          fp_rec[bi] = (bytes + 127) / 128 * 128 + vec_bytes;
          if (fp_rec[bi] <= 48 * 1024) rec_all = std::max(rec_all, fp_rec[bi]);
          fits[bi] = fp[bi] <= smem_cap && nn < 32000 && ni < 32000;
          if (!fits[bi] && unit_kind_h[bi] != 0) body_big[unit_body_h[bi]] = 1;
        }
        // Records staged too (no L2 round trip per level) when that costs no residency: every top
        // tree resident at once, else only tiny ones (config 4's 20000 trees run in waves, where
        // the footprint decides the throughput; measured)
        if (!p.sms) RQ_CUDA(cudaDeviceGetAttribute(&p.sms, cudaDevAttrMultiProcessorCount, p.device));
        const int64_t per_sm = rec_all ? std::min<int64_t>(32, (227 * 1024) / rec_all) : 0;
        int64_t rec_cap = (rec_all && U <= per_sm * std::max(p.sms, 1)) ? rec_all : 16 * 1024;
        if (const char *e = getenv("RQ_TOP_REC_KB")) rec_cap = std::max(0, atoi(e)) * 1024;
        for (int64_t bi = 0; bi < U; bi++) {
          const int first = h_toplvl[h_lvl[bi]], last = h_toplvl[h_lvl[bi + 1]];
          const int nn = last - first, nl = h_lvl[bi + 1] - h_lvl[bi], ni = h_in[last] - h_in[first];
          const int64_t bytes = topblob_bytes(nn, nl, ni, h_rec[last] - h_rec[first]);
          const int64_t smem = fp[bi], smem_rec = fp_rec[bi];
          if (fits[bi] && !body_big[unit_body_h[bi]]) {
            blob_off[bi] = total;
            small_tb.push_back((int32_t)bi);
            small_off.push_back(total);
            total += bytes;
            const int c = smem_rec <= rec_cap ? 0
                        : smem <= 8 * 1024 ? 1 : smem <= 16 * 1024 ? 2 : smem <= 32 * 1024 ? 3 : smem <= 64 * 1024 ? 4 : 5;
            const int64_t sm_c = c == 0 ? smem_rec : smem;
            p.max_topblob_smem = std::max(p.max_topblob_smem, sm_c);
            small_cls.push_back((uint8_t)c);
            small_phase.push_back((uint8_t)(unit_kind_h[bi] == 2 ? 1 : 0));
            p.topclass_smem[c] = std::max(p.topclass_smem[c], sm_c);
            p.topclass_count[c]++;
          } else {
            blob_off[bi] = 0;  // unused
            big_tb.push_back((int32_t)bi);
          }
        }
        p.n_topblob = (int64_t)small_tb.size();
        p.n_topbig = (int64_t)big_tb.size();
        p.h_topblob_off = small_off;
        p.h_topblob_off.push_back(total);
        if (getenv("RQ_VERBOSE")) {
          int mx_nn = 0, mx_nl = 0;
          double s_nn = 0, s_nl = 0;
          int64_t n_split = 0;
          for (int64_t bi = 0; bi < U; bi++) {
            const int nn = h_toplvl[h_lvl[bi + 1]] - h_toplvl[h_lvl[bi]], nl = h_lvl[bi + 1] - h_lvl[bi];
            mx_nn = std::max(mx_nn, nn), mx_nl = std::max(mx_nl, nl), s_nn += nn, s_nl += nl;
            n_split += unit_kind_h[bi] == 2;
          }
          fprintf(stderr, "[rq] top trees: %lld bodies (%lld split) in %lld units, nodes mean %.1f max %d, levels mean "
                  "%.1f max %d; staged %lld, global %lld; classes (count/smem):", (long long)p.n_topbodies,
                  (long long)n_split, (long long)U, s_nn / std::max<int64_t>(1, U), mx_nn,
                  s_nl / std::max<int64_t>(1, U), mx_nl, (long long)p.n_topblob, (long long)p.n_topbig);
          for (int c = 0; c < Plan::N_TOPCLASS; c++)
            fprintf(stderr, " %lld/%lld", (long long)p.topclass_count[c], (long long)p.topclass_smem[c]);
          fprintf(stderr, "\n");
        }
        auto firsts = [&](const std::vector<int32_t> &list, std::vector<int64_t> &out) {
          out.assign(m + 1, (int64_t)list.size());
          for (int64_t i = (int64_t)list.size() - 1; i >= 0; i--) out[unit_body_h[list[i]]] = i;
          for (int64_t j = m - 1; j >= 0; j--) out[j] = std::min(out[j], out[j + 1]);
        };
        firsts(small_tb, p.h_topblob_first);
        firsts(big_tb, p.h_topbig_first);
        p.topblob.alloc(std::max<int64_t>(total, 16));
        p.topblob_off.alloc(std::max<int64_t>(p.n_topblob, 1) * 8);
        p.topblob_body.alloc(std::max<int64_t>(p.n_topblob, 1) * 4);
        p.topblob_class.alloc(std::max<int64_t>(p.n_topblob, 1));
        p.topbig.alloc(std::max<int64_t>(p.n_topbig, 1) * 4);
        // blob indices grouped by class (stable: body order inside a class), so each class launch
        // runs exactly its own blobs
        std::vector<int32_t> cls_order;
        cls_order.reserve(p.n_topblob);
        for (int f = 0; f < 2; f++) {
          for (int c = 0; c < Plan::N_TOPCLASS; c++) {
            p.topclass_first[f][c] = (int64_t)cls_order.size();
            for (int64_t i = 0; i < p.n_topblob; i++)
              if (small_cls[i] == c && small_phase[i] == f) cls_order.push_back((int32_t)i);
          }
          p.topclass_first[f][Plan::N_TOPCLASS] = (int64_t)cls_order.size();
        }
        p.topblob_order.alloc(std::max<int64_t>(p.n_topblob, 1) * 4);
        if (p.n_topblob) {
          RQ_CUDA(cudaMemcpyAsync(p.topblob_off.p, small_off.data(), p.n_topblob * 8, cudaMemcpyHostToDevice, s));
          RQ_CUDA(cudaMemcpyAsync(p.topblob_body.p, small_tb.data(), p.n_topblob * 4, cudaMemcpyHostToDevice, s));
          RQ_CUDA(cudaMemcpyAsync(p.topblob_class.p, small_cls.data(), p.n_topblob, cudaMemcpyHostToDevice, s));
          RQ_CUDA(cudaMemcpyAsync(p.topblob_order.p, cls_order.data(), p.n_topblob * 4, cudaMemcpyHostToDevice, s));
        }
        if (p.n_topbig) RQ_CUDA(cudaMemcpyAsync(p.topbig.p, big_tb.data(), p.n_topbig * 4, cudaMemcpyHostToDevice, s));
        DBuf d_blob_off;
        d_blob_off.alloc(U * 8);
        RQ_CUDA(cudaMemcpyAsync(d_blob_off.p, blob_off.data(), U * 8, cudaMemcpyHostToDevice, s));
        if (p.n_topblob) {
          // write every node; nodes of "big" bodies write into a scratch blob that is dropped
          DBuf dummy;
          int64_t big_bytes = 0;
          std::vector<int64_t> off2(blob_off);
          for (auto bi : big_tb) {
            const int first = h_toplvl[h_lvl[bi]], last = h_toplvl[h_lvl[bi + 1]];
            off2[bi] = total + big_bytes;
            big_bytes += topblob_bytes(last - first, h_lvl[bi + 1] - h_lvl[bi], h_in[last] - h_in[first],
                                       h_rec[last] - h_rec[first]);
          }
          DBuf all_blob;
          all_blob.alloc(total + big_bytes + 16);
          RQ_CUDA(cudaMemcpyAsync(d_blob_off.p, off2.data(), U * 8, cudaMemcpyHostToDevice, s));
          k_top_blob<<<nblk(nt), NT, 0, s>>>(p.top.as<TopNode>(), nt, tunit.as<int32_t>(), p.topbody_lvl.as<int32_t>(),
                                              unit_kind.as<int32_t>(), p.toplvl.as<int32_t>(), slot2loc.as<int32_t>(),
                                              slot2unit.as<int32_t>(), in_scan.as<int32_t>(), rec_scan.as<int64_t>(),
                                              d_blob_off.as<int64_t>(), p.rec.as<double>(), p.perm.as<int32_t>(), boff,
                                              all_blob.as<uint8_t>());
          RQ_CUDA(cudaMemcpyAsync(p.topblob.p, all_blob.p, total, cudaMemcpyDeviceToDevice, s));
          RQ_CUDA(cudaStreamSynchronize(s));
        }
        // dataflow top trees (bodies whose top tree does not fit shared memory)
        p.top_parent.alloc(std::max<int64_t>(nt, 1) * 4);
        p.top_need.alloc(std::max<int64_t>(nt, 1) * 4);
        RQ_CUDA(cudaMemsetAsync(p.top_need.p, 0, std::max<int64_t>(nt, 1) * 4, s));
        RQ_CUDA(cudaMemsetAsync(p.top_parent.p, 0xff, std::max<int64_t>(nt, 1) * 4, s));
        std::vector<int32_t> starts;
        p.h_topstart_first.assign(m + 1, 0);
        if (p.n_topbig) {
          DBuf slot2top, is_start;
          slot2top.alloc(std::max<int64_t>(p.n_slots, 1) * 4);
          is_start.alloc(nt * 4);
          RQ_CUDA(cudaMemsetAsync(slot2top.p, 0xff, std::max<int64_t>(p.n_slots, 1) * 4, s));
          RQ_CUDA(cudaMemsetAsync(is_start.p, 0, nt * 4, s));
          k_top_slot2top<<<nblk(nt), NT, 0, s>>>(p.top.as<TopNode>(), nt, slot2top.as<int32_t>());
          for (auto bi : big_tb) {
            const int64_t q0 = h_toplvl[h_lvl[bi]], q1 = h_toplvl[h_lvl[bi + 1]];
            k_top_links<<<nblk(q1 - q0), NT, 0, s>>>(p.top.as<TopNode>(), q0, q1, slot2top.as<int32_t>(),
                                                     p.top_parent.as<int32_t>(), is_start.as<int32_t>(),
                                                     p.top_need.as<int32_t>());
          }
          std::vector<int32_t> hs(nt);
          d2h(hs.data(), is_start.p, nt, s);
          std::vector<int64_t> first_of_body(m + 1, -1);
          for (auto bi : big_tb) {
            const int64_t q0 = h_toplvl[h_lvl[bi]], q1 = h_toplvl[h_lvl[bi + 1]];
            if (first_of_body[unit_body_h[bi]] < 0) first_of_body[unit_body_h[bi]] = (int64_t)starts.size();
            for (int64_t q = q0; q < q1; q++)
              if (hs[q]) starts.push_back((int32_t)q);
          }
          first_of_body[m] = (int64_t)starts.size();
          for (int64_t j = m - 1; j >= 0; j--)
            if (first_of_body[j] < 0) first_of_body[j] = first_of_body[j + 1];
          p.h_topstart_first.assign(first_of_body.begin(), first_of_body.end());
        }
        p.n_top_start = (int64_t)starts.size();
        p.top_start.alloc(std::max<int64_t>(p.n_top_start, 1) * 4);
        if (p.n_top_start)
          RQ_CUDA(cudaMemcpyAsync(p.top_start.p, starts.data(), p.n_top_start * 4, cudaMemcpyHostToDevice, s));
        // root-to-start paths (downward dataflow sweep), CSR over the start nodes
        {
          const int64_t ns = p.n_top_start;
          DBuf plen;
          plen.alloc(std::max<int64_t>(ns, 1) * 8);
          p.top_path_off.alloc((ns + 1) * 8);
          if (ns) k_top_path_len<<<nblk(ns), NT, 0, s>>>(p.top_parent.as<int32_t>(), p.top_start.as<int32_t>(), ns,
                                                       plen.as<int64_t>());
          if (ns) exclusive_scan(plen.as<int64_t>(), p.top_path_off.as<int64_t>(), ns, s);
          const int64_t total = ns ? d2h1<int64_t>(p.top_path_off.as<int64_t>() + ns - 1, s) +
                                         d2h1<int64_t>(plen.as<int64_t>() + ns - 1, s)
                                   : 0;
          RQ_CUDA(cudaMemcpyAsync(p.top_path_off.as<int64_t>() + ns, &total, 8, cudaMemcpyHostToDevice, s));
          p.top_paths.alloc(std::max<int64_t>(total, 1) * 4);
          if (ns) k_top_path_write<<<nblk(ns), NT, 0, s>>>(p.top_parent.as<int32_t>(), p.top_start.as<int32_t>(), ns,
                                                         p.top_path_off.as<int64_t>(), p.top_paths.as<int32_t>());
        }
        RQ_CUDA(cudaStreamSynchronize(s));
      } else {
        p.h_topblob_first.assign(m + 1, 0);
        p.h_topbig_first.assign(m + 1, 0);
        p.h_topstart_first.assign(m + 1, 0);
        p.toplvl.alloc(4);
        p.topbody_lvl.alloc(4);
        p.n_topunits = 0;
        int32_t z = 0;
        RQ_CUDA(cudaMemcpyAsync(p.topbody_lvl.p, &z, 4, cudaMemcpyHostToDevice, s));
        RQ_CUDA(cudaStreamSynchronize(s));
      }
    }
    tm.mark("top");
    // case counts
    {
      DBuf cc;
      cc.alloc(4 * 8);
      RQ_CUDA(cudaMemsetAsync(cc.p, 0, 4 * 8, s));
      k_case_count<<<(unsigned)std::min<int64_t>(nblk(NN), 4 * 148), NT, 0, s>>>(p.flags.as<uint8_t>(), NN,
                                                                             cc.as<unsigned long long>());
      unsigned long long hc[4];
      d2h(hc, cc.p, 4, s);
      for (int c = 0; c < 4; c++) p.n_case[c] = (int64_t)hc[c];
    }
    RQ_CUDA(cudaGetLastError());
    RQ_CUDA(cudaStreamSynchronize(s));
  }
}

int check_duplicates(const double *pos_in, const int64_t *offsets, int64_t m, bool host_input, cudaStream_t s,
                     int64_t *body, int64_t *bi, int64_t *bj, double *tol_out) {
  if (m < 1) throw Error(RQ_ERR_VALUE, "need at least one body");
  for (int64_t j = 0; j < m; j++)
    if (offsets[j + 1] <= offsets[j]) throw Error(RQ_ERR_VALUE, "every body needs n >= 1");
  const int64_t N = offsets[m];
  DBuf pos, off, body_of, bmin, bmax, table, hit, err;
  pos.alloc(N * 24);
  RQ_CUDA(cudaMemcpyAsync(pos.p, pos_in, N * 24, host_input ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, s));
  off.alloc((m + 1) * 8);
  RQ_CUDA(cudaMemcpyAsync(off.p, offsets, (m + 1) * 8, cudaMemcpyHostToDevice, s));
  body_of.alloc(N * 4);
  k_body_of<<<nblk(N), NT, 0, s>>>(off.as<int64_t>(), m, N, body_of.as<int32_t>());
  bmin.alloc(m * 24);
  bmax.alloc(m * 24);
  err.alloc(64);
  RQ_CUDA(cudaMemsetAsync(bmin.p, 0xff, m * 24, s));
  RQ_CUDA(cudaMemsetAsync(bmax.p, 0x00, m * 24, s));
  {
    long long init[8] = {0, 0, 0x7fffffffffffffffLL, 0, 0, 0, 0, 0};
    RQ_CUDA(cudaMemcpyAsync(err.p, init, sizeof(init), cudaMemcpyHostToDevice, s));
  }
  k_bbox<<<nblk(N), NT, 0, s>>>(pos.as<double>(), body_of.as<int32_t>(), N, bmin.as<unsigned long long>(),
                                 bmax.as<unsigned long long>(), err.as<long long>());
  uint64_t cap = 1;
  while (cap < (uint64_t)(2 * N)) cap <<= 1;
  table.alloc(cap * 4);
  RQ_CUDA(cudaMemsetAsync(table.p, 0xff, cap * 4, s));
  hit.alloc(m * 8);
  RQ_CUDA(cudaMemsetAsync(hit.p, 0xff, m * 8, s));
  DupCtx c{pos.as<double>(), body_of.as<int32_t>(), off.as<int64_t>(), bmin.as<unsigned long long>(),
           bmax.as<unsigned long long>(), table.as<int32_t>(), cap - 1, hit.as<unsigned long long>(),
           err.as<long long>()};
  k_dup_insert<<<nblk(N), NT, 0, s>>>(c, N);
  k_dup_query<<<nblk(N), NT, 0, s>>>(c, N);
  RQ_CUDA(cudaGetLastError());
  long long e[3];
  d2h(e, err.p, 3, s);
  if (e[1]) throw Error(RQ_ERR_VALUE, "positions must be finite");
  std::vector<unsigned long long> h(m);
  d2h(h.data(), hit.p, m, s);
  int64_t coincide = e[2];
  for (int64_t j = 0; j < m; j++) {
    if (j == coincide) {
      *body = j; *bi = -1; *bj = -1; *tol_out = 0.0;
      return RQ_ERR_DUPLICATE;
    }
    if (h[j] != ~0ull) {
      *body = j;
      *bi = (int64_t)(h[j] >> 32);
      *bj = (int64_t)(h[j] & 0xffffffffull);
      std::vector<unsigned long long> bb(6);
      d2h(bb.data(), bmin.as<unsigned long long>() + 3 * j, 3, s);
      d2h(bb.data() + 3, bmax.as<unsigned long long>() + 3 * j, 3, s);
      double d2 = 0.0;
      for (int a = 0; a < 3; a++) {
        auto un = [](unsigned long long u) {
          long long v = (long long)((u >> 63) ? (u & 0x7fffffffffffffffull) : ~u);
          double d;
          memcpy(&d, &v, 8);
          return d;
        };
        double ext = un(bb[3 + a]) - un(bb[a]);
        d2 += ext * ext;
      }
      *tol_out = 1e-12 * sqrt(d2);
      return RQ_ERR_DUPLICATE;
    }
  }
  return RQ_OK;
}

void ensure_smem_attr(const void *f, size_t bytes) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int, const void *>, size_t>> set;  // (device, kernel) -> limit
  int dev = 0;
  RQ_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  for (auto &e : set)
    if (e.first.first == dev && e.first.second == f) {
      if (e.second >= bytes) return;
      RQ_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
      e.second = bytes;
      return;
    }
  RQ_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  set.push_back({{dev, f}, bytes});
}

int occupancy_cached(const void *f, int threads, size_t smem) {
  static std::mutex mu;
  static std::vector<std::pair<std::tuple<int, const void *, int, size_t>, int>> memo;  // -> CTAs per SM
  int dev = 0;
  RQ_CUDA(cudaGetDevice(&dev));
  const auto key = std::make_tuple(dev, f, threads, smem);
  std::lock_guard<std::mutex> lk(mu);
  for (auto &e : memo)
    if (e.first == key) return e.second;
  int occ = 0;
  RQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, threads, smem));
  memo.push_back({key, occ});
  return occ;
}

}  // namespace rq
