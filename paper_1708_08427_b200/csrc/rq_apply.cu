// rq_apply.cu -- the hot path: batched fp64 Qv / Q^T w / Q~v / Q~^T g.
//
// Restates upward_apply (Algorithm 2, matfree.py:95-121, merge_infosets
// matfree.py:41-62) and downward_apply (Algorithm 3, matfree.py:124-151,
// split_rvset matfree.py:65-83) as a tile sweep plus a top-tree sweep:
//
//   UP   : k_wave<UP> (rq_wave.cu, all tiles, persistent CTAs) -> k_top2 / k_top_df_up
//   DOWN : k_top2 / k_top_df_down                               -> k_wave<DOWN>
//
// The top trees (nodes with more than S beads) run here: one CTA per body with its
// top tree staged in shared memory (k_top2), or dataflow sweeps over global memory
// for top trees too large for that (k_top_df_*).  Q / Q^T run through the private
// residue layout (Plan::res_base) plus 6 root rows per body (k_expand / k_compress);
// k > 1 columns run as a column loop over transposed blocks, or as the multi-RHS
// kernels of rq_mrhs.cu.  No tensor cores: HBM-bound sweeps of tiny fp64 orthogonal
// transforms (~0.3 flop/B).  DESIGN.md §2 has the full description.
#include <algorithm>
#include <type_traits>
#include <climits>
#include <cuda/atomic>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "rq_nodeops.cuh"
#include "rq_plan.hpp"

namespace rq {
namespace {

constexpr int NT_TOP = 128;  // dataflow top kernels

// ---- PTX helpers: mbarrier + bulk copy ------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Programmatic dependent launch: every apply kernel is launched with programmatic
// stream serialisation (no early trigger: the successor launches when it completes) and waits
// for its predecessor's results (griddepcontrol.wait) only before touching data another
// kernel produces (input/output vectors, exchange slots); plan data is read before.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  uint32_t addr = smem_u32(bar);
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
__device__ __forceinline__ void prefetch_l2(const void *p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

//   UP  : the chunk's bead forces, gathered through perm
//   DOWN: the chunk's residue coefficients (contiguous per tile) + tile-root RV-sets
__device__ __forceinline__ void cp_async16cg_u32(uint32_t dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8_u32(uint32_t dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ---- top tree (nodes with more than tile_leaves beads) ---------------------------------

// Top trees too large for shared memory (e.g. config 3's single 2^20-bead body:
// ~23k top nodes, height ~15) run as dataflow sweeps over global memory, one
// thread per "start" node (both children below the top tree):
//  * upward: a thread merges its node, publishes the info vector (scratch slot),
//    then climbs to the parent only if it is the second child to arrive (per-node
//    arrival counters, self-resetting) -- no level barriers, full parallelism;
//  * downward: every thread recomputes the split chain along its root-to-node
//    path (identical arithmetic, so every path sees identical values) and writes
//    the outputs of the children that leave the top tree (tile roots, beads).
// a node record (global memory, 16-byte aligned) into registers
__device__ __forceinline__ void ldg_rec(int cs, const double *g, double (&R)[rec_size(GENERAL)]) {
  const double2 *g2 = reinterpret_cast<const double2 *>(g);
  const int n2 = rec_size(cs) / 2;
#pragma unroll
  for (int i = 0; i < rec_size(GENERAL) / 2; i++) {
    if (i < n2) {
      const double2 v = __ldg(g2 + i);
      R[2 * i] = v.x;
      R[2 * i + 1] = v.y;
    } else {
      R[2 * i] = 0.0;
      R[2 * i + 1] = 0.0;
    }
  }
}

// a 6-vector at a 16-byte aligned address (48-byte entries of aligned regions)
__device__ __forceinline__ void ld6(const double *p, double (&v)[6]) {
  const double2 *p2 = reinterpret_cast<const double2 *>(p);
  const double2 a = p2[0], b = p2[1], c = p2[2];
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y; v[4] = c.x; v[5] = c.y;
}
__device__ __forceinline__ void st6(double *p, const double (&v)[6]) {
  double2 *p2 = reinterpret_cast<double2 *>(p);
  p2[0] = make_double2(v[0], v[1]);
  p2[1] = make_double2(v[2], v[3]);
  p2[2] = make_double2(v[4], v[5]);
}

// a node record staged in shared memory (generic loads) into registers
__device__ __forceinline__ void lds_rec_any(int cs, const double *g, double (&R)[rec_size(GENERAL)]) {
  const double2 *g2 = reinterpret_cast<const double2 *>(g);
  const int n2 = rec_size(cs) / 2;
#pragma unroll
  for (int i = 0; i < rec_size(GENERAL) / 2; i++) {
    if (i < n2) {
      const double2 v = g2[i];
      R[2 * i] = v.x;
      R[2 * i + 1] = v.y;
    } else {
      R[2 * i] = 0.0;
      R[2 * i + 1] = 0.0;
    }
  }
}

struct TopDfCtx {
  const int32_t *starts;
  int64_t n;
  const int32_t *paths;     // root-to-start paths (downward sweep)
  const int64_t *path_off;
  const TopNode *top;
  const int32_t *parent, *need;
  int32_t *cnt;
  const int32_t *perm;
  const int64_t *bead_off;
  const double *rec;
  const double *in;
  double *out;
  int64_t k, col;
  double *scratch;
  const int64_t *res_base;  // private residue layout (Plan::res_base)
  double *roots;            // body-root 6-vectors (Q / Q^T), nullptr for Q~ / Q~^T
  int S;
};

__device__ __forceinline__ void top_fetch(const TopDfCtx &a, int64_t bead0, int32_t ref, double (&m)[6]) {
  if (ref >= 0) {
#pragma unroll
    for (int r = 0; r < 6; r++) m[r] = __ldcg(&a.scratch[6 * (int64_t)ref + r]);
  } else {
    const int64_t row = (bead0 + a.perm[~(int64_t)ref]) * 3;
    m[0] = a.in[(row + 0) * a.k + a.col];
    m[1] = a.in[(row + 1) * a.k + a.col];
    m[2] = a.in[(row + 2) * a.k + a.col];
    m[3] = m[4] = m[5] = 0.0;
  }
}

__device__ __forceinline__ void top_store(const TopDfCtx &a, int64_t bead0, int32_t ref, const double (&l)[6]) {
  if (ref >= 0) {
#pragma unroll
    for (int r = 0; r < 6; r++) __stcg(&a.scratch[6 * (int64_t)ref + r], l[r]);
  } else {
    const int64_t row = (bead0 + a.perm[~(int64_t)ref]) * 3;
    a.out[(row + 0) * a.k + a.col] = l[0];
    a.out[(row + 1) * a.k + a.col] = l[1];
    a.out[(row + 2) * a.k + a.col] = l[2];
  }
}

__global__ void __launch_bounds__(NT_TOP) k_top_df_up(TopDfCtx a) {
  pdl_wait();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  int q = a.starts[i];
  for (;;) {
    const TopNode T = a.top[q];
    const int par = T.is_root ? -1 : __ldg(&a.parent[q]);
    const int need = par >= 0 ? __ldg(&a.need[par]) : 0;
    const int j = T.body;
    const int64_t bead0 = a.bead_off[j];
    const int64_t sbase = a.res_base[j];
    const int cs = flag_case(T.flags);
    double R[rec_size(GENERAL)];
    ldg_rec(cs, a.rec + T.rec_off, R);
    double aa, bb, mx[6], my[6], mp[6], res[6];
    top_fetch(a, bead0, T.x, mx);
    top_fetch(a, bead0, T.y, my);
    rec_ratios(cs, R, 1, aa, bb);
    merge(cs, R, 1, flag_signs(T.flags), aa, bb, mx, my, mp, res);
    for (int r = 0; r < res_rows(cs); r++) a.out[(sbase + T.res_q + r) * a.k + a.col] = res[r];
    if (T.is_root) {
      if (a.roots)
        for (int r = 0; r < 6; r++) a.roots[6 * (int64_t)j + r] = mp[r];
      return;
    }
#pragma unroll
    for (int r = 0; r < 6; r++) __stcg(&a.scratch[6 * (int64_t)T.self_slot + r], mp[r]);
    if (need == 2) {
      // acq_rel: the first arrival's slot writes are released, the second arrival acquires them
      cuda::atomic_ref<int, cuda::thread_scope_device> c(a.cnt[par]);
      if (c.fetch_add(1, cuda::memory_order_acq_rel) == 0) return;  // the sibling's thread continues
      c.store(0, cuda::memory_order_relaxed);                         // reset for the next application
    }
    q = par;
  }
}

__global__ void __launch_bounds__(NT_TOP) k_top_df_down(TopDfCtx a) {
  pdl_wait();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  // precomputed root-to-start path; the next node's TopNode, record and residue rows are
  // loaded while the current one is split (one node of software pipelining)
  const int32_t *path = a.paths + a.path_off[i];
  const int len = (int)(a.path_off[i + 1] - a.path_off[i]);
  TopNode T = a.top[path[0]];
  const int j = T.body;
  const int64_t bead0 = a.bead_off[j];
  const int64_t sbase = a.res_base[j];
  auto load_node = [&](const TopNode &N, double (&R)[rec_size(GENERAL)], double (&res)[6]) {
    const int cs = flag_case(N.flags);
    ldg_rec(cs, a.rec + N.rec_off, R);
#pragma unroll
    for (int r = 0; r < 6; r++) res[r] = r < res_rows(cs) ? a.in[(sbase + N.res_q + r) * a.k + a.col] : 0.0;
  };
  double lp[6];
  for (int r = 0; r < 6; r++) lp[r] = a.roots ? a.roots[6 * (int64_t)j + r] : 0.0;
  double R[rec_size(GENERAL)], res[6];
  load_node(T, R, res);
  for (int d = 0; d < len; d++) {
    TopNode Tn = T;
    double Rn[rec_size(GENERAL)], resn[6];
    if (d + 1 < len) {
      Tn = a.top[path[d + 1]];
      load_node(Tn, Rn, resn);
    }
    const int cs = flag_case(T.flags);
    double aa, bb, lx[6], ly[6];
    rec_ratios(cs, R, 1, aa, bb);
    split(cs, R, 1, flag_signs(T.flags), aa, bb, lp, res, lx, ly);
    if (d + 1 == len) {  // start node: both children leave the top tree
      top_store(a, bead0, T.x, lx);
      top_store(a, bead0, T.y, ly);
      break;
    }
    const bool x_on_path = T.x >= 0 && T.x == Tn.self_slot;
    // the off-path child: written here unless it is itself a top node (another path's)
    if (x_on_path) {
      if (!T.y_top) top_store(a, bead0, T.y, ly);
#pragma unroll
      for (int r = 0; r < 6; r++) lp[r] = lx[r];
    } else {
      if (!T.x_top) top_store(a, bead0, T.x, lx);
#pragma unroll
      for (int r = 0; r < 6; r++) lp[r] = ly[r];
    }
    T = Tn;
#pragma unroll
    for (int e = 0; e < rec_size(GENERAL); e++) R[e] = Rn[e];
#pragma unroll
    for (int r = 0; r < 6; r++) res[r] = resn[r];
  }
}

// ---- staged top tree: one CTA per body, whole top tree in shared memory --------------

struct Top2Ctx {
  const uint8_t *blob;
  const int64_t *blob_off;
  const int32_t *order;  // this launch's blobs (one shared-memory class): block b runs blob order[b]
  const int64_t *bead_off;
  const double *in;
  double *out;
  int64_t k, col;
  double *scratch;
  const int64_t *res_base;  // private residue layout (Plan::res_base)
  double *roots;            // body-root 6-vectors (Q / Q^T), nullptr for Q~ / Q~^T
};

// NTT threads per top tree: one warp for the small shared-memory classes (top trees
// of config-2 bodies: ~4 nodes per level), 128 for the large ones.  SREC: the records are
// staged with the rest of the blob (small top trees: no L2 round trip per level).
template <bool UP, int NTT, bool SREC>
__global__ void __launch_bounds__(NTT) k_top2(Top2Ctx a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  const uint8_t *gB = a.blob + a.blob_off[a.order[blockIdx.x]];
  // stage the header part (levels, meta, inputs) with one TMA copy; the records stay
  // in global memory (prefetched into L2 here) and are read per node, so the CTA
  // needs little shared memory and many top trees are swept concurrently per SM
  if (tid == 0) {
    const TopHdr *gh = reinterpret_cast<const TopHdr *>(gB);
    const unsigned hbytes = SREC ? (unsigned)gh->bytes : (unsigned)gh->off_rec;
    const unsigned rbytes = (unsigned)gh->bytes - hbytes;
    if (rbytes) prefetch_l2(gB + hbytes, rbytes);
    mbar_init(&bar, 1);
    fence_mbar_init();
    mbar_expect_tx(&bar, hbytes);
    bulk_g2s(smem, gB, hbytes, &bar);
  }
  __syncthreads();

  pdl_wait();
  mbar_wait(&bar, 0);
  const TopHdr h = *reinterpret_cast<const TopHdr *>(smem);
  const int32_t *LB = reinterpret_cast<const int32_t *>(smem + sizeof(TopHdr));
  const TopMeta *MD = reinterpret_cast<const TopMeta *>(smem + h.off_meta);
  const int32_t *INREF = reinterpret_cast<const int32_t *>(smem + h.off_in);
  const double *REC = reinterpret_cast<const double *>((SREC ? smem : gB) + h.off_rec);
  // X | MT: X holds the input info vectors (UP) or the staged residues (DOWN)
  double *IN = reinterpret_cast<double *>(smem + ((SREC ? h.bytes : h.off_rec) + 127) / 128 * 128);
  double *RT = IN;
  double *MT = IN + 6 * max(h.n_inputs, h.n_nodes);
  const int64_t K = a.k, col = a.col;
  const int64_t bead0 = a.bead_off[h.body];
  const int64_t sbase = a.res_base[h.body];
  if (UP) {
    // inputs staged with cp.async, all in flight at once: tile-root vectors (3 x 16 B from
    // L2, .cg) and bead forces (3 x 8 B; the upper half of a bead's info vector is 0)
    for (int q = tid; q < h.n_inputs; q += NTT) {
      const int32_t ref = INREF[q];
      const uint32_t d = smem_u32(IN + 6 * q);
      if (ref >= 0) {
        const double *src = a.scratch + 6 * (int64_t)ref;
        cp_async16cg_u32(d, src);
        cp_async16cg_u32(d + 16, src + 2);
        cp_async16cg_u32(d + 32, src + 4);
      } else {
        const double *src = a.in + ((bead0 + ~(int64_t)ref) * 3) * K + col;
        cp_async8_u32(d, src);
        cp_async8_u32(d + 8, src + K);
        cp_async8_u32(d + 16, src + 2 * K);
        IN[6 * q + 3] = 0.0;
        IN[6 * q + 4] = 0.0;
        IN[6 * q + 5] = 0.0;
      }
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    // one node; CSC = GENERAL: the case is a compile-time constant (nearly every top node: the
    // record loads, the transform and the stores carry no case tests -- ~40% fewer instructions
    // on the one-warp-per-tree critical path), CSC = -1: any case
    auto up_node = [&](auto CSC, int q, const TopMeta &md) {
      constexpr int C = decltype(CSC)::value;
      const int cs = C >= 0 ? C : flag_case(md.flags);
      double recv[rec_size(GENERAL)];
      if (SREC) lds_rec_any(cs, REC + md.rec, recv);
      else ldg_rec(cs, REC + md.rec, recv);
      const double *rec = recv;
      double mx[6], my[6], mp[6], res[6], aa, bb;
      const double *px = md.x >= 0 ? MT + 6 * md.x : IN + 6 * ~(int)md.x;
      const double *py = md.y >= 0 ? MT + 6 * md.y : IN + 6 * ~(int)md.y;
      if (C >= 0) {  // 48-byte entries of a 128-byte aligned region: 16-byte loads
        ld6(px, mx);
        ld6(py, my);
      } else {
#pragma unroll
        for (int r = 0; r < 6; r++) { mx[r] = px[r]; my[r] = py[r]; }
      }
      rec_ratios(cs, rec, 1, aa, bb);
      merge(cs, rec, 1, flag_signs(md.flags), aa, bb, mx, my, mp, res);
      const int rr = res_rows(cs);
      double *o = a.out + (sbase + md.res_q) * K + col;
#pragma unroll
      for (int r = 0; r < 6; r++)
        if (r < rr) o[r * K] = res[r];
      if (md.is_root == 1 && a.roots)
        for (int r = 0; r < 6; r++) a.roots[6 * (int64_t)h.body + r] = mp[r];
      if (md.is_root == 2)  // piece root: its vector goes to the apex through its exchange slot
        for (int r = 0; r < 6; r++) a.scratch[6 * (int64_t)h.root_slot + r] = mp[r];
      if (C >= 0) {
        st6(MT + 6 * q, mp);
      } else {
#pragma unroll
        for (int r = 0; r < 6; r++) MT[6 * q + r] = mp[r];
      }
    };
    for (int lv = 0; lv < h.n_levels; lv++) {
      for (int q = LB[lv] + tid; q < LB[lv + 1]; q += NTT) {
        const TopMeta md = MD[q];
        if (flag_case(md.flags) == GENERAL) up_node(std::integral_constant<int, GENERAL>{}, q, md);
        else up_node(std::integral_constant<int, -1>{}, q, md);
      }
      __syncthreads();
    }
  } else {
    for (int q = tid; q < h.n_nodes; q += NTT) {  // residues staged with cp.async, all in flight
      const TopMeta md = MD[q];
      const int rr = res_rows(flag_case(md.flags));
      const double *src = a.in + (sbase + md.res_q) * K + col;
      const uint32_t d = smem_u32(RT + 6 * q);
      for (int r = 0; r < rr; r++) cp_async8_u32(d + 8u * r, src + r * K);
      if (md.is_root == 1)
        for (int r = 0; r < 6; r++) MT[6 * q + r] = a.roots ? a.roots[6 * (int64_t)h.body + r] : 0.0;
      else if (md.is_root == 2)  // piece root: the RV-set the apex wrote to its exchange slot
        for (int r = 0; r < 6; r++) MT[6 * q + r] = a.scratch[6 * (int64_t)h.root_slot + r];
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    auto dn_node = [&](auto CSC, int q, const TopMeta &md) {
      constexpr int C = decltype(CSC)::value;
      const int cs = C >= 0 ? C : flag_case(md.flags);
      double recv[rec_size(GENERAL)];
      if (SREC) lds_rec_any(cs, REC + md.rec, recv);
      else ldg_rec(cs, REC + md.rec, recv);
      const double *rec = recv;
      double lp[6], res[6] = {0, 0, 0, 0, 0, 0}, lx[6], ly[6], aa, bb;
      if (C >= 0) {
        ld6(MT + 6 * q, lp);
        ld6(RT + 6 * q, res);
      } else {
#pragma unroll
        for (int r = 0; r < 6; r++) lp[r] = MT[6 * q + r];
        const int rr = res_rows(cs);
        for (int r = 0; r < rr; r++) res[r] = RT[6 * q + r];
      }
      rec_ratios(cs, rec, 1, aa, bb);
      split(cs, rec, 1, flag_signs(md.flags), aa, bb, lp, res, lx, ly);
      auto put = [&](int16_t ref, const double (&l)[6]) {
        if (ref >= 0) {
          if (C >= 0) {
            st6(MT + 6 * ref, l);
          } else {
#pragma unroll
            for (int r = 0; r < 6; r++) MT[6 * ref + r] = l[r];
          }
        } else {
          const int32_t in = INREF[~(int)ref];
          if (in >= 0) {
            if (C >= 0) {
              st6(a.scratch + 6 * (int64_t)in, l);
            } else {
              for (int r = 0; r < 6; r++) a.scratch[6 * (int64_t)in + r] = l[r];
            }
          } else {
            const int64_t row = (bead0 + ~(int64_t)in) * 3;
            for (int r = 0; r < 3; r++) a.out[(row + r) * K + col] = l[r];
          }
        }
      };
      put(md.x, lx);
      put(md.y, ly);
    };
    for (int lv = h.n_levels - 1; lv >= 0; lv--) {
      for (int q = LB[lv] + tid; q < LB[lv + 1]; q += NTT) {
        const TopMeta md = MD[q];
        if (flag_case(md.flags) == GENERAL) dn_node(std::integral_constant<int, GENERAL>{}, q, md);
        else dn_node(std::integral_constant<int, -1>{}, q, md);
      }
      __syncthreads();
    }
  }
}

template <class... KArgs, class... Args>
void launch_pdl(void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  RQ_CUDA(cudaLaunchKernelEx(&cfg, kernel, args...));
}

}  // namespace

// Per-stream state is created on a stream's first use and kept for the plan's lifetime
// (the header documents the footprint: applications on many distinct streams each hold
// their own exchange slots and staging).
Plan::StreamState &Plan::state_for(cudaStream_t s) const {
  std::lock_guard<std::mutex> lock(state_mu);
  auto &slot = stream_state[s];
  if (!slot) slot.reset(new StreamState());
  return *slot;
}


// dst (cols, rows) = src (rows, cols)^T, both row-major with leading dimensions lds / ldd;
// 32 x 32 tiles through shared memory, a 1-D grid over tiles (rows can exceed grid.y's limit)
__global__ void k_transpose(const double *src, int64_t R, int64_t Cn, int64_t lds, double *dst, int64_t ldd) {
  __shared__ double t[32][33];
  const int64_t ntc = (Cn + 31) / 32;
  const int64_t r0 = (int64_t)(blockIdx.x / ntc) * 32, c0 = (int64_t)(blockIdx.x % ntc) * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < R && c < Cn) t[i][threadIdx.x] = src[r * lds + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < R && c < Cn) dst[c * ldd + r] = t[threadIdx.x][i];
  }
}

// Q layout <-> private residue layout + roots (one thread per row of the Q layout)
__global__ void k_expand(const double *res, const double *roots, const double *in, const int32_t *body_of,
                         const int64_t *bead_off, const int64_t *res_base, int64_t rows, double *out) {
  pdl_wait();
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= rows) return;
  const int j = body_of[row / 3];
  const int64_t b0 = bead_off[j], loc = row - 3 * b0;
  if (bead_off[j + 1] - b0 == 1) out[row] = in[row];
  else out[row] = loc < 6 ? roots[6 * (int64_t)j + loc] : res[res_base[j] + loc - 6];
}
__global__ void k_compress(const double *in, const int32_t *body_of, const int64_t *bead_off, const int64_t *res_base,
                           int64_t rows, double *res, double *roots, double *out) {
  pdl_wait();
  const int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (row >= rows) return;
  const int j = body_of[row / 3];
  const int64_t b0 = bead_off[j], loc = row - 3 * b0;
  const double v = in[row];
  if (bead_off[j + 1] - b0 == 1) out[row] = v;
  else if (loc < 6) roots[6 * (int64_t)j + loc] = v;
  else res[res_base[j] + loc - 6] = v;
}

void run_apply(const Plan &p, int op, const double *in, double *out, int64_t k, cudaStream_t s, unsigned phases) {
  if (op < 0 || op > 3) throw Error(RQ_ERR_VALUE, "op must be one of ('qv', 'qtv', 'qtilde_v', 'qtilde_tv')");
  if (op >= 2 && p.min_n < 2)
    throw Error(RQ_ERR_BODY_TOO_SMALL, "complement operators need every body to have >= 2 beads");
  if (k < 1) throw Error(RQ_ERR_LENGTH, "k must be >= 1");
  RQ_CUDA(cudaSetDevice(p.device));
  Plan::StreamState &ss = p.state_for(s);
  if (ss.scratch.bytes < (size_t)std::max<int64_t>(p.n_slots, 1) * 48) ss.scratch.alloc(std::max<int64_t>(p.n_slots, 1) * 48);
  if (!ss.top_cnt.p) {  // arrival counters start at zero and reset themselves
    ss.top_cnt.alloc(std::max<int64_t>(p.n_top, 1) * 4);
    RQ_CUDA(cudaMemsetAsync(ss.top_cnt.p, 0, std::max<int64_t>(p.n_top, 1) * 4, s));
  }
  if (use_mrhs(p, k)) {  // column-parallel stack-machine kernels (rq_mrhs.cu)
    run_apply_mrhs(p, op, in, out, k, s, phases, BodyRange());
    return;
  }
  if (k > 1) {
    // Column loop on contiguous columns: transpose the (rows, k) block once, run the K = 1
    // kernels column by column, transpose back (a strided column costs 4x the sectors)
    const bool in_comp = op == RQ_OP_QTILDE_TV, out_comp = op == RQ_OP_QTILDE_V;
    const int64_t ri = 3 * p.N - (in_comp ? 6 * p.m : 0), ro = 3 * p.N - (out_comp ? 6 * p.m : 0);
    // columns padded to an even length: every column starts 16-byte aligned (wave gathers)
    const int64_t li = (ri + 1) & ~(int64_t)1, lo = (ro + 1) & ~(int64_t)1;
    if (ss.col_in.bytes < (size_t)(k * li * 8)) ss.col_in.alloc(k * li * 8);
    if (ss.col_out.bytes < (size_t)(k * lo * 8)) ss.col_out.alloc(k * lo * 8);
    double *ti = ss.col_in.as<double>(), *to = ss.col_out.as<double>();
    auto tiles = [](int64_t R, int64_t Cn) { return (unsigned)(((R + 31) / 32) * ((Cn + 31) / 32)); };
    if (ri > 0) k_transpose<<<tiles(ri, k), dim3(32, 8), 0, s>>>(in, ri, k, k, ti, li);
    for (int64_t c = 0; c < k; c++) run_apply(p, op, ti + c * li, to + c * lo, 1, s, phases);
    if (ro > 0) k_transpose<<<tiles(k, ro), dim3(32, 8), 0, s>>>(to, k, ro, lo, out, k);
    RQ_CUDA(cudaGetLastError());
    return;
  }
  const bool up = (op == RQ_OP_QV || op == RQ_OP_QTILDE_V);
  // Q / Q^T run through the private residue layout (Plan::res_base) plus 6 root rows per
  // body: k_compress splits Q^T's input, k_expand assembles Qv (n = 1 bodies: identity,
  // matfree.py:99-100, 127-128); the sweep kernels themselves only know that layout.
  const bool full = op == RQ_OP_QV || op == RQ_OP_QTV;
  double *roots = nullptr;
  const double *cin = in;
  double *cout = out;
  const int64_t rows3 = 3 * p.N;
  if (full) {
    if (ss.roots.bytes < (size_t)(48 * p.m)) ss.roots.alloc(48 * p.m);
    const int64_t rt = std::max<int64_t>(1, p.res_base[p.m]);
    if (ss.res_tmp.bytes < (size_t)(8 * rt)) ss.res_tmp.alloc(8 * rt);
    roots = ss.roots.as<double>();
    if (up) {
      cout = ss.res_tmp.as<double>();
    } else {
      if (phases & 4u)
        launch_pdl(k_compress, (unsigned)((rows3 + 255) / 256), 256, 0, s, in, (const int32_t *)p.body_of.as<int32_t>(),
                   (const int64_t *)p.bead_off_d.as<int64_t>(), (const int64_t *)p.res_base_d.as<int64_t>(), rows3,
                   ss.res_tmp.as<double>(), roots, out);
      cin = ss.res_tmp.as<double>();
    }
  }
  if (reinterpret_cast<uintptr_t>(cin) & 15) {  // the sweep's 16-byte gathers need an aligned input
    const int64_t len = up ? 3 * p.N : p.res_base[p.m];
    if (ss.in_al.bytes < (size_t)(8 * len)) ss.in_al.alloc(8 * std::max<int64_t>(len, 1));
    RQ_CUDA(cudaMemcpyAsync(ss.in_al.p, cin, 8 * len, cudaMemcpyDeviceToDevice, s));
    cin = ss.in_al.as<double>();
  }
  TopDfCtx t{};
  t.starts = p.top_start.as<int32_t>();
  t.paths = p.top_paths.as<int32_t>();
  t.path_off = p.top_path_off.as<int64_t>();
  t.n = p.n_top_start;
  t.top = p.top.as<TopNode>();
  t.parent = p.top_parent.as<int32_t>();
  t.cnt = ss.top_cnt.as<int32_t>();
  t.need = p.top_need.as<int32_t>();
  t.perm = p.perm.as<int32_t>();
  t.bead_off = p.bead_off_d.as<int64_t>();
  t.rec = p.rec.as<double>();
  t.in = cin;
  t.out = cout;
  t.k = 1;
  t.col = 0;
  t.scratch = ss.scratch.as<double>();
  t.res_base = p.res_base_d.as<int64_t>();
  t.roots = roots;
  t.S = p.tile_leaves;
  Top2Ctx t2{};
  t2.blob = p.topblob.as<uint8_t>();
  t2.blob_off = p.topblob_off.as<int64_t>();
  t2.bead_off = p.bead_off_d.as<int64_t>();
  t2.in = cin;
  t2.out = cout;
  t2.k = 1;
  t2.col = 0;
  t2.scratch = ss.scratch.as<double>();
  t2.res_base = p.res_base_d.as<int64_t>();
  t2.roots = roots;
  if (p.n_topblob && !p.top_attr_set) {
    for (const void *f2 : {(const void *)k_top2<true, 32, true>, (const void *)k_top2<false, 32, true>,
                           (const void *)k_top2<true, 32, false>, (const void *)k_top2<false, 32, false>,
                           (const void *)k_top2<true, 128, false>, (const void *)k_top2<false, 128, false>})
      ensure_smem_attr(f2, (size_t)p.max_topblob_smem);
    p.top_attr_set = true;
  }
  const bool do_sweep = (phases & 1u) && p.wave_streams > 0;
  const bool do_top = (phases & 2u) && (p.n_topblob > 0 || t.n > 0);
  auto top_pass = [&]() {
    // phase 0 (whole top trees, pieces) and phase 1 (apexes of split trees): pieces feed the
    // apex upward, the apex feeds the pieces downward
    for (int i = 0; i < 2 * Plan::N_TOPCLASS; i++) {
      const int f = up ? i / Plan::N_TOPCLASS : 1 - i / Plan::N_TOPCLASS, c = i % Plan::N_TOPCLASS;
      const unsigned nb = (unsigned)(p.topclass_first[f][c + 1] - p.topclass_first[f][c]);
      if (!nb) continue;
      t2.order = p.topblob_order.as<int32_t>() + p.topclass_first[f][c];
      const size_t sm = (size_t)p.topclass_smem[c];
      static const int wide_from = [] {  // classes from here on run 128 threads per top tree
        const char *e = getenv("RQ_TOP_WIDE_CLASS");
        return e ? atoi(e) : 4;  // config 4: the <= 64 KB class's wide levels (measured -5%)
      }();
      if (c >= wide_from) {
        if (up) launch_pdl(k_top2<true, 128, false>, nb, 128, sm, s, t2);
        else launch_pdl(k_top2<false, 128, false>, nb, 128, sm, s, t2);
      } else if (c == 0) {
        if (up) launch_pdl(k_top2<true, 32, true>, nb, 32, sm, s, t2);
        else launch_pdl(k_top2<false, 32, true>, nb, 32, sm, s, t2);
      } else {
        if (up) launch_pdl(k_top2<true, 32, false>, nb, 32, sm, s, t2);
        else launch_pdl(k_top2<false, 32, false>, nb, 32, sm, s, t2);
      }
    }
    if (t.n > 0) {
      const unsigned nb = (unsigned)((t.n + NT_TOP - 1) / NT_TOP);
      if (up) launch_pdl(k_top_df_up, nb, NT_TOP, 0, s, t);
      else launch_pdl(k_top_df_down, nb, NT_TOP, 0, s, t);
    }
  };
  auto sweep = [&]() {
    if (!do_sweep) return;
    const int64_t R = std::max<int64_t>(p.wave_rounds, 1);
    if (!ss.round_ctr.p) {  // monotone counters: zeroed once, targets advance per launch
      ss.round_ctr.alloc((2 * R + 2) * 4);
      RQ_CUDA(cudaMemsetAsync(ss.round_ctr.p, 0, (2 * R + 2) * 4, s));
    }
    const uint32_t epoch = ++ss.wave_epoch[up ? 0 : 1];
    run_wave(p, up, cin, cout, ss.scratch.as<double>(), roots, s,
             ss.round_ctr.as<uint32_t>() + (up ? 0 : p.wave_rounds), epoch,
             ss.round_ctr.as<uint32_t>() + 2 * R + (up ? 0 : 1));
  };
  if (up) {
    sweep();
    if (do_top) top_pass();
  } else {
    if (do_top) top_pass();
    sweep();
  }
  if (full && up && (phases & 4u))
    launch_pdl(k_expand, (unsigned)((rows3 + 255) / 256), 256, 0, s, (const double *)ss.res_tmp.as<double>(),
               (const double *)roots, in, (const int32_t *)p.body_of.as<int32_t>(),
               (const int64_t *)p.bead_off_d.as<int64_t>(), (const int64_t *)p.res_base_d.as<int64_t>(), rows3, out);
  RQ_CUDA(cudaGetLastError());
}



}  // namespace rq
