// rq_apply.cu -- the hot path: batched fp64 Qv / Q^T w / Q~v / Q~^T g.
//
// Restates upward_apply (Algorithm 2, matfree.py:95-121, merge_infosets
// matfree.py:41-62) and downward_apply (Algorithm 3, matfree.py:124-151,
// split_rvset matfree.py:65-83) as a chunk sweep plus a top-tree sweep:
//
//   UP   : k_chunk<UP>   (all chunks, persistent CTAs) -> k_top2<UP> / k_top_df_up
//   DOWN : k_top2<DOWN> / k_top_df_down                 -> k_chunk<DOWN>
//
// A chunk is a set of tiles (maximal subtrees of <= tile_leaves beads) of one
// body.  Per chunk, its head (descriptor | tiles | levels | node meta | perm) is
// TMA bulk-copied into shared memory two chunks ahead, its records prefetched
// into L2, its vector data gathered with cp.async one chunk ahead, and each
// height level's records TMA-copied from L2 one level step ahead; the level
// steps run case-uniform warps (GEN / RB / BB) separated by CTA barriers.
// Tile-root 6-vectors pass to the top-tree kernels through exchange slots.
// No tensor cores: this is an HBM-bound sweep of tiny fp64 orthogonal
// transforms (~0.3 flop/B).  DESIGN.md §2.2 has the full description.
#include <algorithm>
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
constexpr int NLS = 2;  // level-record stages in shared memory (records issued NLS-1 steps ahead)
static_assert((NLS & (NLS - 1)) == 0, "stage indices use & (NLS - 1)");

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

// 32-bit shared-address forms (addresses computed once per kernel)
__device__ __forceinline__ void mbar_expect_tx_u(uint32_t bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s_u(uint32_t dst, const void *src, unsigned bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_u(uint32_t addr, unsigned parity) {
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

struct ApplyCtx {
  const ChunkDesc *chunks;
  const TileDesc *tiles;
  const uint8_t *blob;
  int64_t n_chunks;
  const int64_t *bead_off;
  const double *in;
  double *out;
  int64_t k, col;
  double *scratch;
  int op;
  int head_bytes, lrec_bytes, max_nodes, max_beads, max_res, max_tiles;
  int pf_dist;     // L2 prefetch distance of chunk records (chunks ahead)
  uint32_t sm_head, sm_lrec, sm_v, sm_root, sm_o_lrec, sm_o_v, sm_o_m, sm_o_root;  // smem_map(), host-computed
  unsigned long long *ctr;  // {claim, done}: chunks are claimed dynamically (reset by the last CTA)
  const uint8_t *l2_next;   // upward: the staged top blobs the next kernel sweeps, prefetched into
  int64_t l2_next_bytes;    // L2 by each CTA (a 1/grid slice) once it has no chunk left
  long long *dbg;  // phase timers, only with -DRQ_TIMING (8 per CTA)
};

#ifndef RQ_TIMING
#define RQ_TIMING 0
#endif


// record -> registers with 16-byte loads (records are 16-byte aligned, AoS)
template <int CS>
__device__ __forceinline__ void load_rec(const double *rec, double (&R)[rec_size(CS)]) {
  const double2 *r2 = reinterpret_cast<const double2 *>(rec);
#pragma unroll
  for (int i = 0; i < rec_size(CS) / 2; i++) {
    const double2 v = r2[i];
    R[2 * i] = v.x;
    R[2 * i + 1] = v.y;
  }
}

__device__ __forceinline__ void load6(const double *p, double (&v)[6]) {
  const double2 *p2 = reinterpret_cast<const double2 *>(p);
#pragma unroll
  for (int i = 0; i < 3; i++) {
    const double2 w = p2[i];
    v[2 * i] = w.x;
    v[2 * i + 1] = w.y;
  }
}

__device__ __forceinline__ void store6(double *p, const double (&v)[6]) {
  double2 *p2 = reinterpret_cast<double2 *>(p);
#pragma unroll
  for (int i = 0; i < 3; i++) p2[i] = make_double2(v[2 * i], v[2 * i + 1]);
}

// one node of the upward sweep (merge_infosets, matfree.py:41-62)
// Residues go straight to the output block: row = sbase + tile.res_q - tile.res_local + md.res,
// the chunk-local tile index in md.flags bits 6-15 (OB = out + sbase * K + col).
template <int CS, bool K1>
__device__ __forceinline__ void up_node(int slot, const double *rec, const NodeMeta *ME, double *M, const double *F,
                                        const TileDesc *TD, double *OB, int64_t K) {
  double R[rec_size(CS)];
  load_rec<CS>(rec, R);
  const NodeMeta md = ME[slot];
  double mx[6], my[6];
  if (CS == BEAD_BEAD) {  // both children are beads
    const double *f = F + 3 * (md.x & 0x7fff);
    mx[0] = f[0]; mx[1] = f[1]; mx[2] = f[2]; mx[3] = 0.0; mx[4] = 0.0; mx[5] = 0.0;
  } else {
    load6(M + 6 * md.x, mx);
  }
  if (CS != GENERAL) {  // formula-y of BB / RB is a bead
    const double *f = F + 3 * (md.y & 0x7fff);
    my[0] = f[0]; my[1] = f[1]; my[2] = f[2]; my[3] = 0.0; my[4] = 0.0; my[5] = 0.0;
  } else {
    load6(M + 6 * md.y, my);
  }
  double aa, bb, mp[6], res[6];
  rec_ratios(CS, R, 1, aa, bb);
  merge(CS, R, 1, flag_signs(md.flags), aa, bb, mx, my, mp, res);
  if (CS != BEAD_BEAD) {
    const int64_t kk = K1 ? 1 : K;
    double *o = OB + (int64_t)(TD[md.flags >> 6].res_delta + md.res) * kk;
#pragma unroll
    for (int r = 0; r < res_rows(CS); r++) o[r * kk] = res[r];
  }
  store6(M + 6 * slot, mp);
}

// one node of the downward sweep (split_rvset, matfree.py:65-83)
// Bead velocities go straight to the output block through perm (OB = out + 3 bead0 K + col).
template <int CS, bool K1>
__device__ __forceinline__ void down_node(int slot, const double *rec, const NodeMeta *ME, double *M,
                                          const uint32_t *PERM, double *OB, int64_t K, const double *RES) {
  double R[rec_size(CS)];
  load_rec<CS>(rec, R);
  const NodeMeta md = ME[slot];
  double lp[6], res[6] = {0, 0, 0, 0, 0, 0}, lx[6], ly[6];
  load6(M + 6 * slot, lp);
  if (CS == GENERAL) {
#pragma unroll
    for (int r = 0; r < 6; r++) res[r] = RES[md.res + r];
  }
  else if (CS == RIGID_BEAD) { res[0] = RES[md.res]; res[1] = RES[md.res + 1]; res[2] = RES[md.res + 2]; }
  double aa, bb;
  rec_ratios(CS, R, 1, aa, bb);
  split(CS, R, 1, flag_signs(md.flags), aa, bb, lp, res, lx, ly);
  const int64_t kk = K1 ? 1 : K;
  if (CS == BEAD_BEAD) {
    double *o = OB + 3 * (int64_t)PERM[md.x & 0x7fff] * kk;
    o[0] = lx[0]; o[kk] = lx[1]; o[2 * kk] = lx[2];
  } else {
    store6(M + 6 * md.x, lx);
  }
  if (CS != GENERAL) {
    double *o = OB + 3 * (int64_t)PERM[md.y & 0x7fff] * kk;
    o[0] = ly[0]; o[kk] = ly[1]; o[2 * kk] = ly[2];
  } else {
    store6(M + 6 * md.y, ly);
  }
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Shared-memory map of the chunk kernels (all offsets 128-byte aligned):
//   3 head stages (ChunkDesc | TileDesc[] | LevelDesc[] | NodeMeta[] | perm[])
//   2 level-record stages (one height level's records at a time)
//   2 vector stages (UP: gathered forces; DOWN: gathered residues)
//   M (6 per node) | X (UP: residues; DOWN: velocities) | 2 tile-root stages
// Pointers are derived arithmetically from the extern __shared__ base inside
// the kernel (never stored in arrays) so every access compiles to LDS/STS.
struct SmemMap {
  uint32_t head, lrec, v, x, root;  // section sizes (bytes)
  uint32_t o_lrec, o_v, o_m, o_x, o_root;
};

__host__ __device__ __forceinline__ size_t al128(size_t x) { return (x + 127) / 128 * 128; }

__host__ __device__ __forceinline__ SmemMap smem_map(int head_bytes, int lrec_bytes, int max_beads, int max_res,
                                                     int max_nodes, int max_tiles, bool up) {
  SmemMap m;
  m.head = (uint32_t)al128(head_bytes);
  m.lrec = (uint32_t)al128(lrec_bytes);
  m.v = (uint32_t)al128(8 * (size_t)(up ? 3 * max_beads : max_res));
  m.x = 0u;  // outputs go straight to global memory (residues upward, velocities downward)
  m.root = up ? 0u : (uint32_t)al128(48 * (size_t)max_tiles);  // tile-root RV-sets (DOWN only)
  m.o_lrec = 3 * m.head;
  m.o_v = m.o_lrec + NLS * m.lrec;
  m.o_m = m.o_v + 2 * m.v;
  m.o_x = m.o_m + (uint32_t)al128(48 * (size_t)max_nodes);
  m.o_root = m.o_x + m.x;
  return m;
}

__host__ __device__ inline size_t smem_total(const SmemMap &m) { return m.o_root + 2 * (size_t)m.root; }

struct ChunkView {
  const ChunkDesc *hdr;
  const TileDesc *tiles;
  const LevelDesc *LV;
  const NodeMeta *ME;
  const uint32_t *PERM;
};

__device__ __forceinline__ ChunkView view(const unsigned char *B) {
  ChunkView v;
  v.hdr = reinterpret_cast<const ChunkDesc *>(B);
  v.tiles = reinterpret_cast<const TileDesc *>(B + sizeof(ChunkDesc));
  v.LV = reinterpret_cast<const LevelDesc *>(B + sizeof(ChunkDesc) + sizeof(TileDesc) * v.hdr->n_tiles);
  v.ME = reinterpret_cast<const NodeMeta *>(B + v.hdr->off_meta);
  v.PERM = reinterpret_cast<const uint32_t *>(B + v.hdr->off_perm);
  return v;
}

__device__ __forceinline__ void prefetch_l2(const void *p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Stage the vector data a chunk needs, asynchronously (cp.async, one group):
//   UP  : the chunk's bead forces, gathered through perm
//   DOWN: the chunk's residue coefficients (contiguous per tile) + tile-root RV-sets
__device__ __forceinline__ void cp_async16cg_u32(uint32_t dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8_u32(uint32_t dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}

template <bool UP, int NT, bool K1>
__device__ __forceinline__ void prefetch_vectors(const ApplyCtx &a, const unsigned char *B, double *V, double *ROOT) {
  const ChunkView cv = view(B);
  const ChunkDesc &d = *cv.hdr;
  const int64_t bead0 = d.body_bead0;
  const int64_t K = K1 ? 1 : a.k, col = K1 ? 0 : a.col;  // K1: single right-hand side
  const uint32_t vb = smem_u32(V);
  if (UP) {
    const double *inb = a.in + 3 * bead0 * K + col;
    for (int i = threadIdx.x; i < d.n_beads; i += NT) {
      const uint32_t pp = cv.PERM[i];
      if (!(pp & PERM_FOREIGN)) {
        const double *src = inb + 3 * (int64_t)pp * K;
        const uint32_t dst = vb + 24u * (uint32_t)i;
        cp_async8_u32(dst, src);
        cp_async8_u32(dst + 8, src + K);
        cp_async8_u32(dst + 16, src + 2 * K);
      }
    }
  } else {
    const int64_t sbase = (a.op == RQ_OP_QV || a.op == RQ_OP_QTV) ? d.spec_full : d.spec_comp;
    const uint32_t rb = smem_u32(ROOT);
    // one warp per tile (tiles are independent contiguous residue runs)
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int t = wid; t < d.n_tiles; t += NT / 32) {
      const TileDesc T = cv.tiles[t];
      const double *src = a.in + (sbase + T.res_q + lane) * K + col;
      for (int r = lane; r < T.res_count; r += 32, src += 32 * K) cp_async8_u32(vb + 8u * (uint32_t)(T.res_local + r), src);
      if (lane < 6) {
        if (T.scratch >= 0) cp_async8_u32(rb + 8u * (6 * t + lane), a.scratch + 6 * (int64_t)T.scratch + lane);
        else if (a.op == RQ_OP_QTV) cp_async8_u32(rb + 8u * (6 * t + lane), a.in + (3 * bead0 + lane) * K + col);
        else ROOT[6 * t + lane] = 0.0;  // Q~^T: zero root RV-set (matfree.py:167-168)
      }
    }
  }
  cp_async_commit();
}

__device__ __forceinline__ int level_rec_doubles(const LevelDesc &L) {
  return rec_size(GENERAL) * L.nG + rec_size(RIGID_BEAD) * L.nR + rec_size(BEAD_BEAD) * L.nB;
}

// Persistent chunk sweep.  Pipeline per CTA:
//   * chunk k+2: head (desc | tiles | levels | meta | perm) TMA-copied to smem,
//                records prefetched into L2 (cp.async.bulk.prefetch.L2)
//   * chunk k+1: vectors staged with cp.async
//   * chunk k  : swept level by level; the records of level h+1 are TMA-copied
//                (from L2) into the second record stage while level h runs.
// 128-thread CTAs are bounded to 4 per SM (<= 128 registers): without the bound the
// upward K = 1 specialisation takes 159 registers and drops to 3 CTAs/SM.
#ifndef RQ_MIN_BLOCKS
#define RQ_MIN_BLOCKS 4
#endif
template <bool UP, int NT, bool K1>
__global__ void __launch_bounds__(NT, NT == 128 ? RQ_MIN_BLOCKS : 1) k_chunk(ApplyCtx a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[3 + NLS];  // 0-2 heads, 3.. level-record stages
  const int tid = threadIdx.x;
  // TMA producer: lane 0 of the last warp, whose lanes carry the fewest nodes (case groups
  // fill warps from warp 0), so the producer work stays off the slowest warp's path
  constexpr int PROD = NT - 32;
  const long long t_kernel0 = (RQ_TIMING && a.dbg && tid == 0) ? clock64() : 0;
  // section offsets come precomputed in the launch parameters (recomputing smem_map() from
  // the sizes put ~a dozen dependent instructions in front of every node's first load)
  SmemMap SM;
  SM.head = a.sm_head; SM.lrec = a.sm_lrec; SM.v = a.sm_v; SM.root = a.sm_root; SM.x = 0u;
  SM.o_lrec = a.sm_o_lrec; SM.o_v = a.sm_o_v; SM.o_m = a.sm_o_m; SM.o_x = a.sm_o_root; SM.o_root = a.sm_o_root;
  const uint32_t bar_u = smem_u32(bar), smem_u = smem_u32(smem);
#define BAR(i) (bar_u + 8u * (uint32_t)(i))
#define HEAD_U(i) (smem_u + (uint32_t)(i) * SM.head)
#define LREC_U(i) (smem_u + SM.o_lrec + (uint32_t)(i) * SM.lrec)
#define HEAD(i) (smem + (size_t)(i) * SM.head)
#define LREC(i) reinterpret_cast<double *>(smem + SM.o_lrec + (size_t)(i) * SM.lrec)
#define VBUF(i) reinterpret_cast<double *>(smem + SM.o_v + (size_t)(i) * SM.v)
#define ROOTBUF(i) reinterpret_cast<double *>(smem + SM.o_root + (size_t)(i) * SM.root)
  const int64_t K = K1 ? 1 : a.k, col = K1 ? 0 : a.col;
  // Dynamic schedule: the producer claims chunk indices from a global counter a few
  // iterations ahead (atomicAdd, off the critical path), so CTAs finish within about one
  // chunk of each other (a static round robin left the slowest CTA ~12% behind the mean).
  // s_cid[i & 15] = chunk of iteration i; s_cnt = first iteration without a chunk.
  __shared__ long long s_cid[16];
  __shared__ long long s_cnt;
  int64_t n_claimed = 0, cnt_p = LLONG_MAX;  // producer's view
  const int64_t n_static = 4 + a.pf_dist;      // iterations claimed in the prologue
  auto claim_upto = [&](int64_t i) {
    while (n_claimed <= i && cnt_p == LLONG_MAX) {
      // the prologue's claims are static (round robin; 592 CTAs hitting one counter at
      // launch would serialise ~3000 atomics), later claims come from the counter
      const long long G0 = (long long)gridDim.x;
#ifdef RQ_STATIC_SCHED  // round robin throughout (comparison builds)
      const long long c = (long long)blockIdx.x + n_claimed * G0;
#else
      const long long c = n_claimed < n_static ? (long long)blockIdx.x + n_claimed * G0
                                               : n_static * G0 + (long long)atomicAdd(a.ctr, 1ull);
#endif
      if (c >= a.n_chunks) {
        cnt_p = n_claimed;
        s_cnt = n_claimed;
      } else {
        s_cid[n_claimed & 15] = c;
        n_claimed++;
      }
    }
  };
  if (tid == 0) {
    for (int i = 0; i < 3 + NLS; i++) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  if (tid == PROD) {
    s_cnt = LLONG_MAX;
    claim_upto(3 + a.pf_dist);
  }
  __syncthreads();
  auto finish = [&]() {  // the last CTA to finish resets the counters for a later launch
    if (tid == PROD) {
      __threadfence();
      if (atomicAdd(a.ctr + 1, 1ull) == (unsigned long long)gridDim.x - 1) {
        atomicExch(a.ctr, 0ull);
        atomicExch(a.ctr + 1, 0ull);
      }
    }
  };
  if (*(volatile long long *)&s_cnt == 0) {
    finish();
    return;
  }
  // the producer keeps the descriptors of chunks k+2 and k+3 in registers (loaded
  // one iteration before use, so no global latency sits on the critical path)
  longlong2 dk2 = make_longlong2(0, 0), dk3 = make_longlong2(0, 0);  // {blob_off, off_rec | blob_bytes << 32}
  auto ldesc = [&](int64_t k) -> longlong2 {
    claim_upto(k);
    if (k >= cnt_p) return make_longlong2(0, 0);
    const ChunkDesc *d = &a.chunks[s_cid[k & 15]];
    return make_longlong2(d->blob_off, (long long)(uint32_t)d->off_rec | ((long long)(uint32_t)d->blob_bytes << 32));
  };
  if (tid == PROD) {
    const int64_t cnt = cnt_p;
    for (int64_t k = 0; k < 3 && k < cnt; k++) {
      const longlong2 dd = ldesc(k);
      const unsigned hb = (unsigned)(dd.y & 0xffffffffll), rb = (unsigned)(dd.y >> 32) - hb;
      if (rb && k < a.pf_dist) prefetch_l2(a.blob + dd.x + hb, rb);
      if (k < 2) {
        mbar_expect_tx_u(BAR(k), hb);
        bulk_g2s_u(HEAD_U(k), a.blob + dd.x, hb, BAR(k));
      }
    }
    dk2 = ldesc(2);
    dk3 = ldesc(a.pf_dist);
  }
  unsigned phase = 0;  // parity bit per barrier
  int lctr = 0;        // level steps so far (selects the record stage)

  pdl_wait();  // vectors and exchange slots may come from the previous kernel
  mbar_wait_u(BAR(0), 0);
  phase ^= 1u;
  prefetch_vectors<UP, NT, K1>(a, HEAD(0), VBUF(0), ROOTBUF(0));
  // Level-record pipeline (thread 0): level steps are issued NLS-1 steps ahead of
  // the step being swept, across chunk boundaries as far as heads are resident.
  int64_t pf_k = 0;  // chunk iteration of the next level step to issue
  int pf_s = 0;      // its level step within that chunk
  int pf_n = 0;      // level steps issued so far
  int pf_hs = 0;     // head stage of chunk pf_k (= pf_k % 3, tracked incrementally)
  auto issue_levels = [&](int g, int64_t k_avail) {
    // issue while fewer than NLS steps are in flight beyond the current one
    while (pf_n < g + NLS && pf_k < cnt_p && pf_k <= k_avail) {
      const unsigned char *HB = HEAD(pf_hs);
      const ChunkDesc &nd = *reinterpret_cast<const ChunkDesc *>(HB);
      const int nH = nd.n_levels;
      const LevelDesc *LV = reinterpret_cast<const LevelDesc *>(HB + sizeof(ChunkDesc) + sizeof(TileDesc) * nd.n_tiles);
      const LevelDesc &L2 = LV[UP ? pf_s : nH - 1 - pf_s];
      const double *g2 = reinterpret_cast<const double *>(a.blob + nd.blob_off + nd.off_rec) + L2.recG;
      const unsigned bytes = 8u * (unsigned)level_rec_doubles(L2);
      const int st = pf_n & (NLS - 1);
      mbar_expect_tx_u(BAR(3 + st), bytes);
      bulk_g2s_u(LREC_U(st), g2, bytes, BAR(3 + st));
      pf_n++;
      if (++pf_s == nH) {
        pf_s = 0;
        pf_k++;
        pf_hs = pf_hs == 2 ? 0 : pf_hs + 1;
      }
    }
  };
  if (tid == PROD) issue_levels(0, 0);
  for (int64_t k = 0;; k++) {
    // iteration k+1's chunk was claimed at least two CTA barriers ago
    const int64_t cnt = *(volatile long long *)&s_cnt;
    if (k >= cnt) break;
    const int st = (int)(k % 3), fb = (int)(k & 1);
    if (tid == PROD) {
      if (k + 2 < cnt_p) {  // head of chunk k+2 (stage of chunk k-1, released at the end of k-1)
        const int s2 = (int)((k + 2) % 3);
        const unsigned hb = (unsigned)(dk2.y & 0xffffffffll);
        // WAR on smem (generic reads -> TMA write) is ordered by the barrier; no proxy fence needed
        mbar_expect_tx_u(BAR(s2), hb);
        bulk_g2s_u(HEAD_U(s2), a.blob + dk2.x, hb, BAR(s2));
      }
      if (k + a.pf_dist < cnt_p) {  // records of chunk k+pf_dist into L2
        const unsigned hb = (unsigned)(dk3.y & 0xffffffffll), rb = (unsigned)(dk3.y >> 32) - hb;
        if (rb) prefetch_l2(a.blob + dk3.x + hb, rb);
      }
      dk2 = ldesc(k + 3);
      dk3 = ldesc(k + 1 + a.pf_dist);
    }
    long long tc0 = (RQ_TIMING && a.dbg && tid == 0) ? clock64() : 0;
    if (k + 1 < cnt) {
      const int s1 = (int)((k + 1) % 3);
      mbar_wait_u(BAR(s1), (phase >> s1) & 1u);
      phase ^= 1u << s1;
      prefetch_vectors<UP, NT, K1>(a, HEAD(s1), VBUF(fb ^ 1), ROOTBUF(fb ^ 1));
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (RQ_TIMING && a.dbg && tid == 0) { a.dbg[8 * blockIdx.x + 3] += clock64() - tc0; a.dbg[8 * blockIdx.x + 6] += 1; }
    const ChunkView cv = view(HEAD(st));
    const ChunkDesc &d = *cv.hdr;
    const int64_t bead0 = d.body_bead0;
    const int64_t sbase = (a.op == RQ_OP_QV || a.op == RQ_OP_QTV) ? d.spec_full : d.spec_comp;
    double *M = reinterpret_cast<double *>(smem + SM.o_m);
    const int H = d.n_levels;
    const long long t_lv0 = (RQ_TIMING && a.dbg && tid == 0) ? clock64() : 0;
    if (!UP) {
      for (int i = tid; i < 6 * d.n_tiles; i += NT) M[6 * cv.tiles[i / 6].root_slot + i % 6] = ROOTBUF(fb)[i];
      __syncthreads();
    }
    for (int s = 0; s < H; s++, lctr++) {
      const int h = UP ? s : H - 1 - s;
      const int ls = lctr & (NLS - 1);
      const LevelDesc L = cv.LV[h];
      if (tid == PROD) issue_levels(lctr, k + 1 < cnt ? k + 1 : k);
      __shared__ unsigned long long t_max_node, t_step0, t_grp[4];
      if (RQ_TIMING && a.dbg && tid == 0) { t_max_node = 0; t_step0 = clock64(); t_grp[0] = t_grp[1] = t_grp[2] = t_grp[3] = 0; }
      if (RQ_TIMING && a.dbg) __syncthreads();
      long long tw0 = (RQ_TIMING && a.dbg && tid == 0) ? clock64() : 0;
      mbar_wait_u(BAR(3 + ls), (phase >> (3 + ls)) & 1u);
      phase ^= 1u << (3 + ls);
      long long tw1 = (RQ_TIMING && a.dbg && tid == 0) ? clock64() : 0;
      const long long tn0 = (RQ_TIMING && a.dbg) ? clock64() : 0;
      const double *R = LREC(ls);
      const int oR = rec_size(GENERAL) * L.nG, oB = oR + rec_size(RIGID_BEAD) * L.nR;
      // case-uniform warps: GEN and RB groups each padded to whole warps
      const int gG = (L.nG + 31) & ~31, gR = (L.nR + 31) & ~31;
      const int tot = gG + gR + L.nB;
      if (UP) {
        const double *F = VBUF(fb);
        double *OB = a.out + sbase * K + col;
        for (int q = tid; q < tot; q += NT) {
          if (q < gG) {
            if (q < L.nG)
              up_node<GENERAL, K1>(L.slot_begin + q, R + q * rec_size(GENERAL), cv.ME, M, F, cv.tiles, OB, K);
          } else if (q < gG + gR) {
            const int qq = q - gG;
            if (qq < L.nR)
              up_node<RIGID_BEAD, K1>(L.slot_begin + L.nG + qq, R + oR + qq * rec_size(RIGID_BEAD), cv.ME, M, F,
                                      cv.tiles, OB, K);
          } else {
            const int qq = q - gG - gR;
            up_node<BEAD_BEAD, K1>(L.slot_begin + L.nG + L.nR + qq, R + oB + qq * rec_size(BEAD_BEAD), cv.ME, M, F,
                                   cv.tiles, OB, K);
          }
        }
      } else {
        const double *RES = VBUF(fb);
        double *OB = a.out + 3 * bead0 * K + col;
        for (int q = tid; q < tot; q += NT) {
          if (q < gG) {
            if (q < L.nG)
              down_node<GENERAL, K1>(L.slot_begin + q, R + q * rec_size(GENERAL), cv.ME, M, cv.PERM, OB, K, RES);
          } else if (q < gG + gR) {
            const int qq = q - gG;
            if (qq < L.nR)
              down_node<RIGID_BEAD, K1>(L.slot_begin + L.nG + qq, R + oR + qq * rec_size(RIGID_BEAD), cv.ME, M, cv.PERM,
                                        OB, K, RES);
          } else {
            const int qq = q - gG - gR;
            down_node<BEAD_BEAD, K1>(L.slot_begin + L.nG + L.nR + qq, R + oB + qq * rec_size(BEAD_BEAD), cv.ME, M,
                                     cv.PERM, OB, K, RES);
          }
        }
      }
      long long tw2 = (RQ_TIMING && a.dbg && tid == 0) ? clock64() : 0;
      if (RQ_TIMING && a.dbg && (tid & 31) == 0) {
        const unsigned long long dt = (unsigned long long)(clock64() - (long long)t_step0);
        atomicMax(&t_max_node, dt);
        // per-group slowest: 0 GEN, 1 RB, 2 BB, 3 idle
        const int q = tid;
        const int grp = q < gG ? (q < L.nG ? 0 : 3) : (q < gG + gR ? (q - gG < L.nR ? 1 : 3) : (q - gG - gR < L.nB ? 2 : 3));
        atomicMax(&t_grp[grp], dt);
      }
      (void)tn0;
      __syncthreads();
      if (RQ_TIMING && a.dbg && tid == 0) {
        long long tw3 = clock64();
        a.dbg[8 * blockIdx.x + 0] += tw1 - tw0;  // level record wait
        a.dbg[8 * blockIdx.x + 1] += tw2 - tw1;  // tid0 node work
        a.dbg[8 * blockIdx.x + 5] += (long long)t_max_node;  // slowest warp finishes (from step start)
        (void)tw3;
        a.dbg[8 * blockIdx.x + 4] += 1;          // level steps
        for (int g = 0; g < 4; g++)
          if (t_grp[g]) { a.dbg[8 * (gridDim.x + blockIdx.x) + g] += (long long)t_grp[g]; a.dbg[8 * (gridDim.x + blockIdx.x) + 4 + g] += 1; }
      }
    }
    long long to0 = (RQ_TIMING && a.dbg && tid == 0) ? clock64() : 0;
    if (RQ_TIMING && a.dbg && tid == 0) a.dbg[8 * blockIdx.x + 2] += to0 - t_lv0;  // whole level loop
    if (UP) {
      const int wid = tid >> 5, lane = tid & 31;
      for (int t = wid; t < d.n_tiles; t += NT / 32) {  // tile-root info vectors
        const TileDesc T = cv.tiles[t];
        if (lane < 6) {
          const double v = M[6 * T.root_slot + lane];
          if (T.scratch >= 0) a.scratch[6 * (int64_t)T.scratch + lane] = v;
          else if (a.op == RQ_OP_QV) a.out[(3 * bead0 + lane) * K + col] = v;
        }
      }
    }
    __syncthreads();
    (void)to0;
  }
  if (UP && a.l2_next_bytes > 0 && tid == PROD) {
    const int64_t per = (a.l2_next_bytes + gridDim.x - 1) / gridDim.x;
    const int64_t b0 = (per * blockIdx.x) & ~(int64_t)15;
    const int64_t b1 = std::min<int64_t>(a.l2_next_bytes, per * (blockIdx.x + 1));
    for (int64_t b = b0; b < b1; b += 32768) {
      const int64_t len = std::min<int64_t>(32768, b1 - b) & ~(int64_t)15;
      if (len > 0) prefetch_l2(a.l2_next + b, (unsigned)len);
    }
  }
  finish();
  if (RQ_TIMING && a.dbg && tid == 0) a.dbg[8 * blockIdx.x + 7] = clock64() - t_kernel0;
#undef BAR
#undef HEAD_U
#undef LREC_U
#undef HEAD
#undef LREC
#undef VBUF
#undef ROOTBUF
}

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
  const uint8_t *cls;  // shared-memory class per staged body; a launch serves one class
  int want;
  long long *dbg;      // per-CTA phase timers, only with -DRQ_TIMING
  const int64_t *bead_off;
  const double *in;
  double *out;
  int64_t k, col;
  double *scratch;
  const int64_t *res_base;  // private residue layout (Plan::res_base)
  double *roots;            // body-root 6-vectors (Q / Q^T), nullptr for Q~ / Q~^T
};

// NTT threads per top tree: one warp for the small shared-memory classes (top trees
// of config-2 bodies: ~7 nodes per level), 128 for the large ones
template <bool UP, int NTT>
__global__ void __launch_bounds__(NTT) k_top2(Top2Ctx a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  if (a.cls[blockIdx.x] != a.want) return;
  const bool TM = RQ_TIMING && a.dbg && tid == 0;
  const long long c0 = TM ? clock64() : 0;
  unsigned long long g0 = 0;
  if (TM) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  const uint8_t *gB = a.blob + a.blob_off[blockIdx.x];
  // stage the header part (levels, meta, inputs) with one TMA copy; the records stay
  // in global memory (prefetched into L2 here) and are read per node, so the CTA
  // needs little shared memory and many top trees are swept concurrently per SM
  if (tid == 0) {
    const TopHdr *gh = reinterpret_cast<const TopHdr *>(gB);
    const unsigned hbytes = (unsigned)gh->off_rec;
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
  const long long c1 = TM ? clock64() : 0;
  const TopHdr h = *reinterpret_cast<const TopHdr *>(smem);
  const int32_t *LB = reinterpret_cast<const int32_t *>(smem + sizeof(TopHdr));
  const TopMeta *MD = reinterpret_cast<const TopMeta *>(smem + h.off_meta);
  const int32_t *INREF = reinterpret_cast<const int32_t *>(smem + h.off_in);
  const double *REC = reinterpret_cast<const double *>(gB + h.off_rec);
  // X | MT: X holds the input info vectors (UP) or the staged residues (DOWN)
  double *IN = reinterpret_cast<double *>(smem + (h.off_rec + 127) / 128 * 128);
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
    const long long c2 = TM ? clock64() : 0;
    for (int lv = 0; lv < h.n_levels; lv++) {
      for (int q = LB[lv] + tid; q < LB[lv + 1]; q += NTT) {
        const TopMeta md = MD[q];
        const int cs = flag_case(md.flags);
        double recv[rec_size(GENERAL)];
        ldg_rec(cs, REC + md.rec, recv);
        const double *rec = recv;
        double mx[6], my[6], mp[6], res[6], aa, bb;
        const double *px = md.x >= 0 ? MT + 6 * md.x : IN + 6 * ~(int)md.x;
        const double *py = md.y >= 0 ? MT + 6 * md.y : IN + 6 * ~(int)md.y;
#pragma unroll
        for (int r = 0; r < 6; r++) { mx[r] = px[r]; my[r] = py[r]; }
        rec_ratios(cs, rec, 1, aa, bb);
        merge(cs, rec, 1, flag_signs(md.flags), aa, bb, mx, my, mp, res);
        const int rr = res_rows(cs);
        for (int r = 0; r < rr; r++) a.out[(sbase + md.res_q + r) * K + col] = res[r];
        if (md.is_root && a.roots)
          for (int r = 0; r < 6; r++) a.roots[6 * (int64_t)h.body + r] = mp[r];
#pragma unroll
        for (int r = 0; r < 6; r++) MT[6 * q + r] = mp[r];
      }
      __syncthreads();
    }
    if (TM) {
      const long long c3 = clock64();
      long long *d = a.dbg + 8 * blockIdx.x;
      unsigned long long g1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
      d[0] = c1 - c0; d[1] = c2 - c1; d[2] = c3 - c2; d[3] = h.n_levels; d[4] = h.n_nodes; d[5] = h.n_inputs;
      d[6] = (long long)g0; d[7] = (long long)g1;
    }
  } else {
    for (int q = tid; q < h.n_nodes; q += NTT) {  // residues staged with cp.async, all in flight
      const TopMeta md = MD[q];
      const int rr = res_rows(flag_case(md.flags));
      const double *src = a.in + (sbase + md.res_q) * K + col;
      const uint32_t d = smem_u32(RT + 6 * q);
      for (int r = 0; r < rr; r++) cp_async8_u32(d + 8u * r, src + r * K);
      if (md.is_root)
        for (int r = 0; r < 6; r++) MT[6 * q + r] = a.roots ? a.roots[6 * (int64_t)h.body + r] : 0.0;
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    for (int lv = h.n_levels - 1; lv >= 0; lv--) {
      for (int q = LB[lv] + tid; q < LB[lv + 1]; q += NTT) {
        const TopMeta md = MD[q];
        const int cs = flag_case(md.flags);
        double recv[rec_size(GENERAL)];
        ldg_rec(cs, REC + md.rec, recv);
        const double *rec = recv;
        double lp[6], res[6] = {0, 0, 0, 0, 0, 0}, lx[6], ly[6], aa, bb;
#pragma unroll
        for (int r = 0; r < 6; r++) lp[r] = MT[6 * q + r];
        const int rr = res_rows(cs);
        for (int r = 0; r < rr; r++) res[r] = RT[6 * q + r];
        rec_ratios(cs, rec, 1, aa, bb);
        split(cs, rec, 1, flag_signs(md.flags), aa, bb, lp, res, lx, ly);
        auto put = [&](int16_t ref, const double (&l)[6]) {
          if (ref >= 0) {
#pragma unroll
            for (int r = 0; r < 6; r++) MT[6 * ref + r] = l[r];
          } else {
            const int32_t in = INREF[~(int)ref];
            if (in >= 0) {
              for (int r = 0; r < 6; r++) a.scratch[6 * (int64_t)in + r] = l[r];
            } else {
              const int64_t row = (bead0 + ~(int64_t)in) * 3;
              for (int r = 0; r < 3; r++) a.out[(row + r) * K + col] = l[r];
            }
          }
        };
        put(md.x, lx);
        put(md.y, ly);
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

struct KernelCfg {
  int grid = 0, threads = 128;
  size_t smem = 0;
  void (*fn)(ApplyCtx) = nullptr;
};

template <bool UP>
void (*chunk_fn(int nt, bool k1))(ApplyCtx) {
  if (k1 && nt == 128) return k_chunk<UP, 128, true>;
  switch (nt) {
    case 32: return k_chunk<UP, 32, false>;
    case 64: return k_chunk<UP, 64, false>;
    case 256: return k_chunk<UP, 256, false>;
    default: return k_chunk<UP, 128, false>;
  }
}

KernelCfg chunk_cfg(const Plan &p, bool up, ApplyCtx &a) {
  int dev = p.device;
  int sms = 0;
  RQ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  a.head_bytes = (int)p.max_head_bytes;
  a.lrec_bytes = (int)p.max_level_rec_bytes;
  a.max_nodes = std::max(1, p.max_chunk_nodes);
  a.max_beads = std::max(1, p.max_chunk_beads);
  a.max_res = std::max(1, p.max_chunk_res);
  a.max_tiles = std::max(1, p.max_chunk_tiles);
  KernelCfg cfg;
  cfg.threads = p.chunk_threads;
  const SmemMap sm = smem_map(a.head_bytes, a.lrec_bytes, a.max_beads, a.max_res, a.max_nodes, a.max_tiles, up);
  a.sm_head = sm.head; a.sm_lrec = sm.lrec; a.sm_v = sm.v; a.sm_root = sm.root;
  a.sm_o_lrec = sm.o_lrec; a.sm_o_v = sm.o_v; a.sm_o_m = sm.o_m; a.sm_o_root = sm.o_root;
  cfg.smem = smem_total(sm);
  cfg.fn = up ? chunk_fn<true>(cfg.threads, a.k == 1) : chunk_fn<false>(cfg.threads, a.k == 1);
  RQ_CUDA(cudaFuncSetAttribute((const void *)cfg.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.smem));
  int occ = 0;
  RQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void *)cfg.fn, cfg.threads, cfg.smem));
  if (occ < 1) throw Error(RQ_ERR_CUDA, "chunk kernel does not fit on an SM (smem " + std::to_string(cfg.smem) + ")");
  if (const char *e = getenv("RQ_CTAS_PER_SM")) occ = std::max(1, std::min(occ, atoi(e)));
  cfg.grid = (int)std::min<int64_t>(std::max<int64_t>(a.n_chunks, 1), (int64_t)sms * occ);
  return cfg;
}

}  // namespace

Plan::StreamState &Plan::state_for(cudaStream_t s) const {
  std::lock_guard<std::mutex> lock(state_mu);
  auto &slot = stream_state[s];
  if (!slot) slot.reset(new StreamState());
  return *slot;
}

void chunk_occupancy(const Plan &p, int ctas[2], int64_t smem[2]) {
  for (int u = 0; u < 2; u++) {
    ApplyCtx a{};
    a.k = 1;
    a.n_chunks = p.n_chunks;
    KernelCfg cfg = chunk_cfg(p, u == 1, a);
    smem[u] = (int64_t)cfg.smem;
    int sms = 0;
    RQ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p.device));
    ctas[u] = sms ? (int)((cfg.grid + sms - 1) / sms) : 0;
  }
}

// dst (cols, rows) = src (rows, cols)^T, both row-major; 32 x 32 tiles through shared memory,
// a 1-D grid over tiles (rows can exceed the 65535 limit of grid.y)
__global__ void k_transpose(const double *src, int64_t R, int64_t Cn, double *dst) {
  __shared__ double t[32][33];
  const int64_t ntc = (Cn + 31) / 32;
  const int64_t r0 = (int64_t)(blockIdx.x / ntc) * 32, c0 = (int64_t)(blockIdx.x % ntc) * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < R && c < Cn) t[i][threadIdx.x] = src[r * Cn + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < R && c < Cn) dst[c * R + r] = t[threadIdx.x][i];
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

void run_apply(const Plan &p, int op, const double *in, double *out, int64_t k, cudaStream_t s, unsigned phases,
               BodyRange range) {
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
    run_apply_mrhs(p, op, in, out, k, s, phases, range);
    return;
  }
  if (k > 1) {
    if (range.j1 >= 0) throw Error(RQ_ERR_VALUE, "body ranges need k == 1");
    // Column loop on contiguous columns: transpose the (rows, k) block once, run the K = 1
    // kernels column by column, transpose back (a strided column costs 4x the sectors)
    const bool in_comp = op == RQ_OP_QTILDE_TV, out_comp = op == RQ_OP_QTILDE_V;
    const int64_t ri = 3 * p.N - (in_comp ? 6 * p.m : 0), ro = 3 * p.N - (out_comp ? 6 * p.m : 0);
    if (ss.col_in.bytes < (size_t)(k * ri * 8)) ss.col_in.alloc(k * ri * 8);
    if (ss.col_out.bytes < (size_t)(k * ro * 8)) ss.col_out.alloc(k * ro * 8);
    double *ti = ss.col_in.as<double>(), *to = ss.col_out.as<double>();
    auto tiles = [](int64_t R, int64_t Cn) { return (unsigned)(((R + 31) / 32) * ((Cn + 31) / 32)); };
    if (ri > 0) k_transpose<<<tiles(ri, k), dim3(32, 8), 0, s>>>(in, ri, k, ti);
    for (int64_t c = 0; c < k; c++) run_apply(p, op, ti + c * ri, to + c * ro, 1, s, phases, range);
    if (ro > 0) k_transpose<<<tiles(k, ro), dim3(32, 8), 0, s>>>(to, k, ro, out);
    RQ_CUDA(cudaGetLastError());
    return;
  }
  const bool up = (op == RQ_OP_QV || op == RQ_OP_QTILDE_V);
  const bool all = range.j1 < 0;
  // Q / Q^T run through the private residue layout (Plan::res_base) plus 6 root rows per
  // body: k_compress splits Q^T's input, k_expand assembles Qv (n = 1 bodies: identity,
  // matfree.py:99-100, 127-128); the sweep kernels themselves only know that layout.
  const bool full = op == RQ_OP_QV || op == RQ_OP_QTV;
  double *roots = nullptr;
  const double *cin = in;
  double *cout = out;
  const int64_t rows3 = 3 * p.N;
  if (full) {
    if (!all) throw Error(RQ_ERR_VALUE, "body ranges need a complement operator");
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
  static const bool old_chunks = getenv("RQ_WAVE") && atoi(getenv("RQ_WAVE")) == 0;  // A/B comparison only
  const bool wave = p.wave_streams > 0 && all && !old_chunks;
  const int64_t j0 = all ? 0 : range.j0, j1 = all ? p.m : range.j1;
  const int64_t c0 = all ? 0 : p.h_chunk_first[j0], c1 = all ? p.n_chunks : p.h_chunk_first[j1];
  const int64_t tb0 = all ? 0 : p.h_topblob_first[j0], tb1 = all ? p.n_topblob : p.h_topblob_first[j1];
  ApplyCtx a{};
  KernelCfg cfg;
  if (!wave) {
    a.chunks = p.chunks.as<ChunkDesc>() + c0;
    a.tiles = p.tiles.as<TileDesc>();
    a.blob = p.blob.as<uint8_t>();
    a.n_chunks = c1 - c0;
    a.bead_off = p.bead_off_d.as<int64_t>();
    a.in = cin;
    a.out = cout;
    a.k = 1;
    a.scratch = ss.scratch.as<double>();
    a.op = up ? RQ_OP_QTILDE_V : RQ_OP_QTILDE_TV;
    cfg = chunk_cfg(p, up, a);
    if (!ss.chunk_ctr.p) {  // claim/done counters start at zero and reset themselves
      ss.chunk_ctr.alloc(4 * sizeof(unsigned long long));
      RQ_CUDA(cudaMemsetAsync(ss.chunk_ctr.p, 0, 4 * sizeof(unsigned long long), s));
    }
    if (up && tb1 > tb0) {  // the top pass that follows reads these blobs
      a.l2_next = p.topblob.as<uint8_t>() + p.h_topblob_off[tb0];
      a.l2_next_bytes = p.h_topblob_off[tb1] - p.h_topblob_off[tb0];
    }
    a.pf_dist = 1;
  }
  TopDfCtx t{};
  const int64_t ts0 = all ? 0 : p.h_topstart_first[j0], ts1 = all ? p.n_top_start : p.h_topstart_first[j1];
  t.starts = p.top_start.as<int32_t>() + ts0;
  t.paths = p.top_paths.as<int32_t>();
  t.path_off = p.top_path_off.as<int64_t>() + ts0;
  t.n = ts1 - ts0;
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
  t2.blob_off = p.topblob_off.as<int64_t>() + tb0;
  t2.cls = p.topblob_class.as<uint8_t>() + tb0;
  t2.bead_off = p.bead_off_d.as<int64_t>();
  t2.in = cin;
  t2.out = cout;
  t2.k = 1;
  t2.col = 0;
  t2.scratch = ss.scratch.as<double>();
  t2.res_base = p.res_base_d.as<int64_t>();
  t2.roots = roots;
  if (p.n_topblob && !p.top_attr_set) {
    for (const void *f2 : {(const void *)k_top2<true, 32>, (const void *)k_top2<false, 32>,
                           (const void *)k_top2<true, 128>, (const void *)k_top2<false, 128>})
      RQ_CUDA(cudaFuncSetAttribute(f2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.max_topblob_smem));
    p.top_attr_set = true;
  }
  const bool do_chunks = (phases & 1u) && (wave ? p.wave_streams > 0 : a.n_chunks > 0);
  const bool do_top = (phases & 2u) && (tb1 > tb0 || t.n > 0);
  auto top_pass = [&]() {
    for (int c = 0; c < 4 && tb1 > tb0; c++) {
      if (!p.topclass_count[c]) continue;
      t2.want = c;
      const size_t sm = (size_t)p.topclass_smem[c];
      if (c < 2) {
        if (up) launch_pdl(k_top2<true, 32>, (unsigned)(tb1 - tb0), 32, sm, s, t2);
        else launch_pdl(k_top2<false, 32>, (unsigned)(tb1 - tb0), 32, sm, s, t2);
      } else {
        if (up) launch_pdl(k_top2<true, 128>, (unsigned)(tb1 - tb0), 128, sm, s, t2);
        else launch_pdl(k_top2<false, 128>, (unsigned)(tb1 - tb0), 128, sm, s, t2);
      }
    }
    if (t.n > 0) {
      const unsigned nb = (unsigned)((t.n + NT_TOP - 1) / NT_TOP);
      if (up) launch_pdl(k_top_df_up, nb, NT_TOP, 0, s, t);
      else launch_pdl(k_top_df_down, nb, NT_TOP, 0, s, t);
    }
  };
  auto sweep = [&]() {
    if (!do_chunks) return;
    if (wave) {
      run_wave(p, up, cin, cout, ss.scratch.as<double>(), roots, s);
    } else {
      a.ctr = ss.chunk_ctr.as<unsigned long long>() + 2 * (ss.chunk_epoch++ & 1u);
      launch_pdl(cfg.fn, (unsigned)cfg.grid, (unsigned)cfg.threads, cfg.smem, s, a);
    }
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


void run_apply_host(const Plan &p, int op, const double *in, double *out, int64_t k) {
  if (op < 0 || op > 3) throw Error(RQ_ERR_VALUE, "op must be one of ('qv', 'qtv', 'qtilde_v', 'qtilde_tv')");
  if (k < 1) throw Error(RQ_ERR_LENGTH, "k must be >= 1");
  if (op >= 2 && p.min_n < 2)
    throw Error(RQ_ERR_BODY_TOO_SMALL, "complement operators need every body to have >= 2 beads");
  RQ_CUDA(cudaSetDevice(p.device));
  std::lock_guard<std::mutex> lock(p.host_mu);
  if (!p.host_stream) {
    for (auto *st : {&p.host_stream, &p.host_stream2, &p.host_stream3})
      RQ_CUDA(cudaStreamCreateWithFlags(st, cudaStreamNonBlocking));
  }
  const bool in_comp = op == RQ_OP_QTILDE_TV, out_comp = op == RQ_OP_QTILDE_V;
  const int64_t ri = 3 * p.N - (in_comp ? 6 * p.m : 0), ro = 3 * p.N - (out_comp ? 6 * p.m : 0);
  const size_t bi = (size_t)ri * k * 8, bo = (size_t)ro * k * 8;
  if (p.stage_in.bytes < bi) p.stage_in.alloc(bi);
  if (p.stage_out.bytes < bo) p.stage_out.alloc(bo);
  cudaStream_t s_k = p.host_stream2;
  double *din = p.stage_in.as<double>(), *dout = p.stage_out.as<double>();
  RQ_CUDA(cudaMemcpyAsync(din, in, bi, cudaMemcpyHostToDevice, s_k));
  run_apply(p, op, din, dout, k, s_k);
  RQ_CUDA(cudaMemcpyAsync(out, dout, bo, cudaMemcpyDeviceToHost, s_k));
  RQ_CUDA(cudaStreamSynchronize(s_k));
}

}  // namespace rq
