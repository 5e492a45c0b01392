// rq_apply.cu -- the hot path: batched fp64 Qv / Q^T w / Q~v / Q~^T g.
//
// Restates upward_apply (Algorithm 2, matfree.py:95-121, merge_infosets
// matfree.py:41-62) and downward_apply (Algorithm 3, matfree.py:124-151,
// split_rvset matfree.py:65-83) as two kernels each:
//
//   UP   : k_chunk_up (all chunks, persistent CTAs) -> k_top_up (per body)
//   DOWN : k_top_down (per body)                     -> k_chunk_down
//
// A chunk blob (level table | node meta | perm | SoA factor records) is moved
// HBM -> shared memory with one cp.async.bulk (TMA bulk copy) per chunk,
// double-buffered on an mbarrier so the next chunk streams in while the
// current one is swept level by level (one thread per node, nodes of a level
// are independent).  Children exchange their 6-long info/RV vectors through
// shared memory; the beads' forces/velocities are gathered/scattered through
// perm once per chunk.  No tensor cores: this is an HBM-bound sweep of tiny
// orthogonal transforms (~0.3-0.6 flop/B).
#include <algorithm>
#include <cstdio>

#include "rq_nodeops.cuh"
#include "rq_plan.hpp"

namespace rq {
namespace {

constexpr int NT_TOP = 128;

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
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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
  int buf_bytes, max_nodes, max_beads, max_res;
};

__device__ __forceinline__ int64_t spec_base(int op, const int64_t *bead_off, int j) {
  // first residue row of body j in the op's spectral layout
  return (op == RQ_OP_QV || op == RQ_OP_QTV) ? 3 * bead_off[j] + 6 : 3 * bead_off[j] - 6 * (int64_t)j;
}

__device__ __forceinline__ void issue_chunk(const ApplyCtx &a, int64_t c, void *dst, uint64_t *bar) {
  const ChunkDesc *d = &a.chunks[c];
  unsigned bytes = (unsigned)d->blob_bytes;
  mbar_expect_tx(bar, bytes);
  bulk_g2s(dst, a.blob + d->blob_off, bytes, bar);
}

// one node of the upward sweep (merge_infosets, matfree.py:41-62)
template <int CS>
__device__ __forceinline__ void up_node(int slot, const double *rec, int st, const NodeMeta *ME, double *M,
                                        const double *F, double *RES) {
  const NodeMeta md = ME[slot];
  double mx[6], my[6];
  if (md.x & SRC_BEAD) {
    const double *f = F + 3 * (md.x & 0x7fff);
    mx[0] = f[0]; mx[1] = f[1]; mx[2] = f[2]; mx[3] = 0.0; mx[4] = 0.0; mx[5] = 0.0;
  } else {
#pragma unroll
    for (int r = 0; r < 6; r++) mx[r] = M[6 * md.x + r];
  }
  if (CS != GENERAL && (md.y & SRC_BEAD)) {  // formula-y of BB / RB is always a bead
    const double *f = F + 3 * (md.y & 0x7fff);
    my[0] = f[0]; my[1] = f[1]; my[2] = f[2]; my[3] = 0.0; my[4] = 0.0; my[5] = 0.0;
  } else {
#pragma unroll
    for (int r = 0; r < 6; r++) my[r] = M[6 * md.y + r];
  }
  double aa, bb, mp[6], res[6];
  rec_ratios(CS, rec, st, aa, bb);
  merge(CS, rec, st, flag_signs(md.flags), aa, bb, mx, my, mp, res);
#pragma unroll
  for (int r = 0; r < res_rows(CS); r++) RES[md.res + r] = res[r];
#pragma unroll
  for (int r = 0; r < 6; r++) M[6 * slot + r] = mp[r];
}

// one node of the downward sweep (split_rvset, matfree.py:65-83)
template <int CS>
__device__ __forceinline__ void down_node(int slot, const double *rec, int st, const NodeMeta *ME, double *M,
                                          double *F, const double *RES) {
  const NodeMeta md = ME[slot];
  double lp[6], res[6] = {0, 0, 0, 0, 0, 0}, lx[6], ly[6];
#pragma unroll
  for (int r = 0; r < 6; r++) lp[r] = M[6 * slot + r];
#pragma unroll
  for (int r = 0; r < res_rows(CS); r++) res[r] = RES[md.res + r];
  double aa, bb;
  rec_ratios(CS, rec, st, aa, bb);
  split(CS, rec, st, flag_signs(md.flags), aa, bb, lp, res, lx, ly);
  if (md.x & SRC_BEAD) {
    double *f = F + 3 * (md.x & 0x7fff);
    f[0] = lx[0]; f[1] = lx[1]; f[2] = lx[2];
  } else {
#pragma unroll
    for (int r = 0; r < 6; r++) M[6 * md.x + r] = lx[r];
  }
  if (md.y & SRC_BEAD) {
    double *f = F + 3 * (md.y & 0x7fff);
    f[0] = ly[0]; f[1] = ly[1]; f[2] = ly[2];
  } else {
#pragma unroll
    for (int r = 0; r < 6; r++) M[6 * md.y + r] = ly[r];
  }
}

template <bool UP, int NT_CHUNK>
__global__ void __launch_bounds__(NT_CHUNK) k_chunk(ApplyCtx a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[2];
  const int tid = threadIdx.x;
  unsigned char *buf0 = smem, *buf1 = smem + a.buf_bytes;
  double *M = reinterpret_cast<double *>(smem + 2 * a.buf_bytes);
  double *F = M + 6 * a.max_nodes;
  double *RES = F + 3 * a.max_beads;
  const int64_t K = a.k, col = a.col;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  int64_t c = blockIdx.x;
  if (c < a.n_chunks && tid == 0) issue_chunk(a, c, buf0, &bar[0]);
  unsigned phase0 = 0, phase1 = 0;
  for (int it = 0; c < a.n_chunks; c += gridDim.x, it++) {
    const int b = it & 1;
    const int64_t cn = c + gridDim.x;
    if (cn < a.n_chunks && tid == 0) {
      fence_proxy_async();
      issue_chunk(a, cn, b ? buf0 : buf1, b ? &bar[0] : &bar[1]);
    }
    const ChunkDesc d = a.chunks[c];
    const int j = d.body;
    const int64_t bead0 = a.bead_off[j];
    const int64_t sbase = spec_base(a.op, a.bead_off, j);
    if (b) { mbar_wait(&bar[1], phase1); phase1 ^= 1u; }
    else { mbar_wait(&bar[0], phase0); phase0 ^= 1u; }
    const unsigned char *B = b ? buf1 : buf0;
    const LevelDesc *LV = reinterpret_cast<const LevelDesc *>(B);
    const NodeMeta *ME = reinterpret_cast<const NodeMeta *>(B + d.off_meta);
    const uint32_t *PERM = reinterpret_cast<const uint32_t *>(B + d.off_perm);
    const double *REC = reinterpret_cast<const double *>(B + d.off_rec);

    if (UP) {
      for (int i = tid; i < d.n_beads; i += NT_CHUNK) {
        uint32_t pp = PERM[i];
        if (!(pp & PERM_FOREIGN)) {
          const int64_t row = (bead0 + pp) * 3;
          F[i * 3 + 0] = a.in[(row + 0) * K + col];
          F[i * 3 + 1] = a.in[(row + 1) * K + col];
          F[i * 3 + 2] = a.in[(row + 2) * K + col];
        }
      }
      __syncthreads();
      for (int h = 0; h < d.n_levels; h++) {
        const LevelDesc L = LV[h];
        // case-uniform warps: each case group is padded to whole warps
        const int gG = (L.nG + 31) & ~31, gR = (L.nR + 31) & ~31;
        const int tot = gG + gR + L.nB;
        for (int q = tid; q < tot; q += NT_CHUNK) {
          if (q < gG) {
            if (q < L.nG) up_node<GENERAL>(L.slot_begin + q, REC + L.recG + q, L.nG, ME, M, F, RES);
          } else if (q < gG + gR) {
            const int qq = q - gG;
            if (qq < L.nR) up_node<RIGID_BEAD>(L.slot_begin + L.nG + qq, REC + L.recR + qq, L.nR, ME, M, F, RES);
          } else {
            const int qq = q - gG - gR;
            up_node<BEAD_BEAD>(L.slot_begin + L.nG + L.nR + qq, REC + L.recB + qq, L.nB, ME, M, F, RES);
          }
        }
        __syncthreads();
      }
      // residues (contiguous per tile) and tile-root info vectors
      for (int t = 0; t < d.n_tiles; t++) {
        const TileDesc T = a.tiles[d.tile_begin + t];
        for (int r = tid; r < T.res_count; r += NT_CHUNK)
          a.out[(sbase + T.res_q + r) * K + col] = RES[T.res_local + r];
        if (tid < 6) {
          const double v = M[6 * T.root_slot + tid];
          if (T.scratch >= 0) a.scratch[6 * (int64_t)T.scratch + tid] = v;
          else if (a.op == RQ_OP_QV) a.out[(3 * bead0 + tid) * K + col] = v;
        }
      }
    } else {
      for (int t = 0; t < d.n_tiles; t++) {
        const TileDesc T = a.tiles[d.tile_begin + t];
        for (int r = tid; r < T.res_count; r += NT_CHUNK)
          RES[T.res_local + r] = a.in[(sbase + T.res_q + r) * K + col];
        if (tid < 6) {
          double v;
          if (T.scratch >= 0) v = a.scratch[6 * (int64_t)T.scratch + tid];
          else v = (a.op == RQ_OP_QTV) ? a.in[(3 * bead0 + tid) * K + col] : 0.0;
          M[6 * T.root_slot + tid] = v;
        }
      }
      __syncthreads();
      for (int h = d.n_levels - 1; h >= 0; h--) {
        const LevelDesc L = LV[h];
        const int gG = (L.nG + 31) & ~31, gR = (L.nR + 31) & ~31;
        const int tot = gG + gR + L.nB;
        for (int q = tid; q < tot; q += NT_CHUNK) {
          if (q < gG) {
            if (q < L.nG) down_node<GENERAL>(L.slot_begin + q, REC + L.recG + q, L.nG, ME, M, F, RES);
          } else if (q < gG + gR) {
            const int qq = q - gG;
            if (qq < L.nR) down_node<RIGID_BEAD>(L.slot_begin + L.nG + qq, REC + L.recR + qq, L.nR, ME, M, F, RES);
          } else {
            const int qq = q - gG - gR;
            down_node<BEAD_BEAD>(L.slot_begin + L.nG + L.nR + qq, REC + L.recB + qq, L.nB, ME, M, F, RES);
          }
        }
        __syncthreads();
      }
      for (int i = tid; i < d.n_beads; i += NT_CHUNK) {
        uint32_t pp = PERM[i];
        if (!(pp & PERM_FOREIGN)) {
          const int64_t row = (bead0 + pp) * 3;
          a.out[(row + 0) * K + col] = F[i * 3 + 0];
          a.out[(row + 1) * K + col] = F[i * 3 + 1];
          a.out[(row + 2) * K + col] = F[i * 3 + 2];
        }
      }
    }
    __syncthreads();
  }
}

// ---- top tree (nodes with more than tile_leaves beads) ---------------------------------

struct TopCtx {
  const TopNode *top;
  const int32_t *topbody, *topbody_lvl, *toplvl, *perm;
  const int64_t *bead_off;
  const double *rec;
  const double *in;
  double *out;
  int64_t k, col;
  double *scratch;
  int op;
};

template <bool UP>
__global__ void __launch_bounds__(NT_TOP) k_top(TopCtx a) {
  const int bi = blockIdx.x;
  const int j = a.topbody[bi];
  const int64_t bead0 = a.bead_off[j];
  const int64_t sbase = spec_base(a.op, a.bead_off, j);
  const int64_t K = a.k, col = a.col;
  const int lv0 = a.topbody_lvl[bi], lv1 = a.topbody_lvl[bi + 1];
  for (int s = 0; s < lv1 - lv0; s++) {
    const int lv = UP ? lv0 + s : lv1 - 1 - s;
    const int p0 = a.toplvl[lv], p1 = a.toplvl[lv + 1];
    for (int p = p0 + threadIdx.x; p < p1; p += NT_TOP) {
      const TopNode T = a.top[p];
      const int cs = flag_case(T.flags);
      const unsigned signs = flag_signs(T.flags);
      const double *rec = a.rec + T.rec_off;
      double aa, bb;
      rec_ratios(cs, rec, 1, aa, bb);
      const int rr = res_rows(cs);
      if (UP) {
        double mx[6], my[6], mp[6], res[6];
        auto fetch = [&](int32_t ref, double (&m)[6]) {
          if (ref >= 0) {
#pragma unroll
            for (int r = 0; r < 6; r++) m[r] = __ldcg(&a.scratch[6 * (int64_t)ref + r]);
          } else {
            const int64_t gb = ~(int64_t)ref;
            const int64_t row = (bead0 + a.perm[gb]) * 3;
            m[0] = a.in[(row + 0) * K + col];
            m[1] = a.in[(row + 1) * K + col];
            m[2] = a.in[(row + 2) * K + col];
            m[3] = m[4] = m[5] = 0.0;
          }
        };
        fetch(T.x, mx);
        fetch(T.y, my);
        merge(cs, rec, 1, signs, aa, bb, mx, my, mp, res);
        for (int r = 0; r < rr; r++) a.out[(sbase + T.res_q + r) * K + col] = res[r];
        if (T.is_root) {
          if (a.op == RQ_OP_QV)
            for (int r = 0; r < 6; r++) a.out[(3 * bead0 + r) * K + col] = mp[r];
        } else {
          for (int r = 0; r < 6; r++) a.scratch[6 * (int64_t)T.self_slot + r] = mp[r];
        }
      } else {
        double lp[6], res[6] = {0, 0, 0, 0, 0, 0}, lx[6], ly[6];
        if (T.is_root) {
          for (int r = 0; r < 6; r++) lp[r] = (a.op == RQ_OP_QTV) ? a.in[(3 * bead0 + r) * K + col] : 0.0;
        } else {
          for (int r = 0; r < 6; r++) lp[r] = __ldcg(&a.scratch[6 * (int64_t)T.self_slot + r]);
        }
        for (int r = 0; r < rr; r++) res[r] = a.in[(sbase + T.res_q + r) * K + col];
        split(cs, rec, 1, signs, aa, bb, lp, res, lx, ly);
        auto store = [&](int32_t ref, const double (&l)[6]) {
          if (ref >= 0) {
            for (int r = 0; r < 6; r++) a.scratch[6 * (int64_t)ref + r] = l[r];
          } else {
            const int64_t gb = ~(int64_t)ref;
            const int64_t row = (bead0 + a.perm[gb]) * 3;
            a.out[(row + 0) * K + col] = l[0];
            a.out[(row + 1) * K + col] = l[1];
            a.out[(row + 2) * K + col] = l[2];
          }
        };
        store(T.x, lx);
        store(T.y, ly);
      }
    }
    __syncthreads();
  }
}

// single-bead bodies: Qv and Q^T w are the identity (matfree.py:99-100, 127-128)
__global__ void k_small(const int32_t *bodies, int64_t n, const int64_t *bead_off, const double *in,
                        double *out, int64_t K, int64_t col) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= 3 * n) return;
  int64_t row = 3 * bead_off[bodies[t / 3]] + t % 3;
  out[row * K + col] = in[row * K + col];
}

struct KernelCfg {
  int grid = 0, threads = 128;
  size_t smem = 0;
  void (*fn)(ApplyCtx) = nullptr;
};

template <bool UP>
void (*chunk_fn(int nt))(ApplyCtx) {
  switch (nt) {
    case 32: return k_chunk<UP, 32>;
    case 64: return k_chunk<UP, 64>;
    case 256: return k_chunk<UP, 256>;
    default: return k_chunk<UP, 128>;
  }
}

KernelCfg chunk_cfg(const Plan &p, bool up, ApplyCtx &a) {
  int dev = p.device;
  int sms = 0;
  RQ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  a.buf_bytes = (int)((p.max_blob + 127) / 128 * 128);
  a.max_nodes = std::max(1, p.max_chunk_nodes);
  a.max_beads = std::max(1, p.max_chunk_beads);
  a.max_res = std::max(1, p.max_chunk_res);
  KernelCfg cfg;
  cfg.threads = p.chunk_threads;
  cfg.smem = 2 * (size_t)a.buf_bytes + 8 * (6 * (size_t)a.max_nodes + 3 * (size_t)a.max_beads + (size_t)a.max_res);
  cfg.fn = up ? chunk_fn<true>(cfg.threads) : chunk_fn<false>(cfg.threads);
  RQ_CUDA(cudaFuncSetAttribute((const void *)cfg.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.smem));
  int occ = 0;
  RQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void *)cfg.fn, cfg.threads, cfg.smem));
  if (occ < 1) throw Error(RQ_ERR_CUDA, "chunk kernel does not fit on an SM (smem " + std::to_string(cfg.smem) + ")");
  cfg.grid = (int)std::min<int64_t>(p.n_chunks, (int64_t)sms * occ);
  return cfg;
}

}  // namespace

void run_apply(const Plan &p, int op, const double *in, double *out, int64_t k, cudaStream_t s, unsigned phases) {
  if (op < 0 || op > 3) throw Error(RQ_ERR_VALUE, "op must be one of ('qv', 'qtv', 'qtilde_v', 'qtilde_tv')");
  if (op >= 2 && p.min_n < 2)
    throw Error(RQ_ERR_BODY_TOO_SMALL, "complement operators need every body to have >= 2 beads");
  if (k < 1) throw Error(RQ_ERR_LENGTH, "k must be >= 1");
  RQ_CUDA(cudaSetDevice(p.device));
  if (p.scratch_k < 1 || p.scratch.bytes < (size_t)std::max<int64_t>(p.n_slots, 1) * 48) {
    p.scratch.alloc(std::max<int64_t>(p.n_slots, 1) * 48);
    p.scratch_k = 1;
  }
  const bool up = (op == RQ_OP_QV || op == RQ_OP_QTILDE_V);
  ApplyCtx a{};
  a.chunks = p.chunks.as<ChunkDesc>();
  a.tiles = p.tiles.as<TileDesc>();
  a.blob = p.blob.as<uint8_t>();
  a.n_chunks = p.n_chunks;
  a.bead_off = p.bead_off_d.as<int64_t>();
  a.in = in;
  a.out = out;
  a.k = k;
  a.scratch = p.scratch.as<double>();
  a.op = op;
  KernelCfg cfg = chunk_cfg(p, up, a);
  TopCtx t{};
  t.top = p.top.as<TopNode>();
  t.topbody = p.topbody.as<int32_t>();
  t.topbody_lvl = p.topbody_lvl.as<int32_t>();
  t.toplvl = p.toplvl.as<int32_t>();
  t.perm = p.perm.as<int32_t>();
  t.bead_off = p.bead_off_d.as<int64_t>();
  t.rec = p.rec.as<double>();
  t.in = in;
  t.out = out;
  t.k = k;
  t.scratch = p.scratch.as<double>();
  t.op = op;
  for (int64_t col = 0; col < k; col++) {
    a.col = col;
    t.col = col;
    const bool do_chunks = (phases & 1u) && p.n_chunks, do_top = (phases & 2u) && p.n_topbodies;
    if (up) {
      if (do_chunks) cfg.fn<<<cfg.grid, cfg.threads, cfg.smem, s>>>(a);
      if (do_top) k_top<true><<<(unsigned)p.n_topbodies, NT_TOP, 0, s>>>(t);
    } else {
      if (do_top) k_top<false><<<(unsigned)p.n_topbodies, NT_TOP, 0, s>>>(t);
      if (do_chunks) cfg.fn<<<cfg.grid, cfg.threads, cfg.smem, s>>>(a);
    }
    if ((phases & 4u) && p.n_small && op <= 1)
      k_small<<<(unsigned)((3 * p.n_small + 255) / 256), 256, 0, s>>>(p.small_bodies.as<int32_t>(), p.n_small,
                                                                      p.bead_off_d.as<int64_t>(), in, out, k, col);
  }
  RQ_CUDA(cudaGetLastError());
}

}  // namespace rq
