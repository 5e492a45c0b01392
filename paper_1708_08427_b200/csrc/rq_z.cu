// rq_z.cu -- (c) force/torque reductions Zf and Z^T u (model.py:129-149) and
// the model centroid (BeadModel.centroid = positions.mean(0), model.py:56-61).
//
// Z is never assembled: Zf = [sum f_k ; sum (r_k - c) x f_k] is a segmented
// reduction with a FIXED order (segments of seg_len(n_j) beads -- a function of
// the body's own size only -- tree-reduced inside a CTA, then reduced per body by
// the body's last-arriving CTA in a fixed order), so results do not depend on batch
// composition or GPU count.  All k columns go in one launch (grid.y = column).  Z^T u =
// V + w x (r_k - c) is a streaming per-bead map (48 B/bead).
#include <algorithm>
#include <vector>

#include "rq_plan.hpp"

namespace rq {
namespace {

constexpr int NTZ = 256;
// segment length: 4096 beads, 1024 for bodies of >= 2^18 beads (enough CTAs for one body)
inline int64_t seg_len(int64_t n) { return n >= (int64_t(1) << 18) ? 1024 : 4096; }

template <int W>
__device__ __forceinline__ void block_sum(double (&v)[W], double *sh) {
  // sh: (NTZ / 32) * W doubles; fixed reduction tree (shuffle tree per warp, then warp 0 over
  // the warp sums); the result is valid in thread 0
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int w = 0; w < W; w++) v[w] = __dadd_rn(v[w], __shfl_down_sync(0xffffffffu, v[w], o));
  if (lane == 0)
#pragma unroll
    for (int w = 0; w < W; w++) sh[w * (NTZ / 32) + wid] = v[w];
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int w = 0; w < W; w++) v[w] = lane < NTZ / 32 ? sh[w * (NTZ / 32) + lane] : 0.0;
#pragma unroll
    for (int o = NTZ / 64; o > 0; o >>= 1)
#pragma unroll
      for (int w = 0; w < W; w++) v[w] = __dadd_rn(v[w], __shfl_down_sync(0xffffffffu, v[w], o));
  }
}

__global__ void __launch_bounds__(NTZ) k_seg_possum(const double *pos, const int64_t *seg_begin, double *part) {
  __shared__ double sh[3 * NTZ / 32];
  const int64_t s = blockIdx.x;
  const int64_t b = seg_begin[s], e = seg_begin[s + 1];
  double v[3] = {0, 0, 0};
  for (int64_t i = b + threadIdx.x; i < e; i += NTZ)
    for (int a = 0; a < 3; a++) v[a] += pos[i * 3 + a];
  block_sum<3>(v, sh);
  if (threadIdx.x == 0)
    for (int a = 0; a < 3; a++) part[s * 6 + a] = v[a];
}

__global__ void k_body_mean(const double *part, const int64_t *body_seg, const int64_t *bead_off, int64_t m,
                            double *cen) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  double v[3] = {0, 0, 0};
  for (int64_t s = body_seg[j]; s < body_seg[j + 1]; s++)
    for (int a = 0; a < 3; a++) v[a] += part[s * 6 + a];
  double n = (double)(bead_off[j + 1] - bead_off[j]);
  for (int a = 0; a < 3; a++) cen[j * 3 + a] = v[a] / n;
}

// One launch: a CTA per (segment, column) reduces its segment; the last CTA of a body (per
// column; arrival counter, threadfence) then sums the body's segment partials in a fixed order
// (thread t: segments t, t + NTZ, ...; then the block tree), so the result depends only on
// the body's size.  Single-segment bodies write their sums directly.  The counters reset
// themselves, so back-to-back calls on one stream reuse them.
__global__ void __launch_bounds__(NTZ) k_zf(const double *pos, const int64_t *seg_begin, const int32_t *seg_body,
                                            const int64_t *body_seg, int64_t m, const double *origin, const double *f,
                                            int64_t K, int64_t n_seg, double *part, unsigned *cnt, double *out) {
  __shared__ double sh[6 * NTZ / 32];
  __shared__ int last;
  const int64_t s = blockIdx.x;
  const int64_t col = blockIdx.y;
  const int64_t b = seg_begin[s], e = seg_begin[s + 1];
  const int j = seg_body[s];
  const double cx = origin[j * 3], cy = origin[j * 3 + 1], cz = origin[j * 3 + 2];
  double v[6] = {0, 0, 0, 0, 0, 0};
  // Fixed order, independent of where the body sits in the batch: thread t takes the bead
  // pairs (2q, 2q+1), q = t, t + NTZ, ... of the segment (then thread 0 an odd last bead),
  // followed by the fixed tree of block_sum.  Aligned K = 1 inputs load each pair as
  // 3 x 16 B of positions and of forces; otherwise the same pairs load element-wise.
  // explicit roundings (no FMA contraction), so both load paths compute bit-identically
  auto acc = [&](double x, double y, double z, double fx, double fy, double fz) {
    x = __dsub_rn(x, cx); y = __dsub_rn(y, cy); z = __dsub_rn(z, cz);
    v[0] = __dadd_rn(v[0], fx);
    v[1] = __dadd_rn(v[1], fy);
    v[2] = __dadd_rn(v[2], fz);
    v[3] = __dadd_rn(v[3], __dsub_rn(__dmul_rn(y, fz), __dmul_rn(z, fy)));
    v[4] = __dadd_rn(v[4], __dsub_rn(__dmul_rn(z, fx), __dmul_rn(x, fz)));
    v[5] = __dadd_rn(v[5], __dsub_rn(__dmul_rn(x, fy), __dmul_rn(y, fx)));
  };
  const int64_t npair = (e - b) / 2;
  if (K == 1 && ((b & 1) == 0) && ((reinterpret_cast<uintptr_t>(f) & 15) == 0)) {
    const double2 *P2 = reinterpret_cast<const double2 *>(pos + 3 * b);
    const double2 *F2 = reinterpret_cast<const double2 *>(f + 3 * b);
#pragma unroll 2
    for (int64_t q = threadIdx.x; q < npair; q += NTZ) {
      const double2 p0 = P2[3 * q], p1 = P2[3 * q + 1], p2 = P2[3 * q + 2];
      const double2 f0 = F2[3 * q], f1 = F2[3 * q + 1], f2 = F2[3 * q + 2];
      acc(p0.x, p0.y, p1.x, f0.x, f0.y, f1.x);
      acc(p1.y, p2.x, p2.y, f1.y, f2.x, f2.y);
    }
  } else {
    for (int64_t q = threadIdx.x; q < npair; q += NTZ) {
      for (int h = 0; h < 2; h++) {
        const int64_t i = b + 2 * q + h;
        acc(pos[i * 3], pos[i * 3 + 1], pos[i * 3 + 2], f[(i * 3) * K + col], f[(i * 3 + 1) * K + col],
            f[(i * 3 + 2) * K + col]);
      }
    }
  }
  if (((e - b) & 1) && threadIdx.x == 0) {
    const int64_t i = e - 1;
    acc(pos[i * 3], pos[i * 3 + 1], pos[i * 3 + 2], f[(i * 3) * K + col], f[(i * 3 + 1) * K + col],
        f[(i * 3 + 2) * K + col]);
  }
  block_sum<6>(v, sh);
  const int64_t s0 = body_seg[j], s1 = body_seg[j + 1];
  if (s1 - s0 == 1) {
    if (threadIdx.x == 0)
      for (int a = 0; a < 6; a++) out[(j * 6 + a) * K + col] = v[a];
    return;
  }
  double *P = part + col * n_seg * 6;
  if (threadIdx.x == 0) {
    for (int a = 0; a < 6; a++) P[s * 6 + a] = v[a];
    __threadfence();
    last = atomicAdd(&cnt[col * m + j], 1u) == (unsigned)(s1 - s0 - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int a = 0; a < 6; a++) v[a] = 0.0;
  for (int64_t q = s0 + threadIdx.x; q < s1; q += NTZ)
    for (int a = 0; a < 6; a++) v[a] = __dadd_rn(v[a], __ldcg(&P[q * 6 + a]));
  __syncthreads();  // sh reused
  block_sum<6>(v, sh);
  if (threadIdx.x == 0) {
    for (int a = 0; a < 6; a++) out[(j * 6 + a) * K + col] = v[a];
    cnt[col * m + j] = 0;
  }
}

// K = 1, 16-byte aligned output: a thread maps a bead pair (48 contiguous bytes in and out)
__global__ void k_ztu2(const double *pos, const int32_t *body_of, const double *origin, const double *u, int64_t N,
                       double *out) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (2 * q >= N) return;
  const double2 *P2 = reinterpret_cast<const double2 *>(pos) + 3 * q;
  double2 *O2 = reinterpret_cast<double2 *>(out) + 3 * q;
  const double2 p0 = P2[0], p1 = P2[1], p2 = P2[2];
  double o[6];
  auto map = [&](int64_t i, double x, double y, double z, double *r) {
    const int j = body_of[i];
    x -= origin[j * 3]; y -= origin[j * 3 + 1]; z -= origin[j * 3 + 2];
    const double *U = u + j * 6;
    r[0] = U[0] + (z * U[4] - y * U[5]);
    r[1] = U[1] + (x * U[5] - z * U[3]);
    r[2] = U[2] + (y * U[3] - x * U[4]);
  };
  map(2 * q, p0.x, p0.y, p1.x, o);
  if (2 * q + 1 < N) {
    map(2 * q + 1, p1.y, p2.x, p2.y, o + 3);
    O2[0] = make_double2(o[0], o[1]);
    O2[1] = make_double2(o[2], o[3]);
    O2[2] = make_double2(o[4], o[5]);
  } else {  // odd N: the last bead alone
    out[6 * q] = o[0];
    out[6 * q + 1] = o[1];
    out[6 * q + 2] = o[2];
  }
}

__global__ void k_ztu(const double *pos, const int32_t *body_of, const double *origin, const double *u, int64_t N,
                      int64_t K, double *out) {
  const int64_t col = blockIdx.y;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int j = body_of[i];
  const double x = pos[i * 3] - origin[j * 3], y = pos[i * 3 + 1] - origin[j * 3 + 1],
               z = pos[i * 3 + 2] - origin[j * 3 + 2];
  const double *U = u + (j * 6) * K + col;
  const double V0 = U[0], V1 = U[K], V2 = U[2 * K], w0 = U[3 * K], w1 = U[4 * K], w2 = U[5 * K];
  out[(i * 3) * K + col] = V0 + (z * w1 - y * w2);
  out[(i * 3 + 1) * K + col] = V1 + (x * w2 - z * w0);
  out[(i * 3 + 2) * K + col] = V2 + (y * w0 - x * w1);
}

}  // namespace

void compute_body_centroids(Plan &p, cudaStream_t s) {
  // fixed segment table
  std::vector<int64_t> seg_begin, body_seg(p.m + 1);
  std::vector<int32_t> seg_body;
  for (int64_t j = 0; j < p.m; j++) {
    body_seg[j] = (int64_t)seg_body.size();
    const int64_t sl = seg_len(p.bead_off[j + 1] - p.bead_off[j]);
    for (int64_t b = p.bead_off[j]; b < p.bead_off[j + 1]; b += sl) {
      seg_begin.push_back(b);
      seg_body.push_back((int32_t)j);
    }
  }
  body_seg[p.m] = (int64_t)seg_body.size();
  seg_begin.push_back(p.N);
  p.n_seg = (int64_t)seg_body.size();
  p.seg_body.alloc(p.n_seg * 4);
  p.seg_begin.alloc((p.n_seg + 1) * 8);
  p.body_seg.alloc((p.m + 1) * 8);
  RQ_CUDA(cudaMemcpyAsync(p.seg_body.p, seg_body.data(), p.n_seg * 4, cudaMemcpyHostToDevice, s));
  RQ_CUDA(cudaMemcpyAsync(p.seg_begin.p, seg_begin.data(), (p.n_seg + 1) * 8, cudaMemcpyHostToDevice, s));
  RQ_CUDA(cudaMemcpyAsync(p.body_seg.p, body_seg.data(), (p.m + 1) * 8, cudaMemcpyHostToDevice, s));
  p.body_centroid.alloc(p.m * 24);
  DBuf part;
  part.alloc(p.n_seg * 48);
  k_seg_possum<<<(unsigned)p.n_seg, NTZ, 0, s>>>(p.pos_orig.as<double>(), p.seg_begin.as<int64_t>(),
                                                 part.as<double>());
  k_body_mean<<<(unsigned)((p.m + 127) / 128), 128, 0, s>>>(part.as<double>(), p.body_seg.as<int64_t>(),
                                                            p.bead_off_d.as<int64_t>(), p.m,
                                                            p.body_centroid.as<double>());
  RQ_CUDA(cudaGetLastError());
}

void run_z(const Plan &p, int op, const double *in, double *out, int64_t k, const double *origin_d,
           cudaStream_t s) {
  if (op != RQ_Z_F && op != RQ_Z_TU) throw Error(RQ_ERR_VALUE, "z op must be RQ_Z_F or RQ_Z_TU");
  if (k < 1 || k > 65535) throw Error(RQ_ERR_LENGTH, "k must be in [1, 65535]");
  RQ_CUDA(cudaSetDevice(p.device));
  const double *origin = origin_d ? origin_d : p.body_centroid.as<double>();
  if (op == RQ_Z_F) {
    // per-segment partial sums are per-stream state: Zf calls on different streams never share them
    Plan::StreamState &ss = p.state_for(s);
    const size_t need = (size_t)p.n_seg * 48 * k;
    if (ss.zpart.bytes < need) ss.zpart.alloc(need);
    if (ss.zcnt.bytes < (size_t)p.m * 4 * k) {
      ss.zcnt.alloc((size_t)p.m * 4 * k);
      RQ_CUDA(cudaMemsetAsync(ss.zcnt.p, 0, (size_t)p.m * 4 * k, s));
    }
    k_zf<<<dim3((unsigned)p.n_seg, (unsigned)k), NTZ, 0, s>>>(
        p.pos_orig.as<double>(), p.seg_begin.as<int64_t>(), p.seg_body.as<int32_t>(), p.body_seg.as<int64_t>(), p.m,
        origin, in, k, p.n_seg, ss.zpart.as<double>(), ss.zcnt.as<unsigned>(), out);
  } else if (k == 1 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
    const int64_t np = (p.N + 1) / 2;
    k_ztu2<<<(unsigned)((np + 255) / 256), 256, 0, s>>>(p.pos_orig.as<double>(), p.body_of.as<int32_t>(), origin,
                                                        in, p.N, out);
  } else {
    k_ztu<<<dim3((unsigned)((p.N + 255) / 256), (unsigned)k), 256, 0, s>>>(p.pos_orig.as<double>(),
                                                                         p.body_of.as<int32_t>(), origin, in, p.N, k,
                                                                         out);
  }
  RQ_CUDA(cudaGetLastError());
}

}  // namespace rq
