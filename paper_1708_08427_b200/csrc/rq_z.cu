// rq_z.cu -- (c) force/torque reductions Zf and Z^T u (model.py:129-149) and
// the model centroid (BeadModel.centroid = positions.mean(0), model.py:56-61).
//
// Z is never assembled: Zf = [sum f_k ; sum (r_k - c) x f_k] is a segmented
// reduction with a FIXED order (segments of SEG beads, tree-reduced inside a
// CTA, then summed in segment order per body), so results do not depend on
// batch composition or GPU count.  Z^T u = V + w x (r_k - c) is a streaming
// per-bead map (48 B/bead).
#include <algorithm>
#include <vector>

#include "rq_plan.hpp"

namespace rq {
namespace {

constexpr int SEG = 4096;
constexpr int NTZ = 256;

template <int W>
__device__ __forceinline__ void block_sum(double (&v)[W], double *sh) {
  // sh: NTZ * W doubles; fixed reduction tree
  const int tid = threadIdx.x;
#pragma unroll
  for (int w = 0; w < W; w++) sh[w * NTZ + tid] = v[w];
  __syncthreads();
  for (int o = NTZ / 2; o > 0; o >>= 1) {
    if (tid < o)
#pragma unroll
      for (int w = 0; w < W; w++) sh[w * NTZ + tid] += sh[w * NTZ + tid + o];
    __syncthreads();
  }
#pragma unroll
  for (int w = 0; w < W; w++) v[w] = sh[w * NTZ];
}

__global__ void __launch_bounds__(NTZ) k_seg_possum(const double *pos, const int64_t *seg_begin, double *part) {
  __shared__ double sh[3 * NTZ];
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

__global__ void __launch_bounds__(NTZ) k_seg_zf(const double *pos, const int64_t *seg_begin, const int32_t *seg_body,
                                                const double *origin, const double *f, int64_t K, int64_t col,
                                                double *part) {
  __shared__ double sh[6 * NTZ];
  const int64_t s = blockIdx.x;
  const int64_t b = seg_begin[s], e = seg_begin[s + 1];
  const int j = seg_body[s];
  const double cx = origin[j * 3], cy = origin[j * 3 + 1], cz = origin[j * 3 + 2];
  double v[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t i = b + threadIdx.x; i < e; i += NTZ) {
    const double x = pos[i * 3] - cx, y = pos[i * 3 + 1] - cy, z = pos[i * 3 + 2] - cz;
    const double fx = f[(i * 3) * K + col], fy = f[(i * 3 + 1) * K + col], fz = f[(i * 3 + 2) * K + col];
    v[0] += fx;
    v[1] += fy;
    v[2] += fz;
    v[3] += y * fz - z * fy;
    v[4] += z * fx - x * fz;
    v[5] += x * fy - y * fx;
  }
  block_sum<6>(v, sh);
  if (threadIdx.x == 0)
    for (int a = 0; a < 6; a++) part[s * 6 + a] = v[a];
}

__global__ void k_body_zf(const double *part, const int64_t *body_seg, int64_t m, double *out, int64_t K,
                          int64_t col) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= m) return;
  double v[6] = {0, 0, 0, 0, 0, 0};
  for (int64_t s = body_seg[j]; s < body_seg[j + 1]; s++)
    for (int a = 0; a < 6; a++) v[a] += part[s * 6 + a];
  for (int a = 0; a < 6; a++) out[(j * 6 + a) * K + col] = v[a];
}

__global__ void k_ztu(const double *pos, const int32_t *body_of, const double *origin, const double *u, int64_t N,
                      int64_t K, int64_t col, double *out) {
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
    for (int64_t b = p.bead_off[j]; b < p.bead_off[j + 1]; b += SEG) {
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
  p.zpart.alloc(p.n_seg * 48);
  RQ_CUDA(cudaMemcpyAsync(p.seg_body.p, seg_body.data(), p.n_seg * 4, cudaMemcpyHostToDevice, s));
  RQ_CUDA(cudaMemcpyAsync(p.seg_begin.p, seg_begin.data(), (p.n_seg + 1) * 8, cudaMemcpyHostToDevice, s));
  RQ_CUDA(cudaMemcpyAsync(p.body_seg.p, body_seg.data(), (p.m + 1) * 8, cudaMemcpyHostToDevice, s));
  p.body_centroid.alloc(p.m * 24);
  k_seg_possum<<<(unsigned)p.n_seg, NTZ, 0, s>>>(p.pos_orig.as<double>(), p.seg_begin.as<int64_t>(),
                                                 p.zpart.as<double>());
  k_body_mean<<<(unsigned)((p.m + 127) / 128), 128, 0, s>>>(p.zpart.as<double>(), p.body_seg.as<int64_t>(),
                                                            p.bead_off_d.as<int64_t>(), p.m,
                                                            p.body_centroid.as<double>());
  RQ_CUDA(cudaGetLastError());
}

void run_z(const Plan &p, int op, const double *in, double *out, int64_t k, const double *origin_d,
           cudaStream_t s) {
  if (op != RQ_Z_F && op != RQ_Z_TU) throw Error(RQ_ERR_VALUE, "z op must be RQ_Z_F or RQ_Z_TU");
  if (k < 1) throw Error(RQ_ERR_LENGTH, "k must be >= 1");
  RQ_CUDA(cudaSetDevice(p.device));
  const double *origin = origin_d ? origin_d : p.body_centroid.as<double>();
  for (int64_t col = 0; col < k; col++) {
    if (op == RQ_Z_F) {
      k_seg_zf<<<(unsigned)p.n_seg, NTZ, 0, s>>>(p.pos_orig.as<double>(), p.seg_begin.as<int64_t>(),
                                                 p.seg_body.as<int32_t>(), origin, in, k, col,
                                                 p.zpart.as<double>());
      k_body_zf<<<(unsigned)((p.m + 127) / 128), 128, 0, s>>>(p.zpart.as<double>(), p.body_seg.as<int64_t>(),
                                                              p.m, out, k, col);
    } else {
      k_ztu<<<(unsigned)((p.N + 255) / 256), 256, 0, s>>>(p.pos_orig.as<double>(), p.body_of.as<int32_t>(),
                                                          origin, in, p.N, k, col, out);
    }
  }
  RQ_CUDA(cudaGetLastError());
}

}  // namespace rq
