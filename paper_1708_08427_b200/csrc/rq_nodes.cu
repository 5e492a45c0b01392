// rq_nodes.cu -- single-node primitives of the reference API run on the GPU
// with the same device code as the batched setup / sweeps:
//   small_lq (factor.py:90-109), factor_bead_bead (factor.py:130-168),
//   merge_infosets (matfree.py:41-62), split_rvset (matfree.py:65-83).
// merge/split take an EXPLICIT k x k mixer (NodeFactor.omega) because users
// may hand in any orthogonal matrix; the batched path streams compact records.
#include <vector>

#include "rq_lq.cuh"
#include "rq_plan.hpp"

namespace rq {
namespace {

template <int K>
__device__ void small_lq_one(const double *a, double *t, double *om) {
  double t6[6], rec[WY<K>::SIZE];
  unsigned sg;
  lq_factor<K>(a, t6, rec, sg);
  t[0] = t6[0]; t[1] = 0.0;   t[2] = 0.0;
  t[3] = t6[1]; t[4] = t6[2]; t[5] = 0.0;
  t[6] = t6[3]; t[7] = t6[4]; t[8] = t6[5];
  for (int j = 0; j < K; j++) {
    double y[K];
    for (int i = 0; i < K; i++) y[i] = (i == j) ? 1.0 : 0.0;
    omega_apply<K>(rec, sg, y);
    for (int i = 0; i < K; i++) om[i * K + j] = y[i];
  }
}

__global__ void k_small_lq(const double *a, int k, int64_t batch, double *t, double *om) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= batch) return;
  if (k == 3) small_lq_one<3>(a + b * 9, t + b * 9, om + b * 9);
  else if (k == 6) small_lq_one<6>(a + b * 18, t + b * 9, om + b * 36);
  else small_lq_one<9>(a + b * 27, t + b * 9, om + b * 81);
}

__global__ void k_factor_bb(const double *d, int64_t batch, double *t, double *g) {
  int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= batch) return;
  double t6[6], dd[3] = {d[b * 3], d[b * 3 + 1], d[b * 3 + 2]};
  factor_bead_bead(dd, t6, g + b * 9);
  double *o = t + b * 9;
  o[0] = t6[0]; o[1] = 0.0;   o[2] = 0.0;
  o[3] = t6[1]; o[4] = t6[2]; o[5] = 0.0;
  o[6] = t6[3]; o[7] = t6[4]; o[8] = t6[5];
}

// column c of a (6 x K) block; one thread per column
__global__ void k_node_merge(int cs, const double *om, double a, double b, const double *mx, const double *my,
                             int64_t K, double *mp, double *res) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= K) return;
  double x[6], y[6];
  for (int r = 0; r < 6; r++) { x[r] = mx[r * K + c]; y[r] = my[r * K + c]; }
  double t[3];
  for (int r = 0; r < 3; r++) {
    t[r] = b * x[r] - a * y[r];
    mp[r * K + c] = a * x[r] + b * y[r];
  }
  int k = cs == BEAD_BEAD ? 3 : (cs == RIGID_BEAD ? 6 : 9);
  double in[9];
  if (cs == BEAD_BEAD) { in[0] = t[0]; in[1] = t[1]; in[2] = t[2]; }
  else if (cs == RIGID_BEAD) { for (int r = 0; r < 3; r++) { in[r] = x[3 + r]; in[3 + r] = t[r]; } }
  else { for (int r = 0; r < 3; r++) { in[r] = x[3 + r]; in[3 + r] = y[3 + r]; in[6 + r] = t[r]; } }
  for (int i = 0; i < k; i++) {
    double s = 0.0;
    for (int j = 0; j < k; j++) s += om[i * k + j] * in[j];
    if (i < 3) mp[(3 + i) * K + c] = s;
    else res[(i - 3) * K + c] = s;
  }
}

__global__ void k_node_split(int cs, const double *om, double a, double b, const double *lp, const double *res,
                             int64_t K, double *lx, double *ly) {
  int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= K) return;
  int k = cs == BEAD_BEAD ? 3 : (cs == RIGID_BEAD ? 6 : 9);
  double in[9], u[9];
  for (int r = 0; r < 3; r++) in[r] = lp[(3 + r) * K + c];
  for (int r = 3; r < k; r++) in[r] = res[(r - 3) * K + c];
  for (int i = 0; i < k; i++) {
    double s = 0.0;
    for (int j = 0; j < k; j++) s += om[j * k + i] * in[j];
    u[i] = s;
  }
  const double *tau = u + (k - 3);
  for (int r = 0; r < 3; r++) {
    double l = lp[r * K + c];
    lx[r * K + c] = a * l + b * tau[r];
    ly[r * K + c] = b * l - a * tau[r];
    lx[(3 + r) * K + c] = cs == BEAD_BEAD ? 0.0 : u[r];
    ly[(3 + r) * K + c] = cs == GENERAL ? u[3 + r] : 0.0;
  }
}

struct Dev {
  DBuf b;
  Dev(const double *h, size_t n) {
    b.alloc(n * 8);
    if (h) RQ_CUDA(cudaMemcpy(b.p, h, n * 8, cudaMemcpyHostToDevice));
  }
  double *p() { return b.as<double>(); }
  void get(double *h, size_t n) { RQ_CUDA(cudaMemcpy(h, b.p, n * 8, cudaMemcpyDeviceToHost)); }
};

inline void need_gpu() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw Error(RQ_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
  }
}

}  // namespace

void node_small_lq(const double *a, int k, int64_t batch, double *t, double *om) {
  need_gpu();
  if (k != 3 && k != 6 && k != 9) throw Error(RQ_ERR_VALUE, "small_lq: k must be 3, 6 or 9");
  Dev da(a, batch * 3 * k), dt(nullptr, batch * 9), dom(nullptr, batch * k * k);
  k_small_lq<<<(unsigned)((batch + 63) / 64), 64>>>(da.p(), k, batch, dt.p(), dom.p());
  RQ_CUDA(cudaGetLastError());
  dt.get(t, batch * 9);
  dom.get(om, batch * k * k);
}

void node_factor_bb(const double *d, int64_t batch, double *t, double *g) {
  need_gpu();
  Dev dd(d, batch * 3), dt(nullptr, batch * 9), dg(nullptr, batch * 9);
  k_factor_bb<<<(unsigned)((batch + 63) / 64), 64>>>(dd.p(), batch, dt.p(), dg.p());
  RQ_CUDA(cudaGetLastError());
  dt.get(t, batch * 9);
  dg.get(g, batch * 9);
}

void node_merge(int cs, const double *om, double a, double b, const double *mx, const double *my, int64_t K,
                double *mp, double *res) {
  need_gpu();
  if (cs < 1 || cs > 3) throw Error(RQ_ERR_VALUE, "merge_infosets: not an internal node case");
  int k = cs == 1 ? 3 : (cs == 2 ? 6 : 9);
  Dev dom(om, k * k), dx(mx, 6 * K), dy(my, 6 * K), dp(nullptr, 6 * K), dr(nullptr, std::max(k - 3, 1) * K);
  k_node_merge<<<(unsigned)((K + 127) / 128), 128>>>(cs, dom.p(), a, b, dx.p(), dy.p(), K, dp.p(), dr.p());
  RQ_CUDA(cudaGetLastError());
  dp.get(mp, 6 * K);
  if (k > 3) dr.get(res, (k - 3) * K);
}

void node_split(int cs, const double *om, double a, double b, const double *lp, const double *res, int64_t K,
                double *lx, double *ly) {
  need_gpu();
  if (cs < 1 || cs > 3) throw Error(RQ_ERR_VALUE, "split_rvset: not an internal node case");
  int k = cs == 1 ? 3 : (cs == 2 ? 6 : 9);
  Dev dom(om, k * k), dl(lp, 6 * K), dr(k > 3 ? res : nullptr, std::max(k - 3, 1) * K), dx(nullptr, 6 * K),
      dy(nullptr, 6 * K);
  k_node_split<<<(unsigned)((K + 127) / 128), 128>>>(cs, dom.p(), a, b, dl.p(), dr.p(), K, dx.p(), dy.p());
  RQ_CUDA(cudaGetLastError());
  dx.get(lx, 6 * K);
  dy.get(ly, 6 * K);
}

}  // namespace rq
