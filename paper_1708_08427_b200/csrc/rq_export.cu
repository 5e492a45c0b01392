// rq_export.cu -- parity exports of the device-resident tree / factor table
// (the lazy TreeNode / NodeFactor views of the Python mirror) and the
// explicit hierarchical Q of Algorithm 1 (generate_explicit_q,
// factor.py:362-390; node_rows, factor.py:247-280).
//
// Explicit rows are produced on the device by unit-seeded downward sweeps:
// a residue row r of node X is (Q^T e_row)^T, which is supported on X's beads
// and equals the downward pass over X's subtree seeded with l_X = 0,
// res_X = e_r (all other residues zero); the root rows [E_n; U_root] are the
// sweeps seeded with l_root = e_r.  Total work O(n log n), like Algorithm 1.
#include <algorithm>
#include <vector>

#include "rq_nodeops.cuh"
#include "rq_plan.hpp"

namespace rq {
namespace {

__constant__ int c_axis_cycle2[3] = {2, 1, 0};

__global__ void k_box(const int32_t *start, const int16_t *depth, const double *pos_tree, const double *root_box,
                      int64_t nb, int64_t base, int64_t body, int64_t nn, double *box) {
  int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= nn) return;
  double cl[3], ch[3], p[3];
  for (int a = 0; a < 3; a++) {
    cl[a] = root_box[body * 6 + a];
    ch[a] = root_box[body * 6 + 3 + a];
    p[a] = pos_tree[(base + start[nb + id]) * 3 + a];
  }
  int dep = depth[nb + id];
  for (int d = 0; d < dep; d++) {
    int a = c_axis_cycle2[d % 3];
    double mid = 0.5 * (cl[a] + ch[a]);
    if (p[a] > mid) cl[a] = mid; else ch[a] = mid;
  }
  for (int a = 0; a < 3; a++) {
    box[id * 6 + a] = cl[a];
    box[id * 6 + 3 + a] = ch[a];
  }
}

// explicit omega (k x k, row-major, stride 81 per node) from the compact record
__global__ void k_omega(const uint8_t *flags, const int64_t *rec_off, const double *rec, int64_t nb, int64_t nn,
                        double *out) {
  int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (id >= nn) return;
  unsigned f = flags[nb + id];
  int cs = flag_case(f);
  const double *r = rec + rec_off[nb + id];
  double *o = out + id * 81;
  if (cs == BEAD_BEAD) {
    for (int e = 0; e < 9; e++) o[e] = r[e];
  } else if (cs == RIGID_BEAD) {
    for (int j = 0; j < 6; j++) {
      double y[6] = {0, 0, 0, 0, 0, 0};
      y[j] = 1.0;
      omega_s<6>(r, 1, flag_signs(f), y);
      for (int i = 0; i < 6; i++) o[i * 6 + j] = y[i];
    }
  } else if (cs == GENERAL) {
    for (int j = 0; j < 9; j++) {
      double y[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
      y[j] = 1.0;
      omega_s<9>(r, 1, flag_signs(f), y);
      for (int i = 0; i < 9; i++) o[i * 9 + j] = y[i];
    }
  }
}

struct QJob {
  int32_t node;     // subtree root (body-local id)
  int32_t seed;     // 0..5: root row (l = e_seed); 6..11: residue row seed-6
  int64_t out_off;  // first double of the row in the output
  int64_t l_off;    // scratch (6 * (2L - 1) doubles)
};

// one thread per explicit row: downward sweep over the subtree in reverse postorder
__global__ void k_explicit_rows(const QJob *jobs, int64_t n_jobs, int64_t nb, const int32_t *start,
                                const int32_t *stop, const int32_t *left, const int32_t *right,
                                const uint8_t *flags, const int64_t *rec_off, const double *rec, double *lbuf,
                                double *out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n_jobs) return;
  const QJob J = jobs[t];
  const int X = J.node;
  const int L = stop[nb + X] - start[nb + X];
  const int first = X - 2 * L + 2;
  const int s0 = start[nb + X];
  double *lb = lbuf + J.l_off;  // indexed by (id - first)
  for (int r = 0; r < 6; r++) lb[6 * (X - first) + r] = (J.seed < 6 && r == J.seed) ? 1.0 : 0.0;
  for (int y = X; y >= first; y--) {
    const int64_t g = nb + y;
    double lp[6];
    for (int r = 0; r < 6; r++) lp[r] = lb[6 * (y - first) + r];
    if (left[g] < 0) {
      const int64_t col = 3 * (int64_t)(start[g] - s0);
      for (int a = 0; a < 3; a++) out[J.out_off + col + a] = lp[a];
      continue;
    }
    unsigned f = flags[g];
    int cs = flag_case(f);
    int l = left[g], rr = right[g];
    int xi = l, yi = rr;
    if (flag_swapped(f)) { xi = rr; yi = l; }
    int nx = stop[nb + xi] - start[nb + xi], ny = stop[nb + yi] - start[nb + yi];
    double a, b;
    ratios(nx, ny, a, b);
    double res[6] = {0, 0, 0, 0, 0, 0}, lx[6], ly[6];
    if (y == X && J.seed >= 6) res[J.seed - 6] = 1.0;
    split(cs, rec + rec_off[g], 1, flag_signs(f), a, b, lp, res, lx, ly);
    for (int r = 0; r < 6; r++) {
      lb[6 * (xi - first) + r] = lx[r];
      lb[6 * (yi - first) + r] = ly[r];
    }
  }
}

template <class T>
void d2h(T *dst, const void *src, size_t count) {
  RQ_CUDA(cudaMemcpy(dst, src, count * sizeof(T), cudaMemcpyDeviceToHost));
}

struct BodyView {
  int64_t n, nn, nb, base;
  std::vector<int32_t> start, stop, left, right, parent, res_off;
  std::vector<int16_t> depth;
  std::vector<int8_t> axis;
  std::vector<uint8_t> flags;
};

BodyView body_view(const Plan &p, int64_t body) {
  if (body < 0 || body >= p.m) throw Error(RQ_ERR_VALUE, "body index out of range");
  BodyView v;
  v.base = p.bead_off[body];
  v.n = p.bead_off[body + 1] - v.base;
  v.nn = 2 * v.n - 1;
  v.nb = 2 * v.base - body;
  auto get32 = [&](const DBuf &b, std::vector<int32_t> &dst) {
    dst.resize(v.nn);
    d2h(dst.data(), b.as<int32_t>() + v.nb, v.nn);
  };
  get32(p.start, v.start);
  get32(p.stop, v.stop);
  get32(p.left, v.left);
  get32(p.right, v.right);
  get32(p.parent, v.parent);
  get32(p.res_off, v.res_off);
  v.depth.resize(v.nn);
  d2h(v.depth.data(), p.depth.as<int16_t>() + v.nb, v.nn);
  v.axis.resize(v.nn);
  d2h(v.axis.data(), p.axis.as<int8_t>() + v.nb, v.nn);
  v.flags.resize(v.nn);
  d2h(v.flags.data(), p.flags.as<uint8_t>() + v.nb, v.nn);
  return v;
}

}  // namespace

void export_tree(const Plan &p, int64_t body, int64_t *perm, int64_t *start, int64_t *stop, int64_t *left,
                 int64_t *right, int32_t *split_axis, int32_t *depth, double *centroid, double *box) {
  RQ_CUDA(cudaSetDevice(p.device));
  BodyView v = body_view(p, body);
  if (perm) {
    std::vector<int32_t> pm(v.n);
    d2h(pm.data(), p.perm.as<int32_t>() + v.base, v.n);
    for (int64_t i = 0; i < v.n; i++) perm[i] = pm[i];
  }
  for (int64_t i = 0; i < v.nn; i++) {
    if (start) start[i] = v.start[i];
    if (stop) stop[i] = v.stop[i];
    if (left) left[i] = v.left[i];
    if (right) right[i] = v.right[i];
    if (split_axis) split_axis[i] = v.axis[i];
    if (depth) depth[i] = v.depth[i];
  }
  if (centroid) d2h(centroid, p.centroid.as<double>() + 3 * v.nb, 3 * v.nn);
  if (box) {
    DBuf b;
    b.alloc(v.nn * 48);
    k_box<<<(unsigned)((v.nn + 127) / 128), 128>>>(p.start.as<int32_t>(), p.depth.as<int16_t>(),
                                                    p.pos_tree.as<double>(), p.root_box.as<double>(), v.nb, v.base,
                                                    body, v.nn, b.as<double>());
    RQ_CUDA(cudaGetLastError());
    d2h(box, b.p, 6 * v.nn);
  }
}

int64_t omega_size(const Plan &p, int64_t body) {
  BodyView v = body_view(p, body);
  int64_t s = 0;
  for (auto f : v.flags) {
    int c = f & 3;
    s += c == BEAD_BEAD ? 9 : (c == RIGID_BEAD ? 36 : (c == GENERAL ? 81 : 0));
  }
  return s;
}

void export_factors(const Plan &p, int64_t body, int32_t *ncase, int64_t *n, int64_t *nx, int64_t *ny,
                    uint8_t *swapped, double *t22, double *omega, int64_t *res_offsets, int64_t *total_rows) {
  RQ_CUDA(cudaSetDevice(p.device));
  BodyView v = body_view(p, body);
  for (int64_t i = 0; i < v.nn; i++) {
    unsigned f = v.flags[i];
    int c = f & 3;
    int L = v.stop[i] - v.start[i];
    int64_t a = 0, b = 0;
    if (c != LEAF) {
      int l = v.left[i], r = v.right[i];
      int Ll = v.stop[l] - v.start[l], Lr = v.stop[r] - v.start[r];
      bool sw = flag_swapped(f);
      a = sw ? Lr : Ll;
      b = sw ? Ll : Lr;
    }
    if (ncase) ncase[i] = c;
    if (n) n[i] = L;
    if (nx) nx[i] = a;
    if (ny) ny[i] = b;
    if (swapped) swapped[i] = flag_swapped(f) ? 1 : 0;
    if (res_offsets) res_offsets[i] = v.res_off[i];
  }
  if (total_rows) *total_rows = v.n >= 2 ? 3 * v.n : 3;
  if (t22) {
    std::vector<double> t6(6 * v.nn);
    d2h(t6.data(), p.t22.as<double>() + 6 * v.nb, 6 * v.nn);
    for (int64_t i = 0; i < v.nn; i++) {
      const double *q = &t6[6 * i];
      double *o = t22 + 9 * i;
      o[0] = q[0]; o[1] = 0.0;  o[2] = 0.0;
      o[3] = q[1]; o[4] = q[2]; o[5] = 0.0;
      o[6] = q[3]; o[7] = q[4]; o[8] = q[5];
    }
  }
  if (omega) {
    DBuf b;
    b.alloc(v.nn * 81 * 8);
    k_omega<<<(unsigned)((v.nn + 127) / 128), 128>>>(p.flags.as<uint8_t>(), p.rec_off.as<int64_t>(),
                                                      p.rec.as<double>(), v.nb, v.nn, b.as<double>());
    RQ_CUDA(cudaGetLastError());
    std::vector<double> h(v.nn * 81);
    d2h(h.data(), b.p, v.nn * 81);
    int64_t o = 0;
    for (int64_t i = 0; i < v.nn; i++) {
      int c = v.flags[i] & 3;
      int k = c == BEAD_BEAD ? 3 : (c == RIGID_BEAD ? 6 : (c == GENERAL ? 9 : 0));
      for (int e = 0; e < k * k; e++) omega[o++] = h[81 * i + e];
    }
  }
}

void explicit_q_size(const Plan &p, int64_t body, int64_t *n_blocks, int64_t *n_doubles) {
  BodyView v = body_view(p, body);
  if (v.n < 2) throw Error(RQ_ERR_TOO_SMALL, "explicit Q needs at least 2 beads");
  int64_t nbk = 0, nd = 0;
  for (int64_t i = 0; i < v.nn; i++) {
    int rr = res_rows(v.flags[i] & 3);
    if (rr) { nbk++; nd += (int64_t)rr * 3 * (v.stop[i] - v.start[i]); }
  }
  *n_blocks = nbk;
  *n_doubles = nd;
}

void explicit_q(const Plan &p, int64_t body, double *root_rows, int64_t *block_node, int64_t *block_col,
                int64_t *block_rows, double *block_data) {
  RQ_CUDA(cudaSetDevice(p.device));
  BodyView v = body_view(p, body);
  if (v.n < 2) throw Error(RQ_ERR_TOO_SMALL, "explicit Q needs at least 2 beads");
  std::vector<QJob> jobs;
  int64_t out_off = 0, l_off = 0;
  const int root = (int)v.nn - 1;
  for (int r = 0; r < 6; r++) {
    jobs.push_back({root, r, out_off, l_off});
    out_off += 3 * v.n;
    l_off += 6 * v.nn;
  }
  const int64_t root_doubles = out_off;
  int64_t b = 0;
  for (int64_t i = 0; i < v.nn; i++) {  // postorder emission order
    int rr = res_rows(v.flags[i] & 3);
    if (!rr) continue;
    int L = v.stop[i] - v.start[i];
    block_node[b] = i;
    block_col[b] = 3 * (int64_t)v.start[i];
    block_rows[b] = rr;
    b++;
    for (int r = 0; r < rr; r++) {
      jobs.push_back({(int32_t)i, 6 + r, out_off, l_off});
      out_off += 3 * (int64_t)L;
      l_off += 6 * (2 * (int64_t)L - 1);
    }
  }
  DBuf d_jobs, d_l, d_out;
  d_jobs.alloc(jobs.size() * sizeof(QJob));
  d_l.alloc(l_off * 8);
  d_out.alloc(out_off * 8);
  RQ_CUDA(cudaMemcpy(d_jobs.p, jobs.data(), jobs.size() * sizeof(QJob), cudaMemcpyHostToDevice));
  k_explicit_rows<<<(unsigned)((jobs.size() + 63) / 64), 64>>>(
      d_jobs.as<QJob>(), (int64_t)jobs.size(), v.nb, p.start.as<int32_t>(), p.stop.as<int32_t>(),
      p.left.as<int32_t>(), p.right.as<int32_t>(), p.flags.as<uint8_t>(), p.rec_off.as<int64_t>(),
      p.rec.as<double>(), d_l.as<double>(), d_out.as<double>());
  RQ_CUDA(cudaGetLastError());
  std::vector<double> h(out_off);
  d2h(h.data(), d_out.p, out_off);
  std::copy(h.begin(), h.begin() + root_doubles, root_rows);
  std::copy(h.begin() + root_doubles, h.end(), block_data);
}

}  // namespace rq
