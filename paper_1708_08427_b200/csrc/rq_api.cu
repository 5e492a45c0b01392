// rq_api.cu -- extern "C" boundary (include/rigidq_b200.h).  Every entry
// catches rq::Error / std::exception, records the message in a thread-local
// slot (rq_last_error) and returns the matching RQ_ERR_* code.
#include <cstring>
#include <mutex>
#include <exception>
#include <new>
#include <string>

#include "rq_plan.hpp"

struct rq_plan {
  rq::Plan p;
};

namespace rq {
namespace {
thread_local std::string g_err;
}
void set_error(const std::string &msg) { g_err = msg; }
const char *last_error() { return g_err.c_str(); }
}  // namespace rq

#define RQ_GUARD(...)                                        \
  try {                                                      \
    rq::set_error("");                                       \
    __VA_ARGS__;                                             \
    return RQ_OK;                                            \
  } catch (const rq::Error &e) {                             \
    rq::set_error(e.msg);                                    \
    return e.code;                                           \
  } catch (const std::bad_alloc &) {                         \
    rq::set_error("host allocation failed");                 \
    return RQ_ERR_NOMEM;                                     \
  } catch (const std::exception &e) {                        \
    rq::set_error(e.what());                                 \
    return RQ_ERR_CUDA;                                      \
  }

namespace {
void need_plan(const rq_plan *p) {
  if (!p) throw rq::Error(RQ_ERR_VALUE, "null plan");
}
#define PLAN_DEVICE(plan) rq::DeviceGuard _dev_guard((plan)->p.device)
void need_gpu() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw rq::Error(RQ_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
  }
}
}  // namespace

extern "C" {

const char *rq_last_error(void) { return rq::last_error(); }

int rq_version(void) { return 200; }

int rq_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int rq_setup(const double *positions, const int64_t *offsets, int64_t m, int max_depth, uint32_t flags,
             void *stream, rq_plan **out) {
  RQ_GUARD({
    if (!out || !offsets) throw rq::Error(RQ_ERR_VALUE, "null argument");
    *out = nullptr;
    need_gpu();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (flags & RQ_SETUP_CHECK_DUPS) {
      int64_t b, i, j;
      double tol;
      int rc = rq::check_duplicates(positions, offsets, m, (flags & RQ_SETUP_HOST_INPUT) != 0, s, &b, &i, &j, &tol);
      if (rc != RQ_OK) {
        char msg[256];
        if (i < 0) snprintf(msg, sizeof msg, "body %lld: all beads coincide", (long long)b);
        else
          snprintf(msg, sizeof msg, "body %lld: beads %lld and %lld are closer than %.3e (dup_tol)", (long long)b,
                   (long long)i, (long long)j, tol);
        throw rq::Error(RQ_ERR_DUPLICATE, msg);
      }
    }
    rq_plan *h = new rq_plan();
    try {
      RQ_CUDA(cudaGetDevice(&h->p.device));
      rq::build_plan(h->p, positions, offsets, m, max_depth, (flags & RQ_SETUP_HOST_INPUT) != 0, s);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  })
}

int rq_plan_free(rq_plan *plan) {
  RQ_GUARD({
    if (plan) {
      cudaSetDevice(plan->p.device);
      delete plan;
    }
  })
}

int rq_plan_device(const rq_plan *plan) { return plan ? plan->p.device : -1; }

int rq_plan_release_stream(const rq_plan *plan, void *stream) {
  RQ_GUARD({
    need_plan(plan);
    PLAN_DEVICE(plan);
    const rq::Plan &p = plan->p;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::unique_ptr<rq::Plan::StreamState> st;
    {
      std::lock_guard<std::mutex> lock(p.state_mu);
      auto it = p.stream_state.find(s);
      if (it != p.stream_state.end()) {
        st = std::move(it->second);
        p.stream_state.erase(it);
      }
    }
    if (st) RQ_CUDA(cudaStreamSynchronize(s));  // its buffers may still be in use by queued work
  })
}

int rq_plan_get_info(const rq_plan *plan, rq_plan_info *info) {
  RQ_GUARD({
    need_plan(plan);
    PLAN_DEVICE(plan);
    const rq::Plan &p = plan->p;
    memset(info, 0, sizeof(*info));
    info->m = p.m;
    info->n_beads = p.N;
    info->n_nodes = p.NN;
    info->n_streams = p.wave_streams;
    info->n_steps = p.wave_steps;
    info->n_top = p.n_top;
    info->tile_leaves = p.tile_leaves;
    info->n_tiles = p.n_tiles;
    info->blob_bytes = p.wave_blob_bytes;
    info->sweep_bytes[0] = p.wave_up_bytes;
    info->sweep_bytes[1] = p.wave_down_bytes;
    info->record_doubles = p.rec_doubles;
    info->full_len = 3 * p.N;
    info->comp_len = 3 * p.N - 6 * p.m;
    for (int c = 0; c < 4; c++) info->n_case[c] = p.n_case[c];
    info->device_bytes = p.device_bytes();
    info->rounds = p.wave_rounds;
    info->node_slots = p.wave_mslots;
    info->stage_bytes = p.wave_stage_bytes;
    if (p.wave_streams) {
      info->sweep_smem = (int64_t)rq::wave_smem(p, nullptr, nullptr, nullptr);
      RQ_CUDA(cudaSetDevice(p.device));
      rq::wave_prepare(p);
      info->sweep_ctas_per_sm = p.wave_ctas_per_sm;
    }
    info->top_staged = p.n_topblob;
    info->top_global = p.n_topbig;
    info->mrhs_min_k = p.mrhs_min;
    info->mrhs_units[0] = p.n_tile_units;
    info->mrhs_units[1] = p.n_top_units;
    info->mrhs_bytes[0] = p.mrhs_tile_bytes;
    info->mrhs_bytes[1] = p.mrhs_top_bytes;
  })
}

int rq_apply(const rq_plan *plan, int op, const double *in, double *out, int64_t k, void *stream) {
  RQ_GUARD({
    need_plan(plan);
    PLAN_DEVICE(plan);
    if (!in || !out) throw rq::Error(RQ_ERR_VALUE, "null vector");
    rq::run_apply(plan->p, op, in, out, k, static_cast<cudaStream_t>(stream));
  })
}

int rq_apply_ex(const rq_plan *plan, int op, const double *in, double *out, int64_t k, void *stream,
                uint32_t phases) {
  RQ_GUARD({
    need_plan(plan);
    PLAN_DEVICE(plan);
    if (!in || !out) throw rq::Error(RQ_ERR_VALUE, "null vector");
    rq::run_apply(plan->p, op, in, out, k, static_cast<cudaStream_t>(stream), phases);
  })
}

int rq_launches_per_apply(const rq_plan *plan, int op, int64_t k) {
  if (!plan) return -1;
  const rq::Plan &p = plan->p;
  if (rq::use_mrhs(p, k)) {  // column-parallel kernels: one launch for the tiles, one per top level
    try {
      rq::DeviceGuard g(p.device);
      rq::build_mrhs(p, nullptr);
    } catch (...) {
      return -1;
    }
    const int tiles = p.n_tile_units > 0 ? 1 : 0, tops = p.n_top_units > 0 ? 1 : 0;
    const int levels = p.n_mtop ? (int)p.h_mtop_level.size() - 1 : 0;
    return tiles + tops + levels + ((p.n_small && op <= 1) ? 1 : 0);
  }
  int classes = 0;
  for (int f = 0; f < 2; f++)
    for (int c = 0; c < rq::Plan::N_TOPCLASS; c++) classes += p.topclass_first[f][c + 1] > p.topclass_first[f][c];
  // wavefront sweep + staged top classes + dataflow top + (Q / Q^T) layout pass
  int per_col = (p.wave_streams ? 1 : 0) + classes + (p.n_top_start ? 1 : 0) + (op <= 1 ? 1 : 0);
  return (int)(per_col * k + (k > 1 ? 2 : 0));  // k > 1: the two block transposes
}

int rq_apply_host(const rq_plan *plan, int op, const double *in, double *out, int64_t k) {
  RQ_GUARD({
    need_plan(plan);
    PLAN_DEVICE(plan);
    rq::run_apply_host(plan->p, op, in, out, k);
  })
}

int rq_apply_host_async(const rq_plan *plan, int op, const double *in, double *out, int64_t k) {
  RQ_GUARD({
    need_plan(plan);
    PLAN_DEVICE(plan);
    rq::run_apply_host_async(plan->p, op, in, out, k);
  })
}

int rq_host_wait(const rq_plan *plan) {
  RQ_GUARD({
    need_plan(plan);
    PLAN_DEVICE(plan);
    rq::host_wait(plan->p);
  })
}

int rq_z_apply(const rq_plan *plan, int op, const double *in, double *out, int64_t k, const double *origin,
               void *stream) {
  RQ_GUARD({
    need_plan(plan);
    PLAN_DEVICE(plan);
    const rq::Plan &p = plan->p;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    rq::DBuf dorg;
    if (origin) {
      dorg.alloc(p.m * 24);
      RQ_CUDA(cudaMemcpyAsync(dorg.p, origin, p.m * 24, cudaMemcpyHostToDevice, s));
    }
    rq::run_z(p, op, in, out, k, origin ? dorg.as<double>() : nullptr, s);
    if (origin) RQ_CUDA(cudaStreamSynchronize(s));
  })
}

int rq_z_apply_host(const rq_plan *plan, int op, const double *in, double *out, int64_t k, const double *origin) {
  RQ_GUARD({
    need_plan(plan);
    PLAN_DEVICE(plan);
    const rq::Plan &p = plan->p;
    RQ_CUDA(cudaSetDevice(p.device));
    const int64_t li = (op == RQ_Z_F) ? 3 * p.N : 6 * p.m, lo = (op == RQ_Z_F) ? 6 * p.m : 3 * p.N;
    rq::DBuf din, dout, dorg;
    din.alloc(li * k * 8);
    dout.alloc(lo * k * 8);
    RQ_CUDA(cudaMemcpy(din.p, in, li * k * 8, cudaMemcpyHostToDevice));
    if (origin) {
      dorg.alloc(p.m * 24);
      RQ_CUDA(cudaMemcpy(dorg.p, origin, p.m * 24, cudaMemcpyHostToDevice));
    }
    rq::run_z(p, op, din.as<double>(), dout.as<double>(), k, origin ? dorg.as<double>() : nullptr, 0);
    RQ_CUDA(cudaMemcpy(out, dout.p, lo * k * 8, cudaMemcpyDeviceToHost));
  })
}

int rq_body_centroids(const rq_plan *plan, double *out) {
  RQ_GUARD({
    need_plan(plan);
    PLAN_DEVICE(plan);
    RQ_CUDA(cudaSetDevice(plan->p.device));
    RQ_CUDA(cudaMemcpy(out, plan->p.body_centroid.p, plan->p.m * 24, cudaMemcpyDeviceToHost));
  })
}

int rq_check_duplicates(const double *positions, const int64_t *offsets, int64_t m, uint32_t flags, void *stream,
                        int64_t *body, int64_t *i, int64_t *j, double *tol) {
  try {
    rq::set_error("");
    need_gpu();
    int64_t b = -1, bi = -1, bj = -1;
    double t = 0.0;
    int rc = rq::check_duplicates(positions, offsets, m, (flags & RQ_SETUP_HOST_INPUT) != 0,
                                  static_cast<cudaStream_t>(stream), &b, &bi, &bj, &t);
    if (body) *body = b;
    if (i) *i = bi;
    if (j) *j = bj;
    if (tol) *tol = t;
    if (rc != RQ_OK) {
      char msg[256];
      if (bi < 0) snprintf(msg, sizeof msg, "all beads coincide");
      else snprintf(msg, sizeof msg, "beads %lld and %lld are closer than %.3e (dup_tol)", (long long)bi, (long long)bj, t);
      rq::set_error(msg);
    }
    return rc;
  } catch (const rq::Error &e) {
    rq::set_error(e.msg);
    return e.code;
  } catch (const std::exception &e) {
    rq::set_error(e.what());
    return RQ_ERR_CUDA;
  }
}

int rq_export_tree(const rq_plan *plan, int64_t body, int64_t *perm, int64_t *start, int64_t *stop, int64_t *left,
                   int64_t *right, int32_t *split_axis, int32_t *depth, double *centroid, double *box) {
  RQ_GUARD({
    need_plan(plan);
    PLAN_DEVICE(plan);
    rq::export_tree(plan->p, body, perm, start, stop, left, right, split_axis, depth, centroid, box);
  })
}

int rq_export_factors(const rq_plan *plan, int64_t body, int32_t *ncase, int64_t *n, int64_t *nx, int64_t *ny,
                      uint8_t *swapped, double *t22, double *omega, int64_t *res_offsets, int64_t *total_rows) {
  RQ_GUARD({
    need_plan(plan);
    PLAN_DEVICE(plan);
    rq::export_factors(plan->p, body, ncase, n, nx, ny, swapped, t22, omega, res_offsets, total_rows);
  })
}

int64_t rq_omega_size(const rq_plan *plan, int64_t body) {
  try {
    need_plan(plan);
    PLAN_DEVICE(plan);
    return rq::omega_size(plan->p, body);
  } catch (const rq::Error &e) {
    rq::set_error(e.msg);
    return -1;
  } catch (const std::exception &e) {
    rq::set_error(e.what());
    return -1;
  }
}

int rq_explicit_q_size(const rq_plan *plan, int64_t body, int64_t *n_blocks, int64_t *n_doubles) {
  RQ_GUARD({
    need_plan(plan);
    PLAN_DEVICE(plan);
    rq::explicit_q_size(plan->p, body, n_blocks, n_doubles);
  })
}

int rq_explicit_q(const rq_plan *plan, int64_t body, double *root_rows, int64_t *block_node, int64_t *block_col,
                  int64_t *block_rows, double *block_data) {
  RQ_GUARD({
    need_plan(plan);
    PLAN_DEVICE(plan);
    rq::explicit_q(plan->p, body, root_rows, block_node, block_col, block_rows, block_data);
  })
}

int rq_small_lq(const double *a, int k, int64_t batch, double *t, double *omega) {
  RQ_GUARD({ rq::node_small_lq(a, k, batch, t, omega); })
}

int rq_factor_bead_bead(const double *offset, int64_t batch, double *t22, double *g) {
  RQ_GUARD({ rq::node_factor_bb(offset, batch, t22, g); })
}

int rq_node_merge(int ncase, const double *omega, double a, double b, const double *mx, const double *my, int64_t k,
                  double *mp, double *res) {
  RQ_GUARD({ rq::node_merge(ncase, omega, a, b, mx, my, k, mp, res); })
}

int rq_node_split(int ncase, const double *omega, double a, double b, const double *lp, const double *res, int64_t k,
                  double *lx, double *ly) {
  RQ_GUARD({ rq::node_split(ncase, omega, a, b, lp, res, k, lx, ly); })
}

}  // extern "C"
