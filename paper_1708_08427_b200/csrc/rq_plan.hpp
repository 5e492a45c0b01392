// rq_plan.hpp -- host-side plan object and error plumbing.
#pragma once

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "rigidq_b200.h"
#include "rq_internal.cuh"
#include "rq_wave.cuh"

namespace rq {

// thread-local error message (rq_last_error)
void set_error(const std::string &msg);
const char *last_error();

struct SetupTimer {  // RQ_SETUP_TIMING=1: per-phase wall time of build_plan (synchronises the stream)
  bool on;
  cudaStream_t s;
  std::chrono::steady_clock::time_point t;
  explicit SetupTimer(cudaStream_t st) : on(getenv("RQ_SETUP_TIMING") != nullptr), s(st), t(std::chrono::steady_clock::now()) {}
  void mark(const char *name) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[rq setup] %-14s %9.3f ms\n", name, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

struct Status {
  int code = RQ_OK;
  std::string msg;
  bool ok() const { return code == RQ_OK; }
};

#define RQ_CUDA(expr)                                                              \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess) {                                                       \
      throw ::rq::Error(RQ_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    }                                                                              \
  } while (0)

struct Error {
  int code;
  std::string msg;
  Error(int c, std::string m) : code(c), msg(std::move(m)) {}
};

// Sets the plan's device for the duration of a C-ABI call and restores the caller's.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard &) = delete;
  DeviceGuard &operator=(const DeviceGuard &) = delete;
};

// owning device buffer
struct DBuf {
  void *p = nullptr;
  size_t bytes = 0;
  DBuf() = default;
  DBuf(const DBuf &) = delete;
  DBuf &operator=(const DBuf &) = delete;
  DBuf(DBuf &&o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
  DBuf &operator=(DBuf &&o) noexcept {
    reset();
    p = o.p; bytes = o.bytes; o.p = nullptr; o.bytes = 0;
    return *this;
  }
  ~DBuf() { reset(); }
  // Stream-ordered allocations from the device's default memory pool, configured to
  // retain freed memory: rebuilding plans (and setup temporaries) reuses mapped memory
  // instead of paying cudaMalloc/cudaFree (which synchronise and remap) every time.
  // An allocation is completed before it is returned, so any stream may use it; a free
  // first waits for the device, so no kernel still using the buffer can see it reused.
  void alloc(size_t b) {
    reset();
    if (b == 0) b = 16;
    cudaStream_t s = pool_stream();
    cudaError_t e = cudaMallocAsync(&p, b, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      p = nullptr;
      cudaGetLastError();
      throw Error(RQ_ERR_NOMEM, std::string("cudaMallocAsync(") + std::to_string(b) + "): " + cudaGetErrorString(e));
    }
    bytes = b;
  }
  void reset() {
    if (p) {
      cudaDeviceSynchronize();
      cudaFreeAsync(p, pool_stream());
    }
    p = nullptr; bytes = 0;
  }
  static cudaStream_t pool_stream() {
    static thread_local int dev_cached = -1;
    static thread_local cudaStream_t st = nullptr;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!st || dev != dev_cached) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
      dev_cached = dev;
    }
    return st;
  }
  template <class T> T *as() const { return static_cast<T *>(p); }
};

struct Plan {
  int device = 0;
  int64_t m = 0, N = 0, NN = 0;    // bodies, beads, nodes
  int max_depth = 96;
  int tile_leaves = 128;           // S: tiles are maximal subtrees with <= S beads
  int tile_height = 0;             // tile height cut (0: none)
  std::vector<int64_t> bead_off;   // host copy, m+1
  int64_t n_case[4] = {0, 0, 0, 0};
  int64_t rec_doubles = 0;
  int64_t n_tiles = 0, n_top = 0, n_slots = 0, n_topbodies = 0, n_toplevels = 0;
  int64_t n_topunits = 0;          // top-tree blob units: whole top trees, or pieces + apex of a split one
  int64_t n_small = 0;             // bodies with n == 1
  int64_t min_n = 0;

  // per body
  DBuf bead_off_d, node_off_d;     // int64 [m+1]
  DBuf body_centroid;              // double [3m] (model centroid)
  DBuf root_box;                   // double [6m]
  // per bead (tree order)
  DBuf perm;                       // int32 body-local original index
  DBuf pos_tree;                   // double [3N]
  DBuf pos_orig;                   // double [3N] (original order, for Z ops)
  DBuf body_of;                    // int32 [N] (original/tree order share bodies)
  // per node (global postorder id)
  DBuf start, stop, left, right, parent;  // int32 body-local
  DBuf depth;                      // int16
  DBuf axis;                       // int8
  DBuf flags;                      // uint8
  DBuf height;                     // int32
  DBuf centroid;                   // double [3NN]
  DBuf t22;                        // double [6NN] lower triangle
  DBuf rec_off;                    // int64 [NN]
  DBuf res_off;                    // int32 [NN] body-relative spectral offsets
  DBuf rec;                        // double [rec_doubles] compact records (postorder)
  // top trees
  DBuf top;                        // TopNode [n_top], sorted by (body, height)
  DBuf topbody;                    // int32 [n_topbodies]: body ids needing the top kernels
  DBuf topbody_lvl;                // int32 [n_topunits+1]: level CSR into toplvl (per blob unit)
  DBuf toplvl;                     // int32 [n_toplevels+1]: top index ranges per level
  DBuf small_bodies;               // int32 [n_small]
  // staged top tree (bodies whose top blob fits shared memory)
  int64_t n_topblob = 0, max_topblob_smem = 0;
  DBuf topblob;                    // bytes
  DBuf topblob_off;                // int64 [n_topblob]: blob byte offsets
  DBuf topblob_body;               // int32 [n_topblob]: top-body index (into topbody)
  DBuf topblob_class;              // uint8 [n_topblob]: shared-memory class (one k_top2 launch per class)
  DBuf topblob_order;              // int32 [n_topblob]: blob indices grouped by class (k_top2 block -> blob)
  // classes: 0 = records staged too; 1..4 = header part staged, <= 8 / 16 / 32 / 64 KB (one warp);
  // 5 = <= 112 KB (128 threads).  Each launch allocates its class's largest footprint.
  static constexpr int N_TOPCLASS = 6;
  int64_t topclass_smem[N_TOPCLASS] = {}, topclass_count[N_TOPCLASS] = {};
  // phase 0: whole top trees and pieces; phase 1: apexes (after the pieces upward, before downward).
  // Phase f, class c: topblob_order[first[f][c], first[f][c+1])
  int64_t topclass_first[2][N_TOPCLASS + 1] = {};
  DBuf topbig;                     // int32 [n_topbig]: top-body indices handled by the global k_top
  int64_t n_topbig = 0;
  // dataflow sweep of those big top trees (k_top_df): parent links, arrival counters, start nodes
  DBuf top_parent;                 // int32 [n_top]: parent top index, -1 for roots / staged bodies
  DBuf top_need;                   // int32 [n_top]: children inside the top tree (arrivals to wait for)
  DBuf top_start;                  // int32 [n_top_start]: top nodes whose children are both below the top tree
  int64_t n_top_start = 0;
  DBuf top_paths, top_path_off;    // int32 root-to-start paths, int64 [n_top_start+1] CSR offsets
  std::vector<int64_t> h_topstart_first;  // [m+1]
  // host-side body -> work-list ranges (segmented / pipelined applications)
  std::vector<int64_t> h_topblob_first, h_topbig_first, h_small_first;  // [m+1] each
  std::vector<int64_t> h_topblob_off;  // [n_topblob+1]: staged top blob byte offsets (host copy)
  DBuf err;                        // int64 [8] device error flags
  // deterministic per-body reductions (centroid, Zf): fixed segments
  int64_t n_seg = 0;
  DBuf seg_body;                   // int32 [n_seg]
  DBuf seg_begin;                  // int64 [n_seg + 1] bead ranges
  DBuf body_seg;                   // int64 [m + 1] segment CSR
  // host-buffer entry points (rq_host.cu): three streams (H2D, kernels, D2H) and two staging
  // slots, so consecutive applications overlap
  mutable cudaStream_t host_stream = nullptr, host_stream2 = nullptr, host_stream3 = nullptr;
  struct HostSlot {
    bool busy = false;
    DBuf din, dout;                          // device staging
    cudaEvent_t e_in = nullptr, e_k = nullptr, e_out = nullptr;
    double *pin_in = nullptr, *pin_out = nullptr;  // pinned staging of pageable buffers
    size_t pin_in_cap = 0, pin_out_cap = 0;
    std::vector<cudaEvent_t> piece_ev;       // per-piece D2H events (pageable results)
    double *defer_out = nullptr;             // pageable result delivered by the next wait
    size_t defer_bytes = 0;
  };
  static constexpr int MAX_HOST_SLOTS = 4;
  mutable HostSlot hslot[MAX_HOST_SLOTS];
  mutable int host_next = 0;
  mutable int host_slots = 0;  // slots in use (RQ_HOST_SLOTS, default 2), set on first use

  mutable std::mutex host_mu;
  // Per-stream exchange state: applications of one plan on different streams may run
  // concurrently (matfree.py:16-17: applies on one fitted tree are safe), so the tile-root
  // exchange slots, the multi-RHS exchange block and the top-tree arrival counters are
  // owned per stream.
  struct StreamState {
    DBuf scratch, mrhs_scratch, mrhs_tx, top_cnt;  // mrhs_tx: multi-RHS top exchange [top][6][k]
    DBuf col_in, col_out;     // column-major copies of a (rows, k) block for the column loop
    DBuf res_tmp, roots;      // Q / Q^T: residues in the private layout and the 6 root rows per body
    DBuf in_al;               // 16-byte aligned copy of a misaligned input
    DBuf round_ctr;           // wave round-window arrival counters [2][rounds] (up, down) + 2 abandon flags
    uint32_t wave_epoch[2] = {0, 0};
    DBuf zpart;               // Zf per-segment partial sums
    DBuf zcnt;                // Zf per-(column, body) arrival counters (self-resetting)
  };
  mutable std::mutex state_mu;
  mutable std::map<cudaStream_t, std::unique_ptr<StreamState>> stream_state;
  StreamState &state_for(cudaStream_t s) const;
  // multi-RHS unit programs (rq_mrhs.cu), built on the first k >= mrhs_min application
  int mrhs_min = 5;                // k at which the column-parallel kernels beat the column loop (measured)
  int mrhs_tile = 64;              // leaves per multi-RHS tile unit
  mutable std::mutex mrhs_mu;
  mutable bool mrhs_built = false;
  mutable int64_t mrhs_entries = 0, n_tile_units = 0, n_top_units = 0;
  mutable int64_t mrhs_tile_bytes = 0, mrhs_top_bytes = 0;  // entry header + record bytes per column group
  mutable int mrhs_depth_tile = 1, mrhs_depth_top = 1;
  mutable DBuf mrhs_units, mrhs_prog, mtop;  // mtop: multi-RHS top nodes by height
  mutable int64_t n_mtop = 0;
  mutable std::vector<int64_t> h_mtop_level;
  mutable std::vector<int64_t> h_tile_unit_first, h_top_unit_first;
  // private residue layout: body j's residues start at res_base[j] = sum_{i<j} max(0, 3 n_i - 6)
  // (the Q~ layout when every body has n >= 2; Q / Q^T go through it plus 6 root rows per body)
  std::vector<int64_t> res_base;   // host copy, m+1
  DBuf res_base_d;                 // int64 [m+1]
  // wavefront apply streams (rq_wave.cu)
  int64_t wave_streams = 0, wave_steps = 0, wave_blob_bytes = 0, wave_nodes = 0;
  int64_t wave_up_bytes = 0, wave_down_bytes = 0;  // bytes one upward / downward sweep streams
  int64_t wave_stage_bytes = 0, wave_rounds = 1;
  int wave_window = 0;                  // run-time round window (rounds)
  mutable int sms = 0;                  // SM count of the plan's device
  int wave_mslots = 0, wave_nst = 2;  // TMA stages (fixed 2: the headers locate the block two steps ahead)
  WaveCaps wave_caps;
  DBuf wave_desc;                  // StepDesc [wave_steps]
  DBuf wave_stream_first;          // int64 [wave_streams + 1]
  DBuf wave_blob;                  // step blocks
  mutable bool wave_ready = false;
  mutable bool top_attr_set = false;  // k_top2 shared-memory attribute set
  mutable int wave_ctas_per_sm = 0;
  int64_t device_bytes() const;
  ~Plan() {
    for (cudaStream_t st : {host_stream, host_stream2, host_stream3})
      if (st) cudaStreamDestroy(st);
    for (auto &S : hslot) {
      for (cudaEvent_t e : {S.e_in, S.e_k, S.e_out})
        if (e) cudaEventDestroy(e);
      for (cudaEvent_t e : S.piece_ev) cudaEventDestroy(e);
      if (S.pin_in) cudaFreeHost(S.pin_in);
      if (S.pin_out) cudaFreeHost(S.pin_out);
    }
  }
};

void build_plan(Plan &p, const double *pos, const int64_t *offsets, int64_t m, int max_depth,
                bool host_input, cudaStream_t s);
struct WaveBuildIn {
  int64_t n_tiles;
  const int64_t *tile_root;  // global node id of every tile root, in tile order
  const int64_t *node_off, *bead_off, *rec_off, *res_base;
  const int32_t *node_body, *start, *stop, *left, *right, *parent, *height, *res_off, *perm, *slot_scan;
  const uint8_t *flags;
  const double *rec;
};
// Raise kernel f's dynamic shared-memory limit on the current device to at least `bytes`.
// The attribute is process-wide, so it only ever grows: a plan with a smaller footprint never
// lowers it under a bigger plan's launches (other threads included).
void ensure_smem_attr(const void *f, size_t bytes);
// CTAs per SM of kernel f at (threads, dynamic smem) on the current device, memoised (the
// multi-RHS launches ask on every application)
int occupancy_cached(const void *f, int threads, size_t smem);
void build_wave(Plan &p, const WaveBuildIn &in, cudaStream_t s);
size_t wave_smem(const Plan &p, uint32_t *o_m, uint32_t *o_v, uint32_t *vreg);
void wave_prepare(const Plan &p);
// tile part of one upward / downward sweep over all bodies (rq_wave.cu); residues in the
// private layout, body-root vectors to / from `roots` (nullptr: dropped / zero)
void run_wave(const Plan &p, bool up, const double *in, double *out, double *scratch, double *roots,
              cudaStream_t s, uint32_t *round_ctr = nullptr, uint32_t epoch = 0, uint32_t *abandon = nullptr);
// bodies [j0, j1) of a plan (all work lists are in body order)
struct BodyRange {
  int64_t j0 = 0, j1 = -1;  // j1 < 0: all bodies
};
void run_apply(const Plan &p, int op, const double *in, double *out, int64_t k, cudaStream_t s,
               unsigned phases = 7u);
void build_mrhs(const Plan &p, cudaStream_t s);
void run_apply_mrhs(const Plan &p, int op, const double *in, double *out, int64_t k, cudaStream_t s,
                    unsigned phases = 7u, BodyRange range = BodyRange());
bool use_mrhs(const Plan &p, int64_t k);
// Host-buffer applications (rq_host.cu): H2D -> kernels -> D2H on three streams and two
// staging slots; the async form returns once queued (pageable results are delivered by
// host_wait), so consecutive applications overlap their copies.
void run_apply_host(const Plan &p, int op, const double *in, double *out, int64_t k);
void run_apply_host_async(const Plan &p, int op, const double *in, double *out, int64_t k);
void host_wait(const Plan &p);
void run_z(const Plan &p, int op, const double *in, double *out, int64_t k, const double *origin_d,
           cudaStream_t s);
int check_duplicates(const double *pos, const int64_t *offsets, int64_t m, bool host_input,
                     cudaStream_t s, int64_t *body, int64_t *i, int64_t *j, double *tol);
void export_tree(const Plan &p, int64_t body, int64_t *perm, int64_t *start, int64_t *stop,
                 int64_t *left, int64_t *right, int32_t *split_axis, int32_t *depth,
                 double *centroid, double *box);
void export_factors(const Plan &p, int64_t body, int32_t *ncase, int64_t *n, int64_t *nx,
                    int64_t *ny, uint8_t *swapped, double *t22, double *omega,
                    int64_t *res_offsets, int64_t *total_rows);
int64_t omega_size(const Plan &p, int64_t body);
void explicit_q_size(const Plan &p, int64_t body, int64_t *n_blocks, int64_t *n_doubles);
void explicit_q(const Plan &p, int64_t body, double *root_rows, int64_t *block_node,
                int64_t *block_col, int64_t *block_rows, double *block_data);

void node_small_lq(const double *a, int k, int64_t batch, double *t, double *om);
void node_factor_bb(const double *d, int64_t batch, double *t, double *g);
void node_merge(int cs, const double *om, double a, double b, const double *mx, const double *my, int64_t K,
                double *mp, double *res);
void node_split(int cs, const double *om, double a, double b, const double *lp, const double *res, int64_t K,
                double *lx, double *ly);

// pageable -> pinned staging copy (non-temporal AVX-512 stores when available; rq_host.cu)
void stage_copy(void *dst, const void *src, size_t n);

}  // namespace rq
