// rq_host.cu -- operator application on HOST buffers (rq_apply_host), pipelined.
//
// The reference API is host-side (numpy arrays in and out, matfree.py:86-92), so
// the drop-in path pays PCIe both ways.  For the complement operators the wave
// layout's host segments (groups of rounds, rq_wave.cuh) let the copies overlap
// the sweep and each other:
//
//   Q~v    s_in : H2D of segment e's bead rows, then a flag write (copy engine)
//          s_k  : k_wave<UP> (gathers of a segment wait for its flag) -> top trees
//          s_out: wait(counter[e] = G * epoch) -> D2H of the residue rows of the
//                 bodies whose tiles are all done; the top-tree residues (written
//                 by the top pass at the end) come back compacted and are scattered
//                 into the host buffer by host threads
//   Q~^T g the top trees run first from their residue rows, gathered on the host
//          into a compact pinned buffer; then H2D of the segments in reverse order
//          (the downward sweep runs the rounds backwards), k_wave<DOWN> waiting on
//          their flags, and D2H of each segment's bead rows once it is done.
//
// Flags and counters are monotone (targets = epoch, G * epoch), so nothing is
// reset between calls.  Stream memory operations (cuStreamWriteValue32 /
// cuStreamWaitValue32) need no SM, so the persistent sweep can never wait on
// work that cannot be scheduled.  Q / Q^T and k > 1 take the plain path
// (H2D, apply, D2H).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <mutex>
#include <thread>
#include <vector>

#include "rq_plan.hpp"

namespace rq {
namespace {

PFN_cuStreamWriteValue32_v11070 p_write = nullptr;
PFN_cuStreamWaitValue32_v11070 p_wait = nullptr;

void load_stream_ops() {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q1, q2;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", (void **)&p_write, cudaEnableDefault, &q1) != cudaSuccess ||
        q1 != cudaDriverEntryPointSuccess)
      p_write = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", (void **)&p_wait, cudaEnableDefault, &q2) != cudaSuccess ||
        q2 != cudaDriverEntryPointSuccess)
      p_wait = nullptr;
    cudaGetLastError();
  });
}

void write_value(cudaStream_t s, const void *addr, uint32_t v) {
  const CUresult r = p_write((CUstream)s, (CUdeviceptr)addr, v, 0);
  if (r != CUDA_SUCCESS) throw Error(RQ_ERR_CUDA, "cuStreamWriteValue32 failed (CUresult " + std::to_string((int)r) + ")");
}
void wait_value(cudaStream_t s, const void *addr, uint32_t v) {
  const CUresult r = p_wait((CUstream)s, (CUdeviceptr)addr, v, CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) throw Error(RQ_ERR_CUDA, "cuStreamWaitValue32 failed (CUresult " + std::to_string((int)r) + ")");
}

// top-tree residue rows <-> compact buffer
__global__ void k_top_rr(const TopNode *top, int64_t nt, const int64_t *res_base, int64_t *row, int64_t *cnt) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= nt) return;
  const TopNode T = top[q];
  const int rr = res_rows(flag_case(T.flags));
  cnt[q] = rr;
  row[q] = rr ? res_base[T.body] + T.res_q : 0;
}
__global__ void k_top_pack(const double *v, const int64_t *row, const int64_t *coff, int64_t nt, double *compact) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= nt) return;
  const int64_t c0 = coff[q], n = coff[q + 1] - c0;
  for (int64_t r = 0; r < n; r++) compact[c0 + r] = v[row[q] + r];
}
__global__ void k_top_unpack(const double *compact, const int64_t *row, const int64_t *coff, int64_t nt, double *v) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= nt) return;
  const int64_t c0 = coff[q], n = coff[q + 1] - c0;
  for (int64_t r = 0; r < n; r++) v[row[q] + r] = compact[c0 + r];
}

void build_top_rows(const Plan &p, cudaStream_t s) {
  if (p.n_top_rows >= 0) return;
  const int64_t nt = p.n_top;
  p.h_top_rows.assign(nt, 0);
  p.h_top_coff.assign(nt + 1, 0);
  if (nt > 0) {
    DBuf row, cnt;
    row.alloc(nt * 8);
    cnt.alloc(nt * 8);
    k_top_rr<<<(unsigned)((nt + 255) / 256), 256, 0, s>>>(p.top.as<TopNode>(), nt, p.res_base_d.as<int64_t>(),
                                                         row.as<int64_t>(), cnt.as<int64_t>());
    std::vector<int64_t> hc(nt);
    RQ_CUDA(cudaMemcpyAsync(p.h_top_rows.data(), row.p, nt * 8, cudaMemcpyDeviceToHost, s));
    RQ_CUDA(cudaMemcpyAsync(hc.data(), cnt.p, nt * 8, cudaMemcpyDeviceToHost, s));
    RQ_CUDA(cudaStreamSynchronize(s));
    for (int64_t q = 0; q < nt; q++) p.h_top_coff[q + 1] = p.h_top_coff[q] + hc[q];
  }
  p.top_compact_doubles = p.h_top_coff[nt];
  p.top_rows_d.alloc(std::max<int64_t>(nt, 1) * 8);
  p.top_coff_d.alloc((nt + 1) * 8);
  p.top_compact.alloc(std::max<int64_t>(p.top_compact_doubles, 1) * 8);
  if (nt) RQ_CUDA(cudaMemcpyAsync(p.top_rows_d.p, p.h_top_rows.data(), nt * 8, cudaMemcpyHostToDevice, s));
  RQ_CUDA(cudaMemcpyAsync(p.top_coff_d.p, p.h_top_coff.data(), (nt + 1) * 8, cudaMemcpyHostToDevice, s));
  RQ_CUDA(cudaHostAlloc((void **)&p.top_pinned, std::max<int64_t>(p.top_compact_doubles, 1) * 8, cudaHostAllocPortable));
  RQ_CUDA(cudaStreamSynchronize(s));
  p.n_top_rows = nt;
}

// host threads over the top nodes: compact <- v rows (pack) or v rows <- compact (unpack)
void host_top_rows(const Plan &p, double *v, bool pack) {
  const int64_t nt = p.n_top_rows;
  if (nt <= 0) return;
  const int T = (int)std::max<int64_t>(1, std::min<int64_t>(8, nt / 4096));
  auto work = [&](int t) {
    const int64_t q0 = nt * t / T, q1 = nt * (t + 1) / T;
    for (int64_t q = q0; q < q1; q++) {
      const int64_t c0 = p.h_top_coff[q], n = p.h_top_coff[q + 1] - c0, r0 = p.h_top_rows[q];
      for (int64_t r = 0; r < n; r++) {
        if (pack) p.top_pinned[c0 + r] = v[r0 + r];
        else v[r0 + r] = p.top_pinned[c0 + r];
      }
    }
  };
  if (T == 1) { work(0); return; }
  std::vector<std::thread> th;
  for (int t = 0; t < T; t++) th.emplace_back(work, t);
  for (auto &x : th) x.join();
}

// RQ_HOST_TRACE=1: event timeline of one host application (diagnostics)
struct Trace {
  bool on = getenv("RQ_HOST_TRACE") != nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> ev;
  cudaEvent_t t0 = nullptr;
  void start(cudaStream_t s) {
    if (!on) return;
    cudaEventCreate(&t0);
    cudaEventRecord(t0, s);
  }
  void mark(const std::string &name, cudaStream_t s) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.emplace_back(name, e);
  }
  void print() {
    if (!on) return;
    for (auto &x : ev) {
      float ms = 0;
      cudaEventElapsedTime(&ms, t0, x.second);
      fprintf(stderr, "[rq host] %-24s %8.3f ms\n", x.first.c_str(), ms);
      cudaEventDestroy(x.second);
    }
    cudaEventDestroy(t0);
  }
};

bool host_pinned(const void *ptr) {
  cudaPointerAttributes at{};
  const bool ok = cudaPointerGetAttributes(&at, ptr) == cudaSuccess && at.type == cudaMemoryTypeHost;
  cudaGetLastError();
  return ok;
}

}  // namespace

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
  cudaStream_t s_in = p.host_stream, s_k = p.host_stream2, s_out = p.host_stream3;
  double *din = p.stage_in.as<double>(), *dout = p.stage_out.as<double>();
  load_stream_ops();
  const bool pipelined = (op == RQ_OP_QTILDE_V || op == RQ_OP_QTILDE_TV) && k == 1 && p.wave_streams > 0 &&
                         p_write && p_wait && host_pinned(in) && host_pinned(out) && !getenv("RQ_HOST_PLAIN");
  if (!pipelined) {
    RQ_CUDA(cudaMemcpyAsync(din, in, bi, cudaMemcpyHostToDevice, s_k));
    run_apply(p, op, din, dout, k, s_k);
    RQ_CUDA(cudaMemcpyAsync(out, dout, bo, cudaMemcpyDeviceToHost, s_k));
    RQ_CUDA(cudaStreamSynchronize(s_k));
    return;
  }
  const int E = p.wave_nseg;
  Trace tr;
  const int64_t m = p.m;
  if (!p.host_sync) {  // plain cudaMalloc: stream memory operations on pool memory are refused
    RQ_CUDA(cudaMalloc(&p.host_sync, 8 * (size_t)E));
    RQ_CUDA(cudaMemset(p.host_sync, 0, 8 * (size_t)E));
  }
  build_top_rows(p, s_k);
  const uint32_t epoch = ++p.host_epoch;
  const uint32_t target = (uint32_t)(p.wave_streams * (int64_t)epoch);
  const uint32_t *flags = static_cast<uint32_t *>(p.host_sync);
  uint32_t *counters = static_cast<uint32_t *>(p.host_sync) + E;
  WaveSync sync{flags, counters, epoch, nullptr};
  // body cut points of the segments (bodies are contiguous in tile order)
  std::vector<int64_t> hi_pref(E), lo_suf(E + 1);  // 1 + max body in segs <= e;  min body in segs >= e
  {
    int64_t h = 0;
    for (int e = 0; e < E; e++) {
      if (p.wave_seg_maxb[e] >= 0) h = std::max<int64_t>(h, p.wave_seg_maxb[e] + 1);
      hi_pref[e] = h;
    }
    int64_t l = m;
    lo_suf[E] = m;
    for (int e = E - 1; e >= 0; e--) {
      if (p.wave_seg_maxb[e] >= 0) l = std::min<int64_t>(l, p.wave_seg_minb[e]);
      lo_suf[e] = l;
    }
  }
  auto rows_full = [&](int64_t j) { return 3 * p.bead_off[j]; };
  auto rows_res = [&](int64_t j) { return p.res_base[j]; };
  if (!p.host_ev) RQ_CUDA(cudaEventCreateWithFlags(&p.host_ev, cudaEventDisableTiming));
  // the previous call's kernels are complete (this function synchronises before returning)
  RQ_CUDA(cudaStreamSynchronize(s_in));
  tr.start(s_in);
  if (op == RQ_OP_QTILDE_V) {
    // inputs: segment e needs the bead rows of bodies < hi_pref[e]
    int64_t prev = 0;
    for (int e = 0; e < E; e++) {
      const int64_t j1 = e == E - 1 ? m : hi_pref[e];
      if (j1 > prev) {
        const int64_t r0 = rows_full(prev), r1 = rows_full(j1);
        RQ_CUDA(cudaMemcpyAsync(din + r0, in + r0, (size_t)(r1 - r0) * 8, cudaMemcpyHostToDevice, s_in));
        prev = j1;
      }
      write_value(s_in, flags + e, epoch);
      tr.mark("h2d seg " + std::to_string(e), s_in);
    }
    // the top pass also reads bead rows (beads directly under top nodes): all copies first
    RQ_CUDA(cudaEventRecord(p.host_ev, s_in));
    sync.before_top = p.host_ev;
    run_apply(p, op, din, dout, 1, s_k, 7u, &sync);
    tr.mark("kernels", s_k);
    // outputs: after segment e, bodies < lo_suf[e + 1] have no tile left
    prev = 0;
    for (int e = 0; e < E; e++) {
      const int64_t j1 = e == E - 1 ? m : lo_suf[e + 1];
      wait_value(s_out, counters + e, target);
      if (j1 > prev) {
        const int64_t r0 = rows_res(prev), r1 = rows_res(j1);
        RQ_CUDA(cudaMemcpyAsync(out + r0, dout + r0, (size_t)(r1 - r0) * 8, cudaMemcpyDeviceToHost, s_out));
        prev = j1;
      }
      tr.mark("d2h seg " + std::to_string(e), s_out);
    }
    // top-tree residues (the top pass ran after the sweep): compact copy, host scatter
    if (p.top_compact_doubles > 0) {
      const int64_t nt = p.n_top_rows;
      k_top_pack<<<(unsigned)((nt + 255) / 256), 256, 0, s_k>>>(dout, p.top_rows_d.as<int64_t>(), p.top_coff_d.as<int64_t>(),
                                                               nt, p.top_compact.as<double>());
      RQ_CUDA(cudaMemcpyAsync(p.top_pinned, p.top_compact.p, p.top_compact_doubles * 8, cudaMemcpyDeviceToHost, s_k));
    }
    RQ_CUDA(cudaStreamSynchronize(s_out));
    RQ_CUDA(cudaStreamSynchronize(s_k));
    host_top_rows(p, out, false);
  } else {  // Q~^T g
    // top trees first: their residue rows, gathered on the host
    if (p.top_compact_doubles > 0) {
      host_top_rows(p, const_cast<double *>(in), true);
      const int64_t nt = p.n_top_rows;
      RQ_CUDA(cudaMemcpyAsync(p.top_compact.p, p.top_pinned, p.top_compact_doubles * 8, cudaMemcpyHostToDevice, s_k));
      k_top_unpack<<<(unsigned)((nt + 255) / 256), 256, 0, s_k>>>(p.top_compact.as<double>(), p.top_rows_d.as<int64_t>(),
                                                                 p.top_coff_d.as<int64_t>(), nt, din);
    }
    // inputs in reverse segment order: segment e needs the residue rows of bodies >= lo_suf[e]
    int64_t prev = m;
    for (int e = E - 1; e >= 0; e--) {
      const int64_t j0 = e == 0 ? 0 : lo_suf[e];
      if (j0 < prev) {
        const int64_t r0 = rows_res(j0), r1 = rows_res(prev);
        RQ_CUDA(cudaMemcpyAsync(din + r0, in + r0, (size_t)(r1 - r0) * 8, cudaMemcpyHostToDevice, s_in));
        prev = j0;
      }
      write_value(s_in, flags + e, epoch);
      tr.mark("h2d seg " + std::to_string(e), s_in);
    }
    run_apply(p, op, din, dout, 1, s_k, 7u, &sync);
    tr.mark("kernels", s_k);
    // outputs: once segments >= e are done, bodies >= hi_pref[e - 1] have no tile left
    prev = m;
    for (int e = E - 1; e >= 0; e--) {
      const int64_t j0 = e == 0 ? 0 : hi_pref[e - 1];
      wait_value(s_out, counters + e, target);
      if (j0 < prev) {
        const int64_t r0 = rows_full(j0), r1 = rows_full(prev);
        RQ_CUDA(cudaMemcpyAsync(out + r0, dout + r0, (size_t)(r1 - r0) * 8, cudaMemcpyDeviceToHost, s_out));
        prev = j0;
      }
      tr.mark("d2h seg " + std::to_string(e), s_out);
    }
    // bodies without tiles (their top pass wrote everything): covered by the last piece;
    // the top pass itself precedes the sweep on s_k, so its bead rows are in place
    RQ_CUDA(cudaStreamSynchronize(s_out));
    RQ_CUDA(cudaStreamSynchronize(s_k));
  }
  RQ_CUDA(cudaStreamSynchronize(s_in));
  tr.print();
}

}  // namespace rq
