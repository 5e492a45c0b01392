// rq_host.cu -- operator application on HOST buffers (rq_apply_host / _async).
//
// The reference API is host-side (numpy arrays in and out, matfree.py:86-92), so
// the drop-in path pays PCIe both ways; the kernels are ~5% of it.  What pays is
// keeping both copy directions busy:
//
//  * an application is H2D (stream s_in) -> kernels (s_k) -> D2H (s_out) on one of
//    two staging slots (RQ_HOST_SLOTS), so consecutive applications overlap: the
//    H2D of the next operands runs while the previous results come back, and the link
//    runs full duplex (98 GB/s for both directions on the B200 hosts vs 55-57 alone)
//    (rq_apply_host_async + rq_host_wait; rq_apply_host is both).
//  * pageable (numpy) buffers are staged through pinned memory in 4 MiB pieces by
//    host threads, each piece's DMA queued as soon as its memcpy is done (and the
//    reverse on the way out, piece by piece behind per-piece events), so the host
//    copies overlap the PCIe transfers.
//
// (A segment-pipelined variant in which the persistent sweep consumed input segments
// as the copy engine flagged them was measured slower on these hosts: the top-tree
// residue rows it had to gather and scatter on the host cost more than the ~15%
// that overlapping both directions inside one application gains; see
// profiles/r02_notes.md.)
#include <immintrin.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "rq_plan.hpp"

namespace rq {
namespace {

constexpr size_t PIECE = size_t(4) << 20;

bool host_pinned(const void *ptr) {
  cudaPointerAttributes at{};
  const bool ok = cudaPointerGetAttributes(&at, ptr) == cudaSuccess && at.type == cudaMemoryTypeHost;
  cudaGetLastError();  // plain malloc'd memory may report an error
  return ok;
}

int host_threads() {
  // 8 threads: 35 GB/s of pageable -> pinned memcpy on the B200 hosts; 16 reach 41 GB/s alone
  // but slow the concurrent DMA down (net loss, profiles/r02_notes.md)
  static const int T = [] {
    int t = (int)std::min(8u, std::max(1u, std::thread::hardware_concurrency()));
    if (const char *e = getenv("RQ_HOST_THREADS")) t = std::max(1, std::min(32, atoi(e)));
    return t;
  }();
  return T;
}

// pageable -> pinned staging copy with non-temporal stores: the staging buffer is read next by
// the copy engine, not by this core, so the stores skip the read-for-ownership of their lines
// (the host memory bus is what the staging competes for with the concurrent DMA).  Falls back
// to memcpy without AVX-512 or for unaligned pieces.
__attribute__((target("avx512f"))) void stream_copy_avx512(char *dst, const char *src, size_t n) {
  size_t i = 0;
  for (; i + 256 <= n; i += 256) {
    const __m512i a = _mm512_loadu_si512(src + i), b = _mm512_loadu_si512(src + i + 64);
    const __m512i c = _mm512_loadu_si512(src + i + 128), d = _mm512_loadu_si512(src + i + 192);
    _mm512_stream_si512(reinterpret_cast<__m512i *>(dst + i), a);
    _mm512_stream_si512(reinterpret_cast<__m512i *>(dst + i + 64), b);
    _mm512_stream_si512(reinterpret_cast<__m512i *>(dst + i + 128), c);
    _mm512_stream_si512(reinterpret_cast<__m512i *>(dst + i + 192), d);
  }
  _mm_sfence();
  if (i < n) memcpy(dst + i, src + i, n - i);
}

}  // namespace

void stage_copy(void *dst, const void *src, size_t n) {
  static const bool nt = [] {
    const char *e = getenv("RQ_HOST_NT");
    return __builtin_cpu_supports("avx512f") && !(e && atoi(e) == 0);
  }();
  if (nt && (reinterpret_cast<uintptr_t>(dst) & 63) == 0)
    stream_copy_avx512(static_cast<char *>(dst), static_cast<const char *>(src), n);
  else
    memcpy(dst, src, n);
}

namespace {

void ensure_pinned(double *&buf, size_t &cap, size_t bytes) {
  if (cap >= bytes) return;
  if (buf) cudaFreeHost(buf);
  buf = nullptr;
  cap = 0;
  RQ_CUDA(cudaHostAlloc((void **)&buf, bytes, cudaHostAllocPortable));
  cap = bytes;
}

void ensure_events(std::vector<cudaEvent_t> &ev, size_t n) {
  while (ev.size() < n) {
    cudaEvent_t e;
    RQ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ev.push_back(e);
  }
}

// finish a slot: wait for its D2H and deliver a pageable result (piece by piece)
void finish_slot(const Plan &p, Plan::HostSlot &S) {
  if (!S.busy) return;
  S.busy = false;
  if (!S.defer_out) {
    RQ_CUDA(cudaEventSynchronize(S.e_out));
    return;
  }
  const size_t bytes = S.defer_bytes, np = (bytes + PIECE - 1) / PIECE;
  const int T = (int)std::min<size_t>(host_threads(), np);
  std::vector<std::thread> th;
  std::vector<int> fail(T, 0);
  for (int t = 0; t < T; t++)
    th.emplace_back([&, t] {
      for (size_t i = (size_t)t; i < np; i += (size_t)T) {
        if (cudaEventSynchronize(S.piece_ev[i]) != cudaSuccess) { fail[t] = 1; return; }
        const size_t off = i * PIECE, len = std::min(PIECE, bytes - off);
        memcpy((char *)S.defer_out + off, (const char *)S.pin_out + off, len);
      }
    });
  for (auto &x : th) x.join();
  S.defer_out = nullptr;
  for (int t = 0; t < T; t++)
    if (fail[t]) throw Error(RQ_ERR_CUDA, "device-to-host copy failed");
  (void)p;
}

}  // namespace

void host_wait(const Plan &p) {
  std::lock_guard<std::mutex> lock(p.host_mu);
  RQ_CUDA(cudaSetDevice(p.device));
  for (auto &S : p.hslot) finish_slot(p, S);
}

void run_apply_host_async(const Plan &p, int op, const double *in, double *out, int64_t k) {
  if (op < 0 || op > 3) throw Error(RQ_ERR_VALUE, "op must be one of ('qv', 'qtv', 'qtilde_v', 'qtilde_tv')");
  if (k < 1) throw Error(RQ_ERR_LENGTH, "k must be >= 1");
  if (op >= 2 && p.min_n < 2)
    throw Error(RQ_ERR_BODY_TOO_SMALL, "complement operators need every body to have >= 2 beads");
  if (!in || !out) throw Error(RQ_ERR_VALUE, "null vector");
  RQ_CUDA(cudaSetDevice(p.device));
  std::lock_guard<std::mutex> lock(p.host_mu);
  if (!p.host_stream) {
    for (auto *st : {&p.host_stream, &p.host_stream2, &p.host_stream3})
      RQ_CUDA(cudaStreamCreateWithFlags(st, cudaStreamNonBlocking));
  }
  cudaStream_t s_in = p.host_stream, s_k = p.host_stream2, s_out = p.host_stream3;
  const bool in_comp = op == RQ_OP_QTILDE_TV, out_comp = op == RQ_OP_QTILDE_V;
  const int64_t ri = 3 * p.N - (in_comp ? 6 * p.m : 0), ro = 3 * p.N - (out_comp ? 6 * p.m : 0);
  const size_t bi = (size_t)ri * k * 8, bo = (size_t)ro * k * 8;
  if (!p.host_slots) {
    p.host_slots = 2;  // 3 or 4 measured the same on config 2; each holds both device vectors
    if (const char *e = getenv("RQ_HOST_SLOTS")) p.host_slots = std::max(1, std::min(Plan::MAX_HOST_SLOTS, atoi(e)));
  }
  p.host_next = (p.host_next + 1) % p.host_slots;
  Plan::HostSlot &S = p.hslot[p.host_next];
  finish_slot(p, S);  // the slot's previous application is delivered before its buffers are reused
  if (!S.e_in) {
    for (auto *e : {&S.e_in, &S.e_k, &S.e_out}) RQ_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  }
  if (S.din.bytes < bi) S.din.alloc(bi);
  if (S.dout.bytes < bo) S.dout.alloc(bo);
  double *din = S.din.as<double>(), *dout = S.dout.as<double>();
  // H2D (the slot's device input is free once its previous kernels ran: finish_slot waited
  // for the D2H that followed them)
  if (host_pinned(in)) {
    RQ_CUDA(cudaMemcpyAsync(din, in, bi, cudaMemcpyHostToDevice, s_in));
  } else {
    ensure_pinned(S.pin_in, S.pin_in_cap, bi);
    const size_t np = (bi + PIECE - 1) / PIECE;
    const int T = (int)std::min<size_t>(host_threads(), np);
    std::vector<std::thread> th;
    std::vector<int> fail(T, 0);
    for (int t = 0; t < T; t++)
      th.emplace_back([&, t] {
        for (size_t i = (size_t)t; i < np; i += (size_t)T) {
          const size_t off = i * PIECE, len = std::min(PIECE, bi - off);
          stage_copy((char *)S.pin_in + off, (const char *)in + off, len);
          if (cudaMemcpyAsync((char *)din + off, (char *)S.pin_in + off, len, cudaMemcpyHostToDevice, s_in) !=
              cudaSuccess) { fail[t] = 1; return; }
        }
      });
    for (auto &x : th) x.join();
    for (int t = 0; t < T; t++)
      if (fail[t]) throw Error(RQ_ERR_CUDA, "staged host-to-device copy failed");
  }
  RQ_CUDA(cudaEventRecord(S.e_in, s_in));
  RQ_CUDA(cudaStreamWaitEvent(s_k, S.e_in, 0));
  run_apply(p, op, din, dout, k, s_k);
  RQ_CUDA(cudaEventRecord(S.e_k, s_k));
  RQ_CUDA(cudaStreamWaitEvent(s_out, S.e_k, 0));
  if (host_pinned(out)) {
    RQ_CUDA(cudaMemcpyAsync(out, dout, bo, cudaMemcpyDeviceToHost, s_out));
  } else {  // pageable: D2H into pinned staging piece by piece; delivered by finish_slot
    ensure_pinned(S.pin_out, S.pin_out_cap, bo);
    const size_t np = (bo + PIECE - 1) / PIECE;
    ensure_events(S.piece_ev, np);
    for (size_t i = 0; i < np; i++) {
      const size_t off = i * PIECE, len = std::min(PIECE, bo - off);
      RQ_CUDA(cudaMemcpyAsync((char *)S.pin_out + off, (char *)dout + off, len, cudaMemcpyDeviceToHost, s_out));
      RQ_CUDA(cudaEventRecord(S.piece_ev[i], s_out));
    }
    S.defer_out = out;
    S.defer_bytes = bo;
  }
  RQ_CUDA(cudaEventRecord(S.e_out, s_out));
  S.busy = true;
}

void run_apply_host(const Plan &p, int op, const double *in, double *out, int64_t k) {
  run_apply_host_async(p, op, in, out, k);
  host_wait(p);
}

}  // namespace rq
