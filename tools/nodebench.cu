// Latency of one merge (up_node) as compiled for the chunk kernel, per case,
// measured in isolation: 1 warp, chained through M so iterations serialize.
#include <cstdio>
#include "../paper_1708_08427_b200/csrc/rq_nodeops.cuh"
using namespace rq;
template <int CS>
__global__ void kb(const double *grec, long long *cyc, double *sink, int iters) {
  __shared__ __align__(16) double REC[64 * 26];
  __shared__ __align__(16) double M[64 * 6];
  __shared__ __align__(16) double F[64 * 3];
  __shared__ __align__(16) double RES[64 * 6];
  __shared__ NodeMeta ME[64];
  for (int i = threadIdx.x; i < 64 * 26; i += blockDim.x) REC[i] = grec[i % 26];
  for (int i = threadIdx.x; i < 64 * 6; i += blockDim.x) M[i] = 0.1 * i;
  for (int i = threadIdx.x; i < 64 * 3; i += blockDim.x) F[i] = 0.2 * i;
  if (threadIdx.x < 64) { ME[threadIdx.x].x = CS == BEAD_BEAD ? (SRC_BEAD | threadIdx.x) : threadIdx.x; ME[threadIdx.x].y = CS == GENERAL ? threadIdx.x : (SRC_BEAD | threadIdx.x); ME[threadIdx.x].res = 6 * threadIdx.x; ME[threadIdx.x].flags = CS; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    const int q = threadIdx.x, slot = threadIdx.x;
    const double *rec = REC + q * rec_size(CS);
    double R[rec_size(CS)];
    const double2 *r2 = reinterpret_cast<const double2 *>(rec);
#pragma unroll
    for (int i = 0; i < rec_size(CS) / 2; i++) { double2 v = r2[i]; R[2 * i] = v.x; R[2 * i + 1] = v.y; }
    const NodeMeta md = ME[slot];
    double mx[6], my[6];
    const double2 *p2 = reinterpret_cast<const double2 *>(M + 6 * (md.x & 0x7fff));
#pragma unroll
    for (int i = 0; i < 3; i++) { double2 w = p2[i]; mx[2 * i] = w.x; mx[2 * i + 1] = w.y; }
    const double2 *q2 = reinterpret_cast<const double2 *>(M + 6 * (md.y & 0x7fff));
#pragma unroll
    for (int i = 0; i < 3; i++) { double2 w = q2[i]; my[2 * i] = w.x; my[2 * i + 1] = w.y; }
    double aa, bb, mp[6], res[6];
    rec_ratios(CS, R, 1, aa, bb);
    merge(CS, R, 1, flag_signs(md.flags), aa, bb, mx, my, mp, res);
#pragma unroll
    for (int r = 0; r < 6; r++) RES[md.res + r] = res[r];
    double2 *o2 = reinterpret_cast<double2 *>(M + 6 * slot);
#pragma unroll
    for (int i = 0; i < 3; i++) o2[i] = make_double2(mp[2 * i] * 1e-3, mp[2 * i + 1] * 1e-3);
    __syncwarp();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  sink[threadIdx.x] = M[threadIdx.x];
}
int main() {
  double h[26]; for (int i = 0; i < 26; i++) h[i] = 0.01 * (i + 1);
  double *g, *s; long long *c; cudaMalloc(&g, 26 * 8); cudaMalloc(&s, 8192); cudaMalloc(&c, 8);
  cudaMemcpy(g, h, 26 * 8, cudaMemcpyHostToDevice);
  int it = 2000; long long cy;
  kb<GENERAL><<<1, 32>>>(g, c, s, it); cudaDeviceSynchronize(); kb<GENERAL><<<1, 32>>>(g, c, s, it); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
  printf("GENERAL   %.1f cycles/node-step\n", cy / (double)it);
  kb<RIGID_BEAD><<<1, 32>>>(g, c, s, it); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
  printf("RIGID     %.1f cycles/node-step\n", cy / (double)it);
  kb<BEAD_BEAD><<<1, 32>>>(g, c, s, it); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
  printf("BEADBEAD  %.1f cycles/node-step\n", cy / (double)it);
  return 0;
}
