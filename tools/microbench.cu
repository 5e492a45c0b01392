// Latency probes on the B200 (fp64 FMA chain, shared-memory load chain,
// __syncthreads round trip, clock64 overhead).  nvcc -arch=sm_100a microbench.cu
#include <cstdio>
__global__ void k(double *out, long long *cyc, int n) {
  __shared__ double sh[1024];
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sh[i] = 1.0 + i * 1e-9; idx[i] = (i * 7 + 1) & 1023; }
  __syncthreads();
  double a = out[threadIdx.x], b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) { a = fma(a, b, c); }
  long long t1 = clock64();
  int j = threadIdx.x;
  for (int i = 0; i < n; i++) { j = idx[j]; }
  long long t2 = clock64();
  for (int i = 0; i < n; i++) { __syncthreads(); }
  long long t3 = clock64();
  double s = 0;
  for (int i = 0; i < n; i++) { s += sh[(j + i) & 1023]; }
  long long t4 = clock64();
  double q = a;
  for (int i = 0; i < n; i++) { q = sqrt(q) + 1.0; }
  long long t5 = clock64();
  double r = a;
  for (int i = 0; i < n; i++) { r = 1.0 / (r + 1.0); }
  long long t6 = clock64();
  out[threadIdx.x] = a + j + s + q + r;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; }
}
int main() {
  double *o; long long *c; cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64); cudaMemset(o, 0, 8192);
  int n = 4096;
  for (int nt : {32, 128, 256}) {
    k<<<1, nt>>>(o, c, n); cudaDeviceSynchronize();
    k<<<1, nt>>>(o, c, n);
    long long h[6]; cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
    printf("threads %d: DFMA chain %.1f cyc, LDS chain %.1f cyc, syncthreads %.1f cyc, LDS+DADD %.1f, sqrt chain %.1f, div chain %.1f\n", nt,
           h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n, h[5] / (double)n);
  }
  return 0;
}
