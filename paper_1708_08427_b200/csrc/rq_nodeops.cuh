// rq_nodeops.cuh -- per-node contractions of the matrix-free passes:
// merge_infosets (matfree.py:41-62) and split_rvset (matfree.py:65-83) with
// the node mixer omega applied from its compact Householder record
// (omega = S H2 H1 H0; records may be strided, SoA inside chunk blobs).
#pragma once

#include "rq_internal.cuh"

namespace rq {

// y <- omega y (S Q^T y) and y <- omega^T y (Q S y) from a compact-WY record
template <int K>
__device__ __forceinline__ void omega_s(const double *rec, int st, unsigned signs, double (&y)[K]) {
  omega_wy<K>(rec, st, signs, y);
}
template <int K>
__device__ __forceinline__ void omega_t_s(const double *rec, int st, unsigned signs, double (&y)[K]) {
  omega_t_wy<K>(rec, st, signs, y);
}

// ratios stored in the record (RIGID_BEAD / GENERAL) or the BEAD_BEAD constant
__device__ __forceinline__ void rec_ratios(int cs, const double *rec, int st, double &a, double &b) {
  if (cs == GENERAL) { a = rec[WY<9>::RA * st]; b = rec[WY<9>::RB * st]; }
  else if (cs == RIGID_BEAD) { a = rec[WY<6>::RA * st]; b = rec[WY<6>::RB * st]; }
  else { a = BB_RATIO; b = BB_RATIO; }
}

__device__ __forceinline__ void ratios(int nx, int ny, double &a, double &b) {
  double n = (double)(nx + ny);  // NodeFactor.ratios (factor.py:85-87)
  a = sqrt((double)nx / n);
  b = sqrt((double)ny / n);
}

// merge_infosets (matfree.py:41-62). res gets residue_rows entries.
#ifndef RQ_SKIP_MATH
#define RQ_SKIP_MATH 0
#endif
__device__ __forceinline__ void merge(int cs, const double *rec, int st, unsigned signs, double a, double b,
                                      const double (&mx)[6], const double (&my)[6], double (&mp)[6],
                                      double (&res)[6]) {
  if (RQ_SKIP_MATH) {  // profiling experiment only: data movement without the transform
#pragma unroll
    for (int r = 0; r < 6; r++) { mp[r] = mx[r] + my[r] + rec[r * st]; res[r] = mx[r] * a + b; }
    return;
  }
  double t[3];
#pragma unroll
  for (int r = 0; r < 3; r++) {
    t[r] = b * mx[r] - a * my[r];
    mp[r] = a * mx[r] + b * my[r];
  }
  if (cs == GENERAL) {
    double y[9] = {mx[3], mx[4], mx[5], my[3], my[4], my[5], t[0], t[1], t[2]};
    omega_s<9>(rec, st, signs, y);
    mp[3] = y[0]; mp[4] = y[1]; mp[5] = y[2];
#pragma unroll
    for (int r = 0; r < 6; r++) res[r] = y[3 + r];
  } else if (cs == RIGID_BEAD) {
    double y[6] = {mx[3], mx[4], mx[5], t[0], t[1], t[2]};
    omega_s<6>(rec, st, signs, y);
    mp[3] = y[0]; mp[4] = y[1]; mp[5] = y[2];
    res[0] = y[3]; res[1] = y[4]; res[2] = y[5];
  } else {  // BEAD_BEAD: m_p[3:] = g @ t
#pragma unroll
    for (int i = 0; i < 3; i++) {
      double s = rec[(3 * i) * st] * t[0];
      s = fma(rec[(3 * i + 1) * st], t[1], s);
      s = fma(rec[(3 * i + 2) * st], t[2], s);
      mp[3 + i] = s;
    }
  }
}

// split_rvset (matfree.py:65-83).
__device__ __forceinline__ void split(int cs, const double *rec, int st, unsigned signs, double a, double b,
                                      const double (&lp)[6], const double (&res)[6], double (&lx)[6],
                                      double (&ly)[6]) {
  double tau[3];
  if (cs == GENERAL) {
    double y[9] = {lp[3], lp[4], lp[5], res[0], res[1], res[2], res[3], res[4], res[5]};
    omega_t_s<9>(rec, st, signs, y);
    lx[3] = y[0]; lx[4] = y[1]; lx[5] = y[2];
    ly[3] = y[3]; ly[4] = y[4]; ly[5] = y[5];
    tau[0] = y[6]; tau[1] = y[7]; tau[2] = y[8];
  } else if (cs == RIGID_BEAD) {
    double y[6] = {lp[3], lp[4], lp[5], res[0], res[1], res[2]};
    omega_t_s<6>(rec, st, signs, y);
    lx[3] = y[0]; lx[4] = y[1]; lx[5] = y[2];
    ly[3] = 0.0; ly[4] = 0.0; ly[5] = 0.0;
    tau[0] = y[3]; tau[1] = y[4]; tau[2] = y[5];
  } else {  // tau = g^T l_p[3:]
#pragma unroll
    for (int j = 0; j < 3; j++) {
      double s = rec[j * st] * lp[3];
      s = fma(rec[(3 + j) * st], lp[4], s);
      s = fma(rec[(6 + j) * st], lp[5], s);
      tau[j] = s;
    }
    lx[3] = lx[4] = lx[5] = 0.0;
    ly[3] = ly[4] = ly[5] = 0.0;
  }
#pragma unroll
  for (int r = 0; r < 3; r++) {
    lx[r] = a * lp[r] + b * tau[r];
    ly[r] = b * lp[r] - a * tau[r];
  }
}

}  // namespace rq
