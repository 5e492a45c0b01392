// rq_lq.cuh -- per-node factorization math (device), restating factor.py.
//
// The LQ of a 3 x K coupling matrix (small_lq, factor.py:90-109) is computed
// as numpy does it: Householder QR of a^T through LAPACK dgeqr2 (dlarfg /
// dlarf branch structure, reached from factor.py:103 via np.linalg.qr).  We
// keep the reflectors in compact form (the apply path streams them) instead
// of forming omega = Q^T explicitly with dorg2r; omega is formed only for
// parity exports.  This translation unit is compiled with --fmad=false so the
// centroid recursion (tree.py:126) and the closed forms round exactly where
// the reference rounds.
#pragma once

#include "rq_internal.cuh"

namespace rq {

__host__ __device__ inline double lq_dnrm2(int n, const double *x) {
  double s = 0.0;
  for (int i = 0; i < n; i++) s += x[i] * x[i];
  return sqrt(s);
}

__host__ __device__ inline double lq_dlapy2(double x, double y) {
  double xa = fabs(x), ya = fabs(y);
  double w = fmax(xa, ya), z = fmin(xa, ya);
  if (z == 0.0 || w > 1.7976931348623157e308) return w;
  double q = z / w;
  return w * sqrt(1.0 + q * q);
}

// dlarfg(n, alpha, x, 1, tau)
__host__ __device__ inline void lq_dlarfg(int n, double &alpha, double *x, double &tau) {
  if (n <= 1) { tau = 0.0; return; }
  double xnorm = lq_dnrm2(n - 1, x);
  if (xnorm == 0.0) { tau = 0.0; return; }
  double beta = -copysign(lq_dlapy2(alpha, xnorm), alpha);
  const double safmin = 2.2250738585072014e-308 / 1.1102230246251565e-16;
  int knt = 0;
  if (fabs(beta) < safmin) {
    const double rsafmn = 1.0 / safmin;
    do {
      knt++;
      for (int i = 0; i < n - 1; i++) x[i] *= rsafmn;
      beta *= rsafmn;
      alpha *= rsafmn;
    } while (fabs(beta) < safmin && knt < 20);
    xnorm = lq_dnrm2(n - 1, x);
    beta = -copysign(lq_dlapy2(alpha, xnorm), alpha);
  }
  tau = (beta - alpha) / beta;
  double scal = 1.0 / (alpha - beta);
  for (int i = 0; i < n - 1; i++) x[i] *= scal;
  for (int j = 0; j < knt; j++) beta *= safmin;
  alpha = beta;
}

// dlarf('Left') on the column-major m x n block C (ldc) with v (v[0] == 1).
__host__ __device__ inline void lq_dlarf_left(int m, int n, const double *v, double tau, double *C, int ldc) {
  int lastv = 0, lastc = 0;
  if (tau != 0.0) {
    lastv = m;
    while (lastv > 0 && v[lastv - 1] == 0.0) lastv--;
    if (n > 0 && lastv > 0) {
      if (C[(n - 1) * ldc] != 0.0 || C[(n - 1) * ldc + lastv - 1] != 0.0) {
        lastc = n;
      } else {
        for (int col = n; col >= 1 && lastc == 0; col--)
          for (int i = 0; i < lastv; i++)
            if (C[(col - 1) * ldc + i] != 0.0) { lastc = col; break; }
      }
    }
  }
  if (lastv > 0 && lastc > 0) {
    double w[3];
    for (int j = 0; j < lastc; j++) {
      double s = 0.0;
      for (int i = 0; i < lastv; i++) s += C[j * ldc + i] * v[i];
      w[j] = s;
    }
    for (int j = 0; j < lastc; j++) {
      double temp = -tau * w[j];
      for (int i = 0; i < lastv; i++) C[j * ldc + i] += v[i] * temp;
    }
  }
}

// small_lq in compact form.  a: row-major 3 x K (== column-major K x 3 A = a^T).
// Outputs t (lower-triangular, packed t00,t10,t11,t20,t21,t22), the compact-WY
// record (WY<K> layout, without the ratios) and the sign bits s_i = -1.
template <int K>
__host__ __device__ inline void lq_factor(const double *a, double t6[6], double *rec, unsigned &signs) {
  bool any = false;
  for (int i = 0; i < 3 * K; i++) any |= (a[i] != 0.0);
  for (int i = 0; i < WY<K>::RA; i++) rec[i] = 0.0;
  signs = 0;
  if (!any) { // factor.py:100-101: t = 0, omega = I_k  (V = 0, T = 0)
    for (int i = 0; i < 6; i++) t6[i] = 0.0;
    return;
  }
  double A[3 * K];
  for (int i = 0; i < 3 * K; i++) A[i] = a[i];
  double tau[3];
  // dgeqr2(K, 3)
  for (int i = 0; i < 3; i++) {
    int i1 = (i + 1 < K) ? i + 1 : K - 1;
    lq_dlarfg(K - i, A[i * K + i], &A[i * K + i1], tau[i]);
    if (i < 2) {
      double aii = A[i * K + i];
      A[i * K + i] = 1.0;
      lq_dlarf_left(K - i, 2 - i, &A[i * K + i], tau[i], &A[(i + 1) * K + i], K);
      A[i * K + i] = aii;
    }
  }
  double s[3];
  for (int i = 0; i < 3; i++) {
    double d = A[i * K + i];
    s[i] = (d < 0.0) ? -1.0 : 1.0; // np.sign with 0 -> +1
    if (d < 0.0) signs |= 1u << i;
  }
  // t = (R[:3,:3] * s[:, None]).T : t[i][j] = R[j][i] * s[j], R[j][i] = A(j, i) = A[i*K + j]
  t6[0] = A[0 * K + 0] * s[0];
  t6[1] = A[1 * K + 0] * s[0];
  t6[2] = A[1 * K + 1] * s[1];
  t6[3] = A[2 * K + 0] * s[0];
  t6[4] = A[2 * K + 1] * s[1];
  t6[5] = A[2 * K + 2] * s[2];
  // V (rows below the diagonal) and T (dlarft forward/columnwise)
  int o = 0;
  for (int i = 0; i < 3; i++)
    for (int r = i + 1; r < K; r++) rec[o++] = A[i * K + r];
  auto vdot = [&](int i, int j) {  // v_i^T v_j for i < j (v_i[i] = 1, v_j[j] = 1, v_j[r < j] = 0)
    double d = (j < K) ? A[i * K + j] : 0.0;
    for (int r = j + 1; r < K; r++) d += A[i * K + r] * A[j * K + r];
    return d;
  };
  const double T00 = tau[0], T11 = tau[1], T22 = tau[2];
  const double T01 = -tau[1] * T00 * vdot(0, 1);
  const double t0 = vdot(0, 2), t1 = vdot(1, 2);
  const double T02 = -tau[2] * (T00 * t0 + T01 * t1);
  const double T12 = -tau[2] * (T11 * t1);
  rec[WY<K>::T + 0] = T00;
  rec[WY<K>::T + 1] = T01;
  rec[WY<K>::T + 2] = T02;
  rec[WY<K>::T + 3] = T11;
  rec[WY<K>::T + 4] = T12;
  rec[WY<K>::T + 5] = T22;
}

// y <- omega y  = S Q^T y   (record with unit stride)
template <int K>
__host__ __device__ inline void omega_apply(const double *rec, unsigned signs, double (&y)[K]) {
  omega_wy<K>(rec, 1, signs, y);
}

// y <- omega^T y = Q S y
template <int K>
__host__ __device__ inline void omega_apply_t(const double *rec, unsigned signs, double (&y)[K]) {
  omega_t_wy<K>(rec, 1, signs, y);
}

__host__ __device__ inline void skew3(const double r[3], double A[9]) { // model.py:25-30
  A[0] = 0.0;   A[1] = -r[2]; A[2] = r[1];
  A[3] = r[2];  A[4] = 0.0;   A[5] = -r[0];
  A[6] = -r[1]; A[7] = r[0];  A[8] = 0.0;
}

// factor_bead_bead (factor.py:130-168) in the cyclic frame axes = (A0, A1, A2)
// (compile-time, so every array index below is static).
template <int A0, int A1, int A2>
__host__ __device__ inline void factor_bead_bead_frame(const double d[3], double t6[6], double g[9]) {
  const double a = d[A0], b = d[A1], c = d[A2];
  const double bc2 = b * b + c * c;
  const double ell = a * a + bc2;
  const double sq2 = sqrt(2.0);
  const double sbc2 = sqrt(bc2);
  const double r2l = sqrt(2.0 * ell / bc2);
  const double tp[9] = {sqrt(2.0 * bc2), 0.0, 0.0,
                        -sq2 * a * b / sbc2, c * r2l, 0.0,
                        -sq2 * a * c / sbc2, -b * r2l, 0.0};
  const double den0 = sqrt(2.0 * bc2), den1 = sqrt(2.0 * ell * bc2), den2 = sqrt(2.0 * ell);
  const double uh[9] = {0.0 / den0, -c / den0, b / den0,
                        bc2 / den1, -a * b / den1, -a * c / den1,
                        -a / den2, -b / den2, -c / den2};
  constexpr int ax[3] = {A0, A1, A2};
  double m[9], gh[9];
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) {
      m[ax[i] * 3 + j] = tp[i * 3 + j];   // m[perm, :] = t_prime
      gh[i * 3 + ax[j]] = uh[i * 3 + j];  // g_half[:, perm] = u_half
    }
  double rec3[WY<3>::SIZE];
  unsigned sg;
  lq_factor<3>(m, t6, rec3, sg);
  double om3[9];
#pragma unroll
  for (int j = 0; j < 3; j++) {  // om3 e_j
    double y[3] = {0.0, 0.0, 0.0};
    y[j] = 1.0;
    omega_apply<3>(rec3, sg, y);
#pragma unroll
    for (int i = 0; i < 3; i++) om3[i * 3 + j] = y[i];
  }
#pragma unroll
  for (int i = 0; i < 3; i++)
#pragma unroll
    for (int j = 0; j < 3; j++) {
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < 3; l++) s += om3[i * 3 + l] * gh[l * 3 + j];
      g[i * 3 + j] = sq2 * s;  // g = sqrt(2) * (om3 @ g_half)
    }
}

// _CYCLIC = {2: (0,1,2), 0: (1,2,0), 1: (2,0,1)} keyed by argmax|d| (first maximum)
__host__ __device__ inline void factor_bead_bead(const double d[3], double t6[6], double g[9]) {
  int am = 0;
  if (fabs(d[1]) > fabs(d[am])) am = 1;
  if (fabs(d[2]) > fabs(d[am])) am = 2;
  if (am == 2) factor_bead_bead_frame<0, 1, 2>(d, t6, g);
  else if (am == 0) factor_bead_bead_frame<1, 2, 0>(d, t6, g);
  else factor_bead_bead_frame<2, 0, 1>(d, t6, g);
}

}  // namespace rq
