/*
 * rq_oracle.c -- CPU restatement of the reference `rigidq` hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see rq_oracle.h).  It restates, in plain C, the
 * algorithms of /root/reference/pkg/src/rigidq (tree.py, factor.py,
 * matfree.py, model.py) including the LAPACK dgeqr2/dorg2r/dlarfg branch
 * structure that numpy's np.linalg.qr reaches through scipy-openblas 0.3.30
 * (factor.py:103).  Compiled with -ffp-contract=off so every product/sum is
 * rounded exactly where the reference's numpy expression rounds.
 */
#include "rq_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------ */
/* LAPACK emulation (reference semantics of dnrm2, dlapy2, dlarfg, dlarf,     */
/* dgeqr2, dorg2r), reached from factor.py:103 via numpy qr(mode=complete).   */
/* ------------------------------------------------------------------------ */

static double lp_dnrm2(int n, const double *x) {
  /* OpenBLAS x86_64 dnrm2 accumulates in x87 extended precision. */
  long double s = 0.0L;
  for (int i = 0; i < n; i++) s += (long double)x[i] * (long double)x[i];
  return (double)sqrtl(s);
}

static double lp_dlapy2(double x, double y) {
  double xa = fabs(x), ya = fabs(y);
  double w = xa > ya ? xa : ya;
  double z = xa < ya ? xa : ya;
  if (z == 0.0 || w > DBL_MAX) return w;
  double q = z / w;
  return w * sqrt(1.0 + q * q);
}

/* dlarfg(n, alpha, x, 1, tau): H*(alpha;x) = (beta;0). */
static void lp_dlarfg(int n, double *alpha, double *x, double *tau) {
  if (n <= 1) { *tau = 0.0; return; }
  double xnorm = lp_dnrm2(n - 1, x);
  if (xnorm == 0.0) { *tau = 0.0; return; }
  double beta = -copysign(lp_dlapy2(*alpha, xnorm), *alpha);
  const double safmin = DBL_MIN / (DBL_EPSILON * 0.5);
  int knt = 0;
  if (fabs(beta) < safmin) {
    const double rsafmn = 1.0 / safmin;
    do {
      knt++;
      for (int i = 0; i < n - 1; i++) x[i] *= rsafmn;
      beta *= rsafmn;
      *alpha *= rsafmn;
    } while (fabs(beta) < safmin && knt < 20);
    xnorm = lp_dnrm2(n - 1, x);
    beta = -copysign(lp_dlapy2(*alpha, xnorm), *alpha);
  }
  *tau = (beta - *alpha) / beta;
  double scal = 1.0 / (*alpha - beta);
  for (int i = 0; i < n - 1; i++) x[i] *= scal;
  for (int j = 0; j < knt; j++) beta *= safmin;
  *alpha = beta;
}

/* dlarf('Left', m, n, v, 1, tau, C, ldc): C := (I - tau v v^T) C. */
static void lp_dlarf_left(int m, int n, const double *v, double tau, double *C, int ldc) {
  int lastv = 0, lastc = 0;
  if (tau != 0.0) {
    lastv = m;
    while (lastv > 0 && v[lastv - 1] == 0.0) lastv--;
    /* iladlc(lastv, n, C, ldc) */
    lastc = 0;
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
    double w[16];
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

/* dgeqr2 on A (m x n, column major, lda = m). */
static void lp_dgeqr2(int m, int n, double *A, double *tau) {
  int k = m < n ? m : n;
  for (int i = 0; i < k; i++) {
    int i1 = (i + 1 < m) ? i + 1 : m - 1;
    lp_dlarfg(m - i, &A[i * m + i], &A[i * m + i1], &tau[i]);
    if (i < n - 1) {
      double aii = A[i * m + i];
      A[i * m + i] = 1.0;
      lp_dlarf_left(m - i, n - i - 1, &A[i * m + i], tau[i], &A[(i + 1) * m + i], m);
      A[i * m + i] = aii;
    }
  }
}

/* dorg2r(m, n, k, A, lda=m, tau): form the m x n Q = H(0)...H(k-1). */
static void lp_dorg2r(int m, int n, int k, double *A, const double *tau) {
  for (int j = k; j < n; j++) {
    for (int l = 0; l < m; l++) A[j * m + l] = 0.0;
    A[j * m + j] = 1.0;
  }
  for (int i = k - 1; i >= 0; i--) {
    if (i < n - 1) {
      A[i * m + i] = 1.0;
      lp_dlarf_left(m - i, n - i - 1, &A[i * m + i], tau[i], &A[(i + 1) * m + i], m);
    }
    if (i < m - 1)
      for (int l = i + 1; l < m; l++) A[i * m + l] *= -tau[i];
    A[i * m + i] = 1.0 - tau[i];
    for (int l = 0; l < i; l++) A[i * m + l] = 0.0;
  }
}

/* small_lq (factor.py:90-109).  a: row-major 3 x k.  The column-major k x 3
 * matrix a^T has exactly a's row-major storage (lda = k). */
void rqo_small_lq(const double *a, int k, double *t, double *omega) {
  int any = 0;
  for (int i = 0; i < 3 * k; i++) if (a[i] != 0.0) { any = 1; break; }
  if (!any) { /* factor.py:100-101 */
    memset(t, 0, 9 * sizeof(double));
    for (int i = 0; i < k; i++)
      for (int j = 0; j < k; j++) omega[i * k + j] = (i == j) ? 1.0 : 0.0;
    return;
  }
  double q[81], tau[3];
  memcpy(q, a, 3 * k * sizeof(double)); /* first 3 columns of the k x k work */
  lp_dgeqr2(k, 3, q, tau);
  double r[9]; /* R[i][j] = A(i,j), i <= j */
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) r[i * 3 + j] = (i <= j) ? q[j * k + i] : 0.0;
  lp_dorg2r(k, k, 3, q, tau);
  double s[3];
  for (int i = 0; i < 3; i++) {
    double d = r[i * 3 + i];
    s[i] = (d > 0.0) ? 1.0 : (d < 0.0 ? -1.0 : 1.0); /* np.sign, 0 -> 1 */
  }
  /* t = (R[:3,:3] * s[:,None]).T */
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) t[i * 3 + j] = r[j * 3 + i] * s[j];
  /* omega = Q^T: omega[i][j] = Q(j,i) = q[i*k + j]; rows 0..2 scaled by s */
  for (int i = 0; i < k; i++)
    for (int j = 0; j < k; j++) omega[i * k + j] = q[i * k + j] * (i < 3 ? s[i] : 1.0);
}

/* ------------------------------------------------------------------------ */
/* tree (tree.py:73-134)                                                      */
/* ------------------------------------------------------------------------ */

static const int AXIS_CYCLE[3] = {2, 1, 0}; /* tree.py:27 */

typedef struct {
  const double *pos; /* original order */
  rqo_body *b;
  int64_t nnodes;   /* nodes appended so far */
  int64_t nleaf;    /* len(leaf_seq) */
  int max_depth;
  int err;
  int64_t *scratch; /* partition scratch */
} build_ctx;

static int64_t build_rec(build_ctx *c, int64_t *idx, int64_t cnt, const double box[6], int depth) {
  rqo_body *b = c->b;
  if (c->err) return -1;
  if (cnt == 1) { /* tree.py:87-93 */
    int64_t id = c->nnodes++;
    int64_t s = c->nleaf++;
    b->perm[s] = idx[0];
    b->start[id] = s; b->stop[id] = s + 1;
    b->left[id] = b->right[id] = -1;
    for (int a = 0; a < 3; a++) b->centroid[id * 3 + a] = c->pos[idx[0] * 3 + a];
    memcpy(&b->box[id * 6], box, 6 * sizeof(double));
    b->split_axis[id] = -1;
    b->depth[id] = depth;
    return id;
  }
  double cell[6];
  memcpy(cell, box, sizeof(cell));
  int d = depth, axis = 0;
  double mid = 0.0;
  int64_t nlow = 0;
  for (;;) { /* tree.py:96-114 */
    if (d >= c->max_depth) { c->err = RQO_ERR_DUPLICATE; return -1; }
    axis = AXIS_CYCLE[d % 3];
    mid = 0.5 * (cell[axis] + cell[3 + axis]);
    nlow = 0;
    for (int64_t i = 0; i < cnt; i++) nlow += (c->pos[idx[i] * 3 + axis] <= mid);
    if (nlow == cnt) cell[3 + axis] = mid;
    else if (nlow == 0) cell[axis] = mid;
    else break;
    d++;
  }
  double low_box[6], high_box[6];
  memcpy(low_box, cell, sizeof(cell)); low_box[3 + axis] = mid;
  memcpy(high_box, cell, sizeof(cell)); high_box[axis] = mid;
  /* stable partition idx -> [low..., high...] (idx[low], idx[~low]) */
  int64_t *tmp = c->scratch;
  int64_t lo = 0, hi = nlow;
  for (int64_t i = 0; i < cnt; i++) {
    if (c->pos[idx[i] * 3 + axis] <= mid) tmp[lo++] = idx[i];
    else tmp[hi++] = idx[i];
  }
  memcpy(idx, tmp, cnt * sizeof(int64_t));
  int64_t start = c->nleaf;
  int64_t l = build_rec(c, idx, nlow, low_box, d + 1);
  int64_t r = build_rec(c, idx + nlow, cnt - nlow, high_box, d + 1);
  if (c->err) return -1;
  int64_t nl = b->stop[l] - b->start[l], nr = b->stop[r] - b->start[r];
  int64_t id = c->nnodes++;
  b->start[id] = start; b->stop[id] = c->nleaf;
  b->left[id] = l; b->right[id] = r;
  for (int a = 0; a < 3; a++) /* tree.py:126 */
    b->centroid[id * 3 + a] =
        ((double)nl * b->centroid[l * 3 + a] + (double)nr * b->centroid[r * 3 + a]) / (double)(nl + nr);
  memcpy(&b->box[id * 6], box, 6 * sizeof(double));
  b->split_axis[id] = axis;
  b->depth[id] = depth;
  return id;
}

static void *xcalloc(size_t n, size_t s) { return calloc(n ? n : 1, s); }

/* ------------------------------------------------------------------------ */
/* factor (factor.py:112-244)                                                 */
/* ------------------------------------------------------------------------ */

static void skew(const double r[3], double A[9]) { /* model.py:25-30 */
  A[0] = 0.0;   A[1] = -r[2]; A[2] = r[1];
  A[3] = r[2];  A[4] = 0.0;   A[5] = -r[0];
  A[6] = -r[1]; A[7] = r[0];  A[8] = 0.0;
}

/* factor_bead_bead (factor.py:130-168): offset d -> t22, g (3x3). */
static void factor_bead_bead(const double d[3], double t22[9], double g[9]) {
  static const int CYC[3][3] = {{1, 2, 0}, {2, 0, 1}, {0, 1, 2}}; /* _CYCLIC[argmax] */
  int am = 0; /* np.argmax(np.abs(d)): first maximum */
  for (int i = 1; i < 3; i++) if (fabs(d[i]) > fabs(d[am])) am = i;
  const int *axes = CYC[am];
  double a = d[axes[0]], b = d[axes[1]], c = d[axes[2]];
  double bc2 = b * b + c * c;
  double ell = a * a + bc2;
  double sq2 = sqrt(2.0);
  double sbc2 = sqrt(bc2);
  double r2l = sqrt(2.0 * ell / bc2);
  double tp[9] = {sqrt(2.0 * bc2), 0.0, 0.0,
                  -sq2 * a * b / sbc2, c * r2l, 0.0,
                  -sq2 * a * c / sbc2, -b * r2l, 0.0};
  double den[3] = {sqrt(2.0 * bc2), sqrt(2.0 * ell * bc2), sqrt(2.0 * ell)};
  double uh[9] = {0.0 / den[0], -c / den[0], b / den[0],
                  bc2 / den[1], -a * b / den[1], -a * c / den[1],
                  -a / den[2], -b / den[2], -c / den[2]};
  double m[9], gh[9];
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) {
      m[axes[i] * 3 + j] = tp[i * 3 + j];
      gh[i * 3 + axes[j]] = uh[i * 3 + j];
    }
  double om3[9];
  rqo_small_lq(m, 3, t22, om3);
  for (int i = 0; i < 3; i++)
    for (int j = 0; j < 3; j++) {
      double s = 0.0;
      for (int l = 0; l < 3; l++) s += om3[i * 3 + l] * gh[l * 3 + j];
      g[i * 3 + j] = sq2 * s;
    }
}

static void factor_all(rqo_body *b) {
  int64_t nn = b->nn;
  /* omega storage: at most 81 per internal node */
  int64_t total = 0;
  for (int64_t id = 0; id < nn; id++) {
    if (b->left[id] < 0) { b->omega_off[id] = -1; b->omega_k[id] = 0; continue; }
    int64_t l = b->left[id], r = b->right[id];
    int64_t nl = b->stop[l] - b->start[l], nr = b->stop[r] - b->start[r];
    int k = (nl == 1 && nr == 1) ? 3 : ((nl == 1 || nr == 1) ? 6 : 9);
    b->omega_off[id] = total; b->omega_k[id] = k;
    total += (int64_t)k * k;
  }
  b->omega = (double *)xcalloc(total, sizeof(double));
  for (int64_t id = 0; id < nn; id++) { /* factor.py:217-243, postorder */
    double *t22 = &b->t22[id * 9];
    if (b->left[id] < 0) { /* factor_leaf, factor.py:122-123 */
      b->fcase[id] = RQO_LEAF; b->fn[id] = 1; b->fnx[id] = 0; b->fny[id] = 0;
      memset(t22, 0, 9 * sizeof(double));
      continue;
    }
    int64_t l = b->left[id], r = b->right[id];
    int64_t nl = b->stop[l] - b->start[l], nr = b->stop[r] - b->start[r];
    const double *cp = &b->centroid[id * 3];
    double *om = &b->omega[b->omega_off[id]];
    b->fn[id] = nl + nr;
    if (nl == 1 && nr == 1) {
      double d[3];
      for (int a = 0; a < 3; a++) d[a] = b->pos[b->start[l] * 3 + a] - cp[a];
      factor_bead_bead(d, t22, om);
      b->fcase[id] = RQO_BEAD_BEAD; b->fnx[id] = 1; b->fny[id] = 1;
    } else if (nl == 1 || nr == 1) { /* factor_rigid_bead, factor.py:171-178 */
      int sw = (nl == 1);
      int64_t rig = sw ? r : l;
      int64_t nx = sw ? nr : nl;
      int64_t n = nx + 1;
      double dr[3], R[9];
      for (int a = 0; a < 3; a++) dr[a] = b->centroid[rig * 3 + a] - cp[a];
      skew(dr, R);
      double sc = sqrt((double)(nx * n));
      double cpl[18];
      for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
          cpl[i * 6 + j] = b->t22[rig * 9 + i * 3 + j];
          cpl[i * 6 + 3 + j] = sc * R[i * 3 + j];
        }
      rqo_small_lq(cpl, 6, t22, om);
      b->fcase[id] = RQO_RIGID_BEAD; b->fnx[id] = nx; b->fny[id] = 1; b->swapped[id] = (uint8_t)sw;
    } else { /* factor_general, factor.py:181-188 */
      int64_t n = nl + nr;
      double dr[3], R[9];
      for (int a = 0; a < 3; a++) dr[a] = b->centroid[l * 3 + a] - cp[a];
      skew(dr, R);
      double sc = sqrt((double)(nl * n) / (double)nr);
      double cpl[27];
      for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
          cpl[i * 9 + j] = b->t22[l * 9 + i * 3 + j];
          cpl[i * 9 + 3 + j] = b->t22[r * 9 + i * 3 + j];
          cpl[i * 9 + 6 + j] = sc * R[i * 3 + j];
        }
      rqo_small_lq(cpl, 9, t22, om);
      b->fcase[id] = RQO_GENERAL; b->fnx[id] = nl; b->fny[id] = nr;
    }
  }
  /* FactorTable residue offsets, factor.py:195-204 */
  int64_t pos = b->n >= 2 ? 6 : 3;
  for (int64_t id = 0; id < nn; id++) {
    b->res_offsets[id] = pos;
    int c = b->fcase[id];
    pos += (c == RQO_RIGID_BEAD) ? 3 : (c == RQO_GENERAL ? 6 : 0);
  }
  b->total_rows = pos;
}

void rqo_body_free(rqo_body *b) {
  free(b->perm); free(b->pos); free(b->start); free(b->stop); free(b->left); free(b->right);
  free(b->split_axis); free(b->depth); free(b->centroid); free(b->box);
  free(b->fcase); free(b->fn); free(b->fnx); free(b->fny); free(b->swapped); free(b->t22);
  free(b->omega_off); free(b->omega_k); free(b->omega); free(b->res_offsets);
  memset(b, 0, sizeof(*b));
}

int rqo_body_setup(const double *pos, int64_t n, int max_depth, rqo_body *b) {
  memset(b, 0, sizeof(*b));
  if (n < 1) return RQO_ERR_VALUE;
  int64_t nn = 2 * n - 1;
  b->n = n; b->nn = nn; b->root = nn - 1;
  b->perm = (int64_t *)xcalloc(n, sizeof(int64_t));
  b->pos = (double *)xcalloc(3 * n, sizeof(double));
  b->start = (int64_t *)xcalloc(nn, sizeof(int64_t));
  b->stop = (int64_t *)xcalloc(nn, sizeof(int64_t));
  b->left = (int64_t *)xcalloc(nn, sizeof(int64_t));
  b->right = (int64_t *)xcalloc(nn, sizeof(int64_t));
  b->split_axis = (int32_t *)xcalloc(nn, sizeof(int32_t));
  b->depth = (int32_t *)xcalloc(nn, sizeof(int32_t));
  b->centroid = (double *)xcalloc(3 * nn, sizeof(double));
  b->box = (double *)xcalloc(6 * nn, sizeof(double));
  b->fcase = (int32_t *)xcalloc(nn, sizeof(int32_t));
  b->fn = (int64_t *)xcalloc(nn, sizeof(int64_t));
  b->fnx = (int64_t *)xcalloc(nn, sizeof(int64_t));
  b->fny = (int64_t *)xcalloc(nn, sizeof(int64_t));
  b->swapped = (uint8_t *)xcalloc(nn, 1);
  b->t22 = (double *)xcalloc(9 * nn, sizeof(double));
  b->omega_off = (int64_t *)xcalloc(nn, sizeof(int64_t));
  b->omega_k = (int32_t *)xcalloc(nn, sizeof(int32_t));
  b->res_offsets = (int64_t *)xcalloc(nn, sizeof(int64_t));
  if (!b->perm || !b->res_offsets) { rqo_body_free(b); return RQO_ERR_NOMEM; }

  /* root cube, tree.py:78-81 */
  double lo[3], hi[3];
  for (int a = 0; a < 3; a++) { lo[a] = pos[a]; hi[a] = pos[a]; }
  for (int64_t i = 1; i < n; i++)
    for (int a = 0; a < 3; a++) {
      double x = pos[i * 3 + a];
      if (x < lo[a]) lo[a] = x;
      if (x > hi[a]) hi[a] = x;
    }
  double ext = 0.0;
  for (int a = 0; a < 3; a++) { double e = hi[a] - lo[a]; if (a == 0 || e > ext) ext = e; }
  double half = ext * (1.0 + 1e-9) / 2.0;
  double box[6];
  for (int a = 0; a < 3; a++) {
    double c = (lo[a] + hi[a]) / 2.0;
    box[a] = c - half; box[3 + a] = c + half;
  }
  int64_t *idx = (int64_t *)xcalloc(n, sizeof(int64_t));
  int64_t *scratch = (int64_t *)xcalloc(n, sizeof(int64_t));
  for (int64_t i = 0; i < n; i++) idx[i] = i;
  build_ctx c = {pos, b, 0, 0, max_depth, 0, scratch};
  build_rec(&c, idx, n, box, 0);
  free(idx); free(scratch);
  if (c.err) { rqo_body_free(b); return c.err; }
  for (int64_t i = 0; i < n; i++)
    for (int a = 0; a < 3; a++) b->pos[i * 3 + a] = pos[b->perm[i] * 3 + a];
  factor_all(b);
  return RQO_OK;
}

/* model.py:65-78 (cKDTree.query_pairs(tol) restated as a sorted sweep). */
static const double *g_sort_pos;
static int cmp_x(const void *a, const void *b) {
  double xa = g_sort_pos[*(const int64_t *)a * 3], xb = g_sort_pos[*(const int64_t *)b * 3];
  if (xa < xb) return -1;
  if (xa > xb) return 1;
  int64_t ia = *(const int64_t *)a, ib = *(const int64_t *)b;
  return (ia > ib) - (ia < ib);
}
int rqo_check_duplicates(const double *pos, int64_t n, int64_t *pi, int64_t *pj) {
  if (n < 2) return 0;
  double lo[3], hi[3];
  for (int a = 0; a < 3; a++) lo[a] = hi[a] = pos[a];
  for (int64_t i = 1; i < n; i++)
    for (int a = 0; a < 3; a++) {
      if (pos[i * 3 + a] < lo[a]) lo[a] = pos[i * 3 + a];
      if (pos[i * 3 + a] > hi[a]) hi[a] = pos[i * 3 + a];
    }
  double d0 = hi[0] - lo[0], d1 = hi[1] - lo[1], d2 = hi[2] - lo[2];
  double diag = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
  if (diag == 0.0) { *pi = 0; *pj = 1; return 1; }
  double tol = 1e-12 * diag;
  int64_t *ord = (int64_t *)xcalloc(n, sizeof(int64_t));
  for (int64_t i = 0; i < n; i++) ord[i] = i;
  g_sort_pos = pos;
  qsort(ord, n, sizeof(int64_t), cmp_x);
  int found = 0;
  int64_t bi = 0, bj = 0;
  for (int64_t s = 0; s < n; s++) {
    int64_t i = ord[s];
    for (int64_t t = s + 1; t < n; t++) {
      int64_t j = ord[t];
      double dx = pos[j * 3] - pos[i * 3];
      if (dx > tol) break;
      double dy = pos[j * 3 + 1] - pos[i * 3 + 1], dz = pos[j * 3 + 2] - pos[i * 3 + 2];
      if (sqrt(dx * dx + dy * dy + dz * dz) <= tol) {
        int64_t a = i < j ? i : j, b2 = i < j ? j : i;
        if (!found || a < bi || (a == bi && b2 < bj)) { bi = a; bj = b2; }
        found = 1;
      }
    }
  }
  free(ord);
  if (found) { *pi = bi; *pj = bj; }
  return found;
}

/* ------------------------------------------------------------------------ */
/* matfree (matfree.py:33-151)                                                */
/* ------------------------------------------------------------------------ */

/* y = omega @ x, omega k x k row-major, x/y: k rows of K columns (row stride K) */
static void matvec_k(const double *om, int k, const double *x, double *y, int64_t K) {
  for (int i = 0; i < k; i++)
    for (int64_t c = 0; c < K; c++) {
      double s = 0.0;
      for (int j = 0; j < k; j++) s += om[i * k + j] * x[j * K + c];
      y[i * K + c] = s;
    }
}
static void matvec_kT(const double *om, int k, const double *x, double *y, int64_t K) {
  for (int i = 0; i < k; i++)
    for (int64_t c = 0; c < K; c++) {
      double s = 0.0;
      for (int j = 0; j < k; j++) s += om[j * k + i] * x[j * K + c];
      y[i * K + c] = s;
    }
}

static void upward_ws(const rqo_body *b, const double *v, double *out, int64_t K, double *m);
void rqo_upward(const rqo_body *b, const double *v, double *out, int64_t K) {
  double *m = (double *)malloc((size_t)(b->nn * 6 * K + 1) * sizeof(double));
  upward_ws(b, v, out, K, m);
  free(m);
}
/* m: caller-provided workspace of nn*6*K doubles (reused across bodies). */
static void upward_ws(const rqo_body *b, const double *v, double *out, int64_t K, double *m) {
  int64_t n = b->n;
  if (n == 1) { memcpy(out, v, 3 * K * sizeof(double)); return; } /* matfree.py:99-100 */
  double x[9 * 64], y[9 * 64];
  double *xb = K <= 64 ? x : (double *)malloc(9 * K * sizeof(double));
  double *yb = K <= 64 ? y : (double *)malloc(9 * K * sizeof(double));
  for (int64_t id = 0; id < b->nn; id++) { /* matfree.py:106-119, postorder */
    double *mp = &m[id * 6 * K];
    if (b->left[id] < 0) {
      int64_t src = b->perm[b->start[id]];
      for (int r = 0; r < 3; r++)
        for (int64_t c = 0; c < K; c++) { mp[r * K + c] = v[(src * 3 + r) * K + c]; mp[(3 + r) * K + c] = 0.0; }
      continue;
    }
    int64_t xi = b->left[id], yi = b->right[id];
    if (b->swapped[id]) { int64_t t = xi; xi = yi; yi = t; }
    const double *mx = &m[xi * 6 * K], *my = &m[yi * 6 * K];
    double a = sqrt((double)b->fnx[id] / (double)b->fn[id]); /* NodeFactor.ratios */
    double bb = sqrt((double)b->fny[id] / (double)b->fn[id]);
    int c = b->fcase[id];
    int k = b->omega_k[id];
    const double *om = &b->omega[b->omega_off[id]];
    /* merge_infosets, matfree.py:41-62 */
    double *t = xb + (k - 3) * K;
    for (int r = 0; r < 3; r++)
      for (int64_t q = 0; q < K; q++) {
        t[r * K + q] = bb * mx[r * K + q] - a * my[r * K + q];
        mp[r * K + q] = a * mx[r * K + q] + bb * my[r * K + q];
      }
    if (c == RQO_BEAD_BEAD) {
      matvec_k(om, 3, xb, yb, K);
      for (int64_t q = 0; q < 3 * K; q++) mp[3 * K + q] = yb[q];
      continue;
    }
    memcpy(xb, mx + 3 * K, 3 * K * sizeof(double));
    if (c == RQO_GENERAL) memcpy(xb + 3 * K, my + 3 * K, 3 * K * sizeof(double));
    matvec_k(om, k, xb, yb, K);
    for (int64_t q = 0; q < 3 * K; q++) mp[3 * K + q] = yb[q];
    int64_t off = b->res_offsets[id];
    memcpy(&out[off * K], yb + 3 * K, (size_t)(k - 3) * K * sizeof(double));
  }
  memcpy(out, &m[b->root * 6 * K], 6 * K * sizeof(double));
  if (xb != x) free(xb);
  if (yb != y) free(yb);
}

static void downward_ws(const rqo_body *b, const double *w, double *out, int64_t K, double *l);
void rqo_downward(const rqo_body *b, const double *w, double *out, int64_t K) {
  double *l = (double *)malloc((size_t)(b->nn * 6 * K + 1) * sizeof(double));
  downward_ws(b, w, out, K, l);
  free(l);
}
static void downward_ws(const rqo_body *b, const double *w, double *out, int64_t K, double *l) {
  int64_t n = b->n;
  if (n == 1) { memcpy(out, w, 3 * K * sizeof(double)); return; } /* matfree.py:127-128 */
  double x[9 * 64], u[9 * 64];
  double *xb = K <= 64 ? x : (double *)malloc(9 * K * sizeof(double));
  double *ub = K <= 64 ? u : (double *)malloc(9 * K * sizeof(double));
  memcpy(&l[b->root * 6 * K], w, 6 * K * sizeof(double));
  for (int64_t id = b->nn - 1; id >= 0; id--) { /* matfree.py:135-147 */
    double *lp = &l[id * 6 * K];
    if (b->left[id] < 0) {
      int64_t dst = b->perm[b->start[id]];
      for (int r = 0; r < 3; r++)
        for (int64_t c = 0; c < K; c++) out[(dst * 3 + r) * K + c] = lp[r * K + c];
      continue;
    }
    int64_t xi = b->left[id], yi = b->right[id];
    if (b->swapped[id]) { int64_t t = xi; xi = yi; yi = t; }
    double *lx = &l[xi * 6 * K], *ly = &l[yi * 6 * K];
    double a = sqrt((double)b->fnx[id] / (double)b->fn[id]);
    double bb = sqrt((double)b->fny[id] / (double)b->fn[id]);
    int c = b->fcase[id];
    int k = b->omega_k[id];
    const double *om = &b->omega[b->omega_off[id]];
    /* split_rvset, matfree.py:65-83 */
    memcpy(xb, lp + 3 * K, 3 * K * sizeof(double));
    if (k > 3) memcpy(xb + 3 * K, &w[b->res_offsets[id] * K], (size_t)(k - 3) * K * sizeof(double));
    matvec_kT(om, k, xb, ub, K);
    const double *tau = ub + (k - 3) * K;
    for (int r = 0; r < 3; r++)
      for (int64_t q = 0; q < K; q++) {
        double lpq = lp[r * K + q], tq = tau[r * K + q];
        lx[r * K + q] = a * lpq + bb * tq;
        ly[r * K + q] = bb * lpq - a * tq;
        lx[(3 + r) * K + q] = (c == RQO_BEAD_BEAD) ? 0.0 : ub[r * K + q];
        ly[(3 + r) * K + q] = (c == RQO_GENERAL) ? ub[(3 + r) * K + q] : 0.0;
      }
  }
  if (xb != x) free(xb);
  if (ub != u) free(ub);
}

/* ------------------------------------------------------------------------ */
/* batched front end (matfree.py:212-247) and Z reductions (model.py:129-149) */
/* ------------------------------------------------------------------------ */

int rqo_batch_setup(const double *pos, const int64_t *offsets, int64_t m,
                    int max_depth, int nthreads, rqo_batch *out) {
  out->m = m;
  out->offsets = (int64_t *)xcalloc(m + 1, sizeof(int64_t));
  memcpy(out->offsets, offsets, (m + 1) * sizeof(int64_t));
  out->bodies = (rqo_body *)xcalloc(m, sizeof(rqo_body));
  int err = 0;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads) reduction(| : err)
#endif
  for (int64_t j = 0; j < m; j++) {
    int e = rqo_body_setup(pos + 3 * offsets[j], offsets[j + 1] - offsets[j], max_depth, &out->bodies[j]);
    err |= e;
  }
  (void)nthreads;
  return err;
}

void rqo_batch_free(rqo_batch *b) {
  for (int64_t j = 0; j < b->m; j++) rqo_body_free(&b->bodies[j]);
  free(b->bodies); free(b->offsets);
  memset(b, 0, sizeof(*b));
}

int rqo_batch_apply(const rqo_batch *b, int op, const double *in, double *out,
                    int64_t K, int nthreads) {
  if (op >= 2)
    for (int64_t j = 0; j < b->m; j++)
      if (b->bodies[j].n < 2) return RQO_ERR_TOO_SMALL;
  int64_t nmax = 1;
  for (int64_t j = 0; j < b->m; j++) if (b->bodies[j].n > nmax) nmax = b->bodies[j].n;
#ifdef _OPENMP
#pragma omp parallel num_threads(nthreads)
#endif
  {
    /* per-thread workspaces reused across bodies (no per-body page faults) */
    double *ws = (double *)malloc((size_t)(2 * nmax * 6 * K + 1) * sizeof(double));
    double *tmp = (double *)malloc((size_t)(3 * nmax * K + 1) * sizeof(double));
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
    for (int64_t j = 0; j < b->m; j++) {
      const rqo_body *bd = &b->bodies[j];
      int64_t n = bd->n, o = b->offsets[j];
      int64_t full = 3 * o, comp = 3 * o - 6 * j;
      if (op == 0) upward_ws(bd, in + full * K, out + full * K, K, ws);
      else if (op == 1) downward_ws(bd, in + full * K, out + full * K, K, ws);
      else if (op == 2) {
        upward_ws(bd, in + full * K, tmp, K, ws);
        memcpy(out + comp * K, tmp + 6 * K, (3 * n - 6) * K * sizeof(double));
      } else {
        memset(tmp, 0, 6 * K * sizeof(double));
        memcpy(tmp + 6 * K, in + comp * K, (3 * n - 6) * K * sizeof(double));
        downward_ws(bd, tmp, out + full * K, K, ws);
      }
    }
    free(ws);
    free(tmp);
  }
  (void)nthreads;
  return RQO_OK;
}

static void body_centroid(const double *p, int64_t n, double c[3]) {
  /* BeadModel.centroid = positions.mean(axis=0), model.py:56-61 */
  double s[3] = {0, 0, 0};
  for (int64_t i = 0; i < n; i++)
    for (int a = 0; a < 3; a++) s[a] += p[i * 3 + a];
  for (int a = 0; a < 3; a++) c[a] = s[a] / (double)n;
}

void rqo_batch_zf(const double *pos, const int64_t *offsets, int64_t m,
                  const double *f, double *out, int nthreads) {
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads)
#endif
  for (int64_t j = 0; j < m; j++) {
    int64_t o = offsets[j], n = offsets[j + 1] - o;
    const double *p = pos + 3 * o, *fj = f + 3 * o;
    double c[3];
    body_centroid(p, n, c);
    double acc[6] = {0, 0, 0, 0, 0, 0};
    for (int64_t i = 0; i < n; i++) {
      double x = p[i * 3] - c[0], y = p[i * 3 + 1] - c[1], z = p[i * 3 + 2] - c[2];
      double fx = fj[i * 3], fy = fj[i * 3 + 1], fz = fj[i * 3 + 2];
      acc[0] += fx; acc[1] += fy; acc[2] += fz;
      acc[3] += -z * fy + y * fz;
      acc[4] += z * fx - x * fz;
      acc[5] += -y * fx + x * fy;
    }
    memcpy(out + 6 * j, acc, sizeof(acc));
  }
  (void)nthreads;
}

void rqo_batch_ztu(const double *pos, const int64_t *offsets, int64_t m,
                   const double *u, double *out, int nthreads) {
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads)
#endif
  for (int64_t j = 0; j < m; j++) {
    int64_t o = offsets[j], n = offsets[j + 1] - o;
    const double *p = pos + 3 * o;
    const double *uj = u + 6 * j;
    double c[3];
    body_centroid(p, n, c);
    for (int64_t i = 0; i < n; i++) {
      double x = p[i * 3] - c[0], y = p[i * 3 + 1] - c[1], z = p[i * 3 + 2] - c[2];
      double *o3 = out + 3 * (o + i);
      o3[0] = uj[0] + z * uj[4] - y * uj[5];
      o3[1] = uj[1] - z * uj[3] + x * uj[5];
      o3[2] = uj[2] + y * uj[3] - x * uj[4];
    }
  }
  (void)nthreads;
}
