/* c_abi_check.c -- a plain C host (no Python, no torch) driving librigidq_b200.so through
 * include/rigidq_b200.h, as a non-Python binding of the reference API would: setup of a
 * batch of bodies from host positions, Q~v / Q~^T g / Zf on host buffers, errors through
 * rq_last_error.  Results are checked against the CPU oracle (test infrastructure,
 * oracle/rq_oracle.c) to the north-star tolerance of 1e-12 relative per body.
 *
 * Build (tests/c_abi/Makefile): gcc ... -lrigidq_b200 oracle/rq_oracle.c
 * Run on a GPU box: tests/c_abi/c_abi_check   (exit status 0 = pass)
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "rigidq_b200.h"
#include "rq_oracle.h"

static uint64_t lcg = 12345;
static double urand(void) {  /* uniform [0, 1) */
  lcg = lcg * 6364136223846793005ULL + 1442695040888963407ULL;
  return (double)(lcg >> 11) * (1.0 / 9007199254740992.0);
}

static double body_rel(const double *a, const double *b, int64_t n) {
  double d = 0, r = 0;
  for (int64_t i = 0; i < n; i++) {
    d += (a[i] - b[i]) * (a[i] - b[i]);
    r += b[i] * b[i];
  }
  return r > 0 ? sqrt(d / r) : sqrt(d);
}

int main(void) {
  if (rq_device_count() < 1) {
    fprintf(stderr, "no CUDA device: %s\n", rq_last_error());
    return 2;
  }
  const int64_t m = 6;
  const int64_t counts[6] = {4096, 3, 700, 129, 20000, 1000};
  int64_t off[7] = {0};
  for (int64_t j = 0; j < m; j++) off[j + 1] = off[j] + counts[j];
  const int64_t N = off[m];
  double *pos = malloc(sizeof(double) * 3 * N);
  for (int64_t j = 0; j < m; j++) {  /* ellipsoid shells, centroid-shifted */
    const double ax = 0.5 + 1.5 * urand(), ay = 0.5 + 1.5 * urand(), az = 0.5 + 1.5 * urand();
    double c[3] = {0, 0, 0};
    for (int64_t i = off[j]; i < off[j + 1]; i++) {
      const double th = M_PI * urand(), ph = 2 * M_PI * urand();
      pos[3 * i] = ax * sin(th) * cos(ph);
      pos[3 * i + 1] = ay * sin(th) * sin(ph);
      pos[3 * i + 2] = az * cos(th);
      for (int a = 0; a < 3; a++) c[a] += pos[3 * i + a];
    }
    for (int64_t i = off[j]; i < off[j + 1]; i++)
      for (int a = 0; a < 3; a++) pos[3 * i + a] -= c[a] / (double)counts[j];
  }
  rq_plan *plan = NULL;
  if (rq_setup(pos, off, m, 96, RQ_SETUP_HOST_INPUT | RQ_SETUP_CHECK_DUPS, NULL, &plan) != RQ_OK) {
    fprintf(stderr, "rq_setup: %s\n", rq_last_error());
    return 1;
  }
  rqo_batch ref;
  if (rqo_batch_setup(pos, off, m, 96, 4, &ref) != 0) {
    fprintf(stderr, "oracle setup failed\n");
    return 1;
  }
  const int64_t nf = 3 * N, nc = 3 * N - 6 * m;
  double *v = malloc(sizeof(double) * nf), *g = malloc(sizeof(double) * nc);
  double *o1 = malloc(sizeof(double) * nf), *o2 = malloc(sizeof(double) * nf);
  for (int64_t i = 0; i < nf; i++) v[i] = urand() - 0.5;
  for (int64_t i = 0; i < nc; i++) g[i] = urand() - 0.5;
  double worst = 0;
  /* Q~v: per-body blocks of 3n - 6 rows */
  if (rq_apply_host(plan, RQ_OP_QTILDE_V, v, o1, 1) != RQ_OK) { fprintf(stderr, "%s\n", rq_last_error()); return 1; }
  rqo_batch_apply(&ref, RQ_OP_QTILDE_V, v, o2, 1, 4);
  for (int64_t j = 0, r = 0; j < m; r += 3 * counts[j] - 6, j++) {
    const double e = body_rel(o1 + r, o2 + r, 3 * counts[j] - 6);
    worst = e > worst ? e : worst;
  }
  /* Q~^T g: per-body blocks of 3n rows */
  if (rq_apply_host(plan, RQ_OP_QTILDE_TV, g, o1, 1) != RQ_OK) { fprintf(stderr, "%s\n", rq_last_error()); return 1; }
  rqo_batch_apply(&ref, RQ_OP_QTILDE_TV, g, o2, 1, 4);
  for (int64_t j = 0; j < m; j++) {
    const double e = body_rel(o1 + 3 * off[j], o2 + 3 * off[j], 3 * counts[j]);
    worst = e > worst ? e : worst;
  }
  /* Zf about each body's centroid: 6 per body */
  if (rq_z_apply_host(plan, RQ_Z_F, v, o1, 1, NULL) != RQ_OK) { fprintf(stderr, "%s\n", rq_last_error()); return 1; }
  rqo_batch_zf(pos, off, m, v, o2, 4);
  double zerr = body_rel(o1, o2, 6 * m);
  /* error path: an unknown op comes back as RQ_ERR_VALUE with a message */
  const int bad = rq_apply_host(plan, 7, v, o1, 1);
  printf("c_abi_check: %lld beads in %lld bodies, worst per-body rel err Q~v/Q~^T g %.2e, Zf %.2e; "
         "bad op -> %d (%s)\n", (long long)N, (long long)m, worst, zerr, bad, rq_last_error());
  rq_plan_free(plan);
  rqo_batch_free(&ref);
  free(pos); free(v); free(g); free(o1); free(o2);
  return (worst < 1e-12 && zerr < 1e-12 && bad == RQ_ERR_VALUE) ? 0 : 1;
}
