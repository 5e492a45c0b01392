/*
 * rigidq_b200.h -- C ABI of the B200-native hierarchical orthogonal-complement
 * operators (arxiv 1708.08427), the drop-in boundary under the Python mirror
 * of the reference package `rigidq` (paper_1708_08427_b200/).
 *
 * The reference has no FFI: its boundary is the Python API of
 * /root/reference/pkg/src/rigidq.  Each entry point below names the reference
 * function(s) it replaces (file:line, relative to that directory).
 *
 * Conventions
 *  - plain pointers and sizes; fp64 everywhere; int64 counts.
 *  - vectors are (len, k) row-major (numpy C order of a (len,) or (len, k)
 *    array), bodies concatenated in body order, beads in ORIGINAL order at
 *    the boundary (matfree.py:86-92, 102, 149).
 *  - "device" pointers are CUDA device (or managed) memory on the plan's
 *    device; `stream` is a cudaStream_t (NULL = legacy default stream).
 *  - every call returns RQ_OK or an error code; rq_last_error() gives the
 *    message of the last failure on the calling thread.  Error codes map
 *    one-to-one onto the reference exception classes (errors.py:4-33).
 *  - a plan (tree + factors + apply layout) is immutable after rq_setup;
 *    concurrent rq_apply calls on distinct streams are safe (matfree.py:16-17).
 *    Each stream a plan is used on gets its own exchange state on first use, kept
 *    until rq_plan_release_stream or rq_plan_free: 48 B per tile root + 4 B per top
 *    node, plus (k > 1 column loop) two k-column staging blocks and (Zf) 48 B per
 *    segment and column.
 *  - every entry point runs on the plan's device and restores the caller's
 *    current device before returning.
 */
#ifndef RIGIDQ_B200_H
#define RIGIDQ_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RQ_OK 0
#define RQ_ERR_DUPLICATE 1      /* DuplicateBeadsError   (errors.py:8)  */
#define RQ_ERR_VALUE 2          /* ValueError                           */
#define RQ_ERR_BODY_TOO_SMALL 3 /* BodyTooSmallError     (errors.py:16) */
#define RQ_ERR_LENGTH 4         /* LengthMismatchError   (errors.py:24) */
#define RQ_ERR_TOO_SMALL 5      /* TooSmallError         (errors.py:12) */
#define RQ_ERR_SIZE_GUARD 6     /* SizeGuardError        (errors.py:20) */
#define RQ_ERR_CUDA 7           /* RuntimeError (CUDA failure / no device) */
#define RQ_ERR_NOMEM 8          /* MemoryError                          */

/* operator codes, matfree.py:209 (_OP_NAMES) */
#define RQ_OP_QV 0        /* upward_apply            matfree.py:95  */
#define RQ_OP_QTV 1       /* downward_apply          matfree.py:124 */
#define RQ_OP_QTILDE_V 2  /* qtilde_apply            matfree.py:154 */
#define RQ_OP_QTILDE_TV 3 /* qtilde_transpose_apply  matfree.py:161 */

/* Z reductions (model.py:129-149 + the caller's dense Z @ f / Z.T @ u) */
#define RQ_Z_F 0  /* f (3N x k) -> Zf (6m x k) */
#define RQ_Z_TU 1 /* u (6m x k) -> Z^T u (3N x k) */

/* rq_setup flags */
#define RQ_SETUP_HOST_INPUT 1u   /* positions pointer is host memory */
#define RQ_SETUP_CHECK_DUPS 2u   /* also run the model.py:65-78 duplicate check */

typedef struct rq_plan rq_plan;

typedef struct rq_plan_info {
  int64_t m;               /* bodies */
  int64_t n_beads;         /* total beads */
  int64_t n_nodes;         /* total nodes (sum 2n_j - 1) */
  int64_t n_streams;       /* wavefront streams = persistent sweep CTAs */
  int64_t n_steps;         /* barrier steps over all streams */
  int64_t n_top;           /* nodes above the tiles */
  int64_t tile_leaves;     /* tile size limit S */
  int64_t n_tiles;         /* tiles with >= 2 beads */
  int64_t blob_bytes;      /* wave blob (records + both sweeps' metadata and gather lists) */
  int64_t sweep_bytes[2];  /* blob bytes one upward / downward sweep streams */
  int64_t record_doubles;  /* compact factor records */
  int64_t full_len;        /* 3N            */
  int64_t comp_len;        /* 3N - 6m       */
  int64_t n_case[4];       /* node counts per case (leaf, BB, RB, GEN) */
  int64_t device_bytes;    /* device memory held by the plan */
  int64_t rounds;          /* tile rounds (all streams work inside one round at a time) */
  int64_t node_slots;      /* node 6-vector slots per sweep CTA (shared memory) */
  int64_t stage_bytes;     /* shared-memory stage of one step block */
  int64_t sweep_smem;      /* dynamic shared memory per sweep CTA */
  int64_t sweep_ctas_per_sm; /* resident sweep CTAs per SM */
  int64_t top_staged;      /* bodies whose top tree is staged in shared memory */
  int64_t top_global;      /* bodies whose top tree is swept from global memory */
  int64_t mrhs_min_k;      /* k at and above which the column-parallel (multi-RHS) kernels run */
  int64_t mrhs_units[2];   /* multi-RHS unit programs: tiles, top trees (0 until the first k >= mrhs_min_k apply) */
  int64_t mrhs_bytes[2];   /* program bytes read per column group: tile units, top units */
} rq_plan_info;

/* Last error message of the calling thread ("" if none). */
const char *rq_last_error(void);
/* Number of CUDA devices visible (0 without a GPU; never fails). */
int rq_device_count(void);
/* ABI version (major*100 + minor). */
int rq_version(void);

/*
 * Per-body setup for a batch of m bodies: tree + factors + apply layout.
 * Replaces BodyOperator.__init__ / MultiBodyOperator.__init__
 * (matfree.py:177-180, 219-221), i.e. build_tree (tree.py:73-134) followed
 * by factor_all (factor.py:213-244) for every body.
 *   positions : (N, 3) row-major, bodies concatenated (device memory unless
 *               RQ_SETUP_HOST_INPUT)
 *   offsets   : HOST int64[m+1], offsets[0] = 0, offsets[m] = N (the
 *               MultiBodyModel.offsets of model.py:98)
 *   max_depth : split depth guard (tree.py:29, default 96)
 * Errors: RQ_ERR_VALUE (bad shape/non-finite), RQ_ERR_DUPLICATE (tree.py:99-103,
 * or model.py:65-78 with RQ_SETUP_CHECK_DUPS).
 */
int rq_setup(const double *positions, const int64_t *offsets, int64_t m, int max_depth,
             uint32_t flags, void *stream, rq_plan **out);
int rq_plan_free(rq_plan *plan);
int rq_plan_get_info(const rq_plan *plan, rq_plan_info *info);
/* Device ordinal the plan lives on. */
int rq_plan_device(const rq_plan *plan);
/* Drop the per-stream exchange state the plan holds for `stream` (after synchronising it),
 * e.g. before a caller destroys a stream it applied the plan on; the next application on
 * that stream allocates it again.  No reference counterpart (resource management). */
int rq_plan_release_stream(const rq_plan *plan, void *stream);

/*
 * Operator application on device buffers (replaces upward_apply /
 * downward_apply / qtilde_apply / qtilde_transpose_apply, matfree.py:95-170,
 * and MultiBodyOperator.apply, matfree.py:235-247).
 *   in  : (in_len, k) row-major device buffer
 *   out : (out_len, k) row-major device buffer (fully overwritten)
 * Lengths: QV/QTV 3N -> 3N; QTILDE_V 3N -> 3N-6m; QTILDE_TV 3N-6m -> 3N.
 * Errors: RQ_ERR_BODY_TOO_SMALL for Q~ ops when a body has n < 2
 * (matfree.py:157,165,229); RQ_ERR_VALUE for an unknown op (matfree.py:236).
 */
int rq_apply(const rq_plan *plan, int op, const double *in, double *out, int64_t k,
             void *stream);
/* Phase-selective variant for profiling (bench.py times the tile sweep
 * alone): phases is a mask of RQ_PHASE_*; rq_apply == all phases. */
#define RQ_PHASE_SWEEP 1u   /* k_wave: the tiles */
#define RQ_PHASE_TOP 2u     /* k_top2 / k_top_df: the top trees */
#define RQ_PHASE_LAYOUT 4u  /* Q / Q^T: root rows <-> private residue layout */
int rq_apply_ex(const rq_plan *plan, int op, const double *in, double *out, int64_t k,
                void *stream, uint32_t phases);
/* Number of kernel launches one rq_apply issues. */
int rq_launches_per_apply(const rq_plan *plan, int op, int64_t k);
/* Same on HOST buffers (pinned or pageable): H2D copy, apply, D2H copy; returns when
 * `out` holds the result (the numpy path of the reference API, matfree.py:86-92). */
int rq_apply_host(const rq_plan *plan, int op, const double *in, double *out, int64_t k);
/* Asynchronous form: returns once the copies and kernels are queued on the plan's own
 * streams (two staging slots), so the H2D of the next application overlaps the D2H of
 * this one.  `in` and `out` must stay valid until rq_host_wait (pageable results are
 * delivered by it; a third application implicitly completes the first). */
int rq_apply_host_async(const rq_plan *plan, int op, const double *in, double *out, int64_t k);
int rq_host_wait(const rq_plan *plan);

/*
 * Force/torque reductions about each body's centroid (or `origin`, host
 * double[3m] or NULL): assemble_z (model.py:129-149) contracted on the fly.
 *   RQ_Z_F : f (3N, k) -> (6m, k) = [sum f ; sum (r - c) x f] per body
 *   RQ_Z_TU: u (6m, k) -> (3N, k) = V + w x (r - c) per bead
 */
int rq_z_apply(const rq_plan *plan, int op, const double *in, double *out, int64_t k,
               const double *origin, void *stream);
int rq_z_apply_host(const rq_plan *plan, int op, const double *in, double *out, int64_t k,
                    const double *origin);
/* Model centroids (BeadModel.centroid, model.py:56-61) -> host double[3m]. */
int rq_body_centroids(const rq_plan *plan, double *out);

/*
 * Duplicate-bead check of BeadModel (model.py:65-78): beads closer than
 * 1e-12 * bbox diagonal.  On a hit returns RQ_ERR_DUPLICATE and the first
 * body and the lexicographically smallest pair (i, j) of it (body-local).
 */
int rq_check_duplicates(const double *positions, const int64_t *offsets, int64_t m,
                        uint32_t flags, void *stream, int64_t *body, int64_t *i,
                        int64_t *j, double *tol);

/*
 * Parity exports of one body (host arrays, body-local ids, postorder).
 * Tree (tree.py:32-70): perm[n]; start, stop, left, right[nn] (-1 = none);
 * split_axis (-1 leaf), depth[nn]; centroid[3nn]; box[6nn] (lo xyz, hi xyz).
 */
int rq_export_tree(const rq_plan *plan, int64_t body, int64_t *perm, int64_t *start,
                   int64_t *stop, int64_t *left, int64_t *right, int32_t *split_axis,
                   int32_t *depth, double *centroid, double *box);
/* Factor table (factor.py:60-87, 191-210): case (0 leaf, 1 BB, 2 RB, 3 GEN),
 * n, n_x, n_y, swapped, t22[9nn], omega packed k*k per internal node in
 * postorder (k = 3, 6, 9), res_offsets[nn], total_rows. omega may be NULL. */
int rq_export_factors(const rq_plan *plan, int64_t body, int32_t *ncase, int64_t *n,
                      int64_t *nx, int64_t *ny, uint8_t *swapped, double *t22,
                      double *omega, int64_t *res_offsets, int64_t *total_rows);
/* Number of doubles rq_export_factors writes to omega for `body`. */
int64_t rq_omega_size(const rq_plan *plan, int64_t body);

/*
 * Explicit hierarchical Q (Algorithm 1; generate_explicit_q, factor.py:362-390):
 * root_rows (6 x 3n, tree-order columns) and the residue blocks in postorder
 * emission order: block_node[b], block_col[b] (= 3*start), block_rows[b], and
 * block_data (rows x 3*n_node each, concatenated).  Query sizes with
 * rq_explicit_q_size.  Errors: RQ_ERR_TOO_SMALL for n < 2 (factor.py:368-369).
 */
int rq_explicit_q_size(const rq_plan *plan, int64_t body, int64_t *n_blocks,
                       int64_t *n_doubles);
int rq_explicit_q(const rq_plan *plan, int64_t body, double *root_rows, int64_t *block_node,
                  int64_t *block_col, int64_t *block_rows, double *block_data);

/*
 * Single-node primitives (HOST buffers), same device code as the batched path.
 *  rq_small_lq          small_lq (factor.py:90-109): batch of row-major 3 x k
 *                       (k = 3, 6, 9) -> t (3x3) and explicit omega (k x k)
 *  rq_factor_bead_bead  factor_bead_bead (factor.py:130-168): batch of offsets
 *                       d[3] -> t22 (3x3), g (3x3)
 *  rq_node_merge        merge_infosets (matfree.py:41-62) with an explicit
 *                       k x k omega: m_x, m_y (6 x k cols) -> m_p (6 x k),
 *                       res ((kk-3) x k)
 *  rq_node_split        split_rvset (matfree.py:65-83): l_p (6 x k),
 *                       res ((kk-3) x k) -> l_x, l_y (6 x k)
 * ncase: 1 BEAD_BEAD, 2 RIGID_BEAD, 3 GENERAL; a, b = NodeFactor.ratios.
 */
int rq_small_lq(const double *a, int k, int64_t batch, double *t, double *omega);
int rq_factor_bead_bead(const double *offset, int64_t batch, double *t22, double *g);
int rq_node_merge(int ncase, const double *omega, double a, double b, const double *mx, const double *my,
                  int64_t k, double *mp, double *res);
int rq_node_split(int ncase, const double *omega, double a, double b, const double *lp, const double *res,
                  int64_t k, double *lx, double *ly);

#ifdef __cplusplus
}
#endif
#endif /* RIGIDQ_B200_H */
