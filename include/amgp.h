/*
 * amgp.h -- C ABI of the B200-native polynomial-smoother / AMG V-cycle / PCG
 * library (libamgp.so, sm_100a).
 *
 * Every entry point replaces one function of the reference package
 * (/root/reference/pkg/src/amgpoly, cited file:line below) on the hot path
 * named by BASELINE.json's north_star.  Plain pointers and sizes only:
 *   - "host" arrays are ordinary CPU memory,
 *   - "device" arrays are CUDA device pointers on the context's device
 *     (e.g. torch.Tensor.data_ptr()).
 * All work is enqueued on the context's stream; functions that return data
 * to the host synchronise that stream.
 *
 * Return value: AMGP_OK (0) or a negative status; amgp_last_error() gives the
 * thread-local message.  The Python shim maps AMGP_EINVAL to ValueError (the
 * reference's convention, e.g. sparse.py:121-122, smoothers.py:100-101) and
 * the others to RuntimeError.
 */
#ifndef AMGP_H
#define AMGP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AMGP_OK 0
#define AMGP_EINVAL (-1) /* dimension mismatch / invalid configuration */
#define AMGP_ECUDA (-2)  /* CUDA runtime error */
#define AMGP_ENOMEM (-3) /* device allocation failed */
#define AMGP_ENCCL (-4)  /* NCCL error */

/* smoothers.py:28 FAMILIES */
enum { AMGP_L1_JACOBI = 0, AMGP_CHEB4 = 1, AMGP_OPT_CHEB4 = 2, AMGP_OPT_CHEB1 = 3 };

/* krylov.py:15-26 KrylovConfig.variant; AMGP_PCG1 = single-reduction PCG
 * (Chronopoulos-Gear; one global reduction per iteration) */
enum { AMGP_PCG = 0, AMGP_FCG = 1, AMGP_PCG1 = 2 };

/* amg.py:65 AmgHierarchy.coarse_solver; AMGP_COARSE_SMOOTHER applies the
 * coarsest level's own smoother from a zero guess, which turns a one-level
 * hierarchy into smoothers.py:193-199 as_preconditioner. */
enum { AMGP_COARSE_L1_JACOBI = 0, AMGP_COARSE_DENSE_DIRECT = 1, AMGP_COARSE_SMOOTHER = 2 };

typedef struct amgp_ctx amgp_ctx;   /* device + stream (+ optional NCCL communicator) */
typedef struct amgp_mat amgp_mat;   /* device matrix in SELL-32 layout */
typedef struct amgp_hier amgp_hier; /* device AMG hierarchy */

/* smoothers.py:52-85 PolySmootherConfig after __post_init__ resolution. */
typedef struct {
    int32_t family;      /* AMGP_* family */
    int32_t degree;      /* k >= 1 */
    double a;            /* opt_cheb1 interval end, 0 < a < 1 */
    double rho_scale;    /* > 0; 1 for l1-Jacobi */
    const double *beta;  /* host, `degree` entries (opt_cheb4 only; else NULL) */
} amgp_smoother_cfg;

/* krylov.py:29-38 SolveReport */
typedef struct {
    int32_t iterations;
    int32_t converged;
    int32_t breakdown;
    int32_t spmv_count;
    int32_t precond_count;
    int32_t n_history;
    double final_relres;
    double elapsed_s;
} amgp_solve_report;

const char *amgp_last_error(void);
int amgp_version(void);

/* ---- context ----------------------------------------------------------- */
/* stream: a cudaStream_t (NULL = create a private non-blocking stream). */
int amgp_ctx_create(int device, void *stream, amgp_ctx **out);
int amgp_ctx_destroy(amgp_ctx *ctx);
int amgp_ctx_set_stream(amgp_ctx *ctx, void *stream);
int amgp_ctx_sync(amgp_ctx *ctx);
/* number of kernels this context has launched (graph replays count their nodes) */
int amgp_ctx_launch_count(amgp_ctx *ctx, int64_t *count);
int amgp_malloc(amgp_ctx *ctx, int64_t bytes, void **dptr);
int amgp_free(amgp_ctx *ctx, void *dptr);
int amgp_memcpy_h2d(amgp_ctx *ctx, void *dst_dev, const void *src_host, int64_t bytes);
int amgp_memcpy_d2h(amgp_ctx *ctx, void *dst_host, const void *src_dev, int64_t bytes);

/* ---- matrices (sparse.py:32-115 CsrMatrix) ----------------------------- */
/* Upload a host CSR (row_ptr int64[nrows+1], col_idx int64[nnz], values
 * f64[nnz]; columns sorted per row as CsrMatrix guarantees, sparse.py:43-75)
 * and pack it into SELL-32 (SELL-C-sigma where rows of very different
 * lengths share slices, see amgp_mat_from_dcsr).  Per-row entry order is
 * kept, so the device SpMV accumulates in exactly the reference's order. */
int amgp_mat_from_csr(amgp_ctx *ctx, int64_t nrows, int64_t ncols, const int64_t *row_ptr,
                      const int64_t *col_idx, const double *values, amgp_mat **out);
/* Rows [row_begin, row_end) of the 3D Poisson matrix on an m^3 grid generated
 * directly on the device (problems.py:32-60 conventions: x-fastest ordering,
 * Dirichlet rows eliminated, diagonal 6 and -1 per neighbour for stencil 7;
 * diagonal 26 and -1 per neighbour for stencil 27).  Columns are global. */
int amgp_mat_poisson3d(amgp_ctx *ctx, int64_t m, int stencil, int64_t row_begin,
                       int64_t row_end, amgp_mat **out);
int amgp_mat_destroy(amgp_mat *A);
/* stored = padded SELL slots; bytes = device bytes of the matrix arrays */
int amgp_mat_info(const amgp_mat *A, int64_t *nrows, int64_t *ncols, int64_t *nnz,
                  int64_t *stored, int64_t *bytes);
/* Download back to host CSR (row_ptr[nrows+1], col_idx[nnz], values[nnz]). */
int amgp_mat_to_csr(amgp_mat *A, int64_t *row_ptr, int64_t *col_idx, double *values);
/* smoothers.py:38-49 l1_jacobi_diag: m_i = sum_j |a_ij| - |a_ii| + a_ii,
 * written to device m[nrows]; AMGP_EINVAL for a non-positive diagonal. */
int amgp_mat_l1_diag(amgp_mat *A, double *m_dev);

/* ---- hot-path kernels --------------------------------------------------- */
/* sparse.py:118-125 spmv: y = A x (device vectors). */
int amgp_spmv(amgp_ctx *ctx, const amgp_mat *A, const double *x, double *y);
/* sparse.py:128-139 fused_update: r -= s; d = d*(rho*rho_prev) + c*r; x += d. */
int amgp_fused_update(amgp_ctx *ctx, int64_t n, double rho, double rho_prev, double c,
                      const double *s, double *r, double *d, double *x);
/* smoothers.py:92-137 smoother_apply: x = S(b, x0), exactly `degree` SpMVs
 * (logically; the x0 == NULL SpMV of a zero vector is skipped on device).
 * x0 == NULL means a zero initial guess; x0 may equal x. */
int amgp_smoother_apply(amgp_ctx *ctx, amgp_mat *A, const double *m,
                        const amgp_smoother_cfg *cfg, const double *b, const double *x0,
                        double *x);

/* out = a + s*b (sign > 0) or a - s*b (sign < 0), the product rounded
 * first: numpy's axpy expressions of krylov.py:101-119 (the PCG of a solve
 * whose preconditioner is a user callable). */
int amgp_vec_update(amgp_ctx *ctx, int64_t n, double s, const double *a, const double *b, double *out,
                    int sign);
/* smoother_apply over HOST buffers, napply independent applications
 * (cfgs[i], b_host[i], x0_host[i] (NULL: zero guess) -> x_host[i]); uploads,
 * kernels and downloads of consecutive applications overlap (two device
 * slots, two copy streams, full-duplex PCIe); returns when every x_host[i]
 * is written.  Results equal amgp_smoother_apply's bit for bit. */
int amgp_smoother_apply_host(amgp_ctx *ctx, amgp_mat *A, const double *m, int napply,
                             const amgp_smoother_cfg *cfgs, const double *const *b_host,
                             const double *const *x0_host, double *const *x_host);

/* ---- V-cycle (amg.py:47-91, 293-319) ----------------------------------- */
/* Levels fine->coarse: A[l], m[l] (device l1 diagonals), P[l] (n_l x n_{l+1})
 * and R[l] = P[l]^T (amg.py:56-59) for l < nlevels-1.  The hierarchy keeps
 * references to the matrices and diagonals (caller keeps them alive). */
int amgp_hier_create(amgp_ctx *ctx, int nlevels, amgp_mat *const *A, const double *const *m,
                     amgp_mat *const *P, amgp_mat *const *R, int coarse_solver,
                     int coarse_sweeps, amgp_hier **out);
/* Smoother of one level (level < 0: all levels), amg.py:51 Level.smoother. */
int amgp_hier_set_smoother(amgp_hier *h, int level, const amgp_smoother_cfg *cfg);
/* dense_direct coarse solver: host column-major Cholesky factor L (n x n,
 * lower) of the coarsest A; solves run on the device (amg.py:295-298). */
int amgp_hier_set_coarse_cholesky(amgp_hier *h, const double *L_colmajor);
/* Capture the V-cycle into a CUDA graph on the next apply (1) or not (0). */
int amgp_hier_use_graph(amgp_hier *h, int enable);
/* Number of levels. */
int amgp_hier_info(amgp_hier *h, int *nlevels);
int amgp_hier_destroy(amgp_hier *h);
/* amg.py:303-315 vcycle_apply: z = V(r), r and z device vectors of n_0. */
int amgp_vcycle_apply(amgp_hier *h, const double *r, double *z);

/* ---- Krylov (krylov.py:45-120) ----------------------------------------- */
/* Solve A x = b with PCG/FCG preconditioned by the V-cycle of h (NULL: none).
 * x is the initial guess when x0_given, else it is zeroed.  history_host may
 * be NULL, else it receives up to itmax+1 relative residuals. */
int amgp_pcg_solve(amgp_ctx *ctx, amgp_mat *A, amgp_hier *h, const double *b, double *x,
                   int x0_given, int variant, double tol, int itmax, double *history_host,
                   amgp_solve_report *report);

/* ---- multi-GPU: one process per GPU, row-block partitions ---
 * The reference is single-process; this is the paper's MPI+CUDA layer
 * rebuilt on NCCL over NVLink.  NCCL is dlopen'ed. */
/* 128-byte ncclUniqueId (rank 0 creates it and shares it out of band) */
int amgp_comm_unique_id(char *id128);
int amgp_ctx_init_comm(amgp_ctx *ctx, int nranks, int rank, const char *id128);
int amgp_ctx_comm_info(amgp_ctx *ctx, int *nranks, int *rank);
/* Attach a halo plan: local columns [0, nown) index the rank's own operand
 * entries, [nown, ncols) the halo, received per SpMV from `peers` (recv_cnt
 * each, in peer order); this rank sends send_cnt[q] own entries
 * (send_idx, concatenated in peer order) to peers[q].  Slices whose columns
 * stay below nown run while the exchange is in flight. */
int amgp_mat_set_halo(amgp_mat *A, int64_t nown, int npeers, const int *peers,
                      const int64_t *send_cnt, const int64_t *send_idx, const int64_t *recv_cnt);
int amgp_mat_halo_info(const amgp_mat *A, int64_t *nown, int64_t *nhalo, int64_t *n_interior,
                       int64_t *n_boundary);
/* Rewrite the global columns of a generated row block to local ones: owned
 * [own_lo, own_hi) first, then halo segments [seg_lo[q], seg_hi[q]) in order. */
int amgp_mat_localize(amgp_mat *A, int64_t own_lo, int64_t own_hi, int nseg,
                      const int64_t *seg_lo, const int64_t *seg_hi);

/* ---- host-side helpers (no device needed; used by CPU tests) ------------ */
/* Pack a CSR into SELL-32 on the host.  Call with outputs NULL to get
 * *nslices and *stored; then with arrays slice_ptr[nslices+1], col[stored]
 * (int32, -1 = padding), val[stored]. */
int amgp_sell_pack_host(int64_t nrows, const int64_t *row_ptr, const int64_t *col_idx,
                        const double *values, int64_t *nslices, int64_t *stored,
                        int64_t *slice_ptr, int32_t *col, double *val);
/* Per-step scalars of smoother_apply computed with the reference's
 * expressions (smoothers.py:112-135); coef[3*degree]: for cheb4/opt_cheb4
 * (cz_j, cr_j, beta_j); for opt_cheb1 coef[0]=theta and (rho_j*rho_{j-1},
 * 2 rho_j/delta) for j=1..degree-1 at coef[1+2(j-1)].  */
int amgp_smoother_coefficients(const amgp_smoother_cfg *cfg, double *coef);

/* ---- native host setup (amg.py:97-287), bit-exact with the reference ----
 * Host CSR in / out (int64 indices, f64 values).  Results of variable size
 * come back as an opaque amgp_hcsr (query with amgp_hcsr_info, copy out with
 * amgp_hcsr_copy, release with amgp_hcsr_free). */
typedef struct amgp_hcsr amgp_hcsr;
int amgp_setup_set_threads(int threads);
int amgp_hcsr_info(const amgp_hcsr *h, int64_t *nrows, int64_t *ncols, int64_t *nnz);
int amgp_hcsr_copy(const amgp_hcsr *h, int64_t *row_ptr, int64_t *col_idx, double *values);
int amgp_hcsr_free(amgp_hcsr *h);
/* amg.py:102-149 sa_aggregate -> agg[n], *n_agg */
int amgp_setup_sa_aggregate(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                            const double *values, double theta, int64_t *agg, int64_t *n_agg);
/* amg.py:152-191 matching_aggregate -> agg[n], *n_agg */
int amgp_setup_matching_aggregate(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                                  const double *values, int sweeps, int64_t *agg,
                                  int64_t *n_agg);
/* amg.py:219-226 smooth_prolongator(A, P_hat(agg), omega) */
int amgp_setup_smooth_prolongator(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                                  const double *values, const int64_t *agg, int64_t n_agg,
                                  double omega, amgp_hcsr **P);
/* amg.py:229-235 galerkin_rap(A, P) */
int amgp_setup_galerkin(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                        const double *values, int64_t nc, const int64_t *p_row_ptr,
                        const int64_t *p_col_idx, const double *p_values, amgp_hcsr **Ac);
/* numpy float64 dot (x @ y) exactly as OpenBLAS 0.3.30's SkylakeX ddot with
 * `threads` BLAS threads evaluates it (amg.py:211-212 power iteration). */
double amgp_setup_blas_dot(int64_t n, const double *x, const double *y, int threads);
/* host y = A x in stored order (the power iteration of amg.py:194-216) */
int amgp_setup_spmv(int64_t n, const int64_t *row_ptr, const int64_t *col_idx,
                    const double *values, const double *x, double *y);

/* ---- device hierarchy setup (amg.py:97-287 on the GPU; dsetup.cu) --------
 * Device pointers.  Row-producing calls follow a count/fill protocol: with
 * row_ptr == NULL they write each output row's entry count to row_cnt; with
 * row_ptr (exclusive prefix sums of those counts) they write the rows,
 * sorted by column, exact zeros dropped.  Columns of produced rows are
 * global int64 indices; A operands are SELL matrices with local columns
 * (own entries [0, nown), halo after, see amgp_mat_set_halo). */
/* scipy csr_diagonal of the own rows (amg.py:221,267 A.diagonal()) */
int amgp_ds_diag(amgp_mat *A, double *d);
/* amg.py:115-121 strength test, own columns only (decoupled aggregation;
 * every column is own on one GPU): strong neighbours j != i with
 * |a_ij| >= theta sqrt(|a_ii a_jj|), in row order.  rows: optional list of
 * rows (nlist of them); off == NULL: cnt[t] = list length; else write the
 * int32 local columns at off[t] (and |a_ij| to sabs unless NULL). */
int amgp_ds_strength(amgp_mat *A, const double *d, double theta, int64_t nown, const int64_t *rows,
                     int64_t nlist, const int64_t *off, int64_t *cnt, int32_t *scol, double *sabs);
/* numpy float64 dots x.y, x.x, y.y in OpenBLAS 0.3.30 SkylakeX ddot order
 * with `threads` BLAS threads (== amgp_setup_blas_dot); out_host[3] */
int amgp_ds_blas_dot3(amgp_ctx *ctx, int64_t n, const double *x, const double *y, int threads,
                      double *out_host);
/* amg.py:194-216 estimate_lambda_max: v (own rows) holds the start vector
 * and is overwritten; the SpMV exchanges A's halo; fold_ranks: per-rank dots
 * folded in rank order across the communicator (row-distributed A). */
int amgp_ds_lambda_max(amgp_ctx *ctx, amgp_mat *A, const double *d, double *v, int iters, int threads,
                       int fold_ranks, double *lam);
/* amg.py:219-226 smooth_prolongator rows of A's own rows (smooth == 0: the
 * tentative P_hat); agg_own / agg_halo: global coarse index of every own /
 * halo column. */
int amgp_ds_prolongator(amgp_mat *A, const double *d, const int64_t *agg_own, const int64_t *agg_halo,
                        double omega, int smooth, const int64_t *row_ptr, int64_t *row_cnt, int64_t *col,
                        double *val);
/* scipy csr_matmat C = A_side B, per-entry order of the A-side rows (the
 * Galerkin products of amg.py:229-235).  A-side: A_sell (local column c =
 * B row c - b_off) or CSR (a_rp, a_col, a_val); output row t = A-side row
 * a_rows[t] (NULL: t), nout rows. */
int amgp_ds_spgemm(amgp_ctx *ctx, const amgp_mat *A_sell, const int64_t *a_rp, const int64_t *a_col,
                   const double *a_val, const int64_t *a_rows, int64_t nout, const int64_t *b_rp,
                   const int64_t *b_col, const double *b_val, int64_t b_off, const int64_t *row_ptr,
                   int64_t *row_cnt, int64_t *c_col, double *c_val);
/* amg.py:234 (G + G^T) * 0.5 from the sorted rows of G and G^T */
int amgp_ds_symmetrize(amgp_ctx *ctx, int64_t n, const int64_t *g_rp, const int64_t *g_col, const double *g_val,
                       const int64_t *t_rp, const int64_t *t_col, const double *t_val, const int64_t *row_ptr,
                       int64_t *row_cnt, int64_t *col, double *val);
/* one-GPU (G + G^T) * 0.5 without a transposed copy: gt[e] = G[K,J] for
 * entry (J,K) (0.0 when absent), orphans = (K, J, G[J,K]) for absent ones
 * (up to cap written; *norph = their number); then the merge with the
 * orphan rows (sorted CSR o_*), count/fill. */
int amgp_ds_sym_lookup(amgp_ctx *ctx, int64_t n, const int64_t *rp, const int64_t *col, const double *val,
                       double *gt, int64_t *orow, int64_t *ocol, double *oval, int64_t cap, int64_t *norph);
int amgp_ds_symmetrize_lookup(amgp_ctx *ctx, int64_t n, const int64_t *g_rp, const int64_t *g_col,
                              const double *g_val, const double *gt, const int64_t *o_rp, const int64_t *o_col,
                              const double *o_val, const int64_t *row_ptr, int64_t *row_cnt, int64_t *col,
                              double *val);
/* SELL-32 matrix from a device CSR with local int64 columns < 2^31;
 * sigma != 0: SELL-C-sigma (rows sorted by length inside 256-row windows)
 * when that stores >= 5 % fewer slots and the matrix has >= 4096 rows. */
int amgp_mat_from_dcsr(amgp_ctx *ctx, int64_t nrows, int64_t ncols, const int64_t *row_ptr,
                       const int64_t *col, const double *val, int sigma, amgp_mat **out);
int amgp_mat_nown(const amgp_mat *A, int64_t *nown);
/* host greedy passes of amg.py:124-148 over device-computed strength lists */
int amgp_setup_sa_pass1(int64_t n, const int64_t *srp, const int32_t *scol, int64_t *agg, int64_t *n_agg);
int amgp_setup_sa_pass2(int64_t nleft, const int64_t *rows, const int64_t *lrp, const int32_t *lcol,
                        const double *labs, int64_t *agg, int64_t *n_agg);

#ifdef __cplusplus
}
#endif
#endif /* AMGP_H */
