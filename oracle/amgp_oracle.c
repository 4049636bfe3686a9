/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the polynomial-smoother /
 * AMG V-cycle / PCG hot path.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library; the
 * product (paper_2407_09848_b200/) never does.
 *
 * A plain-C restatement of the reference algorithm, pinned against golden
 * vectors produced by the reference itself (tests/golden/make_golden.py):
 *
 *   spmv            reference pkg/src/amgpoly/sparse.py:118-125 (scipy
 *                   csr_matvec: row sum from 0.0, stored order, mul then add)
 *   fused_update    sparse.py:128-139
 *   smoother_apply  smoothers.py:92-137 (all four families)
 *   vcycle_apply    amg.py:293-315 (l1-Jacobi x coarse_sweeps coarse solve)
 *   pcg / fcg       krylov.py:45-120 (dots summed sequentially; numpy's
 *                   OpenBLAS ddot uses another order, hence +-1 iterations)
 *
 * Compile with -ffp-contract=off: every expression is evaluated as separate
 * IEEE-754 binary64 operations, exactly as numpy evaluates it.
 * SpMV row loops may be split over pthreads (oracle_set_threads): per-row
 * arithmetic does not depend on the thread count, so the results are bitwise
 * identical for any thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

enum { OR_L1 = 0, OR_CHEB4 = 1, OR_OPT_CHEB4 = 2, OR_OPT_CHEB1 = 3 };

typedef struct {
    int64_t nrows, ncols;
    const int64_t *rp, *ci;
    const double *v;
} or_csr;

static int g_threads = 1;

void oracle_set_threads(int t) { g_threads = t > 0 ? t : 1; }

int oracle_max_threads(void) {
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

/* sparse.py:118-125 -> scipy csr_matvec: sum = 0; sum += Ax[jj]*x[Aj[jj]] */
static void spmv_rows(const or_csr *A, const double *x, double *y, int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; i++) {
        double s = 0.0;
        for (int64_t jj = A->rp[i]; jj < A->rp[i + 1]; jj++) s += A->v[jj] * x[A->ci[jj]];
        y[i] = s;
    }
}

typedef struct { const or_csr *A; const double *x; double *y; int64_t lo, hi; } spmv_job;

static void *spmv_worker(void *p) {
    spmv_job *j = (spmv_job *)p;
    spmv_rows(j->A, j->x, j->y, j->lo, j->hi);
    return NULL;
}

static void spmv_c(const or_csr *A, const double *x, double *y) {
    int64_t n = A->nrows;
    int t = g_threads;
    if (t <= 1 || n < 4096) { spmv_rows(A, x, y, 0, n); return; }
    if (t > 256) t = 256;
    pthread_t th[256];
    spmv_job jobs[256];
    for (int w = 0; w < t; w++) {
        jobs[w].A = A; jobs[w].x = x; jobs[w].y = y;
        jobs[w].lo = n * w / t; jobs[w].hi = n * (w + 1) / t;
        if (w) pthread_create(&th[w], NULL, spmv_worker, &jobs[w]);
    }
    spmv_worker(&jobs[0]);
    for (int w = 1; w < t; w++) pthread_join(th[w], NULL);
}

void oracle_spmv(int64_t nrows, int64_t ncols, const int64_t *rp, const int64_t *ci,
                 const double *v, const double *x, double *y) {
    or_csr A = {nrows, ncols, rp, ci, v};
    spmv_c(&A, x, y);
}

/* sparse.py:128-139 (each numpy statement is one elementwise pass) */
void oracle_fused_update(int64_t n, double rho, double rho_prev, double c, const double *s,
                         double *r, double *d, double *x) {
    double rp = rho * rho_prev;
    for (int64_t i = 0; i < n; i++) {
        r[i] = r[i] - s[i];
        d[i] = d[i] * rp;
        double t = c * r[i];
        d[i] = d[i] + t;
        x[i] = x[i] + d[i];
    }
}

/*
 * smoothers.py:92-137.  b, x0 are not modified; the result goes to out.
 * x0 == NULL means a zero initial guess (an explicit zero vector is used so
 * that the arithmetic is literally the reference's).
 */
int oracle_smoother_apply(int family, int k, double a, double rho, const double *beta,
                          int64_t n, const int64_t *rp, const int64_t *ci, const double *v,
                          const double *m, const double *b, const double *x0, double *out) {
    or_csr A = {n, n, rp, ci, v};
    double *x = out;
    if (x0) memcpy(x, x0, (size_t)n * sizeof(double));
    else for (int64_t i = 0; i < n; i++) x[i] = 0.0;
    double *y = (double *)malloc((size_t)n * sizeof(double));
    double *r = (double *)malloc((size_t)n * sizeof(double));
    double *z = (double *)malloc((size_t)n * sizeof(double));
    if (!y || !r || !z) { free(y); free(r); free(z); return -1; }

    if (family == OR_L1) { /* smoothers.py:106-110 */
        for (int it = 0; it < k; it++) {
            spmv_c(&A, x, y);
            for (int64_t i = 0; i < n; i++) {
                double ri = b[i] - y[i];
                x[i] = x[i] + ri / m[i];
            }
        }
    } else if (family == OR_CHEB4 || family == OR_OPT_CHEB4) { /* :112-122 */
        spmv_c(&A, x, y);
        for (int64_t i = 0; i < n; i++) { r[i] = b[i] - y[i]; z[i] = 0.0; }
        for (int j = 1; j <= k; j++) {
            double cz = (double)(2 * j - 3) / (double)(2 * j + 1);
            double cr = (double)(8 * j - 4) / (double)(2 * j + 1) / rho;
            double bj = family == OR_OPT_CHEB4 ? beta[j - 1] : 1.0;
            for (int64_t i = 0; i < n; i++) {
                double zi = z[i] * cz;
                double t = cr * (r[i] / m[i]);
                zi = zi + t;
                z[i] = zi;
                x[i] = x[i] + bj * zi;
            }
            if (j < k) {
                spmv_c(&A, z, y);
            for (int64_t i = 0; i < n; i++) r[i] = r[i] - y[i];
            }
        }
    } else if (family == OR_OPT_CHEB1) { /* :124-137, chebyshev.py:82-83 */
        double theta = (1.0 + a) / 2.0, delta = (1.0 - a) / 2.0;
        double sigma1 = theta / delta;
        double *d = z;
        spmv_c(&A, x, y);
            for (int64_t i = 0; i < n; i++) {
            r[i] = (b[i] - y[i]) / m[i] / rho;
            d[i] = r[i] / theta;
            x[i] = x[i] + d[i];
        }
        double rho_prev = 1.0 / sigma1;
        for (int j = 1; j < k; j++) {
            spmv_c(&A, d, y);
            double rho_cur = 1.0 / (2.0 * sigma1 - rho_prev);
            double rp = rho_cur * rho_prev;
            double c = 2.0 * rho_cur / delta;
            for (int64_t i = 0; i < n; i++) {
                double s = y[i] / m[i] / rho;
                r[i] = r[i] - s;
                double di = d[i] * rp;
                double t = c * r[i];
                di = di + t;
                d[i] = di;
                x[i] = x[i] + di;
            }
            rho_prev = rho_cur;
        }
    } else {
        free(y); free(r); free(z);
        return -2;
    }
    free(y); free(r); free(z);
    return 0;
}

/* ---- V-cycle (amg.py:293-315) ------------------------------------------ */

typedef struct {
    int nlev;
    const int64_t *n;          /* rows per level */
    const int64_t **A_rp, **A_ci; const double **A_v;
    const double **m;
    const int64_t **P_rp, **P_ci; const double **P_v;   /* n[l] x n[l+1] */
    const int64_t **R_rp, **R_ci; const double **R_v;   /* n[l+1] x n[l]  */
    int family, k; double a, rho; const double *beta;
    int coarse_sweeps;
} or_hier;

static int vcycle_rec(const or_hier *h, int l, const double *r, double *out) {
    int64_t n = h->n[l];
    if (l == h->nlev - 1) /* amg.py:299-300: l1-Jacobi x coarse_sweeps from 0 */
        return oracle_smoother_apply(OR_L1, h->coarse_sweeps, 0.0, 1.0, NULL, n, h->A_rp[l],
                                     h->A_ci[l], h->A_v[l], h->m[l], r, NULL, out);
    int64_t nc = h->n[l + 1];
    double *x = (double *)malloc((size_t)n * sizeof(double));
    double *res = (double *)malloc((size_t)n * sizeof(double));
    double *rc = (double *)malloc((size_t)nc * sizeof(double));
    double *xc = (double *)malloc((size_t)nc * sizeof(double));
    int st = oracle_smoother_apply(h->family, h->k, h->a, h->rho, h->beta, n, h->A_rp[l],
                                   h->A_ci[l], h->A_v[l], h->m[l], r, NULL, x);
    or_csr A = {n, n, h->A_rp[l], h->A_ci[l], h->A_v[l]};
    or_csr R = {nc, n, h->R_rp[l], h->R_ci[l], h->R_v[l]};
    or_csr P = {n, nc, h->P_rp[l], h->P_ci[l], h->P_v[l]};
    spmv_c(&A, x, res);
    for (int64_t i = 0; i < n; i++) res[i] = r[i] - res[i];
    spmv_c(&R, res, rc);
    if (!st) st = vcycle_rec(h, l + 1, rc, xc);
    spmv_c(&P, xc, res);
    for (int64_t i = 0; i < n; i++) x[i] = x[i] + res[i];
    if (!st)
        st = oracle_smoother_apply(h->family, h->k, h->a, h->rho, h->beta, n, h->A_rp[l],
                                   h->A_ci[l], h->A_v[l], h->m[l], r, x, out);
    free(x); free(res); free(rc); free(xc);
    return st;
}

int oracle_vcycle_apply(const or_hier *h, const double *r, double *z) {
    return vcycle_rec(h, 0, r, z);
}

static double dot_c(int64_t n, const double *a, const double *b) {
    double s = 0.0;
    for (int64_t i = 0; i < n; i++) s += a[i] * b[i];
    return s;
}

/*
 * krylov.py:45-120.  h == NULL means no preconditioner (z = r).
 * Returns iterations; *flags bit0 = converged, bit1 = breakdown.
 * history (may be NULL) receives itmax+1 relres values; *nhist its length.
 */
int oracle_pcg(const or_hier *h, int64_t n, const int64_t *rp, const int64_t *ci,
               const double *v, const double *b, double *x, int x0_given, int fcg,
               double tol, int itmax, double *final_relres, int *flags, double *history,
               int *nhist) {
    or_csr A = {n, n, rp, ci, v};
    if (!x0_given) for (int64_t i = 0; i < n; i++) x[i] = 0.0;
    double *r = (double *)malloc((size_t)n * sizeof(double));
    double *z = (double *)malloc((size_t)n * sizeof(double));
    double *d = (double *)malloc((size_t)n * sizeof(double));
    double *Ad = (double *)malloc((size_t)n * sizeof(double));
    int nh = 0, it = 0;
    *flags = 0;
    double bnorm = sqrt(dot_c(n, b, b));
    if (bnorm == 0.0) {
        for (int64_t i = 0; i < n; i++) x[i] = x[i] * 0.0;
        *final_relres = 0.0; *flags = 1; *nhist = 0;
        free(r); free(z); free(d); free(Ad);
        return 0;
    }
    spmv_c(&A, x, Ad);
    for (int64_t i = 0; i < n; i++) r[i] = b[i] - Ad[i];
    double relres = sqrt(dot_c(n, r, r)) / bnorm;
    if (history) history[nh] = relres;
    nh++;
    if (relres <= tol) { *flags = 1; goto done; }
    if (h) vcycle_rec(h, 0, r, z); else memcpy(z, r, (size_t)n * sizeof(double));
    memcpy(d, z, (size_t)n * sizeof(double));
    double rz = dot_c(n, r, z);
    for (it = 1; it <= itmax; it++) {
        spmv_c(&A, d, Ad);
        double dAd = dot_c(n, d, Ad);
        if (dAd <= 0.0) { it -= 1; *flags = 2; goto done; }
        double alpha = fcg ? dot_c(n, r, d) / dAd : rz / dAd;
        for (int64_t i = 0; i < n; i++) x[i] = x[i] + alpha * d[i];
        for (int64_t i = 0; i < n; i++) r[i] = r[i] - alpha * Ad[i];
        relres = sqrt(dot_c(n, r, r)) / bnorm;
        if (history) history[nh] = relres;
        nh++;
        if (relres <= tol) { *flags = 1; goto done; }
        if (h) vcycle_rec(h, 0, r, z); else memcpy(z, r, (size_t)n * sizeof(double));
        if (!fcg) {
            double rz_new = dot_c(n, r, z);
            double beta = rz_new / rz;
            rz = rz_new;
            for (int64_t i = 0; i < n; i++) d[i] = z[i] + beta * d[i];
        } else {
            double beta = dot_c(n, z, Ad) / dAd;
            for (int64_t i = 0; i < n; i++) d[i] = z[i] - beta * d[i];
        }
    }
    it = itmax;
done:
    *final_relres = relres;
    *nhist = nh;
    free(r); free(z); free(d); free(Ad);
    return it;
}
