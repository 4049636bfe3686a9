// K1/K2: the fused polynomial-smoother step kernels and smoother_apply.
//
// One kernel launch per degree step.  Each launch streams the matrix once
// (SELL-32) and fuses the SpMV of the step's operand with the l1 scaling and
// the recurrence update of r / z|d / x -- the reference's k SpMVs plus 2-4
// numpy passes per step (smoothers.py:106-137) become k passes over HBM.
// The operand is double-buffered: rows gather the previous step's operand
// while the new one is written to the other buffer.  The row schedule
// (thread-per-row or split-slice, rows.cuh) is picked per matrix; both give
// identical bits.
//
// Per-element arithmetic, every operation a
// separate round-to-nearest binary64 op in the reference's order:
//   l1_jacobi  sweep     : y=A x ; x' = x + ((b - y)/m)                 (:106-110)
//   cheb4/opt  step 1    : y=A x0; r=b-y ; z=(0*cz)+cr*(r/m); x=x0+beta z (:112-118)
//              step j>1  : y=A z ; r=r-y ; z=z*cz + cr*(r/m) ; x=x+beta z (:117-122)
//   opt_cheb1  init      : y=A x0; r=((b-y)/m)/rho ; d=r/theta ; x=x0+d    (:128-131)
//              step j    : y=A d ; s=(y/m)/rho ; r=r-s ; d=d*rp + c*r ; x=x+d (:132-136)
// With x0 == 0 the first SpMV is skipped (b - A*0 == b bitwise).
#include <algorithm>

#include "epilogues.cuh"

// sparse.py:128-139 fused_update (elementwise, in place)
__global__ void k_fused_update(int64_t n, double rp, double c, const double *__restrict__ s,
                               double *__restrict__ r, double *__restrict__ d,
                               double *__restrict__ x) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double ri = __dsub_rn(r[i], s[i]);
        const double di = __dadd_rn(__dmul_rn(d[i], rp), __dmul_rn(c, ri));
        r[i] = ri;
        d[i] = di;
        x[i] = __dadd_rn(x[i], di);
    }
}

// ---------------------------------------------------------------- host side
// smoothers.py:112-135 scalars, evaluated as Python evaluates them (binary64,
// one operation per statement; built with -ffp-contract=off).
int make_smoother_plan(const amgp_smoother_cfg *cfg, SmootherPlan *plan) {
    if (!cfg) return amgp_fail(AMGP_EINVAL, "null smoother config");
    if (cfg->family < AMGP_L1_JACOBI || cfg->family > AMGP_OPT_CHEB1)
        return amgp_fail(AMGP_EINVAL, "unknown smoother family");
    if (cfg->degree < 1) return amgp_fail(AMGP_EINVAL, "degree must be >= 1");
    if (!(cfg->rho_scale > 0.0)) return amgp_fail(AMGP_EINVAL, "rho_scale must be positive");
    const int k = cfg->degree;
    plan->family = cfg->family;
    plan->degree = k;
    plan->rho = cfg->rho_scale;
    plan->coef.assign(3 * (size_t)k, 0.0);
    const double rho = cfg->rho_scale;
    if (cfg->family == AMGP_CHEB4 || cfg->family == AMGP_OPT_CHEB4) {
        if (cfg->family == AMGP_OPT_CHEB4 && !cfg->beta)
            return amgp_fail(AMGP_EINVAL, "opt_cheb4 needs a beta table");
        for (int j = 1; j <= k; j++) {
            double num = (double)(8 * j - 4), den = (double)(2 * j + 1);
            double q = num / den;
            double cr = q / rho;
            double cz = (double)(2 * j - 3) / den;
            plan->coef[3 * (j - 1) + 0] = cz;
            plan->coef[3 * (j - 1) + 1] = cr;
            plan->coef[3 * (j - 1) + 2] = cfg->family == AMGP_OPT_CHEB4 ? cfg->beta[j - 1] : 1.0;
        }
    } else if (cfg->family == AMGP_OPT_CHEB1) {
        if (!(cfg->a > 0.0 && cfg->a < 1.0)) return amgp_fail(AMGP_EINVAL, "a must lie in (0, 1)");
        double theta = (1.0 + cfg->a) / 2.0;  // chebyshev.py:82-83
        double delta = (1.0 - cfg->a) / 2.0;
        double sigma1 = theta / delta;
        plan->coef[0] = theta;
        double rho_prev = 1.0 / sigma1;
        for (int j = 1; j < k; j++) {
            double t = 2.0 * sigma1;
            double rho_cur = 1.0 / (t - rho_prev);
            double rp = rho_cur * rho_prev;
            double c2 = 2.0 * rho_cur;
            double c = c2 / delta;
            plan->coef[1 + 2 * (j - 1)] = rp;
            plan->coef[2 + 2 * (j - 1)] = c;
            rho_prev = rho_cur;
        }
    }
    return AMGP_OK;
}

extern "C" int amgp_smoother_coefficients(const amgp_smoother_cfg *cfg, double *coef) {
    SmootherPlan p;
    AMGP_TRY(make_smoother_plan(cfg, &p));
    if (coef) std::copy(p.coef.begin(), p.coef.end(), coef);
    return AMGP_OK;
}

template <bool FIRST, bool LAST>
static int launch_cheb4(amgp_ctx *ctx, const amgp_mat *A, const double *m, const double *b,
                        const double *xg, bool x0, double *r, double *znew, double *x, double cz,
                        double cr, double beta) {
    if (FIRST && x0)
        return launch_rows(ctx, A, xg, Cheb4Step<FIRST, LAST, true>{m, b, xg, r, znew, x, cz, cr, beta});
    return launch_rows(ctx, A, xg, Cheb4Step<FIRST, LAST, false>{m, b, xg, r, znew, x, cz, cr, beta});
}

template <bool FIRST, bool LAST, bool X0>
static int launch_cheb1_x0(amgp_ctx *ctx, const amgp_mat *A, const double *m, const double *b,
                           const double *xg, double *r, double *dnew, double *x, double c0,
                           double c1, double rho) {
    if (rho == 1.0)
        return launch_rows(ctx, A, xg, Cheb1Step<FIRST, LAST, X0, true>{m, b, xg, r, dnew, x, c0, c1, rho});
    return launch_rows(ctx, A, xg, Cheb1Step<FIRST, LAST, X0, false>{m, b, xg, r, dnew, x, c0, c1, rho});
}

template <bool FIRST, bool LAST>
static int launch_cheb1(amgp_ctx *ctx, const amgp_mat *A, const double *m, const double *b,
                        const double *xg, bool x0, double *r, double *dnew, double *x, double c0,
                        double c1, double rho) {
    if (FIRST && x0) return launch_cheb1_x0<FIRST, LAST, true>(ctx, A, m, b, xg, r, dnew, x, c0, c1, rho);
    return launch_cheb1_x0<FIRST, LAST, false>(ctx, A, m, b, xg, r, dnew, x, c0, c1, rho);
}

int smoother_enqueue(amgp_ctx *ctx, const amgp_mat *A, const double *m, const SmootherPlan &p,
                     const double *b, const double *x0, double *x, double *work) {
    const int64_t n = A->nrows;
    if (n == 0) return AMGP_OK;
    const int k = p.degree;
    double *r = work, *buf[2] = {work + 2 * n, work + n}, *tmp = work + 3 * n;
    const bool hx0 = x0 != nullptr;
    if (p.family == AMGP_L1_JACOBI) {
        // sweep s writes x when (k - s) is even, else tmp, so sweep k lands in x
        const double *xin = x0;
        for (int s = 1; s <= k; s++) {
            double *xout = ((k - s) % 2 == 0) ? x : tmp;
            if (s == 1 && !hx0) AMGP_TRY(launch_rows(ctx, A, nullptr, L1Sweep<false>{m, b, nullptr, xout}));
            else AMGP_TRY(launch_rows(ctx, A, xin, L1Sweep<true>{m, b, xin, xout}));
            xin = xout;
        }
        return AMGP_OK;
    }
    if (p.family == AMGP_CHEB4 || p.family == AMGP_OPT_CHEB4) {
        for (int j = 1; j <= k; j++) {
            const double cz = p.coef[3 * (j - 1)], cr = p.coef[3 * (j - 1) + 1],
                         be = p.coef[3 * (j - 1) + 2];
            const double *xg = (j == 1) ? x0 : buf[(j - 1) & 1];
            double *zn = buf[j & 1];
            if (j == 1 && k == 1) AMGP_TRY((launch_cheb4<true, true>(ctx, A, m, b, xg, hx0, r, zn, x, cz, cr, be)));
            else if (j == 1) AMGP_TRY((launch_cheb4<true, false>(ctx, A, m, b, xg, hx0, r, zn, x, cz, cr, be)));
            else if (j == k) AMGP_TRY((launch_cheb4<false, true>(ctx, A, m, b, xg, hx0, r, zn, x, cz, cr, be)));
            else AMGP_TRY((launch_cheb4<false, false>(ctx, A, m, b, xg, hx0, r, zn, x, cz, cr, be)));
        }
        return AMGP_OK;
    }
    // opt_cheb1: launch 0 is the init, launches j = 1..k-1 the fused updates
    for (int j = 0; j < k; j++) {
        const double *xg = (j == 0) ? x0 : buf[j & 1];
        double *dn = buf[(j + 1) & 1];
        const bool last = (j == k - 1);
        if (j == 0) {
            const double theta = p.coef[0];
            if (last) AMGP_TRY((launch_cheb1<true, true>(ctx, A, m, b, xg, hx0, r, dn, x, theta, 0.0, p.rho)));
            else AMGP_TRY((launch_cheb1<true, false>(ctx, A, m, b, xg, hx0, r, dn, x, theta, 0.0, p.rho)));
        } else {
            const double rp = p.coef[1 + 2 * (j - 1)], c = p.coef[2 + 2 * (j - 1)];
            if (last) AMGP_TRY((launch_cheb1<false, true>(ctx, A, m, b, xg, hx0, r, dn, x, rp, c, p.rho)));
            else AMGP_TRY((launch_cheb1<false, false>(ctx, A, m, b, xg, hx0, r, dn, x, rp, c, p.rho)));
        }
    }
    return AMGP_OK;
}

static int ensure_work(amgp_mat *A, int64_t doubles) {
    if (A->work_n >= doubles) return AMGP_OK;
    cudaStreamSynchronize(cur_stream(A->ctx));
    cudaFree(A->work);
    A->work = nullptr;
    A->work_n = 0;
    AMGP_CUDA(cudaMalloc(&A->work, (size_t)doubles * sizeof(double)));
    A->work_n = doubles;
    return AMGP_OK;
}

extern "C" int amgp_smoother_apply(amgp_ctx *ctx, amgp_mat *A, const double *m,
                                   const amgp_smoother_cfg *cfg, const double *b,
                                   const double *x0, double *x) {
    if (!ctx || !A || !cfg) return amgp_fail(AMGP_EINVAL, "amgp_smoother_apply: bad argument");
    if (A->nrows != (A->halo ? A->halo->nown : A->ncols))
        return amgp_fail(AMGP_EINVAL, "dimension mismatch");
    if (A->nrows > 0 && (!m || !b || !x)) return amgp_fail(AMGP_EINVAL, "null vector");
    SmootherPlan p;
    AMGP_TRY(make_smoother_plan(cfg, &p));
    AMGP_CUDA(cudaSetDevice(ctx->device));
    std::lock_guard<std::mutex> cg(ctx->mu);  // API calls share the context stream (see amgp_common.cuh)
    std::lock_guard<std::mutex> g(A->mu);
    const int64_t n = A->nrows;
    AMGP_TRY(ensure_work(A, smoother_work_doubles(n) + n));
    if (x0 && x0 == x) {  // x0 may alias x: keep a private copy of x0
        double *x0c = A->work + smoother_work_doubles(n);
        AMGP_CUDA(cudaMemcpyAsync(x0c, x0, n * sizeof(double), cudaMemcpyDeviceToDevice, cur_stream(ctx)));
        x0 = x0c;
    }
    return smoother_enqueue(ctx, A, m, p, b, x0, x, A->work);
}

// End-to-end path with host buffers (the reference-facing call for host
// data): napply independent applications, apply i reading b_host[i] and
// x0_host[i] (NULL: zero guess) and writing x_host[i].  Two device slots and
// two copy streams pipeline the calls: the upload of apply i+1 and the
// download of apply i-1 run while apply i's kernels stream the matrix, and
// PCIe carries H2D and D2H at once (full duplex).  Pinned host buffers give
// asynchronous DMA; pageable ones still work (the driver stages them).
// Every apply computes exactly what amgp_smoother_apply computes.
extern "C" int amgp_smoother_apply_host(amgp_ctx *ctx, amgp_mat *A, const double *m, int napply,
                                        const amgp_smoother_cfg *cfgs, const double *const *b_host,
                                        const double *const *x0_host, double *const *x_host) {
    if (!ctx || !A || napply < 0 || (napply && (!cfgs || !b_host || !x_host)))
        return amgp_fail(AMGP_EINVAL, "amgp_smoother_apply_host: bad argument");
    if (A->nrows != (A->halo ? A->halo->nown : A->ncols)) return amgp_fail(AMGP_EINVAL, "dimension mismatch");
    const int64_t n = A->nrows;
    if (n > 0 && !m) return amgp_fail(AMGP_EINVAL, "null vector");
    std::vector<SmootherPlan> plans(napply);
    for (int i = 0; i < napply; i++) {
        AMGP_TRY(make_smoother_plan(&cfgs[i], &plans[i]));
        if (n > 0 && (!b_host[i] || !x_host[i])) return amgp_fail(AMGP_EINVAL, "null vector");
    }
    if (napply == 0 || n == 0) return AMGP_OK;
    AMGP_CUDA(cudaSetDevice(ctx->device));
    std::lock_guard<std::mutex> cg(ctx->mu);
    std::lock_guard<std::mutex> g(A->mu);
    AMGP_TRY(ensure_work(A, smoother_work_doubles(n) + n));
    if (A->io_n < 6 * n) {  // two slots of (b, x0, x)
        cudaStreamSynchronize(cur_stream(ctx));
        cudaFree(A->io);
        A->io = nullptr;
        A->io_n = 0;
        AMGP_CUDA(cudaMalloc(&A->io, (size_t)6 * n * sizeof(double)));
        A->io_n = 6 * n;
    }
    if (!ctx->io_h2d) AMGP_CUDA(cudaStreamCreateWithFlags(&ctx->io_h2d, cudaStreamNonBlocking));
    if (!ctx->io_d2h) AMGP_CUDA(cudaStreamCreateWithFlags(&ctx->io_d2h, cudaStreamNonBlocking));
    const size_t bytes = (size_t)n * sizeof(double);
    double *db[2] = {A->io, A->io + 3 * n}, *dx0[2] = {A->io + n, A->io + 4 * n},
           *dx[2] = {A->io + 2 * n, A->io + 5 * n};
    cudaEvent_t ev[4][2] = {};  // in, computed, downloaded, start
    int st = AMGP_OK;
    for (auto &row : ev)
        for (auto &e : row)
            if (st == AMGP_OK && cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
                st = amgp_cuda_fail(cudaGetLastError(), "cudaEventCreate", __FILE__, __LINE__);
    cudaStream_t h2d = ctx->io_h2d, d2h = ctx->io_d2h, cs = cur_stream(ctx);
    auto chk = [&](cudaError_t e, const char *what) {
        if (e != cudaSuccess && st == AMGP_OK) st = amgp_cuda_fail(e, what, __FILE__, __LINE__);
    };
    // the copies must also follow work the caller queued on the compute stream
    chk(cudaEventRecord(ev[3][0], cs), "record");
    chk(cudaStreamWaitEvent(h2d, ev[3][0], 0), "wait");
    for (int i = 0; i < napply && st == AMGP_OK; i++) {
        const int s = i & 1;
        const bool hx0 = x0_host && x0_host[i];
        if (i >= 2) chk(cudaStreamWaitEvent(h2d, ev[1][s], 0), "wait");  // slot's inputs consumed
        chk(cudaMemcpyAsync(db[s], b_host[i], bytes, cudaMemcpyHostToDevice, h2d), "upload b");
        if (hx0) chk(cudaMemcpyAsync(dx0[s], x0_host[i], bytes, cudaMemcpyHostToDevice, h2d), "upload x0");
        chk(cudaEventRecord(ev[0][s], h2d), "record");
        chk(cudaStreamWaitEvent(cs, ev[0][s], 0), "wait");
        if (i >= 2) chk(cudaStreamWaitEvent(cs, ev[2][s], 0), "wait");  // slot's output downloaded
        if (st == AMGP_OK) st = smoother_enqueue(ctx, A, m, plans[i], db[s], hx0 ? dx0[s] : nullptr, dx[s], A->work);
        chk(cudaEventRecord(ev[1][s], cs), "record");
        chk(cudaStreamWaitEvent(d2h, ev[1][s], 0), "wait");
        chk(cudaMemcpyAsync(x_host[i], dx[s], bytes, cudaMemcpyDeviceToHost, d2h), "download x");
        chk(cudaEventRecord(ev[2][s], d2h), "record");
    }
    chk(cudaStreamSynchronize(d2h), "sync");
    chk(cudaStreamSynchronize(h2d), "sync");
    for (auto &row : ev)
        for (auto &e : row)
            if (e) cudaEventDestroy(e);
    return st;
}

// out = a + s*b (sign > 0) or a - s*b (sign < 0): numpy's `a + s * b` with
// the product rounded first (no FMA) -- the axpys of reference krylov.py:101-119.
__global__ void k_vec_update(int64_t n, double s, const double *__restrict__ a, const double *__restrict__ b,
                             double *__restrict__ out, int sign) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double t = __dmul_rn(s, b[i]);
        out[i] = sign > 0 ? __dadd_rn(a[i], t) : __dsub_rn(a[i], t);
    }
}

extern "C" int amgp_vec_update(amgp_ctx *ctx, int64_t n, double s, const double *a, const double *b, double *out,
                               int sign) {
    if (!ctx || n < 0 || (n && (!a || !b || !out)) || sign == 0)
        return amgp_fail(AMGP_EINVAL, "amgp_vec_update: bad argument");
    if (n == 0) return AMGP_OK;
    AMGP_CUDA(cudaSetDevice(ctx->device));
    std::lock_guard<std::mutex> cg(ctx->mu);
    const unsigned g = (unsigned)std::min<int64_t>(grid_for(n, 256), 148 * 16);
    k_vec_update<<<g, 256, 0, cur_stream(ctx)>>>(n, s, a, b, out, sign);
    AMGP_CHECK_LAUNCH(ctx);
    return AMGP_OK;
}

extern "C" int amgp_fused_update(amgp_ctx *ctx, int64_t n, double rho, double rho_prev, double c,
                                 const double *s, double *r, double *d, double *x) {
    if (!ctx || n < 0) return amgp_fail(AMGP_EINVAL, "fused_update: vector length mismatch");
    if (n == 0) return AMGP_OK;
    AMGP_CUDA(cudaSetDevice(ctx->device));
    std::lock_guard<std::mutex> cg(ctx->mu);
    const double rp = rho * rho_prev;  // sparse.py:137 evaluates rho*rho_prev first
    const int blk = 256;
    const unsigned g = (unsigned)std::min<int64_t>(grid_for(n, blk), 148 * 16);
    k_fused_update<<<g, blk, 0, cur_stream(ctx)>>>(n, rp, c, s, r, d, x);
    AMGP_CHECK_LAUNCH(ctx);
    return AMGP_OK;
}
