// Device AMG hierarchy and the symmetric V-cycle (reference amg.py:293-319).
//
// Per level l < L-1 (amg.py:309-315):
//   x   = S_l(r, 0)                 K1/K2 fused smoother steps (first SpMV skipped)
//   res = r - A_l x                 K3 residual (k_spmv<1>)
//   rc  = R_l res                   K4 restriction with the explicit P^T (amg.py:56-59)
//   xc  = V_{l+1}(rc)
//   x   = x + P_l xc                K5 prolongation + correction (k_spmv<2>)
//   z   = S_l(r, x)                 K1/K2 post-smoother
// Coarsest level (amg.py:293-300): l1-Jacobi x coarse_sweeps from 0 -- one
// single-CTA kernel (K6) with the iterate in shared memory when it fits, else
// one launch per sweep; or the dense Cholesky solve.
// The whole V-cycle is captured once into a CUDA graph and replayed.
#include <algorithm>
#include <vector>

#include "epilogues.cuh"

struct amgp_hier {
    amgp_ctx *ctx = nullptr;
    int nlev = 0;
    std::vector<amgp_mat *> A, P, R;
    std::vector<const double *> m;
    std::vector<SmootherPlan> plan;
    SmootherPlan coarse_plan;
    int coarse_solver = AMGP_COARSE_L1_JACOBI;
    int coarse_sweeps = 30;
    // per-level device buffers
    std::vector<double *> rl, zl, xpre, res, work;
    double *cholL = nullptr;  // dense coarse factor (column-major)
    // graph cache
    bool use_graph = true;
    cudaGraphExec_t gexec = nullptr;
    const double *g_r = nullptr;
    double *g_z = nullptr;
    cudaStream_t cap_stream = nullptr;  // graph capture stream (see vcycle_enqueue)
    int64_t g_nodes = 0;
    std::mutex mu;
};

#define COARSE_SMEM_BYTES (227 * 1024)

// K6 for coarsest levels too large for k_coarse_l1_reg (below): all
// l1-Jacobi sweeps in one CTA with the level's SELL values and columns staged
// in shared memory; each row thread forms its products and sums them in slot
// order (padding skipped: contributes +0.0, bitwise neutral -- rows.cuh) and
// updates the row as k_l1_sweep does, so the result is bitwise the
// multi-launch one.
static inline size_t coarse_smem(const amgp_mat *A) {
    return 16 * (size_t)A->nrows + 12 * (size_t)A->stored + 64;
}

__global__ void __launch_bounds__(1024)
k_coarse_l1(SellView A, const double *__restrict__ m, const double *__restrict__ b,
            double *__restrict__ x, int sweeps) {
    extern __shared__ double sh[];
    const int64_t n = A.nrows;
    const int64_t stored = A.slice_ptr[A.nslices];
    double *buf[2] = {sh, sh + n};
    double *pv = sh + 2 * n;
    int32_t *pc = (int32_t *)(pv + stored);
    for (int64_t e = threadIdx.x; e < stored; e += blockDim.x) {
        pv[e] = A.val[e];
        pc[e] = A.col[e];
    }
    __syncthreads();
    for (int s = 1; s <= sweeps; s++) {
        const double *xin = buf[(s - 1) & 1];
        double *xout = buf[s & 1];
        for (int64_t row = threadIdx.x; row < n; row += blockDim.x) {
            double y = 0.0;
            if (s > 1) {
                const int64_t sl = row >> 5;
                const int lane = row & 31;
                const int64_t base = A.slice_ptr[sl];
                const int w = (int)((A.slice_ptr[sl + 1] - base) >> 5);
                const double *vv = pv + base + lane;
                const int32_t *cc = pc + base + lane;
#pragma unroll 8
                for (int j = 0; j < w; j++) {
                    const int32_t c = cc[j * 32];
                    if (c >= 0) y = __dadd_rn(y, __dmul_rn(vv[j * 32], xin[c]));
                }
            }
            const double rr = __dsub_rn(b[row], y);
            xout[row] = __dadd_rn(s > 1 ? xin[row] : 0.0, __ddiv_rn(rr, m[row]));
        }
        __syncthreads();
    }
    for (int64_t row = threadIdx.x; row < n; row += blockDim.x) x[row] = buf[sweeps & 1][row];
}

// K6 for coarsest levels of at most COARSE_REG_SLOTS SELL slots: each of
// the 1024 threads keeps the values of its 16 slots in registers across all
// sweeps (16-bit columns in shared memory), so a sweep is one parallel
// product pass over the shared-memory iterate plus the ordered row sums --
// the same operations in the same order as k_coarse_l1.
#define COARSE_REG_K 16
#define COARSE_REG_SLOTS (1024 * COARSE_REG_K)
__global__ void __launch_bounds__(1024, 1)
k_coarse_l1_reg(SellView A, const double *__restrict__ m, const double *__restrict__ b,
                double *__restrict__ x, int sweeps) {
    extern __shared__ double sh[];
    const int64_t n = A.nrows;
    const int stored = (int)A.slice_ptr[A.nslices];
    double *buf[2] = {sh, sh + n};
    double *prod = sh + 2 * n;
    int16_t *pc = (int16_t *)(prod + stored);  // 16-bit columns (ncols < 32768)
    double vr[COARSE_REG_K];
#pragma unroll
    for (int k = 0; k < COARSE_REG_K; k++) {
        const int e = threadIdx.x + k * 1024;
        if (e < stored) pc[e] = (int16_t)A.col[e];
        vr[k] = e < stored ? A.val[e] : 0.0;
    }
    __syncthreads();
    for (int s = 1; s <= sweeps; s++) {
        const double *xin = buf[(s - 1) & 1];
        double *xout = buf[s & 1];
        if (s > 1) {
#pragma unroll
            for (int k = 0; k < COARSE_REG_K; k++) {
                const int e = threadIdx.x + k * 1024;
                if (e < stored) {
                    const int c = pc[e];
                    prod[e] = c >= 0 ? __dmul_rn(vr[k], xin[c]) : 0.0;
                }
            }
            __syncthreads();
        }
        for (int64_t row = threadIdx.x; row < n; row += blockDim.x) {
            double y = 0.0;
            if (s > 1) {
                const int64_t sl = row >> 5;
                const int lane = row & 31;
                const int64_t base = A.slice_ptr[sl];
                const int w = (int)((A.slice_ptr[sl + 1] - base) >> 5);
                const double *pp = prod + base + lane;
#pragma unroll 8
                for (int j = 0; j < w; j++) y = __dadd_rn(y, pp[j * 32]);
            }
            const double rr = __dsub_rn(__ldg(b + row), y);
            xout[row] = __dadd_rn(s > 1 ? xin[row] : 0.0, __ddiv_rn(rr, __ldg(m + row)));
        }
        __syncthreads();
    }
    for (int64_t row = threadIdx.x; row < n; row += blockDim.x) x[row] = buf[sweeps & 1][row];
}

// Dense coarse solve z = (L L^T)^{-1} r, L column-major lower triangular.
__global__ void __launch_bounds__(1024)
k_chol_solve(int64_t n, const double *__restrict__ L, const double *__restrict__ r,
             double *__restrict__ z) {
    extern __shared__ double y[];
    __shared__ double piv;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) y[i] = r[i];
    __syncthreads();
    for (int64_t j = 0; j < n; j++) {  // L y = r
        if (threadIdx.x == 0) {
            piv = y[j] / L[j + j * n];
            y[j] = piv;
        }
        __syncthreads();
        const double pj = piv;
        for (int64_t i = j + 1 + threadIdx.x; i < n; i += blockDim.x) y[i] -= L[i + j * n] * pj;
        __syncthreads();
    }
    for (int64_t j = n - 1; j >= 0; j--) {  // L^T z = y
        if (threadIdx.x == 0) {
            piv = y[j] / L[j + j * n];
            y[j] = piv;
        }
        __syncthreads();
        const double pj = piv;
        for (int64_t i = threadIdx.x; i < j; i += blockDim.x) y[i] -= L[j + i * n] * pj;
        __syncthreads();
    }
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) z[i] = y[i];
}

static int coarse_enqueue(amgp_hier *h, const double *r, double *z) {
    amgp_ctx *ctx = h->ctx;
    const int l = h->nlev - 1;
    amgp_mat *A = h->A[l];
    const int64_t n = A->nrows;
    if (n == 0) return AMGP_OK;
    if (h->coarse_solver == AMGP_COARSE_DENSE_DIRECT) {
        if (!h->cholL) return amgp_fail(AMGP_EINVAL, "dense_direct coarse solver without factor");
        k_chol_solve<<<1, 256, n * sizeof(double), cur_stream(ctx)>>>(n, h->cholL, r, z);
        AMGP_CHECK_LAUNCH(ctx);
        return AMGP_OK;
    }
    if (h->coarse_solver == AMGP_COARSE_SMOOTHER)
        return smoother_enqueue(ctx, A, h->m[l], h->plan[l], r, nullptr, z, h->work[l]);
    const size_t reg_smem = 16 * (size_t)A->nrows + 10 * (size_t)A->stored + 64;
    // (the single-CTA kernels address rows by SELL position: identity order only)
    if (!A->halo && !A->perm && A->stored <= COARSE_REG_SLOTS && A->ncols < 32768 && reg_smem <= COARSE_SMEM_BYTES) {
        k_coarse_l1_reg<<<1, 1024, reg_smem, cur_stream(ctx)>>>(view_of(A), h->m[l], r, z, h->coarse_sweeps);
        AMGP_CHECK_LAUNCH(ctx);
        return AMGP_OK;
    }
    if (!A->halo && !A->perm && coarse_smem(A) <= COARSE_SMEM_BYTES) {
        k_coarse_l1<<<1, 1024, coarse_smem(A), cur_stream(ctx)>>>(view_of(A), h->m[l], r, z, h->coarse_sweeps);
        AMGP_CHECK_LAUNCH(ctx);
        return AMGP_OK;
    }
    return smoother_enqueue(ctx, A, h->m[l], h->coarse_plan, r, nullptr, z, h->work[l]);
}

static int vcycle_level(amgp_hier *h, int l, const double *r, double *z) {
    if (l == h->nlev - 1) return coarse_enqueue(h, r, z);
    amgp_ctx *ctx = h->ctx;
    amgp_mat *A = h->A[l];
    const SmootherPlan &p = h->plan[l];
    double *x = h->xpre[l];
    AMGP_TRY(smoother_enqueue(ctx, A, h->m[l], p, r, nullptr, x, h->work[l]));
    AMGP_TRY(residual_enqueue(ctx, A, r, x, h->res[l]));
    AMGP_TRY(spmv_enqueue(ctx, h->R[l], h->res[l], h->rl[l + 1]));
    AMGP_TRY(vcycle_level(h, l + 1, h->rl[l + 1], h->zl[l + 1]));
    AMGP_TRY(prolong_add_enqueue(ctx, h->P[l], h->zl[l + 1], x));
    return smoother_enqueue(ctx, A, h->m[l], p, r, x, z, h->work[l]);
}

// Enqueue one V-cycle (graph replay when enabled).  Caller holds h->mu.
int vcycle_enqueue(amgp_hier *h, const double *r, double *z) {
    amgp_ctx *ctx = h->ctx;
    if (!h->use_graph) return vcycle_level(h, 0, r, z);
    if (!h->gexec || h->g_r != r || h->g_z != z) {
        if (h->gexec) {
            cudaGraphExecDestroy(h->gexec);
            h->gexec = nullptr;
        }
        cudaGraph_t graph = nullptr;
        const int64_t before = ctx->launches.load();
        // Capture on the hierarchy's private stream, named by this thread's
        // capture override (amgp_common.cuh): other host threads keep
        // enqueueing on the context stream meanwhile, and none of their work
        // can land in the graph.
        if (!h->cap_stream) AMGP_CUDA(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
        cudaError_t e = cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) return amgp_cuda_fail(e, "cudaStreamBeginCapture", __FILE__, __LINE__);
        amgp_capture = {ctx, h->cap_stream};
        int st = vcycle_level(h, 0, r, z);
        amgp_capture = {};
        e = cudaStreamEndCapture(h->cap_stream, &graph);
        const int64_t nodes = ctx->launches.load() - before;
        ctx->launches.fetch_sub(nodes);  // captured, not launched
        if (st != AMGP_OK) {
            if (graph) cudaGraphDestroy(graph);
            return st;
        }
        if (e != cudaSuccess) return amgp_cuda_fail(e, "cudaStreamEndCapture", __FILE__, __LINE__);
        e = cudaGraphInstantiate(&h->gexec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) {
            h->gexec = nullptr;
            return amgp_cuda_fail(e, "cudaGraphInstantiate", __FILE__, __LINE__);
        }
        h->g_r = r;
        h->g_z = z;
        h->g_nodes = nodes;
    }
    AMGP_CUDA(cudaGraphLaunch(h->gexec, cur_stream(ctx)));
    ctx->launches.fetch_add(h->g_nodes);
    return AMGP_OK;
}

static void hier_free_buffers(amgp_hier *h) {
    for (auto *v : {&h->rl, &h->zl, &h->xpre, &h->res, &h->work})
        for (double *p : *v) cudaFree(p);
    cudaFree(h->cholL);
    if (h->gexec) cudaGraphExecDestroy(h->gexec);
    if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
}

extern "C" int amgp_hier_create(amgp_ctx *ctx, int nlevels, amgp_mat *const *A,
                                const double *const *m, amgp_mat *const *P, amgp_mat *const *R,
                                int coarse_solver, int coarse_sweeps, amgp_hier **out) {
    if (!ctx || !out || nlevels < 1 || !A || !m)
        return amgp_fail(AMGP_EINVAL, "amgp_hier_create: bad argument");
    if (coarse_solver != AMGP_COARSE_L1_JACOBI && coarse_solver != AMGP_COARSE_DENSE_DIRECT &&
        coarse_solver != AMGP_COARSE_SMOOTHER)
        return amgp_fail(AMGP_EINVAL, "unknown coarse solver");
    if (coarse_sweeps < 1) return amgp_fail(AMGP_EINVAL, "coarse_sweeps must be >= 1");
    // operand length of a (possibly distributed) matrix: its own columns
    auto own = [](const amgp_mat *M) { return M->halo ? M->halo->nown : M->ncols; };
    for (int l = 0; l < nlevels; l++) {
        if (!A[l] || A[l]->nrows != own(A[l]) || (A[l]->nrows > 0 && !m[l]))
            return amgp_fail(AMGP_EINVAL, "level matrix must be square with a diagonal");
        if (l < nlevels - 1) {
            if (!P || !R || !P[l] || !R[l]) return amgp_fail(AMGP_EINVAL, "missing prolongator");
            if (P[l]->nrows != A[l]->nrows || own(P[l]) != A[l + 1]->nrows ||
                R[l]->nrows != A[l + 1]->nrows || own(R[l]) != A[l]->nrows)
                return amgp_fail(AMGP_EINVAL, "dimension mismatch in prolongator");
        }
    }
    AMGP_CUDA(cudaSetDevice(ctx->device));
    amgp_hier *h = new amgp_hier();
    h->ctx = ctx;
    h->nlev = nlevels;
    h->coarse_solver = coarse_solver;
    h->coarse_sweeps = coarse_sweeps;
    amgp_smoother_cfg ccfg{AMGP_L1_JACOBI, coarse_sweeps, 0.0, 1.0, nullptr};
    make_smoother_plan(&ccfg, &h->coarse_plan);
    amgp_smoother_cfg dflt{AMGP_L1_JACOBI, 1, 0.0, 1.0, nullptr};
    SmootherPlan dp;
    make_smoother_plan(&dflt, &dp);
    h->rl.assign(nlevels, nullptr);
    h->zl.assign(nlevels, nullptr);
    h->xpre.assign(nlevels, nullptr);
    h->res.assign(nlevels, nullptr);
    h->work.assign(nlevels, nullptr);
    cudaError_t e = cudaSuccess;
    for (int l = 0; l < nlevels; l++) {
        h->A.push_back(A[l]);
        h->m.push_back(m[l]);
        h->P.push_back(l < nlevels - 1 ? P[l] : nullptr);
        h->R.push_back(l < nlevels - 1 ? R[l] : nullptr);
        h->plan.push_back(dp);
        const size_t n = (size_t)std::max<int64_t>(A[l]->nrows, 1);
        if (e == cudaSuccess && l > 0) e = cudaMalloc(&h->rl[l], n * sizeof(double));
        if (e == cudaSuccess && l > 0) e = cudaMalloc(&h->zl[l], n * sizeof(double));
        if (e == cudaSuccess) e = cudaMalloc(&h->xpre[l], n * sizeof(double));
        if (e == cudaSuccess) e = cudaMalloc(&h->res[l], n * sizeof(double));
        if (e == cudaSuccess) e = cudaMalloc(&h->work[l], smoother_work_doubles(n) * sizeof(double));
    }
    if (e != cudaSuccess) {
        hier_free_buffers(h);
        delete h;
        return amgp_cuda_fail(e, "hierarchy buffers", __FILE__, __LINE__);
    }
    // K6 stages the coarsest level in up to 227 KB of dynamic shared memory
    cudaFuncSetAttribute(k_coarse_l1, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         COARSE_SMEM_BYTES);
    cudaFuncSetAttribute(k_coarse_l1_reg, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         COARSE_SMEM_BYTES);
    cudaFuncSetAttribute(k_chol_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    *out = h;
    return AMGP_OK;
}

extern "C" int amgp_hier_set_smoother(amgp_hier *h, int level, const amgp_smoother_cfg *cfg) {
    if (!h) return amgp_fail(AMGP_EINVAL, "null hierarchy");
    SmootherPlan p;
    AMGP_TRY(make_smoother_plan(cfg, &p));
    std::lock_guard<std::mutex> cg(h->ctx->mu);
    std::lock_guard<std::mutex> g(h->mu);
    if (level >= h->nlev) return amgp_fail(AMGP_EINVAL, "level out of range");
    for (int l = 0; l < h->nlev; l++)
        if (level < 0 || l == level) h->plan[l] = p;
    if (h->gexec) {  // invalidate the captured graph
        cudaStreamSynchronize(cur_stream(h->ctx));
        cudaGraphExecDestroy(h->gexec);
        h->gexec = nullptr;
    }
    return AMGP_OK;
}

extern "C" int amgp_hier_set_coarse_cholesky(amgp_hier *h, const double *L) {
    if (!h || !L) return amgp_fail(AMGP_EINVAL, "bad argument");
    const int64_t n = h->A[h->nlev - 1]->nrows;
    if (n * (int64_t)sizeof(double) > 200 * 1024)
        return amgp_fail(AMGP_EINVAL, "coarse level too large for the dense device solve");
    std::lock_guard<std::mutex> cg(h->ctx->mu);
    std::lock_guard<std::mutex> g(h->mu);
    cudaFree(h->cholL);
    h->cholL = nullptr;
    AMGP_CUDA(cudaMalloc(&h->cholL, std::max<int64_t>(n * n, 1) * sizeof(double)));
    AMGP_CUDA(cudaMemcpy(h->cholL, L, n * n * sizeof(double), cudaMemcpyHostToDevice));
    h->coarse_solver = AMGP_COARSE_DENSE_DIRECT;
    if (h->gexec) {
        cudaGraphExecDestroy(h->gexec);
        h->gexec = nullptr;
    }
    return AMGP_OK;
}

extern "C" int amgp_hier_use_graph(amgp_hier *h, int enable) {
    if (!h) return amgp_fail(AMGP_EINVAL, "null hierarchy");
    std::lock_guard<std::mutex> cg(h->ctx->mu);
    std::lock_guard<std::mutex> g(h->mu);
    h->use_graph = enable != 0;
    return AMGP_OK;
}

extern "C" int amgp_hier_info(amgp_hier *h, int *nlevels) {
    if (!h) return amgp_fail(AMGP_EINVAL, "null hierarchy");
    if (nlevels) *nlevels = h->nlev;
    return AMGP_OK;
}

extern "C" int amgp_hier_destroy(amgp_hier *h) {
    if (!h) return AMGP_OK;
    cudaSetDevice(h->ctx->device);
    cudaStreamSynchronize(cur_stream(h->ctx));
    hier_free_buffers(h);
    delete h;
    return AMGP_OK;
}

extern "C" int amgp_vcycle_apply(amgp_hier *h, const double *r, double *z) {
    if (!h) return amgp_fail(AMGP_EINVAL, "null hierarchy");
    if (h->A[0]->nrows > 0 && (!r || !z)) return amgp_fail(AMGP_EINVAL, "null vector");
    if (r == z) return amgp_fail(AMGP_EINVAL, "r and z must not alias");
    AMGP_CUDA(cudaSetDevice(h->ctx->device));
    std::lock_guard<std::mutex> cg(h->ctx->mu);
    std::lock_guard<std::mutex> g(h->mu);
    return vcycle_enqueue(h, r, z);
}

// exposed to pcg.cu
int64_t hier_rows(const amgp_hier *h) { return h->A[0]->nrows; }
std::mutex &hier_mutex(amgp_hier *h) { return h->mu; }
