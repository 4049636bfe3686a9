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
#include <cooperative_groups.h>

#include <algorithm>
#include <vector>

#include "epilogues.cuh"

namespace cg = cooperative_groups;

// ---------------------------------------------------------------- V-cycle tail
// The smallest levels of a hierarchy are latency bound: ~20 us per launch for
// a few thousand rows.  K8 runs the whole bottom of the V-cycle (pre-smooth,
// residual, restriction on every tail level, the coarse solve, prolongation
// and post-smoothing back up) as ONE cooperative kernel: one CTA per SM, every
// step a grid-wide phase separated by grid.sync().  Within a phase each CTA
// takes whole 32-row slices, forms all (row, slot) products in parallel into
// shared memory and sums each row in slot order -- the per-row arithmetic of
// the regular kernels, so the results are bitwise unchanged.
#define TAIL_MAX_LEV 8
#define TAIL_MAX_K 32
#define TAIL_THREADS 512
#define TAIL_CHUNK 192
#define TAIL_MAX_STORED (4LL << 20)
#define TAIL_MAX_ROWS 65536

struct TailLev {
    SellView A, P, R;  // P: this level <- next; R: next <- this
    const double *m;
    const double *r;   // rhs (levels >= 1 of the tail; level 0 comes as a kernel argument)
    double *z, *xpre, *res, *work;
    int64_t n;
    int wA, wP, wR;  // widest slice of A, P, R (picks the phase schedule)
    int family, degree;
    double rho;
    double coef[3 * TAIL_MAX_K];
};

struct TailDesc {
    int nlev, coarse_sweeps;
    TailLev lev[TAIL_MAX_LEV];
};

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
    int64_t g_nodes = 0;
    // cooperative tail (K8)
    // Off by default: measured on B200 (128^3 SA, levels 3-5 in the tail)
    // 12.4 ms vs 11.6 ms per solve -- the grid barriers plus the sequential
    // 300-500-term row sums of the coarse SA levels cost more than the
    // launches they replace (profiles/r01_summary.md).
    bool use_tail = false;
    bool tail_dirty = true;
    int tail_start = -1;  // first level run by the tail kernel (-1: none)
    TailDesc *d_tail = nullptr;
    size_t tail_smem = 0;
    int tail_grid = 0;
    std::mutex mu;
};

#define COARSE_SMEM_BYTES (227 * 1024)
#define TAIL_COARSE_SMEM (200 * 1024)  // K8's coarse phase (products staged)
static inline size_t tail_coarse_smem(const amgp_mat *A) {
    return 16 * (size_t)A->nrows + 20 * (size_t)A->stored + 64;
}

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
        k_chol_solve<<<1, 256, n * sizeof(double), ctx->stream>>>(n, h->cholL, r, z);
        AMGP_CHECK_LAUNCH(ctx);
        return AMGP_OK;
    }
    if (h->coarse_solver == AMGP_COARSE_SMOOTHER)
        return smoother_enqueue(ctx, A, h->m[l], h->plan[l], r, nullptr, z, h->work[l]);
    const size_t reg_smem = 16 * (size_t)A->nrows + 10 * (size_t)A->stored + 64;
    if (!A->halo && A->stored <= COARSE_REG_SLOTS && A->ncols < 32768 && reg_smem <= COARSE_SMEM_BYTES) {
        k_coarse_l1_reg<<<1, 1024, reg_smem, ctx->stream>>>(view_of(A), h->m[l], r, z, h->coarse_sweeps);
        AMGP_CHECK_LAUNCH(ctx);
        return AMGP_OK;
    }
    if (!A->halo && coarse_smem(A) <= COARSE_SMEM_BYTES) {
        k_coarse_l1<<<1, 1024, coarse_smem(A), ctx->stream>>>(view_of(A), h->m[l], r, z, h->coarse_sweeps);
        AMGP_CHECK_LAUNCH(ctx);
        return AMGP_OK;
    }
    return smoother_enqueue(ctx, A, h->m[l], h->coarse_plan, r, nullptr, z, h->work[l]);
}

// ---------------------------------------------------------------- K8 device side
// One grid-wide phase: y = A xg row by row, then epi(row, y).  Short rows
// (the matrix's widest slice <= TAIL_SHORT slots): every thread of the grid
// owns rows (a warp = one slice) and sums its slots in order.  Long rows: a
// CTA owns a slice, its warps form the slot products (8 independent loads in
// flight per thread) into shared memory, warp 0 sums them in slot order.
// Operands written by earlier phases are read with ld.global.cg (L2), never
// through the non-coherent path.
#define TAIL_SHORT 16
template <class Epi>
__device__ void tail_phase(const SellView &A, int wmax, const double *xg, const Epi &epi,
                           double *prod) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (!Epi::kSpmv || wmax <= TAIL_SHORT) {
        const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
        for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < A.nslices * 32;
             row += nthr) {
            double y = 0.0;
            if (Epi::kSpmv) {
                const int64_t s = row >> 5, base = __ldg(A.slice_ptr + s);
                const int w = (int)((__ldg(A.slice_ptr + s + 1) - base) >> 5);
                const int32_t *cp = A.col + base + (row & 31);
                const double *vp = A.val + base + (row & 31);
                int32_t cc[TAIL_SHORT];
                double pv[TAIL_SHORT];
#pragma unroll
                for (int j = 0; j < TAIL_SHORT; j++) cc[j] = j < w ? __ldg(cp + j * 32) : -1;
#pragma unroll
                for (int j = 0; j < TAIL_SHORT; j++)
                    pv[j] = cc[j] >= 0 ? __dmul_rn(__ldg(vp + j * 32), __ldcg(xg + cc[j])) : 0.0;
#pragma unroll
                for (int j = 0; j < TAIL_SHORT; j++)
                    if (cc[j] >= 0) y = __dadd_rn(y, pv[j]);
            }
            if (row < A.nrows) epi(row, y);
        }
        return;
    }
    constexpr int NW = TAIL_THREADS / 32;
    for (int64_t s = blockIdx.x; s < A.nslices; s += gridDim.x) {
        const int64_t row = s * 32 + lane;
        const int64_t base = __ldg(A.slice_ptr + s);
        const int w = (int)((__ldg(A.slice_ptr + s + 1) - base) >> 5);
        double sum = 0.0;
        for (int j0 = 0; j0 < w; j0 += TAIL_CHUNK) {
            const int jn = min(TAIL_CHUNK, w - j0);
            for (int j = warp; j < jn; j += NW * 8) {
                int32_t cc[8];
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const int jj = j + u * NW;
                    cc[u] = jj < jn ? __ldg(A.col + base + (int64_t)(j0 + jj) * 32 + lane) : -2;
                }
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const int jj = j + u * NW;
                    if (cc[u] == -2) continue;
                    const double v = __ldg(A.val + base + (int64_t)(j0 + jj) * 32 + lane);
                    prod[jj * 32 + lane] = cc[u] >= 0 ? __dmul_rn(v, __ldcg(xg + cc[u])) : 0.0;
                }
            }
            __syncthreads();
            if (warp == 0)
                for (int j = 0; j < jn; j++) sum = __dadd_rn(sum, prod[j * 32 + lane]);
            __syncthreads();
        }
        if (warp == 0 && row < A.nrows) epi(row, sum);
    }
}

template <bool FIRST, bool LAST, bool X0>
__device__ __forceinline__ void tail_cheb4(const TailLev &L, const double *b, const double *xg,
                                           double *r, double *zn, double *x, int j, double *prod) {
    const double *c = L.coef + 3 * (j - 1);
    tail_phase(L.A, L.wA, xg, Cheb4Step<FIRST, LAST, X0>{L.m, b, xg, r, zn, x, c[0], c[1], c[2]}, prod);
}

template <bool FIRST, bool LAST, bool X0>
__device__ __forceinline__ void tail_cheb1(const TailLev &L, const double *b, const double *xg,
                                           double *r, double *dn, double *x, int j, double *prod) {
    const double c0 = j == 0 ? L.coef[0] : L.coef[1 + 2 * (j - 1)];
    const double c1 = j == 0 ? 0.0 : L.coef[2 + 2 * (j - 1)];
    if (L.rho == 1.0)
        tail_phase(L.A, L.wA, xg, Cheb1Step<FIRST, LAST, X0, true>{L.m, b, xg, r, dn, x, c0, c1, L.rho}, prod);
    else
        tail_phase(L.A, L.wA, xg, Cheb1Step<FIRST, LAST, X0, false>{L.m, b, xg, r, dn, x, c0, c1, L.rho}, prod);
}

// smoother_enqueue (smoother.cu) as grid-wide phases, same buffers and order
__device__ void tail_smoother(const TailLev &L, const double *b, const double *x0, double *x,
                              double *prod, cg::grid_group &grid) {
    const int64_t n = L.n;
    const int k = L.degree;
    double *r = L.work, *buf[2] = {L.work + 2 * n, L.work + n}, *tmp = L.work + 3 * n;
    const bool hx0 = x0 != nullptr;
    if (L.family == AMGP_L1_JACOBI) {
        const double *xin = x0;
        for (int s = 1; s <= k; s++) {
            double *xout = ((k - s) % 2 == 0) ? x : tmp;
            if (s == 1 && !hx0) tail_phase(L.A, L.wA, nullptr, L1Sweep<false>{L.m, b, nullptr, xout}, prod);
            else tail_phase(L.A, L.wA, xin, L1Sweep<true>{L.m, b, xin, xout}, prod);
            grid.sync();
            xin = xout;
        }
        return;
    }
    if (L.family == AMGP_CHEB4 || L.family == AMGP_OPT_CHEB4) {
        for (int j = 1; j <= k; j++) {
            const double *xg = (j == 1) ? x0 : buf[(j - 1) & 1];
            double *zn = buf[j & 1];
            if (j == 1 && k == 1) {
                if (hx0) tail_cheb4<true, true, true>(L, b, xg, r, zn, x, j, prod);
                else tail_cheb4<true, true, false>(L, b, xg, r, zn, x, j, prod);
            } else if (j == 1) {
                if (hx0) tail_cheb4<true, false, true>(L, b, xg, r, zn, x, j, prod);
                else tail_cheb4<true, false, false>(L, b, xg, r, zn, x, j, prod);
            } else if (j == k) {
                tail_cheb4<false, true, false>(L, b, xg, r, zn, x, j, prod);
            } else {
                tail_cheb4<false, false, false>(L, b, xg, r, zn, x, j, prod);
            }
            grid.sync();
        }
        return;
    }
    for (int j = 0; j < k; j++) {  // opt_cheb1
        const double *xg = (j == 0) ? x0 : buf[j & 1];
        double *dn = buf[(j + 1) & 1];
        const bool last = (j == k - 1);
        if (j == 0) {
            if (last) {
                if (hx0) tail_cheb1<true, true, true>(L, b, xg, r, dn, x, j, prod);
                else tail_cheb1<true, true, false>(L, b, xg, r, dn, x, j, prod);
            } else {
                if (hx0) tail_cheb1<true, false, true>(L, b, xg, r, dn, x, j, prod);
                else tail_cheb1<true, false, false>(L, b, xg, r, dn, x, j, prod);
            }
        } else if (last) {
            tail_cheb1<false, true, false>(L, b, xg, r, dn, x, j, prod);
        } else {
            tail_cheb1<false, false, false>(L, b, xg, r, dn, x, j, prod);
        }
        grid.sync();
    }
}

// coarsest level: k_coarse_l1's arithmetic, run by CTA 0 in shared memory
__device__ void tail_coarse(const TailLev &L, const double *b, double *x, int sweeps, double *sh) {
    const SellView &A = L.A;
    const int64_t n = A.nrows;
    const int64_t stored = A.slice_ptr[A.nslices];
    double *buf[2] = {sh, sh + n};
    double *pv = sh + 2 * n;
    double *prod = pv + stored;
    int32_t *pc = (int32_t *)(prod + stored);
    for (int64_t e = threadIdx.x; e < stored; e += blockDim.x) {
        pv[e] = A.val[e];
        pc[e] = A.col[e];
    }
    __syncthreads();
    for (int s = 1; s <= sweeps; s++) {
        const double *xin = buf[(s - 1) & 1];
        double *xout = buf[s & 1];
        if (s > 1) {
            for (int64_t e = threadIdx.x; e < stored; e += blockDim.x) {
                const int32_t c = pc[e];
                prod[e] = c >= 0 ? __dmul_rn(pv[e], xin[c]) : 0.0;
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
                for (int j = 0; j < w; j++) y = __dadd_rn(y, pp[j * 32]);
            }
            const double rr = __dsub_rn(__ldcg(b + row), y);
            xout[row] = __dadd_rn(s > 1 ? xin[row] : 0.0, __ddiv_rn(rr, L.m[row]));
        }
        __syncthreads();
    }
    for (int64_t row = threadIdx.x; row < n; row += blockDim.x) x[row] = buf[sweeps & 1][row];
}

__global__ void __launch_bounds__(TAIL_THREADS, 1)
k_vcycle_tail(const TailDesc *__restrict__ D, const double *r0, double *z0) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double smem[];
    const int L = D->nlev;
    for (int t = 0; t < L - 1; t++) {  // down: amg.py:310-312
        const TailLev &V = D->lev[t];
        const double *r = t == 0 ? r0 : V.r;
        tail_smoother(V, r, nullptr, V.xpre, smem, grid);
        tail_phase(V.A, V.wA, V.xpre, SpmvEpi<1>{r, V.res}, smem);
        grid.sync();
        tail_phase(V.R, V.wR, V.res, SpmvEpi<0>{nullptr, (double *)D->lev[t + 1].r}, smem);
        grid.sync();
    }
    {  // coarsest: amg.py:299-300
        const TailLev &C = D->lev[L - 1];
        if (blockIdx.x == 0) tail_coarse(C, L == 1 ? r0 : C.r, L == 1 ? z0 : C.z, D->coarse_sweeps, smem);
        grid.sync();
    }
    for (int t = L - 2; t >= 0; t--) {  // up: amg.py:314-315
        const TailLev &V = D->lev[t];
        const double *r = t == 0 ? r0 : V.r;
        tail_phase(V.P, V.wP, D->lev[t + 1].z, SpmvEpi<2>{nullptr, V.xpre}, smem);
        grid.sync();
        tail_smoother(V, r, V.xpre, t == 0 ? z0 : V.z, smem, grid);
    }
}

// ---------------------------------------------------------------- K8 host side
static void tail_plan(amgp_hier *h) {
    h->tail_start = -1;
    if (!h->use_tail || h->coarse_solver != AMGP_COARSE_L1_JACOBI) return;
    const int Lc = h->nlev - 1;
    amgp_mat *C = h->A[Lc];
    if (C->halo || tail_coarse_smem(C) > TAIL_COARSE_SMEM || C->nrows > TAIL_MAX_ROWS) return;
    int start = Lc;
    for (int l = Lc - 1; l >= 0 && Lc - l < TAIL_MAX_LEV; l--) {
        const amgp_mat *A = h->A[l];
        if (A->halo || h->P[l]->halo || h->R[l]->halo) break;
        if (A->stored > TAIL_MAX_STORED || A->nrows > TAIL_MAX_ROWS) break;
        if (h->plan[l].degree > TAIL_MAX_K) break;
        start = l;
    }
    if (start == Lc) return;  // a coarse solve alone is already one kernel
    h->tail_start = start;
}

static int tail_prepare(amgp_hier *h) {
    if (!h->tail_dirty) return AMGP_OK;
    tail_plan(h);
    h->tail_dirty = false;
    if (h->tail_start < 0) return AMGP_OK;
    TailDesc d;
    memset(&d, 0, sizeof(d));
    d.nlev = h->nlev - h->tail_start;
    d.coarse_sweeps = h->coarse_sweeps;
    for (int t = 0; t < d.nlev; t++) {
        const int l = h->tail_start + t;
        TailLev &V = d.lev[t];
        V.A = view_of(h->A[l]);
        V.wA = h->A[l]->max_width;
        if (l < h->nlev - 1) {
            V.P = view_of(h->P[l]);
            V.R = view_of(h->R[l]);
            V.wP = h->P[l]->max_width;
            V.wR = h->R[l]->max_width;
        }
        V.m = h->m[l];
        V.r = h->rl[l];
        V.z = h->zl[l];
        V.xpre = h->xpre[l];
        V.res = h->res[l];
        V.work = h->work[l];
        V.n = h->A[l]->nrows;
        const SmootherPlan &p = (l == h->nlev - 1) ? h->coarse_plan : h->plan[l];
        V.family = p.family;
        V.degree = p.degree;
        V.rho = p.rho;
        std::copy(p.coef.begin(), p.coef.begin() + std::min<size_t>(p.coef.size(), 3 * TAIL_MAX_K), V.coef);
    }
    if (!h->d_tail) AMGP_CUDA(cudaMalloc(&h->d_tail, sizeof(TailDesc)));
    AMGP_CUDA(cudaStreamSynchronize(h->ctx->stream));
    AMGP_CUDA(cudaMemcpy(h->d_tail, &d, sizeof(TailDesc), cudaMemcpyHostToDevice));
    h->tail_smem = std::max<size_t>((size_t)TAIL_CHUNK * 32 * sizeof(double), tail_coarse_smem(h->A[h->nlev - 1]));
    AMGP_CUDA(cudaFuncSetAttribute(k_vcycle_tail, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)h->tail_smem));
    int per_sm = 0, nsm = 0;
    AMGP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_vcycle_tail, TAIL_THREADS,
                                                            h->tail_smem));
    AMGP_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, h->ctx->device));
    if (per_sm < 1) {
        h->tail_start = -1;
        return AMGP_OK;
    }
    h->tail_grid = nsm;  // one CTA per SM
    return AMGP_OK;
}

static int tail_enqueue(amgp_hier *h, const double *r, double *z) {
    amgp_ctx *ctx = h->ctx;
    const TailDesc *d = h->d_tail;
    void *args[] = {(void *)&d, (void *)&r, (void *)&z};
    AMGP_CUDA(cudaLaunchCooperativeKernel((const void *)k_vcycle_tail, dim3(h->tail_grid),
                                          dim3(TAIL_THREADS), args, h->tail_smem, ctx->stream));
    ctx->launches.fetch_add(1);
    return AMGP_OK;
}

static int vcycle_level(amgp_hier *h, int l, const double *r, double *z) {
    if (l == h->tail_start) return tail_enqueue(h, r, z);
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
    if (h->tail_dirty) {  // (re)plan the cooperative tail before any capture
        if (h->gexec) {
            cudaGraphExecDestroy(h->gexec);
            h->gexec = nullptr;
        }
        AMGP_TRY(tail_prepare(h));
    }
    if (!h->use_graph) return vcycle_level(h, 0, r, z);
    if (!h->gexec || h->g_r != r || h->g_z != z) {
        if (h->gexec) {
            cudaGraphExecDestroy(h->gexec);
            h->gexec = nullptr;
        }
        cudaGraph_t graph = nullptr;
        const int64_t before = ctx->launches.load();
        AMGP_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
        int st = vcycle_level(h, 0, r, z);
        cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
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
    AMGP_CUDA(cudaGraphLaunch(h->gexec, ctx->stream));
    ctx->launches.fetch_add(h->g_nodes);
    return AMGP_OK;
}

static void hier_free_buffers(amgp_hier *h) {
    for (auto *v : {&h->rl, &h->zl, &h->xpre, &h->res, &h->work})
        for (double *p : *v) cudaFree(p);
    cudaFree(h->cholL);
    cudaFree(h->d_tail);
    if (h->gexec) cudaGraphExecDestroy(h->gexec);
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
    std::lock_guard<std::mutex> g(h->mu);
    if (level >= h->nlev) return amgp_fail(AMGP_EINVAL, "level out of range");
    for (int l = 0; l < h->nlev; l++)
        if (level < 0 || l == level) h->plan[l] = p;
    h->tail_dirty = true;
    if (h->gexec) {  // invalidate the captured graph
        cudaStreamSynchronize(h->ctx->stream);
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
    std::lock_guard<std::mutex> g(h->mu);
    cudaFree(h->cholL);
    h->cholL = nullptr;
    AMGP_CUDA(cudaMalloc(&h->cholL, std::max<int64_t>(n * n, 1) * sizeof(double)));
    AMGP_CUDA(cudaMemcpy(h->cholL, L, n * n * sizeof(double), cudaMemcpyHostToDevice));
    h->coarse_solver = AMGP_COARSE_DENSE_DIRECT;
    h->tail_dirty = true;
    if (h->gexec) {
        cudaGraphExecDestroy(h->gexec);
        h->gexec = nullptr;
    }
    return AMGP_OK;
}

extern "C" int amgp_hier_use_graph(amgp_hier *h, int enable) {
    if (!h) return amgp_fail(AMGP_EINVAL, "null hierarchy");
    std::lock_guard<std::mutex> g(h->mu);
    h->use_graph = enable != 0;
    return AMGP_OK;
}

extern "C" int amgp_hier_use_tail(amgp_hier *h, int enable) {
    if (!h) return amgp_fail(AMGP_EINVAL, "null hierarchy");
    std::lock_guard<std::mutex> g(h->mu);
    h->use_tail = enable != 0;
    h->tail_dirty = true;
    return AMGP_OK;
}

extern "C" int amgp_hier_info(amgp_hier *h, int *nlevels, int *tail_start) {
    if (!h) return amgp_fail(AMGP_EINVAL, "null hierarchy");
    std::lock_guard<std::mutex> g(h->mu);
    if (h->tail_dirty) AMGP_TRY(tail_prepare(h));
    if (nlevels) *nlevels = h->nlev;
    if (tail_start) *tail_start = h->tail_start;
    return AMGP_OK;
}

extern "C" int amgp_hier_destroy(amgp_hier *h) {
    if (!h) return AMGP_OK;
    cudaSetDevice(h->ctx->device);
    cudaStreamSynchronize(h->ctx->stream);
    hier_free_buffers(h);
    delete h;
    return AMGP_OK;
}

extern "C" int amgp_vcycle_apply(amgp_hier *h, const double *r, double *z) {
    if (!h) return amgp_fail(AMGP_EINVAL, "null hierarchy");
    if (h->A[0]->nrows > 0 && (!r || !z)) return amgp_fail(AMGP_EINVAL, "null vector");
    if (r == z) return amgp_fail(AMGP_EINVAL, "r and z must not alias");
    AMGP_CUDA(cudaSetDevice(h->ctx->device));
    std::lock_guard<std::mutex> g(h->mu);
    return vcycle_enqueue(h, r, z);
}

// exposed to pcg.cu
int64_t hier_rows(const amgp_hier *h) { return h->A[0]->nrows; }
std::mutex &hier_mutex(amgp_hier *h) { return h->mu; }
