// K7: PCG / FCG on the device (reference krylov.py:45-120).
//
// Every PCG scalar stays on the device; the host only reads back the relative
// residual (and the breakdown flag) once per iteration to decide termination.
// Dots are deterministic: a fixed grid, per-thread sequential partials,
// xor-butterfly warp sums, a fixed block tree, and the last block to finish
// (atomic ticket) folds the per-block partials in block order -- the same
// bits on every run.  Across GPUs the per-rank totals are all-gathered and
// folded in rank order (dist.cu), so every rank holds identical scalars.
// The dot order differs from OpenBLAS ddot, hence the reference's +-1
// iteration tolerance.
//
// One iteration (fusions in brackets):
//   [Ad = A d ; d.Ad (; r.d)] -> dAd, alpha, breakdown          k_pcg_spmv_dot
//       (distributed: halo-exchanged SpMV, then k_pcg_dot2)
//   [x += alpha d ; r -= alpha Ad ; r.r] -> relres              k_pcg_update
//   z = V(r)                                                    V-cycle graph
//   [r.z | z.Ad] -> beta                                        k_pcg_dot
//   d = z +- beta d                                             k_pcg_dir
#include <math.h>

#include <algorithm>
#include <chrono>

#include "rows.cuh"

int vcycle_enqueue(amgp_hier *h, const double *r, double *z);
int64_t hier_rows(const amgp_hier *h);
std::mutex &hier_mutex(amgp_hier *h);
int allreduce_sum_ordered(amgp_ctx *ctx, const double *local, int nv, double *out);

enum {
    S_BNORM = 0, S_RZ, S_DAD, S_ALPHA, S_BETA, S_RELRES, S_BRK, S_RR, S_BB, S_AUX,
    S_COUNT,
    S_LOC = 16,  // per-rank reduction totals (distributed)
    S_GLB = 32   // rank-folded totals
};

// what the folded totals of a reduction become (krylov.py line numbers)
enum { OP_BNORM, OP_RELRES, OP_RZ, OP_DAD, OP_DAD_FCG, OP_BETA, OP_BETA_FCG, OP_CG1 };

#define RB 256          // reduction block
#define RGRID_MAX 1184  // 148 SMs x 8

__device__ __forceinline__ void apply_op(int op, const double *t, double *sc) {
    switch (op) {
        case OP_BNORM:  // :67
            sc[S_BNORM] = sqrt(t[0]);
            sc[S_BRK] = 0.0;
            break;
        case OP_RELRES:  // :75, :103
            sc[S_RELRES] = __ddiv_rn(sqrt(t[0]), sc[S_BNORM]);
            break;
        case OP_RZ:  // :92
            sc[S_RZ] = t[0];
            sc[S_BRK] = 0.0;
            break;
        case OP_DAD:
        case OP_DAD_FCG: {  // :96-100
            const double dAd = t[0];
            sc[S_DAD] = dAd;
            if (dAd <= 0.0) sc[S_BRK] = 1.0;
            sc[S_ALPHA] = op == OP_DAD_FCG ? __ddiv_rn(t[1], dAd) : __ddiv_rn(sc[S_RZ], dAd);
            break;
        }
        case OP_BETA:  // :111-113
            sc[S_BETA] = __ddiv_rn(t[0], sc[S_RZ]);
            sc[S_RZ] = t[0];
            break;
        case OP_BETA_FCG:  // :118
            sc[S_BETA] = __ddiv_rn(t[0], sc[S_DAD]);
            break;
        case OP_CG1: {  // single-reduction PCG: t = (r.u, w.u, r.r), u = M r, w = A u
            const double g = t[0], dl = t[1];
            sc[S_RELRES] = __ddiv_rn(sqrt(t[2]), sc[S_BNORM]);
            double beta = 0.0, denom = dl;
            if (sc[S_AUX] != 0.0) {
                beta = __ddiv_rn(g, sc[S_RZ]);
                denom = __dsub_rn(dl, __ddiv_rn(__dmul_rn(beta, g), sc[S_ALPHA]));
            }
            if (denom <= 0.0) sc[S_BRK] = 1.0;  // p.Ap <= 0 (krylov.py:97-99 analogue)
            sc[S_BETA] = beta;
            sc[S_ALPHA] = __ddiv_rn(g, denom);
            sc[S_RZ] = g;
            sc[S_AUX] = 1.0;
            break;
        }
    }
}

__global__ void k_apply_op(int op, double *sc) { apply_op(op, sc + S_GLB, sc); }

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double ws[RB / 32];
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) ws[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < (int)(blockDim.x >> 5) ? ws[lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    }
    return v;  // valid in warp 0
}

// Publish this block's partial(s); the last block folds them in block order
// and either applies `op` (single GPU) or stores the rank totals at S_LOC.
template <int NV>
__device__ void reduce_finish(const double (&acc)[NV], double *partial, unsigned *ticket, int op,
                              bool dist, double *sc) {
    __shared__ bool last;
    double bs[NV];
#pragma unroll
    for (int q = 0; q < NV; q++) bs[q] = block_sum(acc[q]);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < NV; q++) partial[q * RGRID_MAX + blockIdx.x] = bs[q];
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double tot[NV];
#pragma unroll
    for (int q = 0; q < NV; q++) {
        double t = 0.0;
        for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x)
            t = __dadd_rn(t, __ldcg(partial + q * RGRID_MAX + i));
        tot[q] = block_sum(t);
    }
    if (threadIdx.x == 0) {
        *ticket = 0;
        if (dist) {
#pragma unroll
            for (int q = 0; q < NV; q++) sc[S_LOC + q] = tot[q];
        } else {
            apply_op(op, tot, sc);
        }
    }
}

// sum_i a_i b_i (and, with NV = 2, sum_i c_i d_i)
template <int NV>
__global__ void __launch_bounds__(RB)
k_pcg_dot2(int64_t n, const double *__restrict__ a, const double *__restrict__ b,
           const double *__restrict__ c, const double *__restrict__ d, double *partial,
           unsigned *ticket, double *sc, int op, int dist, int skip_on_breakdown) {
    if (skip_on_breakdown && sc[S_BRK] != 0.0) return;
    double acc[NV];
#pragma unroll
    for (int q = 0; q < NV; q++) acc[q] = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB) {
        acc[0] = __dadd_rn(acc[0], __dmul_rn(a[i], b[i]));
        if (NV > 1) acc[NV - 1] = __dadd_rn(acc[NV - 1], __dmul_rn(c[i], d[i]));
    }
    reduce_finish<NV>(acc, partial, ticket, op, dist, sc);
}

// single-GPU fused Ad = A d ; d.Ad (; r.d)
template <bool FCG>
__global__ void __launch_bounds__(RB)
k_pcg_spmv_dot(SellView A, const double *__restrict__ d, double *__restrict__ Ad,
               const double *__restrict__ r, double *partial, unsigned *ticket, double *sc) {
    double acc[2] = {0.0, 0.0};
    const int lane = threadIdx.x & 31;
    for (int64_t s = (int64_t)blockIdx.x * (RB / 32) + (threadIdx.x >> 5); s < A.nslices;
         s += (int64_t)gridDim.x * (RB / 32)) {
        const double y = sell_row_dot<8>(A, s, lane, d);
        const int64_t row = sell_row(A, s * 32 + lane);
        if (row >= 0) {
            Ad[row] = y;
            const double di = d[row];
            acc[0] = __dadd_rn(acc[0], __dmul_rn(di, y));
            if (FCG) acc[1] = __dadd_rn(acc[1], __dmul_rn(r[row], di));
        }
    }
    reduce_finish<2>(acc, partial, ticket, FCG ? OP_DAD_FCG : OP_DAD, false, sc);
}

__global__ void __launch_bounds__(RB)
k_pcg_update(int64_t n, double *__restrict__ x, double *__restrict__ r,
             const double *__restrict__ d, const double *__restrict__ Ad, double *partial,
             unsigned *ticket, double *sc, int dist) {
    if (sc[S_BRK] != 0.0) return;  // breakdown: x, r stay as the reference returns them
    const double alpha = sc[S_ALPHA];
    double acc[1] = {0.0};
    for (int64_t i = (int64_t)blockIdx.x * RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB) {
        x[i] = __dadd_rn(x[i], __dmul_rn(alpha, d[i]));             // krylov.py:101
        const double ri = __dsub_rn(r[i], __dmul_rn(alpha, Ad[i]));  // :102
        r[i] = ri;
        acc[0] = __dadd_rn(acc[0], __dmul_rn(ri, ri));
    }
    reduce_finish<1>(acc, partial, ticket, OP_RELRES, dist, sc);
}

// (r.u, w.u, r.r) in one pass -- the single reduction of the pcg1 variant
__global__ void __launch_bounds__(RB)
k_cg1_dot3(int64_t n, const double *__restrict__ r, const double *__restrict__ u,
           const double *__restrict__ w, double *partial, unsigned *ticket, double *sc, int dist) {
    double acc[3] = {0.0, 0.0, 0.0};
    for (int64_t i = (int64_t)blockIdx.x * RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB) {
        const double ri = r[i], ui = u[i];
        acc[0] = __dadd_rn(acc[0], __dmul_rn(ri, ui));
        acc[1] = __dadd_rn(acc[1], __dmul_rn(w[i], ui));
        acc[2] = __dadd_rn(acc[2], __dmul_rn(ri, ri));
    }
    reduce_finish<3>(acc, partial, ticket, OP_CG1, dist, sc);
}

// p = u + beta p ; s = w + beta s ; x += alpha p ; r -= alpha s
__global__ void k_cg1_update(int64_t n, const double *__restrict__ u, const double *__restrict__ w,
                             double *__restrict__ p, double *__restrict__ s, double *__restrict__ x,
                             double *__restrict__ r, const double *sc) {
    const double alpha = sc[S_ALPHA], beta = sc[S_BETA];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double pi = __dadd_rn(u[i], __dmul_rn(beta, p[i]));
        const double si = __dadd_rn(w[i], __dmul_rn(beta, s[i]));
        p[i] = pi;
        s[i] = si;
        x[i] = __dadd_rn(x[i], __dmul_rn(alpha, pi));
        r[i] = __dsub_rn(r[i], __dmul_rn(alpha, si));
    }
}

template <bool FCG>
__global__ void k_pcg_dir(int64_t n, const double *__restrict__ z, double *__restrict__ d,
                          const double *sc) {
    if (sc[S_BRK] != 0.0) return;
    const double beta = sc[S_BETA];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double bd = __dmul_rn(beta, d[i]);
        d[i] = FCG ? __dsub_rn(z[i], bd) : __dadd_rn(z[i], bd);  // :114 / :119
    }
}

__global__ void k_scale_zero(int64_t n, double *x) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] = __dmul_rn(x[i], 0.0);
}

namespace {
struct PcgWork {  // views into the context's cached PCG workspace
    double *partial = nullptr;
    unsigned *ticket = nullptr;
    double *r = nullptr, *z = nullptr, *d = nullptr, *Ad = nullptr, *s = nullptr;
};

// Grow-only workspace cached on the context: cudaMalloc/cudaFree per solve
// would synchronise the device inside the caller's pipeline.
int pcg_workspace(amgp_ctx *ctx, int64_t n, PcgWork *w) {
    const int64_t need = 5 * std::max<int64_t>(n, 1) + 3 * RGRID_MAX + 8;
    if (ctx->red_partial_n < need) {
        cudaStreamSynchronize(cur_stream(ctx));
        cudaFree(ctx->red_partial);
        ctx->red_partial = nullptr;
        ctx->red_partial_n = 0;
        AMGP_CUDA(cudaMalloc(&ctx->red_partial, need * sizeof(double)));
        ctx->red_partial_n = need;
        AMGP_CUDA(cudaMemsetAsync(ctx->red_partial, 0, need * sizeof(double), cur_stream(ctx)));
    }
    double *p = ctx->red_partial;
    const int64_t nn = std::max<int64_t>(n, 1);
    w->ticket = (unsigned *)p;  // 8 doubles of room for the tickets (zeroed once)
    w->partial = p + 8;
    w->r = w->partial + 3 * RGRID_MAX;
    w->z = w->r + nn;
    w->d = w->z + nn;
    w->Ad = w->d + nn;
    w->s = w->Ad + nn;
    return AMGP_OK;
}
}  // namespace

static unsigned rgrid(int64_t n) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(grid_for(n, RB), RGRID_MAX));
}

extern "C" int amgp_pcg_solve(amgp_ctx *ctx, amgp_mat *A, amgp_hier *h, const double *b,
                              double *x, int x0_given, int variant, double tol, int itmax,
                              double *history, amgp_solve_report *rep) {
    if (!ctx || !A || !rep) return amgp_fail(AMGP_EINVAL, "amgp_pcg_solve: bad argument");
    if (variant != AMGP_PCG && variant != AMGP_FCG && variant != AMGP_PCG1)
        return amgp_fail(AMGP_EINVAL, "unknown Krylov variant");
    if (!(tol > 0.0) || itmax < 1) return amgp_fail(AMGP_EINVAL, "tol must be positive and itmax >= 1");
    const int64_t nown = A->halo ? A->halo->nown : A->ncols;
    if (A->nrows != nown) return amgp_fail(AMGP_EINVAL, "matrix must be square");
    if (h && hier_rows(h) != A->nrows) return amgp_fail(AMGP_EINVAL, "dimension mismatch");
    const int64_t n = A->nrows;
    if (n > 0 && (!b || !x)) return amgp_fail(AMGP_EINVAL, "null vector");
    AMGP_CUDA(cudaSetDevice(ctx->device));
    std::lock_guard<std::mutex> cg(ctx->mu);
    auto t0 = std::chrono::steady_clock::now();
    auto elapsed = [&] {
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    };
    const bool fcg = variant == AMGP_FCG;
    // row-distributed solve: the fine matrix carries a halo plan (a single-GPU
    // solve on a multi-rank context stays local)
    const bool dist = ctx->comm != nullptr && ctx->nranks > 1 && A->halo != nullptr;
    cudaStream_t st = cur_stream(ctx);
    double *sc = ctx->scalars, *hs = ctx->host_scalars;

    PcgWork w;
    const size_t nb = (size_t)std::max<int64_t>(n, 1) * sizeof(double);
    AMGP_TRY(pcg_workspace(ctx, n, &w));
    const unsigned g = rgrid(n);
    const unsigned gs = (unsigned)std::max<int64_t>(1, std::min<int64_t>(grid_for(A->nslices, RB / 32), RGRID_MAX));

    // one reduction: launch the kernel; across ranks, fold the totals and
    // apply the op on every rank
    auto dot = [&](int nv, const double *a, const double *bb, const double *c, const double *d,
                   int op, int skip_brk) -> int {
        if (nv == 1)
            k_pcg_dot2<1><<<g, RB, 0, st>>>(n, a, bb, c, d, w.partial, w.ticket, sc, op, dist, skip_brk);
        else
            k_pcg_dot2<2><<<g, RB, 0, st>>>(n, a, bb, c, d, w.partial, w.ticket, sc, op, dist, skip_brk);
        AMGP_CHECK_LAUNCH(ctx);
        if (dist) {
            AMGP_TRY(allreduce_sum_ordered(ctx, sc + S_LOC, nv, sc + S_GLB));
            k_apply_op<<<1, 1, 0, st>>>(op, sc);
            AMGP_CHECK_LAUNCH(ctx);
        }
        return AMGP_OK;
    };

    *rep = amgp_solve_report{};
    int nh = 0;
    auto fetch = [&]() -> int {
        AMGP_CUDA(cudaMemcpyAsync(hs, sc, S_COUNT * sizeof(double), cudaMemcpyDeviceToHost, st));
        AMGP_CUDA(cudaStreamSynchronize(st));
        return AMGP_OK;
    };

    if (!x0_given) AMGP_CUDA(cudaMemsetAsync(x, 0, nb, st));
    AMGP_TRY(dot(1, b, b, nullptr, nullptr, OP_BNORM, 0));  // bnorm (:67)
    AMGP_TRY(fetch());
    if (hs[S_BNORM] == 0.0) {  // krylov.py:68-69
        k_scale_zero<<<g, RB, 0, st>>>(n, x);
        AMGP_CHECK_LAUNCH(ctx);
        AMGP_CUDA(cudaStreamSynchronize(st));
        rep->converged = 1;
        rep->elapsed_s = elapsed();
        return AMGP_OK;
    }
    AMGP_TRY(residual_enqueue(ctx, A, b, x, w.r));  // r = b - A x (:71)
    int spmv = 1, pc = 0;
    AMGP_TRY(dot(1, w.r, w.r, nullptr, nullptr, OP_RELRES, 0));
    AMGP_TRY(fetch());
    double relres = hs[S_RELRES];
    if (history) history[nh] = relres;
    nh++;
    auto finish = [&](int it, bool conv, bool brk) {
        rep->iterations = it;
        rep->converged = conv;
        rep->breakdown = brk;
        rep->final_relres = relres;
        rep->spmv_count = spmv;
        rep->precond_count = pc;
        rep->n_history = nh;
        rep->elapsed_s = elapsed();
        return AMGP_OK;
    };
    if (relres <= tol) return finish(0, true, false);

    if (variant == AMGP_PCG1) {
        // Chronopoulos-Gear single-reduction PCG (the paper's "CG requiring
        // only one global synchronization"): per iteration
        // u = M r, w = A u and ONE fused reduction (r.u, w.u, r.r); the
        // residual norm of the current iterate arrives with it, so a
        // converged solve costs one extra preconditioner application.
        std::unique_lock<std::mutex> hl1;
        if (h) hl1 = std::unique_lock<std::mutex>(hier_mutex(h));
        double *u = w.z, *ww = w.Ad, *pp = w.d, *ss = w.s;
        AMGP_CUDA(cudaMemsetAsync(sc + S_AUX, 0, sizeof(double), st));
        AMGP_CUDA(cudaMemsetAsync(sc + S_BRK, 0, sizeof(double), st));
        AMGP_CUDA(cudaMemsetAsync(pp, 0, nb, st));
        AMGP_CUDA(cudaMemsetAsync(ss, 0, nb, st));
        for (int it = 0;; it++) {
            if (h) AMGP_TRY(vcycle_enqueue(h, w.r, u));
            else AMGP_CUDA(cudaMemcpyAsync(u, w.r, nb, cudaMemcpyDeviceToDevice, st));
            pc++;
            AMGP_TRY(spmv_enqueue(ctx, A, u, ww));
            spmv++;
            k_cg1_dot3<<<g, RB, 0, st>>>(n, w.r, u, ww, w.partial, w.ticket, sc, dist);
            AMGP_CHECK_LAUNCH(ctx);
            if (dist) {
                AMGP_TRY(allreduce_sum_ordered(ctx, sc + S_LOC, 3, sc + S_GLB));
                k_apply_op<<<1, 1, 0, st>>>(OP_CG1, sc);
                AMGP_CHECK_LAUNCH(ctx);
            }
            AMGP_TRY(fetch());
            if (it > 0) {
                relres = hs[S_RELRES];
                if (history) history[nh] = relres;
                nh++;
                if (relres <= tol) return finish(it, true, false);
            }
            if (hs[S_BRK] != 0.0) return finish(it, false, true);
            if (it == itmax) return finish(itmax, false, false);
            k_cg1_update<<<g, RB, 0, st>>>(n, u, ww, pp, ss, x, w.r, sc);
            AMGP_CHECK_LAUNCH(ctx);
        }
    }

    std::unique_lock<std::mutex> hl;
    if (h) hl = std::unique_lock<std::mutex>(hier_mutex(h));
    auto precond = [&]() -> int {
        if (h) return vcycle_enqueue(h, w.r, w.z);
        AMGP_CUDA(cudaMemcpyAsync(w.z, w.r, nb, cudaMemcpyDeviceToDevice, st));
        return AMGP_OK;
    };
    AMGP_TRY(precond());
    pc++;
    AMGP_CUDA(cudaMemcpyAsync(w.d, w.z, nb, cudaMemcpyDeviceToDevice, st));
    AMGP_TRY(dot(1, w.r, w.z, nullptr, nullptr, OP_RZ, 0));  // rz (:92)

    // next preconditioner application + direction update (krylov.py:108-119)
    auto next_direction = [&]() -> int {
        AMGP_TRY(precond());
        if (fcg) AMGP_TRY(dot(1, w.z, w.Ad, nullptr, nullptr, OP_BETA_FCG, 1));
        else AMGP_TRY(dot(1, w.r, w.z, nullptr, nullptr, OP_BETA, 1));
        if (fcg) k_pcg_dir<true><<<g, RB, 0, st>>>(n, w.z, w.d, sc);
        else k_pcg_dir<false><<<g, RB, 0, st>>>(n, w.z, w.d, sc);
        AMGP_CHECK_LAUNCH(ctx);
        return AMGP_OK;
    };
    struct Ev {
        cudaEvent_t e = nullptr;
        ~Ev() { if (e) cudaEventDestroy(e); }
    } ev;
    AMGP_CUDA(cudaEventCreateWithFlags(&ev.e, cudaEventDisableTiming));
    double rel_prev = relres, rel_prev2 = -1.0;
    for (int it = 1; it <= itmax; it++) {
        if (!dist && !A->halo) {
            if (fcg) k_pcg_spmv_dot<true><<<gs, RB, 0, st>>>(view_of(A), w.d, w.Ad, w.r, w.partial, w.ticket, sc);
            else k_pcg_spmv_dot<false><<<gs, RB, 0, st>>>(view_of(A), w.d, w.Ad, w.r, w.partial, w.ticket, sc);
            AMGP_CHECK_LAUNCH(ctx);
        } else {
            AMGP_TRY(spmv_enqueue(ctx, A, w.d, w.Ad));
            if (fcg) AMGP_TRY(dot(2, w.d, w.Ad, w.r, w.d, OP_DAD_FCG, 0));
            else AMGP_TRY(dot(1, w.d, w.Ad, nullptr, nullptr, OP_DAD, 0));
        }
        spmv++;
        k_pcg_update<<<g, RB, 0, st>>>(n, x, w.r, w.d, w.Ad, w.partial, w.ticket, sc, dist);
        AMGP_CHECK_LAUNCH(ctx);
        if (dist) {  // after a breakdown k_pcg_update returned early: keep relres
            AMGP_TRY(allreduce_sum_ordered(ctx, sc + S_LOC, 1, sc + S_GLB));
            k_apply_op<<<1, 1, 0, st>>>(OP_RELRES, sc);
            AMGP_CHECK_LAUNCH(ctx);
        }
        AMGP_CUDA(cudaMemcpyAsync(hs, sc, S_COUNT * sizeof(double), cudaMemcpyDeviceToHost, st));
        AMGP_CUDA(cudaEventRecord(ev.e, st));
        // While the host waits for relres, keep the GPU busy with the next
        // V-cycle -- unless the residual history predicts convergence at this
        // check (then the V-cycle would be wasted work).  Harmless either
        // way: x and r are final before the event.
        bool spec = true;
        if (rel_prev2 > 0.0) {
            const double ratio = rel_prev / rel_prev2;
            if (rel_prev * ratio <= 2.0 * tol) spec = false;
        }
        if (spec) AMGP_TRY(next_direction());
        AMGP_CUDA(cudaEventSynchronize(ev.e));
        if (hs[S_BRK] != 0.0) {
            AMGP_CUDA(cudaStreamSynchronize(st));
            return finish(it - 1, false, true);
        }
        relres = hs[S_RELRES];
        if (history) history[nh] = relres;
        nh++;
        if (relres <= tol) {
            AMGP_CUDA(cudaStreamSynchronize(st));
            return finish(it, true, false);
        }
        if (!spec) AMGP_TRY(next_direction());
        pc++;
        rel_prev2 = rel_prev;
        rel_prev = relres;
    }
    AMGP_CUDA(cudaStreamSynchronize(st));
    return finish(itmax, false, false);
}
