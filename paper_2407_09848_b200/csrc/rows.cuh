// Row-parallel SELL-32 kernels with pluggable epilogues.
//
// Every hot kernel of the library is "y_i = sum_j a_ij v_j in stored order,
// then an elementwise epilogue on row i".  Two schedules compute y_i with
// the SAME operations in the SAME order (so results are bitwise identical):
//
//   k_thread_rows  one thread per row, slots loaded SM_U at a time -- for
//                  short rows (fine levels: 4-7 nnz), where the grid holds
//                  enough warps to cover memory latency.
//   k_split_rows   one CTA per 32-row slice; its NW warps compute the slot
//                  products a_ij*v_j in parallel (every load independent ->
//                  deep memory-level parallelism) into shared memory, then
//                  each row is summed sequentially from 0.0 by warp 0.  For
//                  coarse AMG levels (tens to hundreds of nnz per row, few
//                  rows), where thread-per-row is latency bound.
// Padding slots contribute +0.0 in k_split_rows and are skipped in
// k_thread_rows: the row sum is never -0.0 (it starts at +0.0 and
// round-to-nearest never produces -0.0 from a non-negative-zero operand),
// so adding +0.0 leaves it unchanged bit for bit.
#pragma once

#include "amgp_common.cuh"

#define ROWS_BLOCK 256
#define ROWS_SLICES (ROWS_BLOCK / 32)
#define ROWS_U 8
#ifndef SPLIT_WARPS
#define SPLIT_WARPS 16  // measured best of {8,16,32} x {4,8} (tools: AMGP_LIB variants)
#endif
#ifndef SPLIT_U
#define SPLIT_U 4  // slot loads in flight per thread
#endif
#define SPLIT_CHUNK 192
#ifndef SPLIT_BULK
#define SPLIT_BULK 0  // 1: bulk-copy (TMA engine) staging for the split schedule (measured: no gain)
#endif  // slots staged per pass: 192 * 32 * 8 B = 48 KB

// GEN = false: slices s0 .. s0+nlist-1, every column local (single-GPU
// matrices, interior slices of distributed ones).  GEN = true: a slice list
// and/or halo columns (boundary slices) -- kept out of the common kernel so
// its gather stays one load per slot.
template <class Epi, bool GEN>
__global__ void __launch_bounds__(ROWS_BLOCK)
k_thread_rows(SellView A, const double *__restrict__ xg, Epi epi) {
    const int64_t idx = (int64_t)blockIdx.x * ROWS_SLICES + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (idx >= A.nlist) return;
    const int64_t s = GEN && A.slist ? (int64_t)A.slist[idx] : A.s0 + idx;
    double y = 0.0;
    if (Epi::kSpmv) y = sell_row_dot<ROWS_U, GEN>(A, s, lane, xg);
    const int64_t row = s * 32 + lane;
    if (row < A.nrows) epi(row, y);
}

// NW warps, U slot loads in flight per thread: SPLIT_WARPS x SPLIT_U for
// levels with enough slices to fill the GPU; a launch with fewer slices than
// two per SM is latency bound (a slice's chunk costs ceil(192 / (NW U))
// dependent column->gather rounds), so it takes 24 warps x 8 = one round.
template <class Epi, bool GEN, int NW, int U>
__global__ void __launch_bounds__(NW * 32)
k_split_rows(SellView A, const double *__restrict__ xg, Epi epi) {
    __shared__ double prod[SPLIT_CHUNK * 32];
    const int64_t s = GEN && A.slist ? (int64_t)A.slist[blockIdx.x] : A.s0 + (int64_t)blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t base = A.slice_ptr[s];
    const int w = (int)((A.slice_ptr[s + 1] - base) >> 5);
    const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
    double sum = 0.0;
    for (int j0 = 0; j0 < w; j0 += SPLIT_CHUNK) {
        const int jn = min(SPLIT_CHUNK, w - j0);
        for (int j = warp; j < jn; j += NW * U) {
            int32_t cc[U];
            double vv[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int jj = j + u * NW;
                const bool ok = jj < jn;
                const int64_t o = base + (int64_t)(j0 + jj) * 32 + lane;
                cc[u] = ok ? ld_stream_s32(A.col + o, pf) : -1;
                vv[u] = ok ? ld_stream_f64(A.val + o, pf) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int jj = j + u * NW;
                if (jj < jn) {
                    double p = 0.0;
                    if (cc[u] >= 0)
                        p = __dmul_rn(vv[u], ld_gather_f64(GEN && cc[u] >= A.nown ? A.xh + (cc[u] - A.nown)
                                                                                   : xg + cc[u], pl));
                    prod[jj * 32 + lane] = p;
                }
            }
        }
        __syncthreads();
        if (warp == 0) {
#pragma unroll 8
            for (int j = 0; j < jn; j++) sum = __dadd_rn(sum, prod[j * 32 + lane]);
        }
        __syncthreads();
    }
    if (warp == 0) {
        const int64_t row = s * 32 + lane;
        if (row < A.nrows) epi(row, sum);
    }
}

// ---------------------------------------------------------------- bulk-copy split schedule
// k_split_bulk: the split schedule with the slice's slots brought into shared
// memory by the Blackwell bulk-copy engine instead of through registers.  A
// slice's slots [j0, j0 + CH) are contiguous in SELL (CH*32 values, CH*32
// columns), so one elected thread issues two cp.async.bulk copies per chunk
// that complete on an mbarrier; chunk c+1 is in flight while chunk c is
// gathered and summed (two stages).  Each thread then gathers the operand
// for its slots of the chunk (every gather independent), overwrites the
// staged value with the product, and warp 0 sums each row in slot order
// exactly as k_split_rows does -- bitwise the same row sums.
#define BULK_CH 56  // slots per stage: 2 stages x 56 x 32 x 12 B = 43 KB (no opt-in)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                         uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

template <class Epi, bool GEN, int NW>
__global__ void __launch_bounds__(NW * 32)
k_split_bulk(SellView A, const double *__restrict__ xg, Epi epi) {
    constexpr int CH = BULK_CH, U = (CH * 32 + NW * 32 - 1) / (NW * 32);
    __shared__ __align__(128) double sv[2][CH * 32];   // values, then products
    __shared__ __align__(128) int32_t sc[2][CH * 32];  // columns
    __shared__ __align__(8) uint64_t bar[2];
    const int64_t s = GEN && A.slist ? (int64_t)A.slist[blockIdx.x] : A.s0 + (int64_t)blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t base = A.slice_ptr[s];
    const int w = (int)((A.slice_ptr[s + 1] - base) >> 5);
    const int nch = (w + CH - 1) / CH;
    const uint64_t pl = policy_evict_last();
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int c) {
        const int jn = min(CH, w - c * CH);
        const int64_t o = base + (int64_t)c * CH * 32;
        const uint64_t pf = policy_evict_first();
        mbar_expect_tx(&bar[c & 1], (uint32_t)jn * 32 * 12);
        bulk_g2s(sv[c & 1], A.val + o, (uint32_t)jn * 32 * 8, &bar[c & 1], pf);
        bulk_g2s(sc[c & 1], A.col + o, (uint32_t)jn * 32 * 4, &bar[c & 1], pf);
    };
    if (threadIdx.x == 0 && nch > 0) issue(0);
    double sum = 0.0;
    for (int c = 0; c < nch; c++) {
        if (threadIdx.x == 0 && c + 1 < nch) issue(c + 1);  // its stage was released below
        const int jn = min(CH, w - c * CH);
        double *v = sv[c & 1];
        const int32_t *col = sc[c & 1];
        mbar_wait(&bar[c & 1], (uint32_t)(c >> 1) & 1);
        int32_t cc[U];
        double xx[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int e = threadIdx.x + u * NW * 32;
            cc[u] = e < jn * 32 ? col[e] : -1;
        }
#pragma unroll
        for (int u = 0; u < U; u++)
            xx[u] = cc[u] < 0 ? 0.0
                              : ld_gather_f64(GEN && cc[u] >= A.nown ? A.xh + (cc[u] - A.nown) : xg + cc[u], pl);
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int e = threadIdx.x + u * NW * 32;
            if (e < jn * 32) v[e] = cc[u] >= 0 ? __dmul_rn(v[e], xx[u]) : 0.0;
        }
        __syncthreads();
        if (warp == 0) {
#pragma unroll 8
            for (int j = 0; j < jn; j++) sum = __dadd_rn(sum, v[j * 32 + lane]);
        }
        // generic-proxy writes/reads of this stage complete before the bulk
        // engine refills it (issued at the top of iteration c+1)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
    }
    if (warp == 0) {
        const int64_t row = s * 32 + lane;
        if (row < A.nrows) epi(row, sum);
    }
}

// Schedule choice: split when rows are long and there are too few slices to
// keep the GPU's warps busy with thread-per-row.
inline bool use_split(const amgp_mat *A) {
    return A->max_width >= 24 && A->nslices < 148 * 64;
}

template <class Epi>
int launch_view(amgp_ctx *ctx, const amgp_mat *A, const SellView &v, const double *xg,
                const Epi &epi) {
    if (v.nlist == 0) return AMGP_OK;
    const bool gen = v.slist || v.xh;
    const unsigned gs = (unsigned)v.nlist, gt = grid_for(v.nlist, ROWS_SLICES);
    if (Epi::kSpmv && use_split(A) && SPLIT_BULK) {
        if (gen) k_split_bulk<Epi, true, 16><<<gs, 16 * 32, 0, ctx->stream>>>(v, xg, epi);
        else k_split_bulk<Epi, false, 16><<<gs, 16 * 32, 0, ctx->stream>>>(v, xg, epi);
    } else if (Epi::kSpmv && use_split(A)) {
        if (v.nlist < 2 * 148) {
            if (gen) k_split_rows<Epi, true, 24, 8><<<gs, 24 * 32, 0, ctx->stream>>>(v, xg, epi);
            else k_split_rows<Epi, false, 24, 8><<<gs, 24 * 32, 0, ctx->stream>>>(v, xg, epi);
        } else {
            if (gen) k_split_rows<Epi, true, SPLIT_WARPS, SPLIT_U><<<gs, SPLIT_WARPS * 32, 0, ctx->stream>>>(v, xg, epi);
            else k_split_rows<Epi, false, SPLIT_WARPS, SPLIT_U><<<gs, SPLIT_WARPS * 32, 0, ctx->stream>>>(v, xg, epi);
        }
    } else {
        if (gen) k_thread_rows<Epi, true><<<gt, ROWS_BLOCK, 0, ctx->stream>>>(v, xg, epi);
        else k_thread_rows<Epi, false><<<gt, ROWS_BLOCK, 0, ctx->stream>>>(v, xg, epi);
    }
    AMGP_CHECK_LAUNCH(ctx);
    return AMGP_OK;
}

// y-rows of A with epilogue epi, gathering operand xg.  For a distributed
// matrix the halo of xg travels over NCCL on the comm stream while the
// interior slices (no halo column) compute; boundary slices run after.
template <class Epi>
int launch_rows(amgp_ctx *ctx, const amgp_mat *A, const double *xg, const Epi &epi) {
    if (A->nslices == 0) return AMGP_OK;
    if (!Epi::kSpmv || !A->halo) return launch_view(ctx, A, view_of(A), xg, epi);
    const HaloPlan &h = *A->halo;
    AMGP_TRY(halo_exchange_begin(ctx, A, xg));
    SellView v = view_of(A);
    // one launch per run when the set is a few contiguous runs, else the list
    auto launch_set = [&](const std::vector<std::pair<int64_t, int64_t>> &runs,
                          const int32_t *list, int64_t n) -> int {
        if (runs.size() <= 2) {
            for (const auto &r : runs) {
                v.slist = nullptr;
                v.s0 = r.first;
                v.nlist = r.second;
                AMGP_TRY(launch_view(ctx, A, v, xg, epi));
            }
            return AMGP_OK;
        }
        v.slist = list;
        v.s0 = 0;
        v.nlist = n;
        return launch_view(ctx, A, v, xg, epi);
    };
    // interior slices have no halo column (slice_maxcol < nown): plain gather
    v.nown = INT64_MAX;
    v.xh = nullptr;
    AMGP_TRY(launch_set(h.interior_runs, h.interior, h.n_interior));
    AMGP_TRY(halo_exchange_end(ctx, A));
    v.nown = h.nown;
    v.xh = h.halo;
    AMGP_TRY(launch_set(h.boundary_runs, h.boundary, h.n_boundary));
    return halo_exchange_done(ctx, A);
}
