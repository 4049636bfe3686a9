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

#include <algorithm>

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
#define SPLIT_CHUNK 192  // slots staged per pass: 192 * 32 * 8 B = 48 KB

// Launch modes.  ROWS_PLAIN: slices of the run table, every column local
// (single-GPU matrices, interior slices of distributed ones).  ROWS_GEN: a
// slice list and/or halo columns (boundary slices) -- kept out of the common
// kernel so its gather stays one load per slot.
enum { ROWS_PLAIN = 0, ROWS_GEN = 1 };

// Rows of launch CTA `cta` (ROWS_SLICES slices): y = A x (halo-aware gather
// when HALO), then the epilogue.
template <class Epi, int MODE, bool HALO>
__device__ __forceinline__ void thread_rows_body(const SellView &A, int64_t cta,
                                                 const double *__restrict__ xg,
                                                 const double *__restrict__ xh, const Epi &epi) {
    const int64_t idx = cta * ROWS_SLICES + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (idx >= A.nlist) return;
    const int64_t s = MODE == ROWS_GEN && A.slist ? (int64_t)A.slist[idx] : run_slice(A, idx);
    double y = 0.0;
    if (Epi::kSpmv) y = sell_row_dot<ROWS_U, HALO>(A, s, lane, xg, xh);
    const int64_t row = sell_row(A, s * 32 + lane);
    if (row >= 0) epi(row, y);
}

template <class Epi, int MODE>
__global__ void __launch_bounds__(ROWS_BLOCK, 8)  // 32 registers: 8 CTAs per SM
k_thread_rows(SellView A, const double *__restrict__ xg, Epi epi) {
    if (MODE == ROWS_PLAIN) {
        thread_rows_body<Epi, MODE, false>(A, blockIdx.x, xg, nullptr, epi);
    } else {
        const double *xh = halo_wait(A);
        thread_rows_body<Epi, MODE, true>(A, blockIdx.x, xg, xh, epi);
        if (A.complete) halo_complete(A, gridDim.x);
    }
}

// NW warps, U slot loads in flight per thread: SPLIT_WARPS x SPLIT_U for
// levels with enough slices to fill the GPU; a launch with fewer slices than
// two per SM is latency bound (a slice's chunk costs ceil(192 / (NW U))
// dependent column->gather rounds), so it takes 24 warps x 8 = one round.
template <class Epi, int MODE, int NW, int U>
__device__ __forceinline__ void split_rows_body(const SellView &A, int64_t cta, const double *__restrict__ xg,
                                                const double *__restrict__ xh, const Epi &epi,
                                                double *__restrict__ prod) {
    const bool halo = MODE == ROWS_GEN && A.xh != nullptr;
    const int64_t s = MODE == ROWS_GEN && A.slist ? (int64_t)A.slist[cta] : run_slice(A, cta);
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
                    const int64_t c = cc[u];
                    if (c >= 0) {
                        const bool hc = halo && c >= A.nown;
                        const double *src = (hc ? xh : xg) + (hc ? c - A.nown : c);
                        p = __dmul_rn(vv[u], halo ? ld_halo_f64(src, pl) : ld_gather_f64(src, pl));
                    }
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
        const int64_t row = sell_row(A, s * 32 + lane);
        if (row >= 0) epi(row, sum);
    }
}

template <class Epi, int MODE, int NW, int U>
__global__ void __launch_bounds__(NW * 32)
k_split_rows(SellView A, const double *__restrict__ xg, Epi epi) {
    __shared__ double prod[SPLIT_CHUNK * 32];
    const double *xh = A.xh;
    if (MODE == ROWS_GEN) xh = halo_wait(A);
    split_rows_body<Epi, MODE, NW, U>(A, blockIdx.x, xg, xh, epi, prod);
    if (MODE == ROWS_GEN && A.complete) halo_complete(A, gridDim.x);
}

// Interior and boundary slices of a distributed matrix (p2p transport) in ONE
// launch: CTAs [0, ncta_p) pack this exchange's halo for the peers (halo_pack;
// ncta_p = 0 when a separate pack kernel does it), then ncta_i CTAs take the
// interior view I (no halo column), the rest the boundary view B, which waits
// for the peers' halo in-kernel.  Packing CTAs come first and wait for nothing
// of this exchange, so every rank's pack makes progress; the boundary CTAs are
// the last ones dispatched, so the peers' stores have had the whole interior
// to land, and they fill the interior's tail wave instead of running as a
// second, dependent launch.  Pack and boundary CTAs all arrive on the
// completion ticket: the last one advances the epoch.
template <class Epi, int IMODE>
__global__ void __launch_bounds__(ROWS_BLOCK, 8)
k_thread_rows_fused(SellView I, SellView B, PackView pk, int64_t ncta_p, int64_t ncta_i,
                    const double *__restrict__ xg, Epi epi) {
    const int64_t b = blockIdx.x;
    const unsigned ndone = gridDim.x - (unsigned)ncta_i;
    if (b < ncta_p) {
        halo_pack(pk, B.sync_slot, B.nranks, xg, b, ncta_p);
        halo_complete(B, ndone);
    } else if (b < ncta_p + ncta_i) {  // IMODE: ROWS_PLAIN (run table) or ROWS_GEN (slice list)
        thread_rows_body<Epi, IMODE, false>(I, b - ncta_p, xg, nullptr, epi);
    } else {
        const double *xh = halo_wait(B);
        thread_rows_body<Epi, ROWS_GEN, true>(B, b - ncta_p - ncta_i, xg, xh, epi);
        halo_complete(B, ndone);
    }
}

template <class Epi, int NW, int U>
__global__ void __launch_bounds__(NW * 32)
k_split_rows_fused(SellView I, SellView B, PackView pk, int64_t ncta_p, int64_t ncta_i,
                   const double *__restrict__ xg, Epi epi) {
    __shared__ double prod[SPLIT_CHUNK * 32];
    const int64_t b = blockIdx.x;
    const unsigned ndone = gridDim.x - (unsigned)ncta_i;
    if (b < ncta_p) {
        halo_pack(pk, B.sync_slot, B.nranks, xg, b, ncta_p);
        halo_complete(B, ndone);
    } else if (b < ncta_p + ncta_i) {
        split_rows_body<Epi, ROWS_GEN, NW, U>(I, b - ncta_p, xg, nullptr, epi, prod);
    } else {
        const double *xh = halo_wait(B);
        split_rows_body<Epi, ROWS_GEN, NW, U>(B, b - ncta_p - ncta_i, xg, xh, epi, prod);
        halo_complete(B, ndone);
    }
}

// Schedule choice, per launch: split when rows are long and the launch has
// too few slices to keep the GPU's warps busy with thread-per-row (e.g. the
// boundary-slice launch of a distributed coarse level: ~800 slices of ~50
// slots, latency bound at one thread per row).
inline bool use_split(const amgp_mat *A, int64_t nslices_launched) {
    return A->max_width >= 24 && nslices_launched < 148 * 64;
}

template <class Epi, int MODE>
void launch_mode(amgp_ctx *ctx, const amgp_mat *A, const SellView &v0, const double *xg,
                 const Epi &epi) {
    SellView v = v0;
    const bool split = Epi::kSpmv && use_split(A, v.nlist);
    const int nw = v.nlist < 2 * 148 ? 24 : SPLIT_WARPS;
    const unsigned grid = split ? (unsigned)v.nlist : grid_for(v.nlist, ROWS_SLICES);
    if (split) {
        if (nw == 24) {
            k_split_rows<Epi, MODE, 24, 8><<<grid, 24 * 32, 0, cur_stream(ctx)>>>(v, xg, epi);
        } else {
            k_split_rows<Epi, MODE, SPLIT_WARPS, SPLIT_U><<<grid, SPLIT_WARPS * 32, 0, cur_stream(ctx)>>>(v, xg, epi);
        }
    } else {
        k_thread_rows<Epi, MODE><<<grid, ROWS_BLOCK, 0, cur_stream(ctx)>>>(v, xg, epi);
    }
}

template <class Epi>
int launch_view(amgp_ctx *ctx, const amgp_mat *A, const SellView &v, const double *xg,
                const Epi &epi) {
    if (v.nlist == 0) return AMGP_OK;
    if (v.slist || v.xh) launch_mode<Epi, ROWS_GEN>(ctx, A, v, xg, epi);
    else launch_mode<Epi, ROWS_PLAIN>(ctx, A, v, xg, epi);
    AMGP_CHECK_LAUNCH(ctx);
    return AMGP_OK;
}

// y-rows of A with epilogue epi, gathering operand xg.  For a distributed
// matrix the halo of xg travels while the interior slices (no halo column)
// compute: interior launch, exchange (NCCL on the comm stream, or the p2p
// pack kernel on the high-priority stream), boundary launch (p2p: in-kernel
// waits; it completes the exchange).
template <class Epi>
int launch_rows(amgp_ctx *ctx, const amgp_mat *A, const double *xg, const Epi &epi) {
    if (!Epi::kSpmv || !A->halo) {
        if (A->nslices == 0) return AMGP_OK;
        return launch_view(ctx, A, view_of(A), xg, epi);
    }
    const HaloPlan &h = *A->halo;
    const bool p2p = ctx->halo_p2p > 0;
    if (A->nslices == 0 && !p2p) return AMGP_OK;
    SellView v = view_of(A);
    // one launch over interior + boundary slices (k_*_rows_fused) where it
    // measured faster (tools/dist_levels.py, 4 GPUs, profiles/r02_halo_fuse.md):
    // coarse levels and long rows (the fine level's short rows ran 8 % slower
    // fused next to a separate pack kernel); with halo_xpack the fused launch
    // packs the halo itself (no pack kernel, no cross-stream events)
    const bool fuse = p2p && A->nslices >= 2 * 148 && h.n_boundary > 0 && h.n_interior > 0 &&
                      (ctx->halo_fuse == 2 ||
                       (ctx->halo_fuse == 1 && (A->nslices < (1 << 18) || A->max_width >= 16)));
    const bool xpack = fuse && ctx->halo_xpack;
    if (!xpack) AMGP_TRY(halo_exchange_begin(ctx, A, xg));
    if (p2p) {
        v.sync_slot = h.sync_slot;
        v.recvp = h.d_recvp;
        v.nrecvp = h.nrecvp;
        v.nranks = ctx->nranks;
        v.consumed_remote = h.d_consumed_remote;
    }
    // a set of at most SELL_RUNS contiguous runs is launched over the run
    // table (no slice-list indirection), else over the list
    auto set_list = [](SellView &w, const std::vector<std::pair<int64_t, int64_t>> &runs, const int32_t *list,
                       int64_t n) {
        if (runs.size() <= SELL_RUNS) {
            w.slist = nullptr;
            w.nruns = (int)runs.size();
            int64_t end = 0;
            for (size_t r = 0; r < runs.size(); r++) {
                w.run_s0[r] = runs[r].first;
                end += runs[r].second;
                w.run_end[r] = end;
            }
            w.nlist = end;
        } else {
            w.slist = list;
            w.nlist = n;
        }
    };
    auto launch_set = [&](const std::vector<std::pair<int64_t, int64_t>> &runs,
                          const int32_t *list, int64_t n) -> int {
        if (n == 0) return AMGP_OK;
        set_list(v, runs, list, n);
        return launch_view(ctx, A, v, xg, epi);
    };
    // a matrix with fewer slices than two per SM is launch-latency bound:
    // splitting it would pay two dependent launches to hide an exchange the
    // interior is too short to cover, so it runs as ONE halo-aware launch
    // over all its slices after the exchange
    if (A->nslices < 2 * 148) {
        AMGP_TRY(halo_exchange_end(ctx, A));
        v.slist = nullptr;
        v.nruns = 1;
        v.run_s0[0] = 0;
        v.run_end[0] = v.nlist = A->nslices;
        v.nown = h.nown;
        v.xh = h.halo;
        v.xh_stride = p2p ? h.nhalo : 0;
        if (p2p && A->nslices > 0) {
            v.complete = 1;
            return launch_view(ctx, A, v, xg, epi);
        }
        if (A->nslices > 0) AMGP_TRY(launch_view(ctx, A, v, xg, epi));
        return halo_exchange_done(ctx, A);
    }
    // interior slices have no halo column (slice_maxcol < nown): plain gather
    v.nown = INT64_MAX;
    v.xh = nullptr;
    const int nrecvp = v.nrecvp;
    v.nrecvp = 0;
    if (fuse) {
        SellView b = v;
        set_list(v, h.interior_runs, h.interior, h.n_interior);
        set_list(b, h.boundary_runs, h.boundary, h.n_boundary);
        b.nown = h.nown;
        b.xh = h.halo;
        b.xh_stride = h.nhalo;
        b.nrecvp = nrecvp;
        b.complete = 1;
        PackView pk;
        if (xpack) pk = pack_view(h);
        if (Epi::kSpmv && use_split(A, v.nlist + b.nlist)) {
            const int64_t cp = xpack && h.nsend > 0 ? std::min<int64_t>(grid_for(h.nsend, SPLIT_WARPS * 32), 148) : 0;
            k_split_rows_fused<Epi, SPLIT_WARPS, SPLIT_U>
                <<<(unsigned)(cp + v.nlist + b.nlist), SPLIT_WARPS * 32, 0, cur_stream(ctx)>>>(v, b, pk, cp, v.nlist,
                                                                                               xg, epi);
        } else {
            const int64_t cp = xpack && h.nsend > 0 ? std::min<int64_t>(grid_for(h.nsend, ROWS_BLOCK), 148) : 0;
            const int64_t ci = (v.nlist + ROWS_SLICES - 1) / ROWS_SLICES;
            const int64_t cb = (b.nlist + ROWS_SLICES - 1) / ROWS_SLICES;
            const unsigned g = (unsigned)(cp + ci + cb);
            if (v.slist)
                k_thread_rows_fused<Epi, ROWS_GEN><<<g, ROWS_BLOCK, 0, cur_stream(ctx)>>>(v, b, pk, cp, ci, xg, epi);
            else
                k_thread_rows_fused<Epi, ROWS_PLAIN><<<g, ROWS_BLOCK, 0, cur_stream(ctx)>>>(v, b, pk, cp, ci, xg, epi);
        }
        AMGP_CHECK_LAUNCH(ctx);
        // a separate pack kernel reads xg: later work on this stream waits for it
        return xpack ? AMGP_OK : halo_exchange_end(ctx, A);
    }
    AMGP_TRY(launch_set(h.interior_runs, h.interior, h.n_interior));
    AMGP_TRY(halo_exchange_end(ctx, A));
    v.nown = h.nown;
    v.xh = h.halo;
    v.xh_stride = p2p ? h.nhalo : 0;  // p2p halo: double-buffered by exchange parity
    v.nrecvp = nrecvp;
    if (p2p && h.n_boundary > 0) {  // the boundary launch completes the exchange itself
        v.complete = 1;
        return launch_set(h.boundary_runs, h.boundary, h.n_boundary);
    }
    AMGP_TRY(launch_set(h.boundary_runs, h.boundary, h.n_boundary));
    return halo_exchange_done(ctx, A);
}
