// Internal declarations shared by the libamgp.so translation units.
//
// Numerics contract: every kernel
// evaluates the reference's numpy expressions element by element with
// separate IEEE-754 binary64 operations -- __dmul_rn / __dadd_rn / __dsub_rn /
// __ddiv_rn, never a contracted FMA (the library is also built with
// -fmad=false) -- and every sparse row sum starts at 0.0 and accumulates in
// stored-entry order, exactly like scipy's csr_matvec behind
// reference sparse.py:125.  One thread owns one row, so the results are
// bitwise identical to the reference's.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/amgp.h"

#define AMGP_SLICE 32  // SELL slice height == warp width

// ---------------------------------------------------------------- errors
void amgp_set_error(const std::string &msg);
int amgp_fail(int code, const std::string &msg);
int amgp_cuda_fail(cudaError_t e, const char *what, const char *file, int line);

#define AMGP_CUDA(call)                                                        \
    do {                                                                       \
        cudaError_t _e = (call);                                               \
        if (_e != cudaSuccess) return amgp_cuda_fail(_e, #call, __FILE__, __LINE__); \
    } while (0)

#define AMGP_CHECK_LAUNCH(ctx)                                                 \
    do {                                                                       \
        cudaError_t _e = cudaGetLastError();                                   \
        if (_e != cudaSuccess) return amgp_cuda_fail(_e, "kernel launch", __FILE__, __LINE__); \
        (ctx)->launches.fetch_add(1, std::memory_order_relaxed);               \
    } while (0)

#define AMGP_TRY(call)                                                         \
    do {                                                                       \
        int _s = (call);                                                       \
        if (_s != AMGP_OK) return _s;                                          \
    } while (0)

// ---------------------------------------------------------------- objects
struct NcclApi;  // dist.cu: NCCL entry points resolved with dlopen

struct amgp_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::atomic<int64_t> launches{0};
    // Serialises the API calls that enqueue work: they share this stream,
    // and a V-cycle graph capture must not see another thread's launches
    // (lock order: ctx->mu, then a matrix's or hierarchy's own mutex).
    std::mutex mu;
    // deterministic-reduction scratch (PCG): partial sums + scalars
    double *red_partial = nullptr;
    int64_t red_partial_n = 0;
    double *scalars = nullptr;       // device scalar block (see pcg.cu)
    double *host_scalars = nullptr;  // pinned mirror
    // multi-GPU (dist.cu): one NCCL communicator per context, its stream and
    // the events that fork/join halo exchanges with the compute stream
    void *comm = nullptr;  // ncclComm_t
    int nranks = 1, rank = 0;
    cudaStream_t comm_stream = nullptr;
    int prio_high = 0;  // greatest stream priority (halo pack kernels)
    cudaEvent_t ev_packed = nullptr, ev_exchanged = nullptr;
    double *gather_buf = nullptr;  // allgather scratch for global dots
    // direct NVLink transport (AMGP_HALO=p2p, dist.cu): peers' halo buffers
    // and synchronisation words mapped through CUDA IPC; the kernels
    // themselves signal and wait (sync_stride words per matrix slot)
    int halo_p2p = 0;  // 0: NCCL, 1: p2p (default)
    // p2p: interior and boundary slices in one launch (rows.cuh launch_rows):
    // AMGP_HALO_FUSE=0 never, 1 where it measured faster (default), 2 always
    int halo_fuse = 1;
    // fused launches also pack the halo in their first CTAs (no pack kernel,
    // no cross-stream events); AMGP_HALO_XPACK=0: the separate pack kernel
    int halo_xpack = 1;
    // copy streams of the host-buffer smoother path (created on first use)
    cudaStream_t io_h2d = nullptr, io_d2h = nullptr;
    unsigned long long *sync = nullptr;            // [AMGP_MAX_SLOTS][sync_stride]
    std::vector<unsigned long long *> peer_sync;   // every rank's sync array (self included)
    int sync_stride = 0;
    int next_slot = 0;
    // p2p ordered all-reduce (dist.cu allreduce_sum_ordered): a region after
    // the slots of every rank's sync array, [2 parities][nranks][32 words]
    // (16 values, word 31 = the sender's epoch flag), then a local epoch word
    unsigned long long *red = nullptr;                   // my region
    unsigned long long *const *d_peer_red = nullptr;     // device [nranks]: every rank's region
    unsigned long long *red_epoch = nullptr;
    int red_ar = 1;  // AMGP_P2P_ALLREDUCE=0: NCCL AllGather + fold instead
};

// Slots are never reused: a freed slot's words may still receive a peer's
// final ready/consumed signal, so reuse would need a collective in
// amgp_mat_destroy (unsafe from garbage-collected owners).  4096 slots of
// 16 words = 512 KB per context; ~3 slots per distributed level.
#ifndef AMGP_MAX_SLOTS
#define AMGP_MAX_SLOTS 4096
#endif
// per-slot synchronisation words of the p2p transport (u64, monotonic):
//   [0, nranks)         ready[src]    -- epoch of the last halo src delivered here
//   [nranks, 2 nranks)  consumed[dst] -- epoch whose halo dst has finished reading
//   [2 nranks]          epoch         -- exchanges completed on this rank
//   [2 nranks + 1]      ticket        -- pack-kernel CTAs done (last one signals)
//   [2 nranks + 2]      ticket        -- boundary launch CTAs done (last one completes)
#ifndef AMGP_SYNC_STRIDE
#define AMGP_SYNC_STRIDE(nr) ((2 * (nr) + 3 + 15) / 16 * 16)
#endif

// Halo plan of a row-distributed matrix (dist.cu).  Columns [0, nown) are
// the rank's own entries of the operand vector; columns >= nown index the
// halo buffer, filled per SpMV by NCCL send/recv with the neighbours.
struct HaloPlan {
    int64_t nown = 0, nhalo = 0, nsend = 0;
    std::vector<int> peers;                       // neighbour ranks (ascending)
    std::vector<int64_t> send_cnt, send_off;      // per peer, into sendbuf
    std::vector<int64_t> recv_cnt, recv_off;      // per peer, into halo
    int64_t *send_idx = nullptr;                  // device [nsend] own indices
    double *sendbuf = nullptr;                    // device [nsend]
    double *halo = nullptr;                       // device [nhalo]
    int32_t *interior = nullptr, *boundary = nullptr;  // device slice lists
    int64_t n_interior = 0, n_boundary = 0;
    // the same sets as runs of consecutive slices (first, count); when a set
    // has few runs (row-block partitions of banded levels: interior = one
    // run, boundary = the two block ends) kernels index slices directly
    // instead of through the list
    std::vector<std::pair<int64_t, int64_t>> interior_runs, boundary_runs;
    // p2p transport: sync slot, per-peer remote destinations of my data
    int slot = -1;
    bool sym = false;                // every send peer is also a receive peer
    double **d_dest = nullptr;       // device [2 npeers] remote base for my segment (parity 0, then 1)
    int64_t *d_seg = nullptr;        // device [npeers + 1] send offsets
    std::vector<void *> opened;      // IPC-opened peer halo allocations
    unsigned long long *sync_slot = nullptr;  // device: this slot's words on this rank
    int *d_sendp = nullptr, *d_recvp = nullptr;  // device: ranks I send to / receive from
    int nsendp = 0, nrecvp = 0;
    unsigned long long **d_ready_remote = nullptr;     // [nsendp] ready[me] on each receiver
    unsigned long long **d_consumed_remote = nullptr;  // [nrecvp] consumed[me] on each sender
};

// The stream library work of a context is enqueued on.  A V-cycle graph is
// captured on a private stream (vcycle.cu) named by this thread-local
// override, so other host threads keep using ctx->stream meanwhile (their
// launches can never end up inside the capture).
struct CaptureOverride {
    const amgp_ctx *ctx = nullptr;
    cudaStream_t stream = nullptr;
};
extern thread_local CaptureOverride amgp_capture;
inline cudaStream_t cur_stream(const amgp_ctx *ctx) {
    return amgp_capture.ctx == ctx ? amgp_capture.stream : ctx->stream;
}

struct amgp_mat {
    amgp_ctx *ctx = nullptr;
    int64_t nrows = 0, ncols = 0, nnz = 0;
    int64_t nslices = 0, stored = 0;
    int64_t *slice_ptr = nullptr;  // [nslices+1] element offsets (multiples of 32)
    int32_t *col = nullptr;        // [stored], -1 = padding
    double *val = nullptr;         // [stored]
    int32_t max_width = 0;
    // SELL-C-sigma: rows sorted by length inside windows of AMGP_SIGMA rows
    // (fewer padded slots); perm[pos] = row stored at SELL position pos (-1:
    // padding), iperm[row] = its position.  Both null: identity order.
    int32_t *perm = nullptr, *iperm = nullptr;
    int64_t row_offset = 0;  // first global row of a generated row block
    std::vector<int64_t> slice_maxcol;  // host: largest column per slice (-1: empty)
    HaloPlan *halo = nullptr;           // non-null: distributed operand
    // per-matrix smoother workspace (r, two operand buffers, x copy)
    double *work = nullptr;
    int64_t work_n = 0;
    // host-buffer path (amgp_smoother_apply_host): two (b, x0, x) slots
    double *io = nullptr;
    int64_t io_n = 0;
    std::mutex mu;
};

// Plain-old-data view passed to kernels.
#define SELL_RUNS 8
struct SellView {
    const int64_t *__restrict__ slice_ptr;
    const int32_t *__restrict__ col;
    const double *__restrict__ val;
    int64_t nrows;
    int64_t nslices;
    const int32_t *__restrict__ perm;   // SELL-C-sigma row order (see amgp_mat), or null
    const int32_t *__restrict__ iperm;
    const int32_t *__restrict__ slist;  // slices to process (nullptr: the run table)
    int64_t nlist;
    int64_t nown;                       // gathers of columns >= nown read xh
    const double *__restrict__ xh;
    // up to SELL_RUNS runs of consecutive slices: launch index i < run_end[0]
    // is slice run_s0[0] + i, etc. (interior / boundary sets of row blocks)
    int nruns;
    int64_t run_s0[SELL_RUNS], run_end[SELL_RUNS];
    // p2p transport: before gathering xh, wait until every rank in recvp has
    // delivered this exchange (sync words of the matrix slot, amgp_ctx); the
    // halo is double-buffered by exchange parity: exchange e lives at
    // xh + (e & 1) * xh_stride
    unsigned long long *sync_slot;
    const int *recvp;
    int nrecvp, nranks;
    int complete;  // ROWS_GEN boundary launch of the p2p transport: last CTA completes
    unsigned long long *const *consumed_remote;
    int64_t xh_stride;
};

inline SellView view_of(const amgp_mat *A) {
    SellView v{};
    v.slice_ptr = A->slice_ptr;
    v.col = A->col;
    v.val = A->val;
    v.perm = A->perm;
    v.iperm = A->iperm;
    v.nrows = A->nrows;
    v.nslices = A->nslices;
    v.nlist = A->nslices;
    v.nown = INT64_MAX;
    v.nruns = 1;
    v.run_s0[0] = 0;
    v.run_end[0] = A->nslices;
    return v;
}

#define AMGP_SIGMA 256  // sorting window of SELL-C-sigma (8 slices)

// row stored at SELL position pos (slice pos / 32, lane pos % 32); -1: padding
__device__ __forceinline__ int64_t sell_row(const SellView &A, int64_t pos) {
    if (A.perm) return A.perm[pos];
    return pos < A.nrows ? pos : -1;
}
// SELL position of row i
__device__ __forceinline__ int64_t sell_pos(const SellView &A, int64_t i) {
    return A.iperm ? (int64_t)A.iperm[i] : i;
}

// slice processed by launch index idx (run table; see SellView)
__device__ __forceinline__ int64_t run_slice(const SellView &A, int64_t idx) {
    int64_t s = A.run_s0[0] + idx;
#pragma unroll
    for (int r = 1; r < SELL_RUNS; r++)
        if (r < A.nruns && idx >= A.run_end[r - 1]) s = A.run_s0[r] + (idx - A.run_end[r - 1]);
    return s;
}

// An opaque copy of p: loads through it cannot be scheduled before this point
// (the halo pointer after halo_wait's barrier).
__device__ __forceinline__ const double *launder_ptr(const double *p) {
    asm volatile("" : "+l"(p)::"memory");
    return p;
}

// system-scope acquire / release on u64 words (peer-mapped synchronisation)
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// polling loads: no acquire (an acquire load also invalidates the SM's L1,
// which the gathers of the CTAs sharing the SM live on); one acquire after
// the condition holds
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_gpu(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Boundary kernels of the p2p transport: one thread per CTA waits until the
// halo of the current exchange (epoch + 1) has arrived from every sender.
// Returns the halo buffer of this exchange: the p2p halo is double-buffered
// by exchange parity (xh_stride = nhalo; 0 for NCCL).  Every thread reads
// the epoch itself: it only advances after every CTA of the launch has
// passed the completion ticket (halo_complete).
__device__ __forceinline__ const double *halo_wait(const SellView &A) {
    if (A.nrecvp == 0) return A.xh;
    const unsigned long long e = ld_relaxed_gpu(A.sync_slot + 2 * A.nranks);
    if (threadIdx.x == 0) {  // relaxed polls, one acquire (an acquire load invalidates the SM's L1)
        for (int i = 0; i < A.nrecvp; i++) {
            const unsigned long long *w = A.sync_slot + A.recvp[i];
            while (ld_relaxed_sys(w) < e + 1) __nanosleep(20);
            (void)ld_acquire_sys(w);
        }
    }
    __syncthreads();
    return launder_ptr(A.xh + (int64_t)(e & 1ull) * A.xh_stride);
}

// End of a boundary launch of the p2p transport, called by its nctas CTAs:
// the last of them advances the epoch and tells every sender its halo has
// been read (all reads precede the ticket).
__device__ __forceinline__ void halo_complete(const SellView &A, unsigned nctas) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long *sync = A.sync_slot;
        __threadfence();
        unsigned long long *ticket = sync + 2 * A.nranks + 2;
        if (atomicAdd(ticket, 1ull) == nctas - 1) {
            *ticket = 0;
            const unsigned long long e = sync[2 * A.nranks] + 1;
            sync[2 * A.nranks] = e;
            __threadfence_system();
            for (int i = 0; i < A.nrecvp; i++) st_release_sys(A.consumed_remote[i], e);
        }
    }
}

// p2p pack of one exchange (the k_pack_p2p kernel, and the first CTAs of the
// fused row kernels, rows.cuh): entry i of the send list goes straight to its
// receiver's halo buffer of this exchange's parity; ncta CTAs share the list
// and the last of them publishes ready = epoch + 1 on every receiver.  Before
// writing, a non-symmetric exchange waits until each receiver consumed
// exchange epoch - 2 (see dist.cu).
struct PackView {
    int64_t n = 0;  // entries to send
    int npeers = 0, nsendp = 0, sym = 1;
    const int64_t *idx = nullptr;
    double *const *dest = nullptr;  // [2 npeers]
    const int64_t *seg = nullptr;   // [npeers + 1]
    const int *sendp = nullptr;
    unsigned long long *const *ready_remote = nullptr;
};

__device__ __forceinline__ void halo_pack(const PackView &pk, unsigned long long *sync, int nranks,
                                          const double *__restrict__ x, int64_t cta, int64_t ncta) {
    const unsigned long long epoch = ld_relaxed_gpu(sync + 2 * nranks);
    if (!pk.sym && epoch >= 2) {
        if (threadIdx.x == 0) {  // relaxed polls, one acquire (an acquire load invalidates the SM's L1)
            for (int i = 0; i < pk.nsendp; i++) {
                const unsigned long long *w = sync + nranks + pk.sendp[i];
                while (ld_relaxed_sys(w) + 1 < epoch) __nanosleep(20);
                (void)ld_acquire_sys(w);
            }
        }
        __syncthreads();
    }
    const int par = (int)(epoch & 1ull);
    for (int64_t i = cta * blockDim.x + threadIdx.x; i < pk.n; i += ncta * blockDim.x) {
        int q = 0;
        while (q + 1 < pk.npeers && i >= pk.seg[q + 1]) q++;
        pk.dest[par * pk.npeers + q][i - pk.seg[q]] = x[pk.idx[i]];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        unsigned long long *ticket = sync + 2 * nranks + 1;
        if (atomicAdd(ticket, 1ull) == (unsigned long long)ncta - 1) {
            *ticket = 0;
            __threadfence_system();
            for (int i = 0; i < pk.nsendp; i++) st_release_sys(pk.ready_remote[i], epoch + 1);
        }
    }
}

PackView pack_view(const HaloPlan &h);  // dist.cu

// Exchange the halo of operand x (own part) for a distributed matrix; after
// it, kernels may gather x through view.xh (dist.cu).
int halo_exchange_begin(amgp_ctx *ctx, const amgp_mat *A, const double *x);
int halo_exchange_end(amgp_ctx *ctx, const amgp_mat *A);
int halo_exchange_done(amgp_ctx *ctx, const amgp_mat *A);  // after the boundary rows
void mat_free_halo(amgp_mat *A);
void ctx_free_comm(amgp_ctx *ctx);  // communicator resources (amgp_ctx_destroy)
int refresh_slice_maxcol(amgp_mat *A);  // recompute A->slice_maxcol from the device columns

// Resolved smoother configuration with host-computed step scalars
// (smoothers.py:112-135 expressions evaluated in binary64 on the host).
struct SmootherPlan {
    int family = AMGP_L1_JACOBI;
    int degree = 1;
    double rho = 1.0;
    std::vector<double> coef;  // layout documented at amgp_smoother_coefficients
};

int make_smoother_plan(const amgp_smoother_cfg *cfg, SmootherPlan *plan);

// Workspace needed by smoother_enqueue for an n-row matrix (doubles).
inline int64_t smoother_work_doubles(int64_t n) { return 4 * n; }

// Enqueue one smoother application on cur_stream(ctx).  x0 == nullptr: zero
// initial guess.  x0 must not alias x.  work: smoother_work_doubles(n).
int smoother_enqueue(amgp_ctx *ctx, const amgp_mat *A, const double *m, const SmootherPlan &p,
                     const double *b, const double *x0, double *x, double *work);

// y = A x ; y = r - A x ; x += P xc  (thread per row, stored order)
int spmv_enqueue(amgp_ctx *ctx, const amgp_mat *A, const double *x, double *y);
int residual_enqueue(amgp_ctx *ctx, const amgp_mat *A, const double *r, const double *x,
                     double *res);
int prolong_add_enqueue(amgp_ctx *ctx, const amgp_mat *P, const double *xc, double *x);

// Grid helpers
inline unsigned grid_for(int64_t nthreads, int block) {
    return (unsigned)((nthreads + block - 1) / block);
}

// ---------------------------------------------------------------- device helpers
// L2 cache policies (createpolicy): matrix slots are streamed once per step
// (evict_first); gathered operands are reused by neighbouring rows
// (evict_last).  The per-load .L2::evict_* qualifiers need 256-bit loads on
// sm_100, so scalar loads carry the policy via .L2::cache_hint.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double ld_stream_f64(const double *p, uint64_t pol) {
    double v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                 : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int32_t ld_stream_s32(const int32_t *p, uint64_t pol) {
    int32_t v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
                 : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld_gather_f64(const double *p, uint64_t pol) {
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
// Gathers of a boundary launch (columns may index the halo, which a peer GPU
// writes while the kernel runs on the p2p transport): never through the
// non-coherent (.nc) path.  A weak ld.global is coherent after the in-kernel
// acquire (halo_wait: ld.acquire.sys, which also invalidates the SM's L1, then
// bar.sync), and it keeps L1 reuse of the neighbouring x entries; the
// compiler cannot hoist it above the wait because the halo pointer comes out
// of halo_wait laundered (launder_ptr, after the barrier).  One load from a
// selected pointer per slot keeps the U gathers a single predicated batch (a
// per-slot branch between two load kinds serialised them: 0.42 vs 0.31 s per
// 635^3 solve on 4 GPUs).  AMGP_HALO_LD_CG: the previous L2-only .cg load with
// a memory clobber (A/B variant).
__device__ __forceinline__ double ld_halo_f64(const double *p, uint64_t pol) {
    double v;
#ifdef AMGP_HALO_LD_CG
    (void)pol;
    asm("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
#else
    asm("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
#endif
    return v;
}

// Row sum of slice row `lane` of slice `s`: sum_j val*x[col] from 0.0 in slot
// order (== CSR stored order).  Slots are loaded U at a time (predicated) so
// a warp keeps 2U streaming loads + U gathers in flight.  Padding slots
// (col < 0) contribute nothing.  HALO: columns >= A.nown read the halo
// buffer A.xh (boundary slices of a distributed matrix); every other launch
// takes the plain single-load gather.
template <int U, bool HALO = false>
__device__ __forceinline__ double sell_row_dot(const SellView &A, int64_t s, int lane,
                                               const double *__restrict__ x,
                                               const double *__restrict__ xh = nullptr) {
    const int64_t base = A.slice_ptr[s];
    const int w = (int)((A.slice_ptr[s + 1] - base) >> 5);
    const int32_t *c = A.col + base + lane;
    const double *v = A.val + base + lane;
    const uint64_t pf = policy_evict_first(), pl = policy_evict_last();
    double sum = 0.0;
    for (int j = 0; j < w; j += U) {
        int32_t cc[U];
        double vv[U], xx[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const bool ok = j + u < w;
            cc[u] = ok ? ld_stream_s32(c + (int64_t)(j + u) * AMGP_SLICE, pf) : -1;
            vv[u] = ok ? ld_stream_f64(v + (int64_t)(j + u) * AMGP_SLICE, pf) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            if (HALO) {
                const int64_t c = cc[u];
                const bool own = c < A.nown;
                const double *p = (own ? x : xh) + (own ? c : c - A.nown);
                xx[u] = c < 0 ? 0.0 : ld_halo_f64(p, pl);
            } else
                xx[u] = cc[u] < 0 ? 0.0 : ld_gather_f64(x + cc[u], pl);
        }
#pragma unroll
        for (int u = 0; u < U; u++)
            if (cc[u] >= 0) sum = __dadd_rn(sum, __dmul_rn(vv[u], xx[u]));
    }
    return sum;
}
