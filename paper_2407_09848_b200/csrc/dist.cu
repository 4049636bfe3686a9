// Multi-GPU plumbing: one process per GPU, row-block partitions, NCCL halo
// exchange overlapped with the interior rows.
//
// NCCL is resolved at run time with dlopen("libnccl.so.2"), so the library
// shares whatever NCCL the process already loaded (torch's when
// torch.distributed is in use) instead of pinning its own copy.
//
// A distributed matrix keeps global row order inside the rank's block and
// local column indices: [0, nown) = the rank's own operand entries,
// [nown, nown + nhalo) = the halo buffer, filled by one grouped
// ncclSend/ncclRecv per SpMV.  Row arithmetic does not change with the
// partition, so every kernel returns the single-GPU bits.
#include <cuda.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "amgp_common.cuh"

// ---------------------------------------------------------------- direct NVLink transport
// AMGP_HALO=p2p: instead of NCCL send/recv, the pack kernel stores each
// neighbour's halo entries straight into the neighbour's halo buffer (CUDA
// IPC mapping, NVLink stores), and stream memory operations hand over
// ownership: the sender waits until the receiver has consumed the previous
// exchange, writes, then sets the receiver's "ready" word; the receiver's
// stream waits on "ready" before its boundary rows and sets the sender's
// "consumed" word after them.  No communication kernel, no proxy thread;
// the waits are done by the stream front end (no spinning kernels).
typedef CUresult (*PFN_streamValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static PFN_streamValue32 g_wait32 = nullptr, g_write32 = nullptr;

static int load_stream_memops() {
    if (g_wait32 && g_write32) return AMGP_OK;
    cudaDriverEntryPointQueryResult q1, q2;
    AMGP_CUDA(cudaGetDriverEntryPoint("cuStreamWaitValue32", (void **)&g_wait32, cudaEnableDefault, &q1));
    AMGP_CUDA(cudaGetDriverEntryPoint("cuStreamWriteValue32", (void **)&g_write32, cudaEnableDefault, &q2));
    if (!g_wait32 || !g_write32 || q1 != cudaDriverEntryPointSuccess || q2 != cudaDriverEntryPointSuccess)
        return amgp_fail(AMGP_ECUDA, "stream memory operations unavailable");
    return AMGP_OK;
}

#define CU_TRY(call)                                                                      \
    do {                                                                                  \
        CUresult _r = (call);                                                             \
        if (_r != CUDA_SUCCESS)                                                           \
            return amgp_fail(AMGP_ECUDA, "driver call failed (CUresult " + std::to_string((int)_r) + "): " #call); \
    } while (0)

static inline CUdeviceptr flag_addr(uint32_t *base, int slot, int nranks, int peer, int which) {
    return (CUdeviceptr)(base + ((size_t)slot * nranks + peer) * 2 + which);
}

struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi *nccl() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
#define SYM(f) api.f = (decltype(api.f))dlsym(h, "nccl" #f)
            SYM(GetUniqueId);
            SYM(CommInitRank);
            SYM(CommDestroy);
            SYM(Send);
            SYM(Recv);
            SYM(GroupStart);
            SYM(GroupEnd);
            SYM(AllGather);
            SYM(GetErrorString);
#undef SYM
            api.ok = api.GetUniqueId && api.CommInitRank && api.Send && api.Recv && api.GroupStart &&
                     api.GroupEnd && api.AllGather;
        }
    }
    return api.ok ? &api : nullptr;
}

#define NCCL_TRY(call)                                                                   \
    do {                                                                                 \
        ncclResult_t _r = (call);                                                        \
        if (_r != ncclSuccess)                                                           \
            return amgp_fail(AMGP_ENCCL, std::string("NCCL error in " #call ": ") +      \
                                             (nccl()->GetErrorString ? nccl()->GetErrorString(_r) : "?")); \
    } while (0)

extern "C" int amgp_comm_unique_id(char *out) {
    NcclApi *api = nccl();
    if (!api) return amgp_fail(AMGP_ENCCL, "libnccl.so.2 not found");
    if (!out) return amgp_fail(AMGP_EINVAL, "null output");
    ncclUniqueId id;
    NCCL_TRY(api->GetUniqueId(&id));
    memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
    return AMGP_OK;
}

// all-gather `bytes` host bytes per rank through NCCL (setup-time collective)
static int allgather_host(amgp_ctx *ctx, const void *mine, size_t bytes, std::vector<char> &all) {
    NcclApi *api = nccl();
    char *d = nullptr;
    AMGP_CUDA(cudaMalloc(&d, bytes * (ctx->nranks + 1)));
    AMGP_CUDA(cudaMemcpy(d + bytes * ctx->nranks, mine, bytes, cudaMemcpyHostToDevice));
    ncclResult_t r = api->AllGather(d + bytes * ctx->nranks, d, bytes, ncclChar,
                                    (ncclComm_t)ctx->comm, ctx->stream);
    if (r != ncclSuccess) {
        cudaFree(d);
        return amgp_fail(AMGP_ENCCL, "allgather failed");
    }
    all.resize(bytes * ctx->nranks);
    AMGP_CUDA(cudaStreamSynchronize(ctx->stream));
    AMGP_CUDA(cudaMemcpy(all.data(), d, all.size(), cudaMemcpyDeviceToHost));
    cudaFree(d);
    return AMGP_OK;
}

static int p2p_init(amgp_ctx *ctx) {
    AMGP_TRY(load_stream_memops());
    const int nr = ctx->nranks;
    const size_t nflags = (size_t)AMGP_MAX_SLOTS * nr * 2;
    AMGP_CUDA(cudaMalloc(&ctx->flags, nflags * sizeof(uint32_t)));
    std::vector<uint32_t> init(nflags, 0);
    for (size_t i = 1; i < nflags; i += 2) init[i] = 1;  // every halo buffer starts consumed
    AMGP_CUDA(cudaMemcpy(ctx->flags, init.data(), nflags * sizeof(uint32_t), cudaMemcpyHostToDevice));
    cudaIpcMemHandle_t mine;
    AMGP_CUDA(cudaIpcGetMemHandle(&mine, ctx->flags));
    std::vector<char> all;
    AMGP_TRY(allgather_host(ctx, &mine, sizeof(mine), all));
    ctx->peer_flags.assign(nr, nullptr);
    for (int r = 0; r < nr; r++) {
        if (r == ctx->rank) {
            ctx->peer_flags[r] = ctx->flags;
            continue;
        }
        cudaIpcMemHandle_t h;
        memcpy(&h, all.data() + r * sizeof(h), sizeof(h));
        void *p = nullptr;
        AMGP_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        ctx->peer_flags[r] = (uint32_t *)p;
    }
    ctx->halo_p2p = 1;
    return AMGP_OK;
}

extern "C" int amgp_ctx_init_comm(amgp_ctx *ctx, int nranks, int rank, const char *id) {
    if (!ctx || !id || nranks < 1 || rank < 0 || rank >= nranks)
        return amgp_fail(AMGP_EINVAL, "amgp_ctx_init_comm: bad argument");
    NcclApi *api = nccl();
    if (!api) return amgp_fail(AMGP_ENCCL, "libnccl.so.2 not found");
    AMGP_CUDA(cudaSetDevice(ctx->device));
    ncclUniqueId uid;
    memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
    ncclComm_t comm;
    NCCL_TRY(api->CommInitRank(&comm, nranks, uid, rank));
    ctx->comm = comm;
    ctx->nranks = nranks;
    ctx->rank = rank;
    // Highest priority: the NCCL kernels of a halo exchange become ready at
    // the same moment as the interior-rows kernel and must get their SMs
    // first, or the exchange would wait for the interior kernel to drain.
    int least = 0, greatest = 0;
    AMGP_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    AMGP_CUDA(cudaStreamCreateWithPriority(&ctx->comm_stream, cudaStreamNonBlocking, greatest));
    AMGP_CUDA(cudaEventCreateWithFlags(&ctx->ev_packed, cudaEventDisableTiming));
    AMGP_CUDA(cudaEventCreateWithFlags(&ctx->ev_exchanged, cudaEventDisableTiming));
    AMGP_CUDA(cudaMalloc(&ctx->gather_buf, (size_t)nranks * 16 * sizeof(double)));
    const char *mode = getenv("AMGP_HALO");
    if (mode && strcmp(mode, "p2p") == 0 && nranks > 1) {
        if (nranks > 64) return amgp_fail(AMGP_EINVAL, "p2p halo transport supports <= 64 ranks");
        AMGP_TRY(p2p_init(ctx));
    }
    return AMGP_OK;
}

extern "C" int amgp_ctx_comm_info(amgp_ctx *ctx, int *nranks, int *rank) {
    if (!ctx) return amgp_fail(AMGP_EINVAL, "null context");
    if (nranks) *nranks = ctx->nranks;
    if (rank) *rank = ctx->rank;
    return AMGP_OK;
}

// ---------------------------------------------------------------- halo plans
static void halo_free(HaloPlan *h) {
    if (!h) return;
    for (void *p : h->opened) cudaIpcCloseMemHandle(p);
    cudaFree(h->d_dest);
    cudaFree(h->d_seg);
    cudaFree(h->send_idx);
    cudaFree(h->sendbuf);
    cudaFree(h->halo);
    cudaFree(h->interior);
    cudaFree(h->boundary);
    delete h;
}

void mat_free_halo(amgp_mat *A) {
    halo_free(A->halo);
    A->halo = nullptr;
}

// Map where this rank's data lands in each receiver's halo buffer.
static int p2p_attach(amgp_ctx *ctx, HaloPlan *h) {
    if (ctx->next_slot >= AMGP_MAX_SLOTS) return amgp_fail(AMGP_EINVAL, "too many distributed matrices");
    h->slot = ctx->next_slot++;
    struct Info {
        cudaIpcMemHandle_t handle;
        int64_t recv_off[64];
        int64_t recv_cnt[64];
    };
    Info mine;
    memset(&mine, 0, sizeof(mine));
    AMGP_CUDA(cudaIpcGetMemHandle(&mine.handle, h->halo));
    for (size_t q = 0; q < h->peers.size(); q++) {
        mine.recv_off[h->peers[q]] = h->recv_off[q];
        mine.recv_cnt[h->peers[q]] = h->recv_cnt[q];
    }
    std::vector<char> all;
    AMGP_TRY(allgather_host(ctx, &mine, sizeof(Info), all));
    const size_t np = h->peers.size();
    std::vector<double *> dest(np, nullptr);
    std::vector<int64_t> seg(np + 1, 0);
    for (size_t q = 0; q < np; q++) {
        seg[q] = h->send_off[q];
        if (h->send_cnt[q] == 0) continue;
        Info peer;
        memcpy(&peer, all.data() + h->peers[q] * sizeof(Info), sizeof(Info));
        if (peer.recv_cnt[ctx->rank] != h->send_cnt[q])
            return amgp_fail(AMGP_EINVAL, "halo plans of neighbouring ranks disagree");
        void *base = nullptr;
        AMGP_CUDA(cudaIpcOpenMemHandle(&base, peer.handle, cudaIpcMemLazyEnablePeerAccess));
        h->opened.push_back(base);
        dest[q] = (double *)base + peer.recv_off[ctx->rank];
    }
    seg[np] = h->nsend;
    AMGP_CUDA(cudaMalloc(&h->d_dest, std::max<size_t>(np, 1) * sizeof(double *)));
    AMGP_CUDA(cudaMalloc(&h->d_seg, (np + 1) * sizeof(int64_t)));
    if (np) AMGP_CUDA(cudaMemcpy(h->d_dest, dest.data(), np * sizeof(double *), cudaMemcpyHostToDevice));
    AMGP_CUDA(cudaMemcpy(h->d_seg, seg.data(), (np + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
    return AMGP_OK;
}

extern "C" int amgp_mat_set_halo(amgp_mat *A, int64_t nown, int npeers, const int *peers,
                                 const int64_t *send_cnt, const int64_t *send_idx,
                                 const int64_t *recv_cnt) {
    if (!A || nown < 0 || npeers < 0 || (npeers && (!peers || !send_cnt || !recv_cnt)))
        return amgp_fail(AMGP_EINVAL, "amgp_mat_set_halo: bad argument");
    amgp_ctx *ctx = A->ctx;
    if (!ctx->comm && npeers) return amgp_fail(AMGP_EINVAL, "context has no communicator");
    auto *h = new HaloPlan();
    h->nown = nown;
    int64_t so = 0, ro = 0;
    for (int q = 0; q < npeers; q++) {
        if (peers[q] < 0 || peers[q] >= ctx->nranks || peers[q] == ctx->rank) {
            halo_free(h);
            return amgp_fail(AMGP_EINVAL, "bad peer rank");
        }
        h->peers.push_back(peers[q]);
        h->send_cnt.push_back(send_cnt[q]);
        h->send_off.push_back(so);
        h->recv_cnt.push_back(recv_cnt[q]);
        h->recv_off.push_back(ro);
        so += send_cnt[q];
        ro += recv_cnt[q];
    }
    h->nsend = so;
    h->nhalo = ro;
    if (nown + ro != A->ncols) {
        halo_free(h);
        return amgp_fail(AMGP_EINVAL, "nown + halo size must equal the local column count");
    }
    for (int64_t i = 0; i < so; i++)
        if (send_idx[i] < 0 || send_idx[i] >= nown) {
            halo_free(h);
            return amgp_fail(AMGP_EINVAL, "send index outside the owned range");
        }
    // interior slices touch only owned columns; boundary slices touch the halo
    std::vector<int32_t> in, bd;
    for (int64_t s = 0; s < A->nslices; s++)
        (A->slice_maxcol[s] >= nown ? bd : in).push_back((int32_t)s);
    h->n_interior = (int64_t)in.size();
    h->n_boundary = (int64_t)bd.size();
    auto runs = [](const std::vector<int32_t> &s) {
        std::vector<std::pair<int64_t, int64_t>> r;
        for (int32_t x : s) {
            if (!r.empty() && r.back().first + r.back().second == x) r.back().second++;
            else r.emplace_back(x, 1);
        }
        return r;
    };
    h->interior_runs = runs(in);
    h->boundary_runs = runs(bd);
    cudaError_t e = cudaSuccess;
    auto up = [&](void **dst, const void *src, size_t bytes) {
        if (e != cudaSuccess) return;
        e = cudaMalloc(dst, std::max<size_t>(bytes, 8));
        if (e == cudaSuccess && bytes) e = cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
    };
    up((void **)&h->send_idx, send_idx, so * sizeof(int64_t));
    up((void **)&h->interior, in.data(), in.size() * sizeof(int32_t));
    up((void **)&h->boundary, bd.data(), bd.size() * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMalloc(&h->sendbuf, std::max<int64_t>(so, 1) * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&h->halo, std::max<int64_t>(ro, 1) * sizeof(double));
    if (e != cudaSuccess) {
        halo_free(h);
        return amgp_cuda_fail(e, "halo plan upload", __FILE__, __LINE__);
    }
    if (ctx->halo_p2p) {  // collective: every rank attaches its plans in the same order
        int st = p2p_attach(ctx, h);
        if (st != AMGP_OK) {
            halo_free(h);
            return st;
        }
    }
    mat_free_halo(A);
    A->halo = h;
    return AMGP_OK;
}

extern "C" int amgp_mat_halo_info(const amgp_mat *A, int64_t *nown, int64_t *nhalo,
                                  int64_t *n_interior, int64_t *n_boundary) {
    if (!A) return amgp_fail(AMGP_EINVAL, "null matrix");
    const HaloPlan *h = A->halo;
    if (nown) *nown = h ? h->nown : A->ncols;
    if (nhalo) *nhalo = h ? h->nhalo : 0;
    if (n_interior) *n_interior = h ? h->n_interior : A->nslices;
    if (n_boundary) *n_boundary = h ? h->n_boundary : 0;
    return AMGP_OK;
}

__global__ void k_pack(int64_t n, const int64_t *__restrict__ idx, const double *__restrict__ x,
                       double *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = x[idx[i]];
}

// p2p pack: entry i of the send list goes straight to its receiver's halo
__global__ void k_pack_p2p(int64_t n, int npeers, const int64_t *__restrict__ idx,
                           const double *__restrict__ x, double *const *__restrict__ dest,
                           const int64_t *__restrict__ seg) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int q = 0;
        while (q + 1 < npeers && i >= seg[q + 1]) q++;
        dest[q][i - seg[q]] = x[idx[i]];
    }
}

static int p2p_begin(amgp_ctx *ctx, const HaloPlan &h, const double *x) {
    CUstream s = (CUstream)ctx->stream;
    const int nr = ctx->nranks, me = ctx->rank;
    for (size_t q = 0; q < h.peers.size(); q++) {  // receiver done with the previous data
        if (h.send_cnt[q] == 0) continue;
        const CUdeviceptr consumed = flag_addr(ctx->flags, h.slot, nr, h.peers[q], 1);
        CU_TRY(g_wait32(s, consumed, 1, CU_STREAM_WAIT_VALUE_EQ));
        CU_TRY(g_write32(s, consumed, 0, CU_STREAM_WRITE_VALUE_DEFAULT));
    }
    if (h.nsend > 0) {
        const unsigned g = (unsigned)std::min<int64_t>(grid_for(h.nsend, 256), 148 * 8);
        k_pack_p2p<<<g, 256, 0, ctx->stream>>>(h.nsend, (int)h.peers.size(), h.send_idx, x, h.d_dest,
                                              h.d_seg);
        AMGP_CHECK_LAUNCH(ctx);
    }
    for (size_t q = 0; q < h.peers.size(); q++) {  // data in place: signal (after a memory fence)
        if (h.send_cnt[q] == 0) continue;
        CU_TRY(g_write32(s, flag_addr(ctx->peer_flags[h.peers[q]], h.slot, nr, me, 0), 1,
                         CU_STREAM_WRITE_VALUE_DEFAULT));
    }
    return AMGP_OK;
}

static int p2p_end(amgp_ctx *ctx, const HaloPlan &h) {
    CUstream s = (CUstream)ctx->stream;
    for (size_t q = 0; q < h.peers.size(); q++) {
        if (h.recv_cnt[q] == 0) continue;
        const CUdeviceptr ready = flag_addr(ctx->flags, h.slot, ctx->nranks, h.peers[q], 0);
        CU_TRY(g_wait32(s, ready, 1, CU_STREAM_WAIT_VALUE_EQ));
        CU_TRY(g_write32(s, ready, 0, CU_STREAM_WRITE_VALUE_DEFAULT));
    }
    return AMGP_OK;
}

int halo_exchange_done(amgp_ctx *ctx, const amgp_mat *A) {
    if (!ctx->halo_p2p) return AMGP_OK;
    const HaloPlan &h = *A->halo;
    CUstream s = (CUstream)ctx->stream;
    for (size_t q = 0; q < h.peers.size(); q++) {  // boundary rows read the halo: release it
        if (h.recv_cnt[q] == 0) continue;
        CU_TRY(g_write32(s, flag_addr(ctx->peer_flags[h.peers[q]], h.slot, ctx->nranks, ctx->rank, 1),
                         1, CU_STREAM_WRITE_VALUE_DEFAULT));
    }
    return AMGP_OK;
}

int halo_exchange_begin(amgp_ctx *ctx, const amgp_mat *A, const double *x) {
    const HaloPlan &h = *A->halo;
    if (ctx->halo_p2p) return p2p_begin(ctx, h, x);
    NcclApi *api = nccl();
    if (!api || !ctx->comm) return amgp_fail(AMGP_ENCCL, "no communicator for the halo exchange");
    if (h.nsend > 0) {
        const unsigned g = (unsigned)std::min<int64_t>(grid_for(h.nsend, 256), 148 * 8);
        k_pack<<<g, 256, 0, ctx->stream>>>(h.nsend, h.send_idx, x, h.sendbuf);
        AMGP_CHECK_LAUNCH(ctx);
    }
    AMGP_CUDA(cudaEventRecord(ctx->ev_packed, ctx->stream));
    AMGP_CUDA(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_packed, 0));
    ncclComm_t comm = (ncclComm_t)ctx->comm;
    NCCL_TRY(api->GroupStart());
    for (size_t q = 0; q < h.peers.size(); q++) {
        if (h.send_cnt[q] > 0)
            NCCL_TRY(api->Send(h.sendbuf + h.send_off[q], (size_t)h.send_cnt[q], ncclDouble, h.peers[q],
                               comm, ctx->comm_stream));
        if (h.recv_cnt[q] > 0)
            NCCL_TRY(api->Recv(h.halo + h.recv_off[q], (size_t)h.recv_cnt[q], ncclDouble, h.peers[q],
                               comm, ctx->comm_stream));
    }
    NCCL_TRY(api->GroupEnd());
    AMGP_CUDA(cudaEventRecord(ctx->ev_exchanged, ctx->comm_stream));
    return AMGP_OK;
}

int halo_exchange_end(amgp_ctx *ctx, const amgp_mat *A) {
    if (ctx->halo_p2p) return p2p_end(ctx, *A->halo);
    AMGP_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_exchanged, 0));
    return AMGP_OK;
}

// Sum of per-rank partials, deterministic: allgather nv doubles per rank,
// then every rank folds them in rank order.
__global__ void k_fold_ranks(const double *__restrict__ g, int nranks, int nv, double *out) {
    const int q = threadIdx.x;
    if (q >= nv) return;
    double s = 0.0;
    for (int r = 0; r < nranks; r++) s = __dadd_rn(s, g[r * nv + q]);
    out[q] = s;
}

int allreduce_sum_ordered(amgp_ctx *ctx, const double *local, int nv, double *out) {
    NcclApi *api = nccl();
    if (!api || !ctx->comm) return amgp_fail(AMGP_ENCCL, "no communicator");
    if (nv > 16) return amgp_fail(AMGP_EINVAL, "too many reduction values");
    NCCL_TRY(api->AllGather(local, ctx->gather_buf, (size_t)nv, ncclDouble, (ncclComm_t)ctx->comm,
                            ctx->stream));
    k_fold_ranks<<<1, 32, 0, ctx->stream>>>(ctx->gather_buf, ctx->nranks, nv, out);
    AMGP_CHECK_LAUNCH(ctx);
    return AMGP_OK;
}

// ---------------------------------------------------------------- localisation
// Map global columns of a generated row block to local ones: [own_lo, own_hi)
// -> c - own_lo; halo segment q [lo_q, hi_q) -> nown + base_q + (c - lo_q).
__global__ void k_localize(int64_t stored, int32_t *col, int64_t own_lo, int64_t own_hi, int nseg,
                           const int64_t *__restrict__ seg) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < stored;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = col[e];
        if (c < 0) continue;
        int64_t out = -2;
        if (c >= own_lo && c < own_hi) {
            out = c - own_lo;
        } else {
            const int64_t nown = own_hi - own_lo;
            for (int q = 0; q < nseg; q++)
                if (c >= seg[3 * q] && c < seg[3 * q + 1]) out = nown + seg[3 * q + 2] + (c - seg[3 * q]);
        }
        col[e] = (int32_t)out;  // -2 marks a column outside every segment (caught below)
    }
}

__global__ void k_slice_maxcol(SellView A, int64_t *out, int *bad) {
    const int64_t s = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (s >= A.nslices) return;
    const int64_t base = A.slice_ptr[s];
    const int w = (int)((A.slice_ptr[s + 1] - base) >> 5);
    int64_t mx = -1;
    for (int j = 0; j < w; j++) {
        const int32_t c = A.col[base + (int64_t)j * 32 + lane];
        if (c == -2) atomicExch(bad, 1);
        mx = max(mx, (int64_t)c);
    }
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, (int64_t)__shfl_xor_sync(0xffffffffu, (long long)mx, o));
    if (lane == 0) out[s] = mx;
}

int refresh_slice_maxcol(amgp_mat *A) {
    amgp_ctx *ctx = A->ctx;
    A->slice_maxcol.assign(A->nslices, -1);
    if (A->nslices == 0) return AMGP_OK;
    int64_t *d = nullptr;
    int *bad = nullptr;
    AMGP_CUDA(cudaMalloc(&d, A->nslices * sizeof(int64_t)));
    AMGP_CUDA(cudaMalloc(&bad, sizeof(int)));
    AMGP_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), ctx->stream));
    k_slice_maxcol<<<grid_for(A->nslices * 32, 256), 256, 0, ctx->stream>>>(view_of(A), d, bad);
    AMGP_CHECK_LAUNCH(ctx);
    int hbad = 0;
    AMGP_CUDA(cudaMemcpyAsync(A->slice_maxcol.data(), d, A->nslices * sizeof(int64_t),
                              cudaMemcpyDeviceToHost, ctx->stream));
    AMGP_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    AMGP_CUDA(cudaStreamSynchronize(ctx->stream));
    cudaFree(d);
    cudaFree(bad);
    if (hbad) return amgp_fail(AMGP_EINVAL, "column outside the owned range and every halo segment");
    return AMGP_OK;
}

extern "C" int amgp_mat_localize(amgp_mat *A, int64_t own_lo, int64_t own_hi, int nseg,
                                 const int64_t *seg_lo, const int64_t *seg_hi) {
    if (!A || own_lo < 0 || own_hi < own_lo || nseg < 0)
        return amgp_fail(AMGP_EINVAL, "amgp_mat_localize: bad argument");
    amgp_ctx *ctx = A->ctx;
    std::vector<int64_t> seg(3 * (size_t)std::max(nseg, 1));
    int64_t base = 0;
    for (int q = 0; q < nseg; q++) {
        seg[3 * q] = seg_lo[q];
        seg[3 * q + 1] = seg_hi[q];
        seg[3 * q + 2] = base;
        base += seg_hi[q] - seg_lo[q];
    }
    int64_t *dseg = nullptr;
    AMGP_CUDA(cudaMalloc(&dseg, seg.size() * sizeof(int64_t)));
    AMGP_CUDA(cudaMemcpy(dseg, seg.data(), seg.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    if (A->stored > 0) {
        const unsigned g = (unsigned)std::min<int64_t>(grid_for(A->stored, 256), 148 * 16);
        k_localize<<<g, 256, 0, ctx->stream>>>(A->stored, A->col, own_lo, own_hi, nseg, dseg);
        AMGP_CHECK_LAUNCH(ctx);
    }
    AMGP_CUDA(cudaStreamSynchronize(ctx->stream));
    cudaFree(dseg);
    A->ncols = (own_hi - own_lo) + base;
    A->row_offset = 0;  // rows now index the local block; diagonal at column = row
    return refresh_slice_maxcol(A);
}
