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
// IPC mapping, NVLink stores) and the kernels hand over ownership through
// monotonic u64 epoch words (amgp_ctx::sync, one slot per distributed
// matrix, peer-mapped):
//   pack (comm stream)  stores into the receiver's halo buffer of parity
//                       epoch & 1 (double-buffered), after consumed[dst] >=
//                       epoch - 1 (dst finished reading exchange epoch - 2;
//                       implied for symmetric exchanges, see k_pack_p2p), and
//                       its last CTA sets ready[me] = epoch + 1 on every
//                       receiver (release.sys)
//   boundary rows       wait ready[src] >= epoch + 1 (acquire.sys) first
//   completion          epoch += 1 and consumed[me] = epoch on every sender:
//                       the boundary launch's last CTA, else k_halo_signal
// Exchange order is the same on every rank (SPMD), so no wait can close a
// cycle; everything is an ordinary kernel and is captured into graphs.
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
                                    (ncclComm_t)ctx->comm, cur_stream(ctx));
    if (r != ncclSuccess) {
        cudaFree(d);
        return amgp_fail(AMGP_ENCCL, "allgather failed");
    }
    all.resize(bytes * ctx->nranks);
    AMGP_CUDA(cudaStreamSynchronize(cur_stream(ctx)));
    AMGP_CUDA(cudaMemcpy(all.data(), d, all.size(), cudaMemcpyDeviceToHost));
    cudaFree(d);
    return AMGP_OK;
}

// Map every rank's synchronisation words.  Collective; when any rank cannot
// map a peer (no CUDA IPC / peer access between the GPUs) every rank stays
// on NCCL.
static int p2p_init(amgp_ctx *ctx) {
    const int nr = ctx->nranks;
    ctx->sync_stride = AMGP_SYNC_STRIDE(nr);
    const size_t slot_words = (size_t)AMGP_MAX_SLOTS * ctx->sync_stride;
    const size_t words = slot_words + (size_t)2 * nr * 32 + 32;  // + the all-reduce region
    AMGP_CUDA(cudaMalloc(&ctx->sync, words * sizeof(unsigned long long)));
    AMGP_CUDA(cudaMemset(ctx->sync, 0, words * sizeof(unsigned long long)));
    cudaIpcMemHandle_t mine;
    AMGP_CUDA(cudaIpcGetMemHandle(&mine, ctx->sync));
    std::vector<char> all;
    AMGP_TRY(allgather_host(ctx, &mine, sizeof(mine), all));
    ctx->peer_sync.assign(nr, nullptr);
    int ok = 1;
    for (int r = 0; r < nr; r++) {
        if (r == ctx->rank) {
            ctx->peer_sync[r] = ctx->sync;
            continue;
        }
        cudaIpcMemHandle_t h;
        memcpy(&h, all.data() + r * sizeof(h), sizeof(h));
        void *p = nullptr;
        if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            cudaGetLastError();
            ok = 0;
            continue;
        }
        ctx->peer_sync[r] = (unsigned long long *)p;
    }
    std::vector<char> oks;
    AMGP_TRY(allgather_host(ctx, &ok, sizeof(ok), oks));
    for (int r = 0; r < nr; r++) ok &= ((const int *)oks.data())[r];
    if (!ok) {
        for (int r = 0; r < nr; r++)
            if (r != ctx->rank && ctx->peer_sync[r]) cudaIpcCloseMemHandle(ctx->peer_sync[r]);
        ctx->peer_sync.clear();
        cudaFree(ctx->sync);
        ctx->sync = nullptr;
        return AMGP_OK;  // halo_p2p stays 0: NCCL transport
    }
    std::vector<unsigned long long *> red(nr);
    for (int r = 0; r < nr; r++) red[r] = ctx->peer_sync[r] + slot_words;
    AMGP_CUDA(cudaMalloc((void **)&ctx->d_peer_red, nr * sizeof(unsigned long long *)));
    AMGP_CUDA(cudaMemcpy((void *)ctx->d_peer_red, red.data(), nr * sizeof(unsigned long long *),
                         cudaMemcpyHostToDevice));
    ctx->red = ctx->sync + slot_words;
    ctx->red_epoch = ctx->red + (size_t)2 * nr * 32;
    AMGP_CUDA(cudaDeviceSynchronize());
    ctx->halo_p2p = 1;
    const char *fz = getenv("AMGP_HALO_FUSE");
    ctx->halo_fuse = fz && fz[0] >= '0' && fz[0] <= '2' ? fz[0] - '0' : 1;
    const char *xp = getenv("AMGP_HALO_XPACK");
    ctx->halo_xpack = !(xp && xp[0] == '0');
    const char *ar = getenv("AMGP_P2P_ALLREDUCE");
    ctx->red_ar = !(ar && ar[0] == '0');
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
    ctx->prio_high = greatest;
    AMGP_CUDA(cudaEventCreateWithFlags(&ctx->ev_packed, cudaEventDisableTiming));
    AMGP_CUDA(cudaEventCreateWithFlags(&ctx->ev_exchanged, cudaEventDisableTiming));
    AMGP_CUDA(cudaMalloc(&ctx->gather_buf, (size_t)nranks * 16 * sizeof(double)));
    // halo transport: direct NVLink (default when every pair of GPUs can
    // map each other, <= 64 ranks) or NCCL (AMGP_HALO=nccl, or fallback)
    const char *mode = getenv("AMGP_HALO");
    const bool want_p2p = !mode || strcmp(mode, "p2p") == 0;
    if (want_p2p && nranks > 1 && nranks <= 64) AMGP_TRY(p2p_init(ctx));
    return AMGP_OK;
}

// Release the communicator side of a context (amgp_ctx_destroy): IPC
// mappings of the peers' synchronisation words, NCCL communicator, streams.
void ctx_free_comm(amgp_ctx *ctx) {
    for (size_t r = 0; r < ctx->peer_sync.size(); r++)
        if ((int)r != ctx->rank && ctx->peer_sync[r]) cudaIpcCloseMemHandle(ctx->peer_sync[r]);
    ctx->peer_sync.clear();
    cudaFree(ctx->sync);
    ctx->sync = nullptr;
    cudaFree((void *)ctx->d_peer_red);
    ctx->d_peer_red = nullptr;
    ctx->red = ctx->red_epoch = nullptr;
    cudaFree(ctx->gather_buf);
    ctx->gather_buf = nullptr;
    if (ctx->ev_packed) cudaEventDestroy(ctx->ev_packed);
    if (ctx->ev_exchanged) cudaEventDestroy(ctx->ev_exchanged);
    ctx->ev_packed = ctx->ev_exchanged = nullptr;
    if (ctx->comm_stream) {
        cudaStreamSynchronize(ctx->comm_stream);
        cudaStreamDestroy(ctx->comm_stream);
        ctx->comm_stream = nullptr;
    }
    NcclApi *api = nccl();
    if (ctx->comm && api && api->CommDestroy) api->CommDestroy((ncclComm_t)ctx->comm);
    ctx->comm = nullptr;
}

extern "C" int amgp_ctx_comm_info(amgp_ctx *ctx, int *nranks, int *rank) {
    if (!ctx) return amgp_fail(AMGP_EINVAL, "null context");
    if (nranks) *nranks = ctx->nranks;
    if (rank) *rank = ctx->rank;
    return AMGP_OK;
}

// ---------------------------------------------------------------- halo plans
// Freeing a plan needs no cross-rank barrier under SPMD use: every peer's
// pack into my halo buffer for an exchange completes before my boundary
// launch of that exchange (which waits for it), so after my stream is idle no
// peer writes my halo buffers; the peers' last consumed/ready signals land in
// the context's sync words, which live as long as the context.
static void halo_free(HaloPlan *h) {
    if (!h) return;
    for (void *p : h->opened) cudaIpcCloseMemHandle(p);
    cudaFree(h->d_dest);
    cudaFree(h->d_seg);
    cudaFree(h->d_sendp);
    cudaFree(h->d_recvp);
    cudaFree(h->d_ready_remote);
    cudaFree(h->d_consumed_remote);
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
    if (ctx->next_slot >= AMGP_MAX_SLOTS)
        return amgp_fail(AMGP_EINVAL, "too many distributed matrices on this context: all " +
                                          std::to_string(AMGP_MAX_SLOTS) +
                                          " p2p synchronisation slots are used (slots are not reused)");
    h->slot = ctx->next_slot++;
    struct Info {
        cudaIpcMemHandle_t handle;
        int64_t recv_off[64];
        int64_t recv_cnt[64];
        int64_t nhalo;
    };
    Info mine;
    memset(&mine, 0, sizeof(mine));
    AMGP_CUDA(cudaIpcGetMemHandle(&mine.handle, h->halo));
    mine.nhalo = h->nhalo;
    for (size_t q = 0; q < h->peers.size(); q++) {
        mine.recv_off[h->peers[q]] = h->recv_off[q];
        mine.recv_cnt[h->peers[q]] = h->recv_cnt[q];
    }
    std::vector<char> all;
    AMGP_TRY(allgather_host(ctx, &mine, sizeof(Info), all));
    const size_t np = h->peers.size();
    std::vector<double *> dest(2 * np, nullptr);
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
        dest[np + q] = dest[q] + peer.nhalo;  // parity-1 buffer
    }
    seg[np] = h->nsend;
    AMGP_CUDA(cudaMalloc(&h->d_dest, std::max<size_t>(2 * np, 1) * sizeof(double *)));
    AMGP_CUDA(cudaMalloc(&h->d_seg, (np + 1) * sizeof(int64_t)));
    if (np) AMGP_CUDA(cudaMemcpy(h->d_dest, dest.data(), 2 * np * sizeof(double *), cudaMemcpyHostToDevice));
    AMGP_CUDA(cudaMemcpy(h->d_seg, seg.data(), (np + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
    // synchronisation words: mine for this slot, and where to signal peers
    const int nr = ctx->nranks, me = ctx->rank, st = ctx->sync_stride;
    h->sync_slot = ctx->sync + (size_t)h->slot * st;
    std::vector<int> sendp, recvp;
    std::vector<unsigned long long *> ready_remote, consumed_remote;
    for (size_t q = 0; q < np; q++) {
        const int r = h->peers[q];
        if (h->send_cnt[q] > 0) {
            sendp.push_back(r);
            ready_remote.push_back(ctx->peer_sync[r] + (size_t)h->slot * st + me);
        }
        if (h->recv_cnt[q] > 0) {
            recvp.push_back(r);
            consumed_remote.push_back(ctx->peer_sync[r] + (size_t)h->slot * st + nr + me);
        }
    }
    h->nsendp = (int)sendp.size();
    h->nrecvp = (int)recvp.size();
    h->sym = std::all_of(sendp.begin(), sendp.end(), [&](int r) {
        return std::find(recvp.begin(), recvp.end(), r) != recvp.end();
    });
    auto upload = [](void **dst, const void *src, size_t bytes) -> cudaError_t {
        cudaError_t e = cudaMalloc(dst, std::max<size_t>(bytes, 8));
        if (e == cudaSuccess && bytes) e = cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
        return e;
    };
    AMGP_CUDA(upload((void **)&h->d_sendp, sendp.data(), sendp.size() * sizeof(int)));
    AMGP_CUDA(upload((void **)&h->d_recvp, recvp.data(), recvp.size() * sizeof(int)));
    AMGP_CUDA(upload((void **)&h->d_ready_remote, ready_remote.data(), ready_remote.size() * sizeof(void *)));
    AMGP_CUDA(upload((void **)&h->d_consumed_remote, consumed_remote.data(),
                     consumed_remote.size() * sizeof(void *)));
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
    // p2p: two halo buffers (exchange parity, see k_pack_p2p)
    if (e == cudaSuccess)
        e = cudaMalloc(&h->halo, std::max<int64_t>(ro, 1) * (ctx->halo_p2p > 0 ? 2 : 1) * sizeof(double));
    if (e != cudaSuccess) {
        halo_free(h);
        return amgp_cuda_fail(e, "halo plan upload", __FILE__, __LINE__);
    }
    if (ctx->halo_p2p > 0) {  // collective: every rank attaches its plans in the same order
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
// buffer of this exchange's parity (double-buffered: exchange e writes
// buffer e & 1, so it only has to wait until each receiver has consumed
// exchange e - 2 -- and not at all when every receiver also sends to me: my
// launches of exchange e - 1 waited for its pack of e - 1, which its stream
// issued after its boundary launch of e - 2; with the pack inside the fused
// row kernel: its kernel of e - 1, boundary included, completed before its
// kernel of e started).  The last CTA to finish publishes the new epoch.
__global__ void k_pack_p2p(PackView pk, const double *__restrict__ x, unsigned long long *sync, int nranks) {
    halo_pack(pk, sync, nranks, x, blockIdx.x, gridDim.x);
}

PackView pack_view(const HaloPlan &h) {
    PackView pk;
    pk.n = h.nsend;
    pk.npeers = (int)h.peers.size();
    pk.idx = h.send_idx;
    pk.dest = h.d_dest;
    pk.seg = h.d_seg;
    pk.sendp = h.d_sendp;
    pk.nsendp = h.nsendp;
    pk.sym = (int)h.sym;
    pk.ready_remote = h.d_ready_remote;
    return pk;
}

// after the boundary rows: this exchange is complete on this rank
__global__ void k_halo_signal(unsigned long long *sync, int nranks, int nrecvp,
                              unsigned long long *const *__restrict__ consumed_remote) {
    if (threadIdx.x != 0) return;
    const unsigned long long e = sync[2 * nranks] + 1;
    sync[2 * nranks] = e;
    __threadfence_system();
    for (int i = 0; i < nrecvp; i++) st_release_sys(consumed_remote[i], e);
}

static int p2p_begin(amgp_ctx *ctx, const HaloPlan &h, const double *x) {
    if (h.nsend == 0) return AMGP_OK;
    cudaStream_t st = ctx->comm_stream;
    AMGP_CUDA(cudaEventRecord(ctx->ev_packed, cur_stream(ctx)));
    AMGP_CUDA(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_packed, 0));
    // launched with the highest priority explicitly (kept when captured into
    // a graph): its CTAs must be scheduled ahead of the interior rows
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)std::min<int64_t>(grid_for(h.nsend, 256), 148 * 4));
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributePriority;
    attr[0].val.priority = ctx->prio_high;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    AMGP_CUDA(cudaLaunchKernelEx(&cfg, k_pack_p2p, pack_view(h), (const double *)x, h.sync_slot, ctx->nranks));
    AMGP_CHECK_LAUNCH(ctx);
    AMGP_CUDA(cudaEventRecord(ctx->ev_exchanged, ctx->comm_stream));
    return AMGP_OK;
}

static int p2p_end(amgp_ctx *ctx, const HaloPlan &h) {
    // the pack kernel must not be overtaken by the next exchange's; the
    // data itself is awaited inside the boundary kernels (halo_wait)
    if (h.nsend > 0) AMGP_CUDA(cudaStreamWaitEvent(cur_stream(ctx), ctx->ev_exchanged, 0));
    return AMGP_OK;
}

int halo_exchange_done(amgp_ctx *ctx, const amgp_mat *A) {
    if (!ctx->halo_p2p) return AMGP_OK;
    const HaloPlan &h = *A->halo;
    if (h.peers.empty()) return AMGP_OK;
    k_halo_signal<<<1, 32, 0, cur_stream(ctx)>>>(h.sync_slot, ctx->nranks, h.nrecvp, h.d_consumed_remote);
    AMGP_CHECK_LAUNCH(ctx);
    return AMGP_OK;
}

int halo_exchange_begin(amgp_ctx *ctx, const amgp_mat *A, const double *x) {
    const HaloPlan &h = *A->halo;
    if (ctx->halo_p2p) return p2p_begin(ctx, h, x);
    NcclApi *api = nccl();
    if (!api || !ctx->comm) return amgp_fail(AMGP_ENCCL, "no communicator for the halo exchange");
    if (h.nsend > 0) {
        const unsigned g = (unsigned)std::min<int64_t>(grid_for(h.nsend, 256), 148 * 8);
        k_pack<<<g, 256, 0, cur_stream(ctx)>>>(h.nsend, h.send_idx, x, h.sendbuf);
        AMGP_CHECK_LAUNCH(ctx);
    }
    AMGP_CUDA(cudaEventRecord(ctx->ev_packed, cur_stream(ctx)));
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
    AMGP_CUDA(cudaStreamWaitEvent(cur_stream(ctx), ctx->ev_exchanged, 0));
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

// The same ordered sum over NVLink (p2p transport): one warp stores my nv
// values into every rank's region (parity epoch & 1), releases my flag there,
// waits for every rank's flag in my region and folds the nranks values in
// rank order -- the NCCL path's exact arithmetic, one ~µs kernel instead of
// an AllGather plus a fold.  Parity reuse is safe: a rank writes exchange e
// only after its kernel of e - 1, which waited for every rank's e - 1 values,
// i.e. after every rank finished reading e - 2.
__global__ void __launch_bounds__(32)
k_p2p_allreduce(const double *__restrict__ local, int nv, double *__restrict__ out,
                unsigned long long *const *__restrict__ peer_red, unsigned long long *red,
                unsigned long long *red_epoch, int nranks, int me) {
    const int t = threadIdx.x;
    const unsigned long long e = *red_epoch;
    const int64_t par = (int64_t)(e & 1ull) * nranks * 32;
    if (t < nv) {
        const unsigned long long bits = (unsigned long long)__double_as_longlong(local[t]);
        for (int r = 0; r < nranks; r++) peer_red[r][par + me * 32 + t] = bits;
    }
    __syncthreads();
    if (t == 0) {
        __threadfence_system();
        for (int r = 0; r < nranks; r++) st_release_sys(peer_red[r] + par + me * 32 + 31, e + 1);
        for (int r = 0; r < nranks; r++) {
            const unsigned long long *w = red + par + r * 32 + 31;
            while (ld_relaxed_sys(w) < e + 1) __nanosleep(20);
            (void)ld_acquire_sys(w);
        }
    }
    __syncthreads();
    if (t < nv) {
        double s = 0.0;
        for (int r = 0; r < nranks; r++)
            s = __dadd_rn(s, __longlong_as_double((long long)ld_relaxed_gpu(red + par + r * 32 + t)));
        out[t] = s;
    }
    __syncthreads();
    if (t == 0) *red_epoch = e + 1;
}

int allreduce_sum_ordered(amgp_ctx *ctx, const double *local, int nv, double *out) {
    if (nv > 16) return amgp_fail(AMGP_EINVAL, "too many reduction values");
    if (ctx->red && ctx->red_ar) {
        k_p2p_allreduce<<<1, 32, 0, cur_stream(ctx)>>>(local, nv, out, ctx->d_peer_red, ctx->red, ctx->red_epoch,
                                                       ctx->nranks, ctx->rank);
        AMGP_CHECK_LAUNCH(ctx);
        return AMGP_OK;
    }
    NcclApi *api = nccl();
    if (!api || !ctx->comm) return amgp_fail(AMGP_ENCCL, "no communicator");
    if (nv > 16) return amgp_fail(AMGP_EINVAL, "too many reduction values");
    NCCL_TRY(api->AllGather(local, ctx->gather_buf, (size_t)nv, ncclDouble, (ncclComm_t)ctx->comm,
                            cur_stream(ctx)));
    k_fold_ranks<<<1, 32, 0, cur_stream(ctx)>>>(ctx->gather_buf, ctx->nranks, nv, out);
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
    AMGP_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), cur_stream(ctx)));
    k_slice_maxcol<<<grid_for(A->nslices * 32, 256), 256, 0, cur_stream(ctx)>>>(view_of(A), d, bad);
    AMGP_CHECK_LAUNCH(ctx);
    int hbad = 0;
    AMGP_CUDA(cudaMemcpyAsync(A->slice_maxcol.data(), d, A->nslices * sizeof(int64_t),
                              cudaMemcpyDeviceToHost, cur_stream(ctx)));
    AMGP_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, cur_stream(ctx)));
    AMGP_CUDA(cudaStreamSynchronize(cur_stream(ctx)));
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
        k_localize<<<g, 256, 0, cur_stream(ctx)>>>(A->stored, A->col, own_lo, own_hi, nseg, dseg);
        AMGP_CHECK_LAUNCH(ctx);
    }
    AMGP_CUDA(cudaStreamSynchronize(cur_stream(ctx)));
    cudaFree(dseg);
    A->ncols = (own_hi - own_lo) + base;
    A->row_offset = 0;  // rows now index the local block; diagonal at column = row
    return refresh_slice_maxcol(A);
}
