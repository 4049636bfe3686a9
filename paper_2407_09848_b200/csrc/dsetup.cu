// Device-resident AMG hierarchy setup (reference amg.py:97-287 on the GPU).
//
// The reference builds each coarse level with Python greedy loops plus
// scipy's C++ sparse kernels.  The greedy aggregation is inherently
// sequential and stays on the host (setup.cpp, fed with strength lists
// computed here); every floating-point product of the setup runs here, with
// the reference's accumulation order restated per ENTRY:
//
//   diagonal            scipy csr_diagonal (amg.py:221, :267)
//   strength lists      |a_ij| >= theta sqrt(|a_ii a_jj|)       (amg.py:115-121)
//   lambda_max          25 power iterations on D^-1/2 A D^-1/2 with the
//                       dots in OpenBLAS ddot order              (amg.py:194-216)
//   smoothed P          P = P_hat - (diags(omega/d) A) P_hat     (amg.py:219-226)
//   Galerkin            (A^T P) -> P^T (A^T P) -> (G + G^T) 0.5  (amg.py:229-235)
//
// Why per-entry order suffices (so no linked lists are needed): in scipy's
// csr_matmat every output entry (r, k) is 0.0 + a_r,j1 b_j1,k + a_r,j2 b_j2,k +
// ... in the order of the A-side row r, because a canonical B row holds k at
// most once; the linked list only decides the STORAGE order of row r, and
// every consumer here either sorts or only uses per-entry values.  Exact
// zeros are dropped (csr_matmat, csr_binop_csr, eliminate_zeros).  All
// arithmetic is separate IEEE-754 binary64 multiply / add (-fmad=false, and
// __dmul_rn / __dadd_rn spelled out), so the hierarchy is bitwise the
// reference's on one GPU.  On several GPUs (dsetup.py) the same kernels run
// per row block with halo rows exchanged over NCCL.
//
// Count/fill convention of the row-producing entry points: with
// row_ptr == NULL the kernel writes the entry count of every output row to
// row_cnt; with row_ptr (exclusive prefix of those counts) it writes the
// sorted entries.  The two passes compute identical rows.
#include <math.h>
#include <stdio.h>

#include <algorithm>
#include <vector>

#include "amgp_common.cuh"

int allreduce_sum_ordered(amgp_ctx *ctx, const double *local, int nv, double *out);
int mat_alloc(amgp_ctx *ctx, int64_t nrows, int64_t ncols, int64_t nnz, int64_t ns, int64_t stored,
              amgp_mat **out);

namespace {

// length of row i (its SELL position: slice pos / 32, lane pos % 32; padding
// slots sit after the row); *base_out = the row's first slot
__device__ __forceinline__ int sell_row_len(const SellView &A, int64_t i, int64_t *base_out) {
    const int64_t pos = sell_pos(A, i);
    const int64_t s = pos >> 5;
    const int lane = (int)(pos & 31);
    const int64_t base = A.slice_ptr[s];
    const int w = (int)((A.slice_ptr[s + 1] - base) >> 5);
    int len = 0;
    while (len < w && A.col[base + (int64_t)len * 32 + lane] >= 0) len++;
    *base_out = base + lane;
    return len;
}

// ---------------------------------------------------------------- diagonal
__global__ void k_ds_diag(SellView A, double *__restrict__ d) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= A.nrows) return;
    int64_t b;
    const int len = sell_row_len(A, i, &b);
    double acc = 0.0;  // scipy csr_diagonal: sums the (single) diagonal entry from 0
    for (int j = 0; j < len; j++)
        if (A.col[b + (int64_t)j * 32] == i) acc = __dadd_rn(acc, A.val[b + (int64_t)j * 32]);
    d[i] = acc;
}

// ---------------------------------------------------------------- strength
// amg.py:115-121 restricted to the rank's own columns (decoupled
// aggregation; every column is own on one GPU).  rows: optional row list.
__global__ void k_ds_strength(SellView A, const double *__restrict__ d, double theta, int64_t nown,
                              const int64_t *__restrict__ rows, int64_t nlist,
                              const int64_t *__restrict__ off, int64_t *__restrict__ cnt,
                              int32_t *__restrict__ scol, double *__restrict__ sabs) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nlist) return;
    const int64_t i = rows ? rows[t] : t;
    int64_t b;
    const int len = sell_row_len(A, i, &b);
    const double di = d[i];
    int64_t k = off ? off[t] : 0, c0 = k;
    for (int j = 0; j < len; j++) {
        const int64_t c = A.col[b + (int64_t)j * 32];
        if (c == i || c >= nown) continue;
        const double v = A.val[b + (int64_t)j * 32];
        const double thr = __dmul_rn(theta, sqrt(fabs(__dmul_rn(di, d[c]))));
        if (fabs(v) >= thr) {
            if (off) {
                scol[k] = (int32_t)c;
                if (sabs) sabs[k] = fabs(v);
            }
            k++;
        }
    }
    if (!off) cnt[t] = k - c0;
}

// ---------------------------------------------------------------- elementwise
__global__ void k_ds_div(int64_t n, const double *__restrict__ a, const double *__restrict__ b,
                         double *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = __ddiv_rn(a[i], b[i]);
}
__global__ void k_ds_sqrt(int64_t n, const double *__restrict__ a, double *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = sqrt(a[i]);
}
// v = w / nrm (nrm on the device; untouched once the iteration has stopped)
__global__ void k_ds_scale(int64_t n, const double *__restrict__ w, const double *__restrict__ sc,
                           double *__restrict__ v) {
    if (sc[2] != 0.0) return;  // stopped (nrm == 0)
    const double nrm = sc[1];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        v[i] = __ddiv_rn(w[i], nrm);
}

// ---------------------------------------------------------------- OpenBLAS ddot
// numpy's float64 dot as OpenBLAS 0.3.30's SkylakeX ddot evaluates it (see
// setup.cpp amgp_setup_blas_dot for the host statement): elements
// [0, n32) feed 32 sequential FMA chains, chain L taking elements L, L+32,
// ... -- exactly one warp lane per chain, so a warp streams both vectors
// fully coalesced.  Then the 8->4 fold, one optional 16-element block, the
// fixed combination tree and the scalar FMA tail.  One CTA per OpenBLAS
// thread chunk; three dots (x.y, x.x, y.y) share one pass.
//
// The chains are latency bound (one dependent FMA per 32 elements per lane),
// so the operands are staged by the bulk-copy engine: one producer thread
// issues cp.async.bulk copies of x and y into a 12-stage shared-memory ring
// (mbarrier complete_tx), the consumer warp runs the chains out of shared
// memory.  Misaligned chunks take the plain-load path (same arithmetic).
#ifndef DOT_STAGES
#define DOT_STAGES 12  // 192 KB in flight for the one-SM chain (8: 128 KB; tools/setup_ab.py, same bits)
#endif
#ifndef DOT_CH
#define DOT_CH 1024  // doubles per stage per operand (8 KB)
#endif

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// exact OpenBLAS combination of the 32 chain accumulators plus the 16-block
// and scalar tail (setup.cpp ddot_chunk), evaluated by one thread
__device__ double blas_finish(const double *acc, int64_t n, int64_t n1, int64_t n32, const double *x,
                              const double *y) {
    double dot = 0.0;
    if (n1) {
        double a0[4], a1[4], a2[4], a3[4];
        for (int l = 0; l < 4; l++) {
            a0[l] = __dadd_rn(acc[l], acc[l + 4]);
            a1[l] = __dadd_rn(acc[8 + l], acc[8 + l + 4]);
            a2[l] = __dadd_rn(acc[16 + l], acc[16 + l + 4]);
            a3[l] = __dadd_rn(acc[24 + l], acc[24 + l + 4]);
        }
        for (int64_t i = n32; i < n1; i += 16)
            for (int l = 0; l < 4; l++) {
                a0[l] = __fma_rn(x[i + l], y[i + l], a0[l]);
                a1[l] = __fma_rn(x[i + 4 + l], y[i + 4 + l], a1[l]);
                a2[l] = __fma_rn(x[i + 8 + l], y[i + 8 + l], a2[l]);
                a3[l] = __fma_rn(x[i + 12 + l], y[i + 12 + l], a3[l]);
            }
        double s[4];
        for (int l = 0; l < 4; l++) s[l] = __dadd_rn(__dadd_rn(__dadd_rn(a0[l], a1[l]), a2[l]), a3[l]);
        dot = __dadd_rn(__dadd_rn(s[0], s[2]), __dadd_rn(s[1], s[3]));
    }
    for (int64_t i = n1; i < n; i++) dot = __fma_rn(y[i], x[i], dot);
    return dot;
}

struct DotChunk {
    int64_t start, len;
};

__global__ void __launch_bounds__(64) k_blas_dot3(const double *__restrict__ x, const double *__restrict__ y,
                                                  const DotChunk *__restrict__ chunks, int use_bulk,
                                                  double *__restrict__ out) {
    extern __shared__ __align__(128) double dsm[];  // [STAGES][CH] x, then [STAGES][CH] y
    __shared__ __align__(8) uint64_t full[DOT_STAGES], empty[DOT_STAGES];
    __shared__ double accs[3][32];
    const DotChunk ch = chunks[blockIdx.x];
    const double *xs = x + ch.start, *ys = y + ch.start;
    const int64_t n = ch.len, n1 = n & ~(int64_t)15, n32 = n1 & ~(int64_t)31;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double axy = 0.0, axx = 0.0, ayy = 0.0;
    if (use_bulk) {
        double *sx = dsm, *sy = dsm + DOT_STAGES * DOT_CH;
        const int64_t nst = (n32 + DOT_CH - 1) / DOT_CH;
        if (threadIdx.x == 0)
            for (int s = 0; s < DOT_STAGES; s++) {
                mbar_init(&full[s], 1);
                mbar_init(&empty[s], 1);
            }
        __syncthreads();
        if (warp == 1) {
            if (lane == 0)
                for (int64_t k = 0; k < nst; k++) {
                    const int s = (int)(k % DOT_STAGES);
                    if (k >= DOT_STAGES) mbar_wait(&empty[s], (unsigned)((k / DOT_STAGES - 1) & 1));
                    const int64_t e0 = k * DOT_CH;
                    const unsigned bytes = (unsigned)(min((int64_t)DOT_CH, n32 - e0) * 8);
                    mbar_expect_tx(&full[s], 2 * bytes);
                    bulk_g2s(sx + s * DOT_CH, xs + e0, bytes, &full[s]);
                    bulk_g2s(sy + s * DOT_CH, ys + e0, bytes, &full[s]);
                }
        } else {
            for (int64_t k = 0; k < nst; k++) {
                const int s = (int)(k % DOT_STAGES);
                mbar_wait(&full[s], (unsigned)((k / DOT_STAGES) & 1));
                const int len = (int)min((int64_t)DOT_CH, n32 - k * DOT_CH);
                const double *px = sx + s * DOT_CH + lane, *py = sy + s * DOT_CH + lane;
#pragma unroll 4
                for (int t = 0; t < len; t += 32) {
                    const double a = px[t], b = py[t];
                    axy = __fma_rn(a, b, axy);
                    axx = __fma_rn(a, a, axx);
                    ayy = __fma_rn(b, b, ayy);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            }
        }
    } else if (warp == 0) {
        for (int64_t i = 0; i < n32; i += 32) {
            const double a = xs[i + lane], b = ys[i + lane];
            axy = __fma_rn(a, b, axy);
            axx = __fma_rn(a, a, axx);
            ayy = __fma_rn(b, b, ayy);
        }
    }
    if (warp == 0) {
        accs[0][lane] = axy;
        accs[1][lane] = axx;
        accs[2][lane] = ayy;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        const int q = threadIdx.x;
        const double *p = q == 0 ? xs : (q == 1 ? xs : ys), *r = q == 0 ? ys : (q == 1 ? xs : ys);
        out[blockIdx.x * 3 + q] = blas_finish(accs[q], n, n1, n32, p, r);
    }
}

// OpenBLAS multi-thread split: chunk dots summed in order from 0.0 (a single
// chunk is returned as is, amgp_setup_blas_dot)
__global__ void k_blas_fold(const double *__restrict__ part, int nchunks, double *__restrict__ out) {
    const int q = threadIdx.x;
    if (q >= 3) return;
    if (nchunks == 1) {
        out[q] = part[q];
        return;
    }
    double s = 0.0;
    for (int c = 0; c < nchunks; c++) s = __dadd_rn(s, part[c * 3 + q]);
    out[q] = s;
}

// lam = (v.w) / (v.v); nrm = sqrt(w.w); stop once nrm == 0 (amg.py:211-215)
__global__ void k_power_scalars(const double *__restrict__ t, double *sc) {
    if (threadIdx.x != 0 || sc[2] != 0.0) return;
    sc[0] = __ddiv_rn(t[0], t[1]);
    const double nrm = sqrt(t[2]);
    sc[1] = nrm;
    if (nrm == 0.0) sc[2] = 1.0;
}

// ---------------------------------------------------------------- smoothed prolongator
// amg.py:219-226 per own row i (thread per row):
//   S row i = reversed A row i, entries 0.0 + (omega/d_i) a_ij, zeros dropped
//   T_ik    = sum over S row i (that order) with agg[j] = k of S_ij * 1.0
//   P_ik    = [k == agg_i] - T_ik  (scipy binop: 1.0 - T, 0.0 - T), zeros dropped
// Unique keys live in a per-thread scratch (capacity = row length + 1),
// output sorted by key (rank = number of smaller kept keys).
__global__ void k_ds_prolong(SellView A, const double *__restrict__ d, const int64_t *__restrict__ agg_own,
                             const int64_t *__restrict__ agg_halo, int64_t nown, double omega, int smooth,
                             const int64_t *__restrict__ rp, int64_t *__restrict__ cnt,
                             int64_t *__restrict__ ocol, double *__restrict__ oval, int64_t *__restrict__ sk,
                             double *__restrict__ sv, int cap) {
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t i = tid; i < A.nrows; i += nthr) {
        const int64_t ai = agg_own[i];
        if (!smooth) {  // P = P_hat
            if (!rp) cnt[i] = 1;
            else {
                ocol[rp[i]] = ai;
                oval[rp[i]] = 1.0;
            }
            continue;
        }
        int64_t b;
        const int len = sell_row_len(A, i, &b);
        const double s = __ddiv_rn(omega, d[i]);
        int u = 0;
        for (int j = len - 1; j >= 0; j--) {
            const int64_t c = A.col[b + (int64_t)j * 32];
            const double sa = __dadd_rn(0.0, __dmul_rn(s, A.val[b + (int64_t)j * 32]));
            if (sa == 0.0) continue;  // dropped from S
            const int64_t key = c < nown ? agg_own[c] : agg_halo[c - nown];
            int q = 0;
            while (q < u && sk[q * nthr + tid] != key) q++;
            if (q == u) {
                sk[q * nthr + tid] = key;
                sv[q * nthr + tid] = 0.0;
                u++;
            }
            sv[q * nthr + tid] = __dadd_rn(sv[q * nthr + tid], __dmul_rn(sa, 1.0));
        }
        // the P_hat key joins the union (T_ik = 0 when absent or cancelled)
        {
            int q = 0;
            while (q < u && sk[q * nthr + tid] != ai) q++;
            if (q == u) {
                sk[q * nthr + tid] = ai;
                sv[q * nthr + tid] = 0.0;
                u++;
            }
        }
        // final values in place: a - b with a = [k == agg_i], b = T (0 if T was dropped)
        for (int q = 0; q < u; q++) {
            const int64_t k = sk[q * nthr + tid];
            const double t = sv[q * nthr + tid];
            sv[q * nthr + tid] = __dsub_rn(k == ai ? 1.0 : 0.0, t);
        }
        int kept = 0;
        for (int q = 0; q < u; q++) {
            const double v = sv[q * nthr + tid];
            if (v == 0.0) continue;
            if (rp) {
                const int64_t k = sk[q * nthr + tid];
                int rank = 0;
                for (int r = 0; r < u; r++)
                    if (sv[r * nthr + tid] != 0.0 && sk[r * nthr + tid] < k) rank++;
                ocol[rp[i] + rank] = k;
                oval[rp[i] + rank] = v;
            }
            kept++;
        }
        if (!rp) cnt[i] = kept;
        (void)cap;
    }
}

// ---------------------------------------------------------------- SpGEMM (hash, warp per row)
// C row r = sum over the A-side entries (b_row, a) of row r IN ORDER of
// a * B[b_row, :].  A canonical B row holds each key once, so the 32 lanes
// take the entries of one B row in parallel (distinct keys: no two lanes
// touch one accumulator) and the warp steps through the A-side entries in
// order (__syncwarp between them): every accumulator sees its contributions
// in the reference's order.  Accumulators live in an open-addressing table
// (shared memory, or a per-warp global-memory table for the few huge rows);
// rows that overflow a table are listed and recomputed with a larger one.
// Output rows are sorted by key with exact zeros dropped.
#define HASH_EMPTY (-1ll)

struct ASide {  // SELL matrix (local columns index B rows) or CSR
    SellView sell;
    int is_sell;
    const int64_t *rp, *col;
    const double *val;
};

struct BRows {  // row b of B is stored at rp[b - off]
    const int64_t *rp, *col;
    const double *val;
    int64_t off;
};

__device__ __forceinline__ unsigned hash_slot(int64_t k, unsigned mask) {
    return (unsigned)(((unsigned long long)k * 0x9E3779B97F4A7C15ull) >> 33) & mask;
}

template <int WARPS, int HC, bool GLOBAL_TABLE>
__global__ void __launch_bounds__(WARPS * 32)
k_ds_spgemm(ASide a, BRows bm, const int64_t *__restrict__ arows, const int64_t *__restrict__ plist,
            int64_t nlist, const int64_t *__restrict__ rp,
            int64_t *__restrict__ cnt, int64_t *__restrict__ ocol, double *__restrict__ oval,
            int64_t *__restrict__ ovf, unsigned long long *__restrict__ novf, int64_t *__restrict__ gkeys,
            double *__restrict__ gvals, int32_t *__restrict__ gslots) {
    constexpr int LIMIT = HC <= 128 ? HC / 2 : HC - 64;  // claims before a row is declared overflowing
    // shared tables (dynamic): keys [WARPS][HC], values [WARPS][HC], claimed slots [WARPS][HC]
    extern __shared__ __align__(16) unsigned char hsm[];
    int64_t *s_keys = reinterpret_cast<int64_t *>(hsm);
    double *s_vals = reinterpret_cast<double *>(hsm + (size_t)WARPS * HC * 8);
    int32_t *s_slots = reinterpret_cast<int32_t *>(hsm + (size_t)WARPS * HC * 16);
    __shared__ int s_nclaim[WARPS], s_ovf[WARPS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t gwarp = (int64_t)blockIdx.x * WARPS + warp;
    const int64_t nwarps = (int64_t)gridDim.x * WARPS;
    int64_t *keys = GLOBAL_TABLE ? gkeys + gwarp * HC : s_keys + warp * HC;
    double *vals = GLOBAL_TABLE ? gvals + gwarp * HC : s_vals + warp * HC;
    int32_t *slots = GLOBAL_TABLE ? gslots + gwarp * HC : s_slots + warp * HC;
    for (int t = lane; t < HC; t += 32) keys[t] = HASH_EMPTY;
    if (lane == 0) s_nclaim[warp] = s_ovf[warp] = 0;
    __syncwarp();
    for (int64_t idx = gwarp; idx < nlist; idx += nwarps) {
        const int64_t p = plist ? plist[idx] : idx;  // output row
        const int64_t r = arows ? arows[p] : p;      // its A-side row
        int64_t abase = 0, aend = 0;
        int astride = 1;
        if (a.is_sell) {
            const int64_t pos = sell_pos(a.sell, r);
            const int64_t s = pos >> 5;
            const int64_t base = a.sell.slice_ptr[s];
            const int w = (int)((a.sell.slice_ptr[s + 1] - base) >> 5);
            abase = base + (pos & 31);
            aend = abase + (int64_t)w * 32;
            astride = 32;
        } else {
            abase = a.rp[r];
            aend = a.rp[r + 1];
        }
        for (int64_t e = abase; e < aend; e += astride) {
            const int64_t ac = a.is_sell ? (int64_t)a.sell.col[e] : a.col[e];
            if (ac < 0) break;  // SELL padding: end of the row
            const int64_t brow = ac - bm.off;
            const double av = a.is_sell ? a.sell.val[e] : a.val[e];
            const int64_t b0 = bm.rp[brow], b1 = bm.rp[brow + 1];
            for (int64_t kk = b0 + lane; kk < b1; kk += 32) {
                if (*(volatile int *)&s_ovf[warp]) break;
                const int64_t k = bm.col[kk];
                const double p = __dmul_rn(av, bm.val[kk]);
                unsigned h = hash_slot(k, HC - 1);
                for (;;) {
                    const int64_t cur = *(volatile int64_t *)&keys[h];
                    if (cur == k) {
                        vals[h] = __dadd_rn(vals[h], p);
                        break;
                    }
                    if (cur == HASH_EMPTY) {
                        if (atomicAdd(&s_nclaim[warp], 0) >= LIMIT) {
                            atomicExch(&s_ovf[warp], 1);
                            break;
                        }
                        const unsigned long long old = atomicCAS(
                            (unsigned long long *)&keys[h], (unsigned long long)HASH_EMPTY, (unsigned long long)k);
                        if (old == (unsigned long long)HASH_EMPTY) {
                            vals[h] = __dadd_rn(0.0, p);
                            slots[atomicAdd(&s_nclaim[warp], 1)] = (int32_t)h;
                            break;
                        }
                        if ((int64_t)old == k) {
                            vals[h] = __dadd_rn(vals[h], p);
                            break;
                        }
                    }
                    h = (h + 1) & (HC - 1);
                }
            }
            __syncwarp();
            if (*(volatile int *)&s_ovf[warp]) break;
        }
        __syncwarp();
        const int nclaim = *(volatile int *)&s_nclaim[warp];
        const bool over = *(volatile int *)&s_ovf[warp] != 0;
        if (!over) {
            int kept = 0;
            for (int t = lane; t < nclaim; t += 32) kept += vals[slots[t]] != 0.0;
            for (int o = 16; o > 0; o >>= 1) kept += __shfl_xor_sync(0xffffffffu, kept, o);
            if (!rp) {
                if (lane == 0) cnt[p] = kept;
            } else {
                const int64_t o0 = rp[p];
                for (int t = lane; t < nclaim; t += 32) {
                    const int h = slots[t];
                    const double v = vals[h];
                    if (v == 0.0) continue;
                    const int64_t k = keys[h];
                    int rank = 0;
                    for (int u = 0; u < nclaim; u++) {
                        const int hu = slots[u];
                        rank += (keys[hu] < k) & (vals[hu] != 0.0);
                    }
                    ocol[o0 + rank] = k;
                    oval[o0 + rank] = v;
                }
            }
        } else if (lane == 0) {
            ovf[atomicAdd(novf, 1ull)] = p;
        }
        __syncwarp();
        for (int t = lane; t < nclaim; t += 32) keys[slots[t]] = HASH_EMPTY;
        __syncwarp();
        if (lane == 0) s_nclaim[warp] = s_ovf[warp] = 0;
        __syncwarp();
    }
}

// ---------------------------------------------------------------- symmetrise
// amg.py:234 (S + S^T) * 0.5 on the merged sorted rows of G and G^T:
// scipy binop res = a + b (missing side 0.0), zeros dropped, then * 0.5 and
// eliminate_zeros (CsrMatrix.from_scipy).
__global__ void k_ds_symmetrize(int64_t n, const int64_t *__restrict__ grp, const int64_t *__restrict__ gcol,
                                const double *__restrict__ gval, const int64_t *__restrict__ trp,
                                const int64_t *__restrict__ tcol, const double *__restrict__ tval,
                                const int64_t *__restrict__ rp, int64_t *__restrict__ cnt,
                                int64_t *__restrict__ ocol, double *__restrict__ oval) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    int64_t i = grp[r], ie = grp[r + 1], j = trp[r], je = trp[r + 1];
    int64_t k = rp ? rp[r] : 0, k0 = k;
    while (i < ie || j < je) {
        const int64_t ci = i < ie ? gcol[i] : INT64_MAX, cj = j < je ? tcol[j] : INT64_MAX;
        const int64_t c = ci < cj ? ci : cj;
        const double a = ci == c ? gval[i++] : 0.0;
        const double b = cj == c ? tval[j++] : 0.0;
        const double s = __dadd_rn(a, b);
        if (s == 0.0) continue;
        const double h = __dmul_rn(s, 0.5);
        if (h == 0.0) continue;
        if (rp) {
            ocol[k] = c;
            oval[k] = h;
        }
        k++;
    }
    if (!rp) cnt[r] = k - k0;
}

// ---------------------------------------------------------------- symmetrise without G^T
// One GPU, square G with sorted rows: for entry (J, K) of row J look J up in
// row K (binary search).  gt[e] = G[K, J] (0.0 when row K lacks J); a missing
// (K, J) makes (row K, column J, value G[J, K]) an "orphan" entry of G^T that
// row K's own entries do not cover (only exact-zero cancellations produce
// them).  Memory: one double per entry instead of a transposed copy.
__global__ void k_ds_sym_lookup(int64_t n, const int64_t *__restrict__ rp, const int64_t *__restrict__ col,
                                const double *__restrict__ val, double *__restrict__ gt,
                                int64_t *__restrict__ orow, int64_t *__restrict__ ocol, double *__restrict__ oval,
                                unsigned long long *__restrict__ norph, unsigned long long cap) {
    const int64_t J = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (J >= n) return;
    const int lane = threadIdx.x & 31;
    for (int64_t e = rp[J] + lane; e < rp[J + 1]; e += 32) {
        const int64_t K = col[e];
        int64_t lo = rp[K], hi = rp[K + 1];
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (col[mid] < J) lo = mid + 1;
            else hi = mid;
        }
        if (lo < rp[K + 1] && col[lo] == J) {
            gt[e] = val[lo];
        } else {
            gt[e] = 0.0;
            const unsigned long long o = atomicAdd(norph, 1ull);
            if (o < cap) {
                orow[o] = K;
                ocol[o] = J;
                oval[o] = val[e];
            }
        }
    }
}

// (G + G^T) * 0.5 from G's rows, the looked-up transpose values and the
// orphan rows (sorted CSR): scipy binop res = a + b (missing side 0.0),
// zeros dropped, then * 0.5 and eliminate_zeros.
__global__ void k_ds_symmetrize_lookup(int64_t n, const int64_t *__restrict__ grp, const int64_t *__restrict__ gcol,
                                       const double *__restrict__ gval, const double *__restrict__ gt,
                                       const int64_t *__restrict__ orp, const int64_t *__restrict__ ocol,
                                       const double *__restrict__ oval, const int64_t *__restrict__ rp,
                                       int64_t *__restrict__ cnt, int64_t *__restrict__ out_col,
                                       double *__restrict__ out_val) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    int64_t i = grp[r], ie = grp[r + 1], j = orp[r], je = orp[r + 1];
    int64_t k = rp ? rp[r] : 0, k0 = k;
    while (i < ie || j < je) {
        const int64_t ci = i < ie ? gcol[i] : INT64_MAX, cj = j < je ? ocol[j] : INT64_MAX;
        double a, b;
        int64_t c;
        if (ci < cj) {
            c = ci;
            a = gval[i];
            b = gt[i];
            i++;
        } else {
            c = cj;
            a = 0.0;
            b = oval[j];
            j++;
        }
        const double s = __dadd_rn(a, b);
        if (s == 0.0) continue;
        const double h = __dmul_rn(s, 0.5);
        if (h == 0.0) continue;
        if (rp) {
            out_col[k] = c;
            out_val[k] = h;
        }
        k++;
    }
    if (!rp) cnt[r] = k - k0;
}

// ---------------------------------------------------------------- device CSR -> SELL
__global__ void k_dcsr_width(int64_t n, const int64_t *__restrict__ rp, int32_t *__restrict__ w) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t ns = (n + 31) / 32;
    if ((i >> 5) >= ns) return;
    int len = i < n ? (int)(rp[i + 1] - rp[i]) : 0;
    for (int o = 16; o > 0; o >>= 1) len = max(len, __shfl_xor_sync(0xffffffffu, len, o));
    if ((i & 31) == 0) w[i >> 5] = len;
}

// SELL-C-sigma: one warp sorts one window of AMGP_SIGMA rows by descending
// length (stable: ties keep the row order) in shared memory, writes the
// window's positions -> rows into perm and the sorted slice widths.
__global__ void __launch_bounds__(128) k_sigma_sort(int64_t n, const int64_t *__restrict__ rp,
                                                     int32_t *__restrict__ perm, int32_t *__restrict__ wsorted) {
    const int64_t npos = (n + 31) / 32 * 32;  // positions of the SELL layout
    __shared__ unsigned long long key[4][AMGP_SIGMA];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t win = (int64_t)blockIdx.x * 4 + warp;
    const int64_t w0 = win * AMGP_SIGMA;
    if (w0 >= n) return;
    unsigned long long *k = key[warp];
    for (int t = lane; t < AMGP_SIGMA; t += 32) {
        const int64_t r = w0 + t;
        // (0x7fffffff - len) high, window offset low: ascending = longest first, stable
        const unsigned long long len = r < n ? (unsigned long long)(rp[r + 1] - rp[r]) : 0ull;
        k[t] = r < n ? ((0x7fffffffull - len) << 32) | (unsigned long long)t : ~0ull;
    }
    __syncwarp();
    for (int size = 2; size <= AMGP_SIGMA; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = lane; t < AMGP_SIGMA; t += 32) {
                const int o = t ^ stride;
                if (o > t) {
                    const bool up = (t & size) == 0;
                    const unsigned long long x = k[t], y = k[o];
                    if ((x > y) == up) {
                        k[t] = y;
                        k[o] = x;
                    }
                }
            }
            __syncwarp();
        }
    for (int t = lane; t < AMGP_SIGMA; t += 32) {
        const int64_t pos = w0 + t;
        if (pos >= npos) break;
        const bool real = k[t] != ~0ull;
        perm[pos] = real ? (int32_t)(w0 + (int64_t)(k[t] & 0xffffffffull)) : -1;
        if ((t & 31) == 0)  // slice width = its first (longest) row
            wsorted[pos >> 5] = real ? (int32_t)(0x7fffffffull - (k[t] >> 32)) : 0;
    }
}

__global__ void k_sigma_iperm(int64_t npos, const int32_t *__restrict__ perm, int32_t *__restrict__ iperm) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npos; p += (int64_t)gridDim.x * blockDim.x)
        if (perm[p] >= 0) iperm[perm[p]] = (int32_t)p;
}

// SELL slots of position i (row perm[i], or i itself without a permutation)
__global__ void k_dcsr_fill(int64_t n, int64_t ncols, const int64_t *__restrict__ rp,
                            const int64_t *__restrict__ col, const double *__restrict__ val,
                            const int32_t *__restrict__ perm, const int64_t *__restrict__ sp,
                            int32_t *__restrict__ scol, double *__restrict__ sval, int *bad) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t s = i >> 5;
    if (s >= (n + 31) / 32) return;
    const int lane = (int)(i & 31);
    const int w = (int)((sp[s + 1] - sp[s]) >> 5);
    const int64_t row = perm ? (int64_t)perm[i] : (i < n ? i : -1);
    const int64_t r0 = row >= 0 ? rp[row] : 0;
    const int len = row >= 0 ? (int)(rp[row + 1] - r0) : 0;
    for (int j = 0; j < w; j++) {
        const int64_t o = sp[s] + (int64_t)j * 32 + lane;
        if (j < len) {
            const int64_t c = col[r0 + j];
            if (c < 0 || c >= ncols || c > INT32_MAX) atomicExch(bad, 1);
            scol[o] = (int32_t)c;
            sval[o] = val[r0 + j];
        } else {
            scol[o] = -1;
            sval[o] = 0.0;
        }
    }
}

size_t spgemm_smem(int warps, int hc) { return (size_t)warps * hc * 20; }

int launch_grid(int64_t n, int block, int64_t cap = 148 * 64) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((n + block - 1) / block, cap));
}

}  // namespace

// ======================================================================== C ABI
extern "C" {

int amgp_ds_diag(amgp_mat *A, double *d) {
    if (!A || (!d && A->nrows)) return amgp_fail(AMGP_EINVAL, "amgp_ds_diag: bad argument");
    amgp_ctx *ctx = A->ctx;
    AMGP_CUDA(cudaSetDevice(ctx->device));
    if (A->nrows == 0) return AMGP_OK;
    k_ds_diag<<<grid_for(A->nrows, 256), 256, 0, cur_stream(ctx)>>>(view_of(A), d);
    AMGP_CHECK_LAUNCH(ctx);
    return AMGP_OK;
}

int amgp_ds_strength(amgp_mat *A, const double *d, double theta, int64_t nown, const int64_t *rows,
                     int64_t nlist, const int64_t *off, int64_t *cnt, int32_t *scol, double *sabs) {
    if (!A || !d || nlist < 0 || (!off && !cnt) || (off && !scol))
        return amgp_fail(AMGP_EINVAL, "amgp_ds_strength: bad argument");
    amgp_ctx *ctx = A->ctx;
    AMGP_CUDA(cudaSetDevice(ctx->device));
    if (nlist == 0) return AMGP_OK;
    k_ds_strength<<<grid_for(nlist, 256), 256, 0, cur_stream(ctx)>>>(view_of(A), d, theta, nown, rows, nlist, off,
                                                                 cnt, scol, sabs);
    AMGP_CHECK_LAUNCH(ctx);
    return AMGP_OK;
}

// Device OpenBLAS-order dots of one vector pair: out (device, 3 doubles) =
// (x.y, x.x, y.y) as numpy with `threads` OpenBLAS threads evaluates them.
static int blas_dot3_enqueue(amgp_ctx *ctx, int64_t n, const double *x, const double *y, int threads,
                             double *part, DotChunk *dchunks, double *out) {
    std::vector<DotChunk> ch;
    if (threads <= 1 || n <= 10000) {
        ch.push_back({0, n});
    } else {
        int64_t i = n, start = 0;
        for (int t = 0; i > 0; t++) {
            const int64_t left = threads - t;
            int64_t width = (i + left - 1) / left;
            i -= width;
            if (i < 0) width += i;
            ch.push_back({start, width});
            start += width;
        }
    }
    bool aligned = true;
    for (const auto &c : ch)
        aligned &= ((reinterpret_cast<uintptr_t>(x + c.start) | reinterpret_cast<uintptr_t>(y + c.start)) & 15) == 0;
    AMGP_CUDA(cudaMemcpyAsync(dchunks, ch.data(), ch.size() * sizeof(DotChunk), cudaMemcpyHostToDevice,
                              cur_stream(ctx)));
    const size_t smem = aligned ? (size_t)2 * DOT_STAGES * DOT_CH * sizeof(double) : 0;
    AMGP_CUDA(cudaFuncSetAttribute(k_blas_dot3, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   2 * DOT_STAGES * DOT_CH * (int)sizeof(double)));
    k_blas_dot3<<<(unsigned)ch.size(), 64, smem, cur_stream(ctx)>>>(x, y, dchunks, aligned ? 1 : 0, part);
    AMGP_CHECK_LAUNCH(ctx);
    k_blas_fold<<<1, 32, 0, cur_stream(ctx)>>>(part, (int)ch.size(), out);
    AMGP_CHECK_LAUNCH(ctx);
    return AMGP_OK;
}

int amgp_ds_blas_dot3(amgp_ctx *ctx, int64_t n, const double *x, const double *y, int threads,
                      double *out_host) {
    if (!ctx || n < 0 || !out_host) return amgp_fail(AMGP_EINVAL, "amgp_ds_blas_dot3: bad argument");
    AMGP_CUDA(cudaSetDevice(ctx->device));
    if (n == 0) {
        out_host[0] = out_host[1] = out_host[2] = 0.0;
        return AMGP_OK;
    }
    double *buf = nullptr;
    DotChunk *dch = nullptr;
    AMGP_CUDA(cudaMalloc(&buf, (3 * 64 + 3) * sizeof(double)));
    AMGP_CUDA(cudaMalloc(&dch, 64 * sizeof(DotChunk)));
    int st = blas_dot3_enqueue(ctx, n, x, y, std::min(threads, 64), buf, dch, buf + 3 * 64);
    if (st == AMGP_OK) {
        cudaError_t e = cudaMemcpyAsync(out_host, buf + 3 * 64, 3 * sizeof(double), cudaMemcpyDeviceToHost,
                                        cur_stream(ctx));
        if (e == cudaSuccess) e = cudaStreamSynchronize(cur_stream(ctx));
        if (e != cudaSuccess) st = amgp_cuda_fail(e, "blas_dot3", __FILE__, __LINE__);
    }
    cudaFree(buf);
    cudaFree(dch);
    return st;
}

// amg.py:194-216 estimate_lambda_max on the device: v (own rows, in/out)
// holds the start vector; A's halo exchange (if any) runs inside the SpMV;
// per-rank OpenBLAS-order dots are folded in rank order across GPUs when
// fold_ranks (row-distributed A; 0 for a level replicated on every rank).
int amgp_ds_lambda_max(amgp_ctx *ctx, amgp_mat *A, const double *d, double *v, int iters, int threads,
                       int fold_ranks, double *lam) {
    if (!ctx || !A || !d || !v || iters < 0 || !lam) return amgp_fail(AMGP_EINVAL, "amgp_ds_lambda_max: bad argument");
    AMGP_CUDA(cudaSetDevice(ctx->device));
    const int64_t n = A->nrows;
    double *buf = nullptr;
    DotChunk *dch = nullptr;
    const int64_t nb = std::max<int64_t>(n, 1);
    AMGP_CUDA(cudaMalloc(&buf, (4 * nb + 3 * 64 + 16) * sizeof(double)));
    AMGP_CUDA(cudaMalloc(&dch, 64 * sizeof(DotChunk)));
    double *ds = buf, *u = buf + nb, *y = buf + 2 * nb, *w = buf + 3 * nb;
    double *part = buf + 4 * nb, *sc = part + 3 * 64;  // sc: lam, nrm, stop, -, dots[3] at 4, folded at 8
    int st = AMGP_OK;
    auto run = [&]() -> int {
        AMGP_CUDA(cudaMemsetAsync(sc, 0, 16 * sizeof(double), cur_stream(ctx)));
        const int g = launch_grid(n, 256);
        if (n) {
            k_ds_sqrt<<<g, 256, 0, cur_stream(ctx)>>>(n, d, ds);
            AMGP_CHECK_LAUNCH(ctx);
        }
        for (int it = 0; it < iters; it++) {
            if (n) {
                k_ds_div<<<g, 256, 0, cur_stream(ctx)>>>(n, v, ds, u);
                AMGP_CHECK_LAUNCH(ctx);
            }
            AMGP_TRY(spmv_enqueue(ctx, A, u, y));
            if (n) {
                k_ds_div<<<g, 256, 0, cur_stream(ctx)>>>(n, y, ds, w);
                AMGP_CHECK_LAUNCH(ctx);
                AMGP_TRY(blas_dot3_enqueue(ctx, n, v, w, std::min(threads, 64), part, dch, sc + 4));
            } else {
                AMGP_CUDA(cudaMemsetAsync(sc + 4, 0, 3 * sizeof(double), cur_stream(ctx)));
            }
            const double *tot = sc + 4;
            if (fold_ranks && ctx->nranks > 1) {
                AMGP_TRY(allreduce_sum_ordered(ctx, sc + 4, 3, sc + 8));
                tot = sc + 8;
            }
            k_power_scalars<<<1, 32, 0, cur_stream(ctx)>>>(tot, sc);
            AMGP_CHECK_LAUNCH(ctx);
            if (n) {
                k_ds_scale<<<g, 256, 0, cur_stream(ctx)>>>(n, w, sc, v);
                AMGP_CHECK_LAUNCH(ctx);
            }
        }
        double h[3] = {1.0, 0.0, 0.0};
        AMGP_CUDA(cudaMemcpyAsync(h, sc, 3 * sizeof(double), cudaMemcpyDeviceToHost, cur_stream(ctx)));
        AMGP_CUDA(cudaStreamSynchronize(cur_stream(ctx)));
        *lam = iters == 0 ? 1.0 : (h[2] != 0.0 ? 0.0 : h[0]);
        return AMGP_OK;
    };
    st = run();
    cudaStreamSynchronize(cur_stream(ctx));
    cudaFree(buf);
    cudaFree(dch);
    return st;
}

// smoothed prolongator rows of the own rows of A (count / fill); agg_halo
// holds the coarse index of every halo column (global coarse numbering)
int amgp_ds_prolongator(amgp_mat *A, const double *d, const int64_t *agg_own, const int64_t *agg_halo,
                        double omega, int smooth, const int64_t *row_ptr, int64_t *row_cnt, int64_t *col,
                        double *val) {
    if (!A || !agg_own || (smooth && !d) || (!row_ptr && !row_cnt) || (row_ptr && (!col || !val)))
        return amgp_fail(AMGP_EINVAL, "amgp_ds_prolongator: bad argument");
    amgp_ctx *ctx = A->ctx;
    AMGP_CUDA(cudaSetDevice(ctx->device));
    const int64_t n = A->nrows;
    if (n == 0) return AMGP_OK;
    const int64_t nown = A->halo ? A->halo->nown : A->ncols;
    const int cap = A->max_width + 1;
    // bounded scratch: cap * nthreads entries of (key, value)
    int64_t nthr = std::min<int64_t>(n, (int64_t)148 * 2048);
    while (nthr > 32 * 1024 && (double)nthr * cap * 16 > 2e9) nthr /= 2;
    const int block = 256;
    const int grid = (int)((nthr + block - 1) / block);
    nthr = (int64_t)grid * block;
    int64_t *sk = nullptr;
    double *sv = nullptr;
    AMGP_CUDA(cudaMalloc(&sk, (size_t)nthr * cap * sizeof(int64_t)));
    AMGP_CUDA(cudaMalloc(&sv, (size_t)nthr * cap * sizeof(double)));
    k_ds_prolong<<<grid, block, 0, cur_stream(ctx)>>>(view_of(A), d, agg_own, agg_halo, nown, omega, smooth, row_ptr,
                                                  row_cnt, col, val, sk, sv, cap);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(cur_stream(ctx));
    cudaFree(sk);
    cudaFree(sv);
    if (e != cudaSuccess) return amgp_cuda_fail(e, "k_ds_prolong", __FILE__, __LINE__);
    ctx->launches.fetch_add(1);
    return AMGP_OK;
}

// C = A_side * B in scipy csr_matmat's per-entry order (count / fill).
// A-side: A_sell (SELL matrix whose local column c is B row c - b_off) or the
// CSR (a_rp, a_col, a_val).  Output row t is A-side row a_rows[t] (a_rows
// NULL: t itself); nout output rows.  B rows: b_rp / b_col (keys >= 0) / b_val.
int amgp_ds_spgemm(amgp_ctx *ctx, const amgp_mat *A_sell, const int64_t *a_rp, const int64_t *a_col,
                   const double *a_val, const int64_t *a_rows, int64_t nout, const int64_t *b_rp,
                   const int64_t *b_col, const double *b_val, int64_t b_off, const int64_t *row_ptr,
                   int64_t *row_cnt, int64_t *c_col, double *c_val) {
    if (!ctx || nout < 0 || (!A_sell && nout && !a_rp) || !b_rp || (!row_ptr && !row_cnt) ||
        (row_ptr && (!c_col || !c_val)))
        return amgp_fail(AMGP_EINVAL, "amgp_ds_spgemm: bad argument");
    AMGP_CUDA(cudaSetDevice(ctx->device));
    ASide a{};
    if (A_sell) {
        a.sell = view_of(A_sell);
        a.is_sell = 1;
    } else {
        a.rp = a_rp;
        a.col = a_col;
        a.val = a_val;
    }
    if (nout == 0) return AMGP_OK;
    const int64_t nrows = nout;
    BRows b{b_rp, b_col, b_val, b_off};
    // overflow lists (rows that did not fit the smaller tables)
    int64_t *ovf = nullptr;
    unsigned long long *novf = nullptr;
    AMGP_CUDA(cudaMalloc(&ovf, 2 * (size_t)nrows * sizeof(int64_t)));
    AMGP_CUDA(cudaMalloc(&novf, 2 * sizeof(unsigned long long)));
    int64_t *gk = nullptr;
    double *gv = nullptr;
    int32_t *gs = nullptr;
    int st = AMGP_OK;
    auto fail = [&](cudaError_t e, const char *what) {
        st = amgp_cuda_fail(e, what, __FILE__, __LINE__);
        return st;
    };
    do {
        cudaError_t e = cudaMemsetAsync(novf, 0, 2 * sizeof(unsigned long long), cur_stream(ctx));
        if (e != cudaSuccess) { fail(e, "memset"); break; }
        // stage 1: 128-slot shared tables, 8 warps per CTA
        k_ds_spgemm<8, 128, false><<<launch_grid(nrows, 8, 148 * 32), 256, spgemm_smem(8, 128), cur_stream(ctx)>>>(
            a, b, a_rows, nullptr, nrows, row_ptr, row_cnt, c_col, c_val, ovf, novf, nullptr, nullptr, nullptr);
        if ((e = cudaGetLastError()) != cudaSuccess) { fail(e, "k_ds_spgemm<128>"); break; }
        unsigned long long h[2] = {0, 0};
        e = cudaMemcpyAsync(h, novf, sizeof(h), cudaMemcpyDeviceToHost, cur_stream(ctx));
        if (e == cudaSuccess) e = cudaStreamSynchronize(cur_stream(ctx));
        if (e != cudaSuccess) { fail(e, "spgemm overflow count"); break; }
        if (h[0] == 0) break;
        // stage 2: 1024-slot shared tables (4 warps x 20 KB)
        e = cudaFuncSetAttribute(k_ds_spgemm<4, 1024, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)spgemm_smem(4, 1024));
        if (e != cudaSuccess) { fail(e, "spgemm smem attribute"); break; }
        k_ds_spgemm<4, 1024, false><<<launch_grid((int64_t)h[0], 4, 148 * 8), 128, spgemm_smem(4, 1024),
                                      cur_stream(ctx)>>>(a, b, a_rows, ovf, (int64_t)h[0], row_ptr, row_cnt, c_col,
                                                     c_val, ovf + nrows, novf + 1, nullptr, nullptr, nullptr);
        if ((e = cudaGetLastError()) != cudaSuccess) { fail(e, "k_ds_spgemm<1024>"); break; }
        e = cudaMemcpyAsync(h, novf, sizeof(h), cudaMemcpyDeviceToHost, cur_stream(ctx));
        if (e == cudaSuccess) e = cudaStreamSynchronize(cur_stream(ctx));
        if (e != cudaSuccess) { fail(e, "spgemm overflow count"); break; }
        if (h[1] == 0) break;
        // stage 3: 65536-slot per-warp tables in global memory
        constexpr int HG = 65536;
        const int nw = (int)std::min<unsigned long long>(h[1], 148 * 4);
        if ((e = cudaMalloc(&gk, (size_t)nw * HG * sizeof(int64_t))) != cudaSuccess) { fail(e, "alloc"); break; }
        if ((e = cudaMalloc(&gv, (size_t)nw * HG * sizeof(double))) != cudaSuccess) { fail(e, "alloc"); break; }
        if ((e = cudaMalloc(&gs, (size_t)nw * HG * sizeof(int32_t))) != cudaSuccess) { fail(e, "alloc"); break; }
        e = cudaMemsetAsync(novf, 0, sizeof(unsigned long long), cur_stream(ctx));
        k_ds_spgemm<1, HG, true><<<nw, 32, 0, cur_stream(ctx)>>>(a, b, a_rows, ovf + nrows, (int64_t)h[1], row_ptr,
                                                              row_cnt, c_col, c_val, ovf, novf, gk, gv, gs);
        if ((e = cudaGetLastError()) != cudaSuccess) { fail(e, "k_ds_spgemm<global>"); break; }
        e = cudaMemcpyAsync(h, novf, sizeof(unsigned long long), cudaMemcpyDeviceToHost, cur_stream(ctx));
        if (e == cudaSuccess) e = cudaStreamSynchronize(cur_stream(ctx));
        if (e != cudaSuccess) { fail(e, "spgemm overflow count"); break; }
        if (h[0] != 0) st = amgp_fail(AMGP_EINVAL, "spgemm: output row exceeds 65472 entries");
    } while (false);
    cudaStreamSynchronize(cur_stream(ctx));
    cudaFree(ovf);
    cudaFree(novf);
    cudaFree(gk);
    cudaFree(gv);
    cudaFree(gs);
    if (st == AMGP_OK) ctx->launches.fetch_add(1);
    return st;
}

int amgp_ds_symmetrize(amgp_ctx *ctx, int64_t n, const int64_t *g_rp, const int64_t *g_col, const double *g_val,
                       const int64_t *t_rp, const int64_t *t_col, const double *t_val, const int64_t *row_ptr,
                       int64_t *row_cnt, int64_t *col, double *val) {
    if (!ctx || n < 0 || (n && (!g_rp || !t_rp)) || (!row_ptr && !row_cnt) || (row_ptr && (!col || !val)))
        return amgp_fail(AMGP_EINVAL, "amgp_ds_symmetrize: bad argument");
    AMGP_CUDA(cudaSetDevice(ctx->device));
    if (n == 0) return AMGP_OK;
    k_ds_symmetrize<<<grid_for(n, 256), 256, 0, cur_stream(ctx)>>>(n, g_rp, g_col, g_val, t_rp, t_col, t_val, row_ptr,
                                                               row_cnt, col, val);
    AMGP_CHECK_LAUNCH(ctx);
    return AMGP_OK;
}

// One-GPU symmetrisation helpers (see k_ds_sym_lookup): gt[nnz] and up to
// cap orphan entries (orow, ocol, oval); *norph (host) = number of orphans
// (call again with a larger cap when it exceeds cap).
int amgp_ds_sym_lookup(amgp_ctx *ctx, int64_t n, const int64_t *rp, const int64_t *col, const double *val,
                       double *gt, int64_t *orow, int64_t *ocol, double *oval, int64_t cap, int64_t *norph) {
    if (!ctx || n < 0 || (n && (!rp || !gt)) || !norph || cap < 0)
        return amgp_fail(AMGP_EINVAL, "amgp_ds_sym_lookup: bad argument");
    AMGP_CUDA(cudaSetDevice(ctx->device));
    *norph = 0;
    if (n == 0) return AMGP_OK;
    unsigned long long *d = nullptr;
    AMGP_CUDA(cudaMalloc(&d, sizeof(unsigned long long)));
    cudaError_t e = cudaMemsetAsync(d, 0, sizeof(unsigned long long), cur_stream(ctx));
    if (e == cudaSuccess) {
        k_ds_sym_lookup<<<grid_for(n * 32, 256), 256, 0, cur_stream(ctx)>>>(n, rp, col, val, gt, orow, ocol, oval, d,
                                                                      (unsigned long long)cap);
        e = cudaGetLastError();
    }
    unsigned long long h = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, cur_stream(ctx));
    if (e == cudaSuccess) e = cudaStreamSynchronize(cur_stream(ctx));
    cudaFree(d);
    if (e != cudaSuccess) return amgp_cuda_fail(e, "k_ds_sym_lookup", __FILE__, __LINE__);
    ctx->launches.fetch_add(1);
    *norph = (int64_t)h;
    return AMGP_OK;
}

int amgp_ds_symmetrize_lookup(amgp_ctx *ctx, int64_t n, const int64_t *g_rp, const int64_t *g_col,
                              const double *g_val, const double *gt, const int64_t *o_rp, const int64_t *o_col,
                              const double *o_val, const int64_t *row_ptr, int64_t *row_cnt, int64_t *col,
                              double *val) {
    if (!ctx || n < 0 || (n && (!g_rp || !o_rp)) || (!row_ptr && !row_cnt) || (row_ptr && (!col || !val)))
        return amgp_fail(AMGP_EINVAL, "amgp_ds_symmetrize_lookup: bad argument");
    AMGP_CUDA(cudaSetDevice(ctx->device));
    if (n == 0) return AMGP_OK;
    k_ds_symmetrize_lookup<<<grid_for(n, 256), 256, 0, cur_stream(ctx)>>>(n, g_rp, g_col, g_val, gt, o_rp, o_col, o_val,
                                                                      row_ptr, row_cnt, col, val);
    AMGP_CHECK_LAUNCH(ctx);
    return AMGP_OK;
}

// SELL-32 matrix from a device CSR (columns already local, sorted per row as
// produced by the setup): per-slice widths on the device, slice offsets on
// the host, one fill launch.  sigma != 0: SELL-C-sigma -- rows sorted by
// length inside windows of AMGP_SIGMA rows when that stores >= 5 % fewer
// slots (coarse AMG levels, restriction operators); the row order inside
// each row is untouched, so every row sum keeps the reference's order.
// Matrices under AMGP_SIGMA_MIN_ROWS rows stay unsorted (coarsest levels:
// the single-CTA coarse solver addresses rows by position).
#ifndef AMGP_SIGMA_MIN_ROWS
#define AMGP_SIGMA_MIN_ROWS 4096
#endif
int amgp_mat_from_dcsr(amgp_ctx *ctx, int64_t nrows, int64_t ncols, const int64_t *rp, const int64_t *col,
                       const double *val, int sigma, amgp_mat **out) {
    if (!ctx || !out || nrows < 0 || ncols < 0 || (nrows && !rp))
        return amgp_fail(AMGP_EINVAL, "amgp_mat_from_dcsr: bad argument");
    if (ncols > (int64_t)INT32_MAX + 1) return amgp_fail(AMGP_EINVAL, "matrix too large for int32 column indices");
    if (nrows > INT32_MAX) return amgp_fail(AMGP_EINVAL, "too many rows for one device matrix");
    AMGP_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t st = cur_stream(ctx);
    const int64_t ns = (nrows + 31) / 32;
    int64_t nnz = 0;
    if (nrows) AMGP_CUDA(cudaMemcpyAsync(&nnz, rp + nrows, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    std::vector<int32_t> w(std::max<int64_t>(ns, 1)), ws(std::max<int64_t>(ns, 1));
    int32_t *dperm = nullptr, *dw = nullptr;
    const bool try_sigma = sigma && nrows >= AMGP_SIGMA_MIN_ROWS;
    if (ns) {
        AMGP_CUDA(cudaMalloc(&dw, 2 * ns * sizeof(int32_t)));
        k_dcsr_width<<<grid_for(ns * 32, 256), 256, 0, st>>>(nrows, rp, dw);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess && try_sigma) {
            e = cudaMalloc(&dperm, (size_t)ns * 32 * sizeof(int32_t));
            const int64_t nwin = (nrows + AMGP_SIGMA - 1) / AMGP_SIGMA;
            if (e == cudaSuccess) {
                k_sigma_sort<<<(unsigned)((nwin + 3) / 4), 128, 0, st>>>(nrows, rp, dperm, dw + ns);
                e = cudaGetLastError();
            }
        }
        if (e == cudaSuccess) e = cudaMemcpyAsync(w.data(), dw, ns * sizeof(int32_t), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess && try_sigma)
            e = cudaMemcpyAsync(ws.data(), dw + ns, ns * sizeof(int32_t), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        cudaFree(dw);
        if (e != cudaSuccess) {
            cudaFree(dperm);
            return amgp_cuda_fail(e, "SELL widths", __FILE__, __LINE__);
        }
    } else {
        AMGP_CUDA(cudaStreamSynchronize(st));
    }
    int64_t stored_u = 0, stored_s = 0;
    for (int64_t s = 0; s < ns; s++) {
        stored_u += (int64_t)w[s] * 32;
        stored_s += (int64_t)ws[s] * 32;
    }
    const bool use_sigma = try_sigma && stored_s * 100 <= stored_u * 95;
    if (!use_sigma) {
        cudaFree(dperm);
        dperm = nullptr;
    } else {
        w.swap(ws);
    }
    std::vector<int64_t> sp(ns + 1);
    int64_t stored = 0;
    int32_t wmax = 0;
    for (int64_t s = 0; s < ns; s++) {
        sp[s] = stored;
        stored += (int64_t)w[s] * 32;
        wmax = std::max(wmax, w[s]);
    }
    sp[ns] = stored;
    amgp_mat *A = nullptr;
    int st_alloc = mat_alloc(ctx, nrows, ncols, nnz, ns, stored, &A);
    if (st_alloc != AMGP_OK) {
        cudaFree(dperm);
        return st_alloc;
    }
    A->max_width = wmax;
    A->perm = dperm;
    int *bad = nullptr;
    cudaError_t e = cudaMemcpyAsync(A->slice_ptr, sp.data(), (ns + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess && dperm) e = cudaMalloc(&A->iperm, std::max<int64_t>(nrows, 1) * sizeof(int32_t));
    if (e == cudaSuccess && dperm) {
        k_sigma_iperm<<<grid_for(ns * 32, 256), 256, 0, st>>>(ns * 32, dperm, A->iperm);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMalloc(&bad, sizeof(int));
    if (e == cudaSuccess) e = cudaMemsetAsync(bad, 0, sizeof(int), st);
    if (e == cudaSuccess && ns) {
        k_dcsr_fill<<<grid_for(ns * 32, 256), 256, 0, st>>>(nrows, ncols, rp, col, val, dperm, A->slice_ptr, A->col,
                                                            A->val, bad);
        e = cudaGetLastError();
    }
    int hbad = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(bad);
    if (e != cudaSuccess) {
        amgp_mat_destroy(A);
        return amgp_cuda_fail(e, "k_dcsr_fill", __FILE__, __LINE__);
    }
    if (hbad) {
        amgp_mat_destroy(A);
        return amgp_fail(AMGP_EINVAL, "column index out of range");
    }
    ctx->launches.fetch_add(ns ? (dperm ? 4 : 2) : 0);
    int rs = refresh_slice_maxcol(A);
    if (rs != AMGP_OK) {
        amgp_mat_destroy(A);
        return rs;
    }
    *out = A;
    return AMGP_OK;
}

// Own columns of a matrix: nown of a distributed matrix (its halo plan), else ncols.
int amgp_mat_nown(const amgp_mat *A, int64_t *nown) {
    if (!A || !nown) return amgp_fail(AMGP_EINVAL, "amgp_mat_nown: bad argument");
    *nown = A->halo ? A->halo->nown : A->ncols;
    return AMGP_OK;
}

}  // extern "C"
