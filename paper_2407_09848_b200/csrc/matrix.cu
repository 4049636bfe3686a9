// Device matrices in SELL-32 layout, the direct Poisson generators, the
// l1-Jacobi diagonal, and the plain SpMV-family kernels (K3/K4/K5).
//
// Layout: rows are grouped in slices of 32
// consecutive rows; slice s stores w_s = max row length of its rows slots,
// slot j of row (32 s + t) at element slice_ptr[s] + 32 j + t.  One warp reads
// one slot of its 32 rows with one coalesced 256 B (values) + 128 B (columns)
// transaction.  Row entries keep the CSR stored order (sorted columns,
// reference sparse.py:43-75), so the in-order row sum is the reference's.
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "epilogues.cuh"

// ---------------------------------------------------------------- host packing
extern "C" int amgp_sell_pack_host(int64_t nrows, const int64_t *row_ptr,
                                   const int64_t *col_idx, const double *values,
                                   int64_t *nslices_out, int64_t *stored_out,
                                   int64_t *slice_ptr, int32_t *col, double *val) {
    if (nrows < 0 || !row_ptr || !nslices_out || !stored_out)
        return amgp_fail(AMGP_EINVAL, "amgp_sell_pack_host: bad argument");
    const int64_t ns = (nrows + AMGP_SLICE - 1) / AMGP_SLICE;
    int64_t stored = 0;
    for (int64_t s = 0; s < ns; s++) {
        int64_t w = 0;
        for (int64_t i = s * AMGP_SLICE; i < std::min(nrows, (s + 1) * AMGP_SLICE); i++) {
            int64_t len = row_ptr[i + 1] - row_ptr[i];
            if (len < 0) return amgp_fail(AMGP_EINVAL, "row_ptr must be nondecreasing");
            w = std::max(w, len);
        }
        if (slice_ptr) slice_ptr[s] = stored;
        if (col && val) {
            for (int64_t j = 0; j < w; j++)
                for (int t = 0; t < AMGP_SLICE; t++) {
                    int64_t i = s * AMGP_SLICE + t;
                    int64_t o = stored + j * AMGP_SLICE + t;
                    if (i < nrows && j < row_ptr[i + 1] - row_ptr[i]) {
                        int64_t c = col_idx[row_ptr[i] + j];
                        if (c < 0 || c > INT32_MAX)
                            return amgp_fail(AMGP_EINVAL, "column index out of int32 range");
                        col[o] = (int32_t)c;
                        val[o] = values[row_ptr[i] + j];
                    } else {
                        col[o] = -1;
                        val[o] = 0.0;
                    }
                }
        }
        stored += w * AMGP_SLICE;
    }
    if (slice_ptr) slice_ptr[ns] = stored;
    *nslices_out = ns;
    *stored_out = stored;
    return AMGP_OK;
}

int mat_alloc(amgp_ctx *ctx, int64_t nrows, int64_t ncols, int64_t nnz, int64_t ns,
                     int64_t stored, amgp_mat **out) {
    amgp_mat *A = new amgp_mat();
    A->ctx = ctx;
    A->nrows = nrows;
    A->ncols = ncols;
    A->nnz = nnz;
    A->nslices = ns;
    A->stored = stored;
    cudaError_t e = cudaMalloc(&A->slice_ptr, (size_t)(ns + 1) * sizeof(int64_t));
    if (e == cudaSuccess) e = cudaMalloc(&A->col, (size_t)std::max<int64_t>(stored, 1) * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMalloc(&A->val, (size_t)std::max<int64_t>(stored, 1) * sizeof(double));
    if (e != cudaSuccess) {
        cudaFree(A->slice_ptr);
        cudaFree(A->col);
        cudaFree(A->val);
        delete A;
        return amgp_cuda_fail(e, "matrix allocation", __FILE__, __LINE__);
    }
    *out = A;
    return AMGP_OK;
}

int amgp_mat_from_dcsr(amgp_ctx *ctx, int64_t nrows, int64_t ncols, const int64_t *rp, const int64_t *col,
                       const double *val, int sigma, amgp_mat **out);

// Host CSR -> device: validated here, uploaded, and packed on the device
// (amgp_mat_from_dcsr, SELL-C-sigma where it saves slots).
extern "C" int amgp_mat_from_csr(amgp_ctx *ctx, int64_t nrows, int64_t ncols,
                                 const int64_t *row_ptr, const int64_t *col_idx,
                                 const double *values, amgp_mat **out) {
    if (!ctx || !out || nrows < 0 || ncols < 0 || !row_ptr)
        return amgp_fail(AMGP_EINVAL, "amgp_mat_from_csr: bad argument");
    if (row_ptr[0] != 0) return amgp_fail(AMGP_EINVAL, "row_ptr endpoints inconsistent with values");
    if (ncols > INT32_MAX || nrows > INT32_MAX)
        return amgp_fail(AMGP_EINVAL, "matrix too large for int32 column indices");
    for (int64_t i = 0; i < nrows; i++)
        if (row_ptr[i + 1] < row_ptr[i]) return amgp_fail(AMGP_EINVAL, "row_ptr must be nondecreasing");
    const int64_t nnz = row_ptr[nrows];
    for (int64_t k = 0; k < nnz; k++) {
        if (col_idx[k] < 0 || col_idx[k] > INT32_MAX) return amgp_fail(AMGP_EINVAL, "column index out of int32 range");
        if (col_idx[k] >= ncols) return amgp_fail(AMGP_EINVAL, "column index >= ncols");
    }
    AMGP_CUDA(cudaSetDevice(ctx->device));
    int64_t *drp = nullptr, *dcol = nullptr;
    double *dval = nullptr;
    cudaError_t e = cudaMalloc(&drp, (nrows + 1) * sizeof(int64_t));
    if (e == cudaSuccess) e = cudaMalloc(&dcol, std::max<int64_t>(nnz, 1) * sizeof(int64_t));
    if (e == cudaSuccess) e = cudaMalloc(&dval, std::max<int64_t>(nnz, 1) * sizeof(double));
    if (e == cudaSuccess) e = cudaMemcpy(drp, row_ptr, (nrows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && nnz) e = cudaMemcpy(dcol, col_idx, nnz * sizeof(int64_t), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && nnz) e = cudaMemcpy(dval, values, nnz * sizeof(double), cudaMemcpyHostToDevice);
    int st = e == cudaSuccess ? amgp_mat_from_dcsr(ctx, nrows, ncols, drp, dcol, dval, 1, out)
                              : amgp_cuda_fail(e, "matrix upload", __FILE__, __LINE__);
    cudaStreamSynchronize(cur_stream(ctx));
    cudaFree(drp);
    cudaFree(dcol);
    cudaFree(dval);
    return st;
}

extern "C" int amgp_mat_destroy(amgp_mat *A) {
    if (!A) return AMGP_OK;
    if (A->ctx) {
        cudaSetDevice(A->ctx->device);
        cudaStreamSynchronize(cur_stream(A->ctx));
        if (A->ctx->comm_stream) cudaStreamSynchronize(A->ctx->comm_stream);  // halo pack kernels
    }
    mat_free_halo(A);
    cudaFree(A->slice_ptr);
    cudaFree(A->col);
    cudaFree(A->val);
    cudaFree(A->work);
    cudaFree(A->io);
    cudaFree(A->perm);
    cudaFree(A->iperm);
    delete A;
    return AMGP_OK;
}

extern "C" int amgp_mat_info(const amgp_mat *A, int64_t *nrows, int64_t *ncols, int64_t *nnz,
                             int64_t *stored, int64_t *bytes) {
    if (!A) return amgp_fail(AMGP_EINVAL, "null matrix");
    if (nrows) *nrows = A->nrows;
    if (ncols) *ncols = A->ncols;
    if (nnz) *nnz = A->nnz;
    if (stored) *stored = A->stored;
    if (bytes) *bytes = A->stored * 12 + (A->nslices + 1) * 8;
    return AMGP_OK;
}

extern "C" int amgp_mat_to_csr(amgp_mat *A, int64_t *row_ptr, int64_t *col_idx, double *values) {
    if (!A || !row_ptr) return amgp_fail(AMGP_EINVAL, "amgp_mat_to_csr: bad argument");
    std::vector<int64_t> sp(A->nslices + 1);
    std::vector<int32_t> col(std::max<int64_t>(A->stored, 1));
    std::vector<double> val(std::max<int64_t>(A->stored, 1));
    std::vector<int32_t> iperm;
    AMGP_CUDA(cudaStreamSynchronize(cur_stream(A->ctx)));
    AMGP_CUDA(cudaMemcpy(sp.data(), A->slice_ptr, sp.size() * sizeof(int64_t), cudaMemcpyDeviceToHost));
    if (A->stored > 0) {
        AMGP_CUDA(cudaMemcpy(col.data(), A->col, A->stored * sizeof(int32_t), cudaMemcpyDeviceToHost));
        AMGP_CUDA(cudaMemcpy(val.data(), A->val, A->stored * sizeof(double), cudaMemcpyDeviceToHost));
    }
    if (A->iperm) {
        iperm.resize(A->nrows);
        AMGP_CUDA(cudaMemcpy(iperm.data(), A->iperm, A->nrows * sizeof(int32_t), cudaMemcpyDeviceToHost));
    }
    int64_t k = 0;
    row_ptr[0] = 0;
    for (int64_t i = 0; i < A->nrows; i++) {
        const int64_t pos = A->iperm ? iperm[i] : i;  // SELL position of row i
        int64_t s = pos / AMGP_SLICE, t = pos % AMGP_SLICE;
        int64_t w = (sp[s + 1] - sp[s]) / AMGP_SLICE;
        for (int64_t j = 0; j < w; j++) {
            int64_t o = sp[s] + j * AMGP_SLICE + t;
            if (col[o] < 0) continue;
            if (k >= A->nnz) return amgp_fail(AMGP_EINVAL, "stored entries exceed nnz");
            if (col_idx) col_idx[k] = col[o];
            if (values) values[k] = val[o];
            k++;
        }
        row_ptr[i + 1] = k;
    }
    return AMGP_OK;
}

// ---------------------------------------------------------------- Poisson generators
// problems.py:32-60: index i = ix + m iy + m^2 iz (x fastest), Dirichlet
// neighbours eliminated; columns emitted in ascending order.
__device__ __forceinline__ int poisson_row(int64_t m, int stencil, int64_t i, int64_t *cols,
                                           double *vals) {
    const int64_t m2 = m * m;
    const int64_t iz = i / m2, iy = (i / m) % m, ix = i % m;
    int len = 0;
    if (stencil == 7) {
        if (iz > 0) { cols[len] = i - m2; vals[len++] = -1.0; }
        if (iy > 0) { cols[len] = i - m; vals[len++] = -1.0; }
        if (ix > 0) { cols[len] = i - 1; vals[len++] = -1.0; }
        cols[len] = i; vals[len++] = 6.0;
        if (ix < m - 1) { cols[len] = i + 1; vals[len++] = -1.0; }
        if (iy < m - 1) { cols[len] = i + m; vals[len++] = -1.0; }
        if (iz < m - 1) { cols[len] = i + m2; vals[len++] = -1.0; }
    } else {
        for (int dz = -1; dz <= 1; dz++) {
            if (iz + dz < 0 || iz + dz >= m) continue;
            for (int dy = -1; dy <= 1; dy++) {
                if (iy + dy < 0 || iy + dy >= m) continue;
                for (int dx = -1; dx <= 1; dx++) {
                    if (ix + dx < 0 || ix + dx >= m) continue;
                    cols[len] = i + dx + dy * m + dz * m2;
                    vals[len++] = (dx == 0 && dy == 0 && dz == 0) ? 26.0 : -1.0;
                }
            }
        }
    }
    return len;
}

__global__ void k_poisson_widths(int64_t m, int stencil, int64_t r0, int64_t nrows,
                                 int32_t *widths) {
    int64_t s = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    int lane = threadIdx.x & 31;
    int64_t nslices = (nrows + 31) / 32;
    if (s >= nslices) return;
    int64_t li = s * 32 + lane;
    int len = 0;
    if (li < nrows) {
        int64_t cols[27];
        double vals[27];
        len = poisson_row(m, stencil, r0 + li, cols, vals);
    }
    for (int o = 16; o > 0; o >>= 1) len = max(len, __shfl_xor_sync(0xffffffffu, len, o));
    if (lane == 0) widths[s] = len;
}

__global__ void k_poisson_fill(int64_t m, int stencil, int64_t r0, int64_t nrows,
                               const int64_t *__restrict__ sp, int32_t *__restrict__ col,
                               double *__restrict__ val) {
    int64_t s = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    int lane = threadIdx.x & 31;
    int64_t nslices = (nrows + 31) / 32;
    if (s >= nslices) return;
    int64_t li = s * 32 + lane;
    int64_t cols[27];
    double vals[27];
    int len = li < nrows ? poisson_row(m, stencil, r0 + li, cols, vals) : 0;
    int w = (int)((sp[s + 1] - sp[s]) / 32);
    for (int j = 0; j < w; j++) {
        int64_t o = sp[s] + (int64_t)j * 32 + lane;
        col[o] = j < len ? (int32_t)cols[j] : -1;
        val[o] = j < len ? vals[j] : 0.0;
    }
}

extern "C" int amgp_mat_poisson3d(amgp_ctx *ctx, int64_t m, int stencil, int64_t row_begin,
                                  int64_t row_end, amgp_mat **out) {
    if (!ctx || !out) return amgp_fail(AMGP_EINVAL, "amgp_mat_poisson3d: bad argument");
    if (m < 2) return amgp_fail(AMGP_EINVAL, "m must be >= 2");
    if (stencil != 7 && stencil != 27) return amgp_fail(AMGP_EINVAL, "stencil must be 7 or 27");
    const int64_t n = m * m * m;
    if (n > INT32_MAX) return amgp_fail(AMGP_EINVAL, "m^3 exceeds int32 column range");
    if (row_begin < 0 || row_end > n || row_begin > row_end)
        return amgp_fail(AMGP_EINVAL, "bad row range");
    AMGP_CUDA(cudaSetDevice(ctx->device));
    const int64_t nrows = row_end - row_begin;
    const int64_t ns = (nrows + 31) / 32;
    int32_t *dw = nullptr;
    AMGP_CUDA(cudaMalloc(&dw, std::max<int64_t>(ns, 1) * sizeof(int32_t)));
    const int blk = 256;
    if (ns > 0) {
        k_poisson_widths<<<grid_for(ns * 32, blk), blk, 0, cur_stream(ctx)>>>(m, stencil, row_begin, nrows, dw);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) { cudaFree(dw); return amgp_cuda_fail(e, "k_poisson_widths", __FILE__, __LINE__); }
    }
    std::vector<int32_t> w(std::max<int64_t>(ns, 1));
    std::vector<int64_t> sp(ns + 1);
    cudaError_t e = cudaMemcpyAsync(w.data(), dw, ns * sizeof(int32_t), cudaMemcpyDeviceToHost, cur_stream(ctx));
    if (e == cudaSuccess) e = cudaStreamSynchronize(cur_stream(ctx));
    cudaFree(dw);
    if (e != cudaSuccess) return amgp_cuda_fail(e, "poisson widths", __FILE__, __LINE__);
    int64_t stored = 0;
    int32_t wmax = 0;
    for (int64_t s = 0; s < ns; s++) {
        sp[s] = stored;
        stored += (int64_t)w[s] * 32;
        wmax = std::max(wmax, w[s]);
    }
    sp[ns] = stored;
    amgp_mat *A = nullptr;
    AMGP_TRY(mat_alloc(ctx, nrows, n, 0, ns, stored, &A));
    A->max_width = wmax;
    A->row_offset = row_begin;
    e = cudaMemcpyAsync(A->slice_ptr, sp.data(), (ns + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, cur_stream(ctx));
    if (e != cudaSuccess) { amgp_mat_destroy(A); return amgp_cuda_fail(e, "slice_ptr upload", __FILE__, __LINE__); }
    if (ns > 0) {
        k_poisson_fill<<<grid_for(ns * 32, blk), blk, 0, cur_stream(ctx)>>>(m, stencil, row_begin, nrows,
                                                                       A->slice_ptr, A->col, A->val);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaStreamSynchronize(cur_stream(ctx));
        if (e != cudaSuccess) { amgp_mat_destroy(A); return amgp_cuda_fail(e, "k_poisson_fill", __FILE__, __LINE__); }
        ctx->launches.fetch_add(2);
    }
    // exact nnz: count per plane analytically (each row's length is the
    // product of its per-axis neighbour counts for 27-point, 1 + #axis
    // neighbours for 7-point)
    int64_t nnz = 0;
    const int64_t m2 = m * m;
    for (int64_t i = row_begin; i < row_end;) {
        // process a run of rows with fixed (iy, iz): ix from i%m to m-1
        int64_t iz = i / m2, iy = (i / m) % m, ix = i % m;
        int64_t run = std::min<int64_t>(m - ix, row_end - i);
        int ny = 1 + (iy > 0) + (iy < m - 1), nz = 1 + (iz > 0) + (iz < m - 1);
        for (int64_t x = ix; x < ix + run; x++) {
            int nx = 1 + (x > 0) + (x < m - 1);
            nnz += stencil == 7 ? (nx + ny + nz - 2) : (int64_t)nx * ny * nz;
        }
        i += run;
    }
    A->nnz = nnz;
    int st = refresh_slice_maxcol(A);
    if (st != AMGP_OK) {
        amgp_mat_destroy(A);
        return st;
    }
    *out = A;
    return AMGP_OK;
}

// ---------------------------------------------------------------- l1 diagonal
// smoothers.py:42-49: m = abs_row - |a_ii| + a_ii with
// abs_row = scipy sum(axis=1) of |A| = numpy add.reduceat over the row:
// a_0 + pairwise_sum(a_1..a_{L-1}) (numpy's pairwise summation: <8 terms
// sequential from 0.0, <=128 terms eight interleaved partials, else split).
__device__ double pw_sum(const double *__restrict__ v, const int32_t *__restrict__ c, int64_t lo,
                         int64_t n) {
    // element k of the row lives at v[(lo + k) * 32]
    if (n < 8) {
        double res = 0.0;
        for (int64_t k = 0; k < n; k++) res = __dadd_rn(res, fabs(v[(lo + k) * 32]));
        return res;
    } else if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = fabs(v[(lo + j) * 32]);
        int64_t k = 8;
        for (; k < n - (n % 8); k += 8)
            for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], fabs(v[(lo + k + j) * 32]));
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; k < n; k++) res = __dadd_rn(res, fabs(v[(lo + k) * 32]));
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(pw_sum(v, c, lo, n2), pw_sum(v, c, lo + n2, n - n2));
}

__global__ void k_l1_diag(SellView A, int64_t row_offset, double *__restrict__ m, int *bad) {
    int64_t s = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    int lane = threadIdx.x & 31;
    if (s >= A.nslices) return;
    const int64_t row = sell_row(A, s * 32 + lane);
    if (row < 0) return;
    const int64_t base = A.slice_ptr[s];
    const int w = (int)((A.slice_ptr[s + 1] - base) >> 5);
    const double *v = A.val + base + lane;
    const int32_t *c = A.col + base + lane;
    int len = 0;
    while (len < w && c[(int64_t)len * 32] >= 0) len++;
    double d = 0.0;
    for (int j = 0; j < len; j++)
        if (c[(int64_t)j * 32] == row + row_offset) d = v[(int64_t)j * 32];
    double absrow = 0.0;
    if (len > 0) absrow = __dadd_rn(fabs(v[0]), pw_sum(v, c, 1, len - 1));
    if (!(d > 0.0)) atomicExch(bad, 1);
    m[row] = __dadd_rn(__dsub_rn(absrow, fabs(d)), d);
}

extern "C" int amgp_mat_l1_diag(amgp_mat *A, double *m_dev) {
    if (!A || !m_dev) return amgp_fail(AMGP_EINVAL, "amgp_mat_l1_diag: bad argument");
    amgp_ctx *ctx = A->ctx;
    // square matrix, or a row block (generated: global columns from
    // row_offset; localized: own columns first, halo after)
    if (A->row_offset + A->nrows > A->ncols) return amgp_fail(AMGP_EINVAL, "matrix must be square");
    int *bad = nullptr;
    AMGP_CUDA(cudaMalloc(&bad, sizeof(int)));
    AMGP_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), cur_stream(ctx)));
    // Generated row blocks store global columns: local row i is global row
    // row_offset + i.
    const int64_t off = A->row_offset;
    if (A->nslices > 0) {
        k_l1_diag<<<grid_for(A->nslices * 32, 256), 256, 0, cur_stream(ctx)>>>(view_of(A), off, m_dev, bad);
        AMGP_CHECK_LAUNCH(ctx);
    }
    int hbad = 0;
    AMGP_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, cur_stream(ctx)));
    AMGP_CUDA(cudaStreamSynchronize(cur_stream(ctx)));
    cudaFree(bad);
    if (hbad) return amgp_fail(AMGP_EINVAL, "non-positive diagonal entry");
    return AMGP_OK;
}

// ---------------------------------------------------------------- SpMV kernels
int spmv_enqueue(amgp_ctx *ctx, const amgp_mat *A, const double *x, double *y) {
    return launch_rows(ctx, A, x, SpmvEpi<0>{nullptr, y});
}
int residual_enqueue(amgp_ctx *ctx, const amgp_mat *A, const double *r, const double *x,
                     double *res) {
    return launch_rows(ctx, A, x, SpmvEpi<1>{r, res});
}
int prolong_add_enqueue(amgp_ctx *ctx, const amgp_mat *P, const double *xc, double *x) {
    return launch_rows(ctx, P, xc, SpmvEpi<2>{nullptr, x});
}

extern "C" int amgp_spmv(amgp_ctx *ctx, const amgp_mat *A, const double *x, double *y) {
    if (!ctx || !A || (!x && A->ncols) || (!y && A->nrows))
        return amgp_fail(AMGP_EINVAL, "amgp_spmv: bad argument");
    AMGP_CUDA(cudaSetDevice(ctx->device));
    std::lock_guard<std::mutex> cg(ctx->mu);
    return spmv_enqueue(ctx, A, x, y);
}
