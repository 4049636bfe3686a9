// Native host-side AMG setup, bit-exact with the reference (amg.py:97-287).
//
// The reference builds its hierarchy with Python greedy loops plus scipy's
// C++ sparse kernels; the values of the coarse operators depend on the exact
// summation order of those kernels.  This file restates, operation for
// operation, what the reference's expressions execute:
//
//   matmat()       scipy sparsetools csr_matmat: per output row, a linked
//                  list of touched columns (head insertion -> output in reverse
//                  first-touch order), sums from 0.0 in operand order, exact
//                  zeros dropped.  csc @ X is csr_matmat on swapped operands.
//   compress_t()   scipy csr_tocsc (transpose of compressed arrays; minor
//                  indices come out ascending).
//   binop()        scipy csr_binop_csr (general path: linked list, op(a, b),
//                  zero results dropped).
//
//   sa_aggregate          amg.py:102-149
//   matching_aggregate    amg.py:152-191 (P_c^T cur P_c with scipy's orders)
//   smooth_prolongator    amg.py:219-226 (diags(w/d) @ A, @ P_hat, P_hat - .)
//   galerkin_rap          amg.py:229-235 ((P^T A) P, (S + S^T) * 0.5)
//
// Rows of a product are independent, so matmat runs row blocks on threads
// without changing a single bit.  All arithmetic is binary64 with separate
// multiply and add (built with -ffp-contract=off).
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <chrono>
#include <functional>
#include <memory>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/amgp.h"

void amgp_set_error(const std::string &msg);
int amgp_fail(int code, const std::string &msg);

namespace {

struct Cmp {  // compressed sparse arrays: major index m -> [p[m], p[m+1])
    int64_t nmajor = 0, nminor = 0;
    std::vector<int64_t> p, i;
    std::vector<double> x;
    int64_t nnz() const { return p.empty() ? 0 : p.back(); }
};

int g_threads = 1;

// AMGP_SETUP_TRACE=1 prints per-phase wall times to stderr.
struct Trace {
    const char *name;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    explicit Trace(const char *n) : name(n) {}
    ~Trace() {
        static const bool on = getenv("AMGP_SETUP_TRACE") != nullptr;
        if (on)
            fprintf(stderr, "[amgp setup] %-28s %8.3f s\n", name,
                    std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
};

void parallel_rows(int64_t n, const std::function<void(int64_t, int64_t, int)> &fn) {
    int t = (int)std::max<int64_t>(1, std::min<int64_t>(g_threads, n / 4096));
    if (t <= 1) {
        fn(0, n, 0);
        return;
    }
    std::vector<std::thread> th;
    for (int w = 0; w < t; w++) th.emplace_back(fn, n * w / t, n * (w + 1) / t, w);
    for (auto &x : th) x.join();
}

int nthreads_for(int64_t work_rows) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(g_threads, work_rows / 4096));
}

// Row-parallel assembly of a compressed matrix.  row_fn(r, scratch, oi, ox)
// appends row r's entries (in their final order) and returns their count;
// every row is produced by exactly the sequential algorithm, so the result
// does not depend on the thread count.
template <class Scratch, class MakeScratch, class RowFn>
Cmp build_rows(int64_t n_row, int64_t n_col, MakeScratch make, RowFn row_fn) {
    const int nt = nthreads_for(n_row);
    std::vector<std::vector<int64_t>> ti(nt);
    std::vector<std::vector<double>> tx(nt);
    std::vector<int64_t> cnt(n_row + 1, 0);
    auto work = [&](int64_t r0, int64_t r1, int w) {
        Scratch sc = make();
        for (int64_t r = r0; r < r1; r++) cnt[r + 1] = row_fn(r, sc, ti[w], tx[w]);
    };
    if (nt <= 1) {
        work(0, n_row, 0);
    } else {
        std::vector<std::thread> th;
        for (int w = 0; w < nt; w++) th.emplace_back(work, n_row * w / nt, n_row * (w + 1) / nt, w);
        for (auto &x : th) x.join();
    }
    Cmp C;
    C.nmajor = n_row;
    C.nminor = n_col;
    C.p.resize(n_row + 1);
    C.p[0] = 0;
    for (int64_t r = 0; r < n_row; r++) C.p[r + 1] = C.p[r] + cnt[r + 1];
    C.i.resize(C.p[n_row]);
    C.x.resize(C.p[n_row]);
    std::vector<int64_t> off(nt + 1, 0);
    for (int w = 0; w < nt; w++) off[w + 1] = off[w] + (int64_t)ti[w].size();
    auto copy = [&](int64_t, int64_t, int w) {
        std::copy(ti[w].begin(), ti[w].end(), C.i.begin() + off[w]);
        std::copy(tx[w].begin(), tx[w].end(), C.x.begin() + off[w]);
        std::vector<int64_t>().swap(ti[w]);
        std::vector<double>().swap(tx[w]);
    };
    if (nt <= 1) {
        copy(0, 0, 0);
    } else {
        std::vector<std::thread> th;
        for (int w = 0; w < nt; w++) th.emplace_back(copy, 0, 0, w);
        for (auto &x : th) x.join();
    }
    return C;
}

struct LinkedRow {  // scipy's per-row accumulator: next list + dense sums
    std::vector<int64_t> next;
    std::vector<double> a, b;
};

// scipy csr_matmat: C = A * B (A: nmajor x K, B: K x nminor)
Cmp matmat(const Cmp &A, const Cmp &B) {
    Trace tr("matmat");
    const int64_t n_col = B.nminor;
    return build_rows<LinkedRow>(
        A.nmajor, n_col, [&] { return LinkedRow{std::vector<int64_t>(n_col, -1), std::vector<double>(n_col, 0.0), {}}; },
        [&](int64_t r, LinkedRow &s, std::vector<int64_t> &oi, std::vector<double> &ox) {
            int64_t head = -2, length = 0;
            for (int64_t jj = A.p[r]; jj < A.p[r + 1]; jj++) {
                const int64_t j = A.i[jj];
                const double v = A.x[jj];
                for (int64_t kk = B.p[j]; kk < B.p[j + 1]; kk++) {
                    const int64_t k = B.i[kk];
                    const double prod = v * B.x[kk];
                    s.a[k] = s.a[k] + prod;
                    if (s.next[k] == -1) {
                        s.next[k] = head;
                        head = k;
                        length++;
                    }
                }
            }
            int64_t c = 0;
            for (int64_t jj = 0; jj < length; jj++) {
                if (s.a[head] != 0) {
                    oi.push_back(head);
                    ox.push_back(s.a[head]);
                    c++;
                }
                const int64_t temp = head;
                head = s.next[head];
                s.next[temp] = -1;
                s.a[temp] = 0;
            }
            return c;
        });
}

// scipy csr_tocsc: compressed-transpose (minor indices ascending in output).
// Threads take contiguous source-row blocks; per-thread column counts give
// each block its slots, so every column keeps ascending source rows.
Cmp compress_t(const Cmp &A) {
    Trace tr("compress_t");
    Cmp B;
    B.nmajor = A.nminor;
    B.nminor = A.nmajor;
    const int64_t nnz = A.nnz(), ncol = A.nminor;
    B.p.assign(ncol + 1, 0);
    B.i.resize(nnz);
    B.x.resize(nnz);
    const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(nthreads_for(A.nmajor),
                                                               (int64_t)(1 << 30) / std::max<int64_t>(ncol, 1) / 8));
    std::vector<std::vector<int64_t>> cnt(nt, std::vector<int64_t>(ncol, 0));
    auto count = [&](int64_t r0, int64_t r1, int w) {
        auto &c = cnt[w];
        for (int64_t jj = A.p[r0]; jj < A.p[r1]; jj++) c[A.i[jj]]++;
    };
    auto run = [&](auto fn) {
        if (nt <= 1) { fn(0, A.nmajor, 0); return; }
        std::vector<std::thread> th;
        for (int w = 0; w < nt; w++) th.emplace_back(fn, A.nmajor * w / nt, A.nmajor * (w + 1) / nt, w);
        for (auto &x : th) x.join();
    };
    run(count);
    // column c: thread 0's entries first, then thread 1's ...
    int64_t acc = 0;
    for (int64_t c = 0; c < ncol; c++) {
        B.p[c] = acc;
        for (int w = 0; w < nt; w++) {
            const int64_t k = cnt[w][c];
            cnt[w][c] = acc;
            acc += k;
        }
    }
    B.p[ncol] = acc;
    auto fill = [&](int64_t r0, int64_t r1, int w) {
        auto &pos = cnt[w];
        for (int64_t r = r0; r < r1; r++)
            for (int64_t jj = A.p[r]; jj < A.p[r + 1]; jj++) {
                const int64_t d = pos[A.i[jj]]++;
                B.i[d] = r;
                B.x[d] = A.x[jj];
            }
    };
    run(fill);
    return B;
}

// scipy csr_binop_csr, general path (the canonical path yields the same
// values; only the storage order differs, and every caller canonicalises).
template <class Op>
Cmp binop(const Cmp &A, const Cmp &B, Op op) {
    Trace tr("binop");
    const int64_t n_col = A.nminor;
    return build_rows<LinkedRow>(
        A.nmajor, n_col,
        [&] { return LinkedRow{std::vector<int64_t>(n_col, -1), std::vector<double>(n_col, 0.0), std::vector<double>(n_col, 0.0)}; },
        [&](int64_t r, LinkedRow &s, std::vector<int64_t> &oi, std::vector<double> &ox) {
            int64_t head = -2, length = 0;
            for (int64_t jj = A.p[r]; jj < A.p[r + 1]; jj++) {
                const int64_t j = A.i[jj];
                s.a[j] = s.a[j] + A.x[jj];
                if (s.next[j] == -1) { s.next[j] = head; head = j; length++; }
            }
            for (int64_t jj = B.p[r]; jj < B.p[r + 1]; jj++) {
                const int64_t j = B.i[jj];
                s.b[j] = s.b[j] + B.x[jj];
                if (s.next[j] == -1) { s.next[j] = head; head = j; length++; }
            }
            int64_t c = 0;
            for (int64_t jj = 0; jj < length; jj++) {
                const double res = op(s.a[head], s.b[head]);
                if (res != 0) {
                    oi.push_back(head);
                    ox.push_back(res);
                    c++;
                }
                const int64_t temp = head;
                head = s.next[head];
                s.next[temp] = -1;
                s.a[temp] = 0;
                s.b[temp] = 0;
            }
            return c;
        });
}

// CsrMatrix.from_scipy canonicalisation: sort_indices + eliminate_zeros
// (duplicates cannot occur in the products used here).
Cmp canonical(const Cmp &A) {
    Trace tr("canonical");
    using Row = std::vector<std::pair<int64_t, double>>;
    return build_rows<Row>(
        A.nmajor, A.nminor, [] { return Row(); },
        [&](int64_t r, Row &row, std::vector<int64_t> &oi, std::vector<double> &ox) {
            row.clear();
            for (int64_t jj = A.p[r]; jj < A.p[r + 1]; jj++)
                if (A.x[jj] != 0) row.emplace_back(A.i[jj], A.x[jj]);
            std::sort(row.begin(), row.end(),
                      [](const std::pair<int64_t, double> &a, const std::pair<int64_t, double> &b) {
                          return a.first < b.first;
                      });
            for (auto &e : row) {
                oi.push_back(e.first);
                ox.push_back(e.second);
            }
            return (int64_t)row.size();
        });
}

// Free an intermediate as soon as its last consumer is done (the setup's
// host-memory peak is the fine level's Galerkin product: n rows of A P).
void release(Cmp &m) { Cmp().p.swap(m.p), Cmp().i.swap(m.i), Cmp().x.swap(m.x); }

Cmp from_host(int64_t nrows, int64_t ncols, const int64_t *rp, const int64_t *ci, const double *v) {
    Cmp A;
    A.nmajor = nrows;
    A.nminor = ncols;
    A.p.assign(rp, rp + nrows + 1);
    A.i.assign(ci, ci + rp[nrows]);
    A.x.assign(v, v + rp[nrows]);
    return A;
}

Cmp prolongator(int64_t n, const int64_t *agg, int64_t n_agg) {  // amg.py:97-99
    Cmp P;
    P.nmajor = n;
    P.nminor = n_agg;
    P.p.resize(n + 1);
    std::iota(P.p.begin(), P.p.end(), 0);
    P.i.assign(agg, agg + n);
    P.x.assign(n, 1.0);
    return P;
}

double diag_of(const Cmp &A, int64_t r) {  // scipy diagonal (sums duplicates)
    double d = 0.0;
    for (int64_t jj = A.p[r]; jj < A.p[r + 1]; jj++)
        if (A.i[jj] == r) d = d + A.x[jj];
    return d;
}

}  // namespace

// ---------------------------------------------------------------- C ABI
struct amgp_hcsr {
    Cmp m;
};

static amgp_hcsr *wrap(Cmp &&m) {
    auto *h = new amgp_hcsr();
    h->m = std::move(m);
    return h;
}

extern "C" {

int amgp_setup_set_threads(int threads) {
    g_threads = threads > 0 ? threads : 1;
    return AMGP_OK;
}

int amgp_hcsr_info(const amgp_hcsr *h, int64_t *nrows, int64_t *ncols, int64_t *nnz) {
    if (!h) return amgp_fail(AMGP_EINVAL, "null host matrix");
    if (nrows) *nrows = h->m.nmajor;
    if (ncols) *ncols = h->m.nminor;
    if (nnz) *nnz = h->m.nnz();
    return AMGP_OK;
}

int amgp_hcsr_copy(const amgp_hcsr *h, int64_t *row_ptr, int64_t *col_idx, double *values) {
    if (!h) return amgp_fail(AMGP_EINVAL, "null host matrix");
    const Cmp &m = h->m;
    if (row_ptr) std::copy(m.p.begin(), m.p.end(), row_ptr);
    if (col_idx) std::copy(m.i.begin(), m.i.end(), col_idx);
    if (values) std::copy(m.x.begin(), m.x.end(), values);
    return AMGP_OK;
}

int amgp_hcsr_free(amgp_hcsr *h) {
    delete h;
    return AMGP_OK;
}

// amg.py:102-149
int amgp_setup_sa_aggregate(int64_t n, const int64_t *rp, const int64_t *ci, const double *v,
                            double theta, int64_t *agg, int64_t *n_agg_out) {
    if (n < 0 || !rp || !agg || !n_agg_out) return amgp_fail(AMGP_EINVAL, "sa_aggregate: bad argument");
    std::vector<double> diag(n);
    for (int64_t i = 0; i < n; i++) {
        double d = 0.0;
        for (int64_t jj = rp[i]; jj < rp[i + 1]; jj++)
            if (ci[jj] == i) d = d + v[jj];
        diag[i] = d;
    }
    auto strong = [&](int64_t i, int64_t jj) {
        const int64_t j = ci[jj];
        if (j == i) return false;
        const double prod = diag[i] * diag[j];
        const double thr = theta * sqrt(fabs(prod));
        return fabs(v[jj]) >= thr;
    };
    std::fill(agg, agg + n, -1);
    int64_t n_agg = 0;
    std::vector<int64_t> neigh;
    for (int64_t i = 0; i < n; i++) {  // seeds in natural order
        if (agg[i] >= 0) continue;
        neigh.clear();
        for (int64_t jj = rp[i]; jj < rp[i + 1]; jj++)
            if (strong(i, jj) && agg[ci[jj]] < 0) neigh.push_back(ci[jj]);
        if (neigh.size() < 2) continue;
        agg[i] = n_agg;
        for (int64_t j : neigh) agg[j] = n_agg;
        n_agg++;
    }
    for (int64_t i = 0; i < n; i++) {  // leftovers: strongest aggregated neighbour
        if (agg[i] >= 0) continue;
        int64_t best = -1;
        double best_w = -1.0;
        for (int64_t jj = rp[i]; jj < rp[i + 1]; jj++) {
            if (!strong(i, jj)) continue;
            const int64_t j = ci[jj];
            if (agg[j] >= 0) {
                double w = -INFINITY;  // max |a_ij| over the entries of column j in row i
                for (int64_t kk = rp[i]; kk < rp[i + 1]; kk++)
                    if (ci[kk] == j) w = std::max(w, fabs(v[kk]));
                if (w > best_w) {
                    best = agg[j];
                    best_w = w;
                }
            }
        }
        if (best >= 0) agg[i] = best;
        else agg[i] = n_agg++;
    }
    *n_agg_out = n_agg;
    return AMGP_OK;
}

// amg.py:124-133, the seeding pass of sa_aggregate over precomputed strength
// lists (the device setup computes them: strong neighbours of row i in row
// order, j != i, own columns).  agg is reset to -1 first.
int amgp_setup_sa_pass1(int64_t n, const int64_t *srp, const int32_t *scol, int64_t *agg,
                        int64_t *n_agg_out) {
    if (n < 0 || !srp || !agg || !n_agg_out) return amgp_fail(AMGP_EINVAL, "sa_pass1: bad argument");
    std::fill(agg, agg + n, -1);
    int64_t n_agg = 0;
    for (int64_t i = 0; i < n; i++) {
        if (agg[i] >= 0) continue;
        int cnt = 0;
        for (int64_t jj = srp[i]; jj < srp[i + 1] && cnt < 2; jj++) cnt += agg[scol[jj]] < 0;
        if (cnt < 2) continue;
        agg[i] = n_agg;
        for (int64_t jj = srp[i]; jj < srp[i + 1]; jj++)
            if (agg[scol[jj]] < 0) agg[scol[jj]] = n_agg;
        n_agg++;
    }
    *n_agg_out = n_agg;
    return AMGP_OK;
}

// amg.py:134-148, the leftover pass: rows[] (ascending) are the rows the
// seeding pass left unaggregated, each with its strength list and |a_ij|;
// a row joins the aggregate of its strongest aggregated strong neighbour
// (strict >, first wins), else becomes a singleton.
int amgp_setup_sa_pass2(int64_t nleft, const int64_t *rows, const int64_t *lrp, const int32_t *lcol,
                        const double *labs, int64_t *agg, int64_t *n_agg) {
    if (nleft < 0 || (nleft && (!rows || !lrp)) || !agg || !n_agg)
        return amgp_fail(AMGP_EINVAL, "sa_pass2: bad argument");
    for (int64_t t = 0; t < nleft; t++) {
        const int64_t i = rows[t];
        if (agg[i] >= 0) continue;
        int64_t best = -1;
        double best_w = -1.0;
        for (int64_t jj = lrp[t]; jj < lrp[t + 1]; jj++) {
            const int64_t j = lcol[jj];
            if (agg[j] >= 0 && labs[jj] > best_w) {
                best = agg[j];
                best_w = labs[jj];
            }
        }
        if (best >= 0) agg[i] = best;
        else agg[i] = (*n_agg)++;
    }
    return AMGP_OK;
}

// amg.py:152-191
int amgp_setup_matching_aggregate(int64_t n0, const int64_t *rp, const int64_t *ci,
                                  const double *v, int sweeps, int64_t *agg_out,
                                  int64_t *n_agg_out) {
    if (n0 < 0 || !rp || !agg_out || sweeps < 1)
        return amgp_fail(AMGP_EINVAL, "matching_aggregate: bad argument");
    std::vector<int64_t> agg(n0);
    std::iota(agg.begin(), agg.end(), 0);
    // cur is held as "compressed over columns" (scipy CSC) after the first
    // sweep; A-operand of the next product is cur's column arrays.
    Cmp cur_csr = from_host(n0, n0, rp, ci, v);
    Cmp cur_cols = compress_t(cur_csr);  // first sweep: CSC(cur) via csr_tocsc
    bool first = true;
    for (int s = 0; s < sweeps; s++) {
        const int64_t n = cur_cols.nmajor;
        // diagonal and upper-triangle edges (triu(cur, 1)); cur_cols holds
        // column c -> rows r.
        std::vector<double> diag(n, 0.0);
        for (int64_t c = 0; c < n; c++)
            for (int64_t jj = cur_cols.p[c]; jj < cur_cols.p[c + 1]; jj++)
                if (cur_cols.i[jj] == c) diag[c] = diag[c] + cur_cols.x[jj];
        struct Edge {
            double w;
            int64_t i, j;
        };
        std::vector<Edge> edges;
        for (int64_t c = 0; c < n; c++)
            for (int64_t jj = cur_cols.p[c]; jj < cur_cols.p[c + 1]; jj++) {
                const int64_t r = cur_cols.i[jj];
                if (r + 1 > c) continue;  // keep row + 1 <= col
                const double two_a = 2.0 * cur_cols.x[jj];
                const double den = diag[r] + diag[c];
                const double q = two_a / den;
                const double w = 1.0 - q;
                if (w > 0.0) edges.push_back({w, r, c});
            }
        std::sort(edges.begin(), edges.end(), [](const Edge &a, const Edge &b) {
            if (a.w != b.w) return a.w > b.w;
            if (a.i != b.i) return a.i < b.i;
            return a.j < b.j;
        });
        std::vector<int64_t> mate(n, -1);
        for (const Edge &e : edges)
            if (mate[e.i] < 0 && mate[e.j] < 0) {
                mate[e.i] = e.j;
                mate[e.j] = e.i;
            }
        std::vector<int64_t> new_idx(n, -1);
        int64_t nc = 0;
        for (int64_t i = 0; i < n; i++) {
            if (new_idx[i] >= 0) continue;
            new_idx[i] = nc;
            if (mate[i] >= 0) new_idx[mate[i]] = nc;
            nc++;
        }
        for (auto &a : agg) a = new_idx[a];
        // cur = Pc^T @ cur @ Pc with scipy's evaluation:
        //   C = csr_matmat(cur column arrays, Pc)   -> (Pc^T cur) as CSC
        //   G = csr_matmat(csr_tocsc(Pc), C)         -> (C Pc) as CSC
        Cmp Pc = prolongator(n, new_idx.data(), nc);
        Cmp C = matmat(cur_cols, Pc);
        Cmp G = matmat(compress_t(Pc), C);
        cur_cols = std::move(G);  // G is CSC: column J -> rows K
        first = false;
        if (nc == n) break;
    }
    (void)first;
    int64_t mx = -1;
    for (int64_t a : agg) mx = std::max(mx, a);
    std::copy(agg.begin(), agg.end(), agg_out);
    *n_agg_out = mx + 1;
    return AMGP_OK;
}

// amg.py:219-226: P = P_hat - (diags(omega/d) @ A) @ P_hat, canonicalised.
int amgp_setup_smooth_prolongator(int64_t n, const int64_t *rp, const int64_t *ci,
                                  const double *v, const int64_t *agg, int64_t n_agg,
                                  double omega, amgp_hcsr **out) {
    if (n < 0 || !rp || !agg || !out) return amgp_fail(AMGP_EINVAL, "smooth_prolongator: bad argument");
    Cmp A = from_host(n, n, rp, ci, v);
    // diags(omega/d).tocsr() has one entry per row (zeros dropped); in
    // csr_matmat(D, A) each output entry gets exactly one contribution
    // 0.0 + s*a_rk, and the head-inserted linked list emits each row of A
    // reversed -- built directly.  S's row order matters: it is the summation
    // order of T = S @ P_hat below.
    std::vector<double> scale(n);
    for (int64_t r = 0; r < n; r++) {
        const double d = diag_of(A, r);
        if (d == 0.0) return amgp_fail(AMGP_EINVAL, "zero diagonal entry");
        scale[r] = omega / d;
    }
    Cmp S = build_rows<int>(
        n, n, [] { return 0; },
        [&](int64_t r, int &, std::vector<int64_t> &oi, std::vector<double> &ox) {
            const double s = scale[r];
            int64_t c = 0;
            if (s == 0) return c;
            for (int64_t jj = A.p[r + 1] - 1; jj >= A.p[r]; jj--) {
                const double prod = s * A.x[jj];
                const double sum = 0.0 + prod;
                if (sum != 0) {
                    oi.push_back(A.i[jj]);
                    ox.push_back(sum);
                    c++;
                }
            }
            return c;
        });
    release(A);
    Cmp Ph = prolongator(n, agg, n_agg);
    Cmp T = matmat(S, Ph);
    release(S);
    Cmp R = binop(Ph, T, [](double a, double b) { return a - b; });
    release(T);
    release(Ph);
    *out = wrap(canonical(R));
    return AMGP_OK;
}

// amg.py:229-235: (P^T A) P, then (S + S^T) * 0.5, canonicalised.
int amgp_setup_galerkin(int64_t n, const int64_t *rp, const int64_t *ci, const double *v,
                        int64_t nc, const int64_t *prp, const int64_t *pci, const double *pv,
                        amgp_hcsr **out) {
    if (n < 0 || !rp || !prp || !out) return amgp_fail(AMGP_EINVAL, "galerkin: bad argument");
    Cmp At;
    {
        Cmp A = from_host(n, n, rp, ci, v);
        At = compress_t(A);
    }
    Cmp P = from_host(n, nc, prp, pci, pv);
    Cmp C = matmat(At, P);  // P^T (CSC) @ A: csr_matmat(csc(A), P)
    release(At);
    Cmp G;
    {
        Cmp Pt = compress_t(P);
        release(P);
        G = matmat(Pt, C);  // C (CSC) @ P:  csr_matmat(csc(P), C)
    }
    release(C);
    // G holds "column J -> rows K" of P^T A P.  S = G + G^T evaluated as CSC:
    // the CSR view G^T converted to CSC is compress_t(G arrays).
    Cmp H = compress_t(G);
    Cmp S = binop(G, H, [](double a, double b) { return a + b; });
    release(G);
    release(H);
    for (double &x : S.x) x = x * 0.5;
    // S is CSC (column t -> rows u); tocsr() == compressed transpose
    Cmp Sr = compress_t(S);
    release(S);
    *out = wrap(canonical(Sr));
    return AMGP_OK;
}

// numpy's float64 dot (v @ w, np.linalg.norm) as the reference executes it:
// OpenBLAS 0.3.30 ddot, SkylakeX kernel (the kernel numpy's bundled
// scipy-openblas dispatches on AVX-512 hosts).  n1 = n & -16 elements go
// through the micro-kernel: four 8-wide FMA accumulators over 32-element
// blocks, folded to four 4-wide ones, 16-element blocks on the four 4-wide
// accumulators, then ((a0+a1)+a2)+a3, 256->128 fold and a horizontal add
// (verified bit-exact against numpy for 1, 3 and 8 BLAS threads); the rest is
// dot = fma(y, x, dot).  With `threads` > 1 and n > 10000, OpenBLAS splits n
// into contiguous chunks (width = ceil(remaining / threads_left)) and sums
// the per-chunk dots in order from 0.0.  The reference's hierarchy therefore
// depends on the host's OpenBLAS thread count; the canonical choice here is
// one thread (SURVEY.md section 8d runs the reference with
// OPENBLAS_NUM_THREADS=1).
static double ddot_chunk(int64_t n, const double *x, const double *y) {
    double dot = 0.0;
    const int64_t n1 = n & -16;
    if (n1) {
        double a05[8] = {0}, a15[8] = {0}, a25[8] = {0}, a35[8] = {0};
        const int64_t n32 = n1 & ~(int64_t)31;
        int64_t i = 0;
        for (; i < n32; i += 32)
            for (int l = 0; l < 8; l++) {
                a05[l] = fma(x[i + l], y[i + l], a05[l]);
                a15[l] = fma(x[i + 8 + l], y[i + 8 + l], a15[l]);
                a25[l] = fma(x[i + 16 + l], y[i + 16 + l], a25[l]);
                a35[l] = fma(x[i + 24 + l], y[i + 24 + l], a35[l]);
            }
        double a0[4], a1[4], a2[4], a3[4];
        for (int l = 0; l < 4; l++) {
            a0[l] = a05[l] + a05[l + 4];
            a1[l] = a15[l] + a15[l + 4];
            a2[l] = a25[l] + a25[l + 4];
            a3[l] = a35[l] + a35[l + 4];
        }
        for (; i < n1; i += 16)
            for (int l = 0; l < 4; l++) {
                a0[l] = fma(x[i + l], y[i + l], a0[l]);
                a1[l] = fma(x[i + 4 + l], y[i + 4 + l], a1[l]);
                a2[l] = fma(x[i + 8 + l], y[i + 8 + l], a2[l]);
                a3[l] = fma(x[i + 12 + l], y[i + 12 + l], a3[l]);
            }
        double s[4];
        for (int l = 0; l < 4; l++) s[l] = ((a0[l] + a1[l]) + a2[l]) + a3[l];
        const double h0 = s[0] + s[2], h1 = s[1] + s[3];
        dot = h0 + h1;
    }
    for (int64_t i = n1; i < n; i++) dot = fma(y[i], x[i], dot);
    return dot;
}

extern "C" double amgp_setup_blas_dot(int64_t n, const double *x, const double *y, int threads) {
    if (n <= 0) return 0.0;
    if (threads <= 1 || n <= 10000) return ddot_chunk(n, x, y);
    double dot = 0.0;
    int64_t i = n, start = 0;
    for (int t = 0; i > 0; t++) {
        const int64_t left = threads - t;
        int64_t width = (i + left - 1) / left;
        i -= width;
        if (i < 0) width += i;
        dot = dot + ddot_chunk(width, x + start, y + start);
        start += width;
    }
    return dot;
}

// In-order host SpMV (scipy csr_matvec order), row blocks on threads.
int amgp_setup_spmv(int64_t n, const int64_t *rp, const int64_t *ci, const double *v,
                    const double *x, double *y) {
    if (n < 0 || !rp) return amgp_fail(AMGP_EINVAL, "spmv: bad argument");
    parallel_rows(n, [&](int64_t r0, int64_t r1, int) {
        for (int64_t r = r0; r < r1; r++) {
            double s = 0.0;
            for (int64_t jj = rp[r]; jj < rp[r + 1]; jj++) {
                const double prod = v[jj] * x[ci[jj]];
                s = s + prod;
            }
            y[r] = s;
        }
    });
    return AMGP_OK;
}

}  // extern "C"
