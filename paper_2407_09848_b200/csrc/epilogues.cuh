// Row epilogues of the SELL kernels (rows.cuh): what each hot kernel does
// with y_i = (A v)_i, in the reference's exact elementwise operation order
// (smoothers.py:106-137, amg.py:311-314).
#pragma once

#include "rows.cuh"

// m, b and the gathered operand are never written by the kernel that reads
// them (the operand already travels through the non-coherent path in
// sell_row_dot), so their row loads take it too.
__device__ __forceinline__ double ro(const double *p, int64_t i) { return __ldg(p + i); }

// ---------------------------------------------------------------- epilogues
template <bool FIRST, bool LAST, bool X0>
struct Cheb4Step {
    static constexpr bool kSpmv = !FIRST || X0;
    const double *m;
    const double *b;
    const double *xg;  // x0 (first step) or z_{j-1}
    double *r;
    double *znew;
    double *x;
    double cz, cr, beta;
    __device__ __forceinline__ void operator()(int64_t row, double y) const {
        const double rr = __dsub_rn(FIRST ? ro(b, row) : r[row], y);
        double z = FIRST ? __dmul_rn(0.0, cz) : __dmul_rn(ro(xg, row), cz);
        z = __dadd_rn(z, __dmul_rn(cr, __ddiv_rn(rr, ro(m, row))));
        const double xo = FIRST ? (X0 ? ro(xg, row) : 0.0) : x[row];
        x[row] = __dadd_rn(xo, __dmul_rn(beta, z));
        if (!LAST) {
            r[row] = rr;
            znew[row] = z;
        }
    }
};

template <bool FIRST, bool LAST, bool X0, bool RHO1>
struct Cheb1Step {
    static constexpr bool kSpmv = !FIRST || X0;
    const double *m;
    const double *b;
    const double *xg;  // x0 (init) or d_{j-1}
    double *r;
    double *dnew;
    double *x;
    double c0, c1, rho;  // init: c0 = theta; step: c0 = rho_j rho_{j-1}, c1 = 2 rho_j / delta
    __device__ __forceinline__ void operator()(int64_t row, double y) const {
        double rr, d, xo;
        if (FIRST) {
            rr = __ddiv_rn(__dsub_rn(ro(b, row), y), ro(m, row));
            if (!RHO1) rr = __ddiv_rn(rr, rho);
            d = __ddiv_rn(rr, c0);
            xo = X0 ? ro(xg, row) : 0.0;
        } else {
            double sv = __ddiv_rn(y, ro(m, row));
            if (!RHO1) sv = __ddiv_rn(sv, rho);
            rr = __dsub_rn(r[row], sv);
            d = __dadd_rn(__dmul_rn(ro(xg, row), c0), __dmul_rn(c1, rr));
            xo = x[row];
        }
        x[row] = __dadd_rn(xo, d);
        if (!LAST) {
            r[row] = rr;
            dnew[row] = d;
        }
    }
};

template <bool X0>
struct L1Sweep {
    static constexpr bool kSpmv = X0;
    const double *m;
    const double *b;
    const double *xin;
    double *xout;
    __device__ __forceinline__ void operator()(int64_t row, double y) const {
        const double rr = __dsub_rn(ro(b, row), y);
        xout[row] = __dadd_rn(X0 ? ro(xin, row) : 0.0, __ddiv_rn(rr, ro(m, row)));
    }
};

// MODE 0: y = A x ; MODE 1: y = r - A x (amg.py:311) ; MODE 2: y = y + A x (amg.py:314)
template <int MODE>
struct SpmvEpi {
    static constexpr bool kSpmv = true;
    const double *r;
    double *y;
    __device__ __forceinline__ void operator()(int64_t row, double sum) const {
        if (MODE == 0) y[row] = sum;
        else if (MODE == 1) y[row] = __dsub_rn(r[row], sum);
        else y[row] = __dadd_rn(y[row], sum);
    }
};

