"""Host-side hierarchy setup driven from Python, arithmetic in native C++.

Mirrors reference amg.py:194-287.  Aggregation, prolongator smoothing and the
Galerkin products run in csrc/setup.cpp (bit-exact restatements of the
reference's Python loops and scipy kernels).  The power iteration for
lambda_max keeps its dot products in numpy on purpose: the reference takes
them through numpy/BLAS (amg.py:211-212), whose summation order is the
host BLAS's, so evaluating them with the same numpy call reproduces the
reference's omega bit for bit on any host.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _native as N
from .smoothers import l1_jacobi_diag
from .sparse import CsrMatrix

_threads_set = False


def _threads():
    global _threads_set
    if not _threads_set:
        N.lib().amgp_setup_set_threads(int(os.environ.get("AMGP_SETUP_THREADS", os.cpu_count() or 1)))
        _threads_set = True


def _arrs(A):
    rp = np.ascontiguousarray(A.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(A.col_idx, dtype=np.int64)
    v = np.ascontiguousarray(A.values, dtype=np.float64)
    return rp, ci, v, rp.ctypes.data_as(N._P64), ci.ctypes.data_as(N._P64), v.ctypes.data_as(N._PD)


def _take(h):
    """Copy an amgp_hcsr out into a CsrMatrix and free it."""
    nr, nc, nnz = C.c_int64(), C.c_int64(), C.c_int64()
    N.check(N.lib().amgp_hcsr_info(h, C.byref(nr), C.byref(nc), C.byref(nnz)))
    rp = np.empty(nr.value + 1, dtype=np.int64)
    ci = np.empty(nnz.value, dtype=np.int64)
    v = np.empty(nnz.value, dtype=np.float64)
    N.check(N.lib().amgp_hcsr_copy(h, rp.ctypes.data_as(N._P64), ci.ctypes.data_as(N._P64),
                                   v.ctypes.data_as(N._PD)))
    N.lib().amgp_hcsr_free(h)
    return CsrMatrix(nr.value, nc.value, rp, ci, v)


def _prolongator(n, agg, n_agg):  # amg.py:97-99
    return CsrMatrix(n, n_agg, np.arange(n + 1), agg, np.ones(n))


def sa_aggregate(A, theta=0.01):
    """Tentative prolongator by greedy strong-neighbour aggregation (amg.py:102-149)."""
    _threads()
    rp, ci, v, prp, pci, pv = _arrs(A)
    agg = np.empty(A.nrows, dtype=np.int64)
    n_agg = C.c_int64()
    N.check(N.lib().amgp_setup_sa_aggregate(A.nrows, prp, pci, pv, float(theta),
                                            agg.ctypes.data_as(N._P64), C.byref(n_agg)))
    return _prolongator(A.nrows, agg, n_agg.value)


def matching_aggregate(A, sweeps=3):
    """Tentative prolongator by repeated greedy pairwise matching (amg.py:152-191)."""
    _threads()
    rp, ci, v, prp, pci, pv = _arrs(A)
    agg = np.empty(A.nrows, dtype=np.int64)
    n_agg = C.c_int64()
    N.check(N.lib().amgp_setup_matching_aggregate(A.nrows, prp, pci, pv, int(sweeps),
                                                  agg.ctypes.data_as(N._P64), C.byref(n_agg)))
    return _prolongator(A.nrows, agg, n_agg.value)


def host_spmv(A, x):
    rp, ci, v, prp, pci, pv = _arrs(A)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(A.nrows)
    N.check(N.lib().amgp_setup_spmv(A.nrows, prp, pci, pv, x.ctypes.data_as(N._PD),
                                    y.ctypes.data_as(N._PD)))
    return y


def blas_threads():
    """OpenBLAS thread count whose ddot order the setup reproduces
    (AMGP_BLAS_THREADS, default 1 -- the reference run single-threaded)."""
    return int(os.environ.get("AMGP_BLAS_THREADS", "1"))


def blas_dot(x, y, threads=None):
    """numpy's float64 dot as OpenBLAS (SkylakeX kernel) evaluates it, host-independent."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    return N.lib().amgp_setup_blas_dot(len(x), x.ctypes.data_as(N._PD), y.ctypes.data_as(N._PD),
                                       int(blas_threads() if threads is None else threads))


def estimate_lambda_max(A, d, iters=25):
    """Power iteration on D^-1/2 A D^-1/2 (amg.py:194-216), same seeded start.

    The dots and the norm use blas_dot: the reference takes them through
    numpy -> OpenBLAS ddot, whose summation order (SIMD accumulators, thread
    split) decides the last bits of lambda and hence of every coarse level.
    """
    if np.any(d <= 0.0):
        raise ValueError("diagonal must be positive")
    _threads()
    ds = np.sqrt(d)
    v = np.ones(A.nrows) + np.random.default_rng(0).uniform(-0.5, 0.5, A.nrows)
    lam = 1.0
    for _ in range(iters):
        w = host_spmv(A, v / ds) / ds
        lam = blas_dot(v, w) / blas_dot(v, v)
        nrm = np.sqrt(blas_dot(w, w))
        if nrm == 0.0:
            return 0.0
        v = w / nrm
    return lam


def smooth_prolongator(A, P_hat, omega):
    """P = (I - omega D^-1 A) P_hat (amg.py:219-226)."""
    _threads()
    rp, ci, v, prp, pci, pv = _arrs(A)
    agg = np.ascontiguousarray(P_hat.col_idx, dtype=np.int64)
    if not (np.array_equal(P_hat.row_ptr, np.arange(A.nrows + 1)) and np.all(P_hat.values == 1.0)):
        raise ValueError("P_hat must be an aggregation prolongator")
    h = N._VP()
    N.check(N.lib().amgp_setup_smooth_prolongator(A.nrows, prp, pci, pv,
                                                  agg.ctypes.data_as(N._P64), P_hat.ncols,
                                                  float(omega), C.byref(h)))
    return _take(h)


def galerkin_rap(A, P):
    """Coarse operator P^T A P, symmetrised (amg.py:229-235)."""
    if A.ncols != P.nrows:
        raise ValueError("dimension mismatch in Galerkin product")
    _threads()
    rp, ci, v, prp, pci, pv = _arrs(A)
    qrp, qci, qv, pqrp, pqci, pqv = _arrs(P)
    h = N._VP()
    N.check(N.lib().amgp_setup_galerkin(A.nrows, prp, pci, pv, P.ncols, pqrp, pqci, pqv,
                                        C.byref(h)))
    return _take(h)


def build_hierarchy(A, coarsening, smoother, max_levels, min_coarse_size, coarse_solver,
                    coarse_sweeps):
    """amg.py:238-287 loop."""
    from .amg import AmgHierarchy, Level

    levels = [Level(A=A, M=l1_jacobi_diag(A), smoother=smoother)]
    stagnated = 0
    while (levels[-1].A.nrows > min_coarse_size and len(levels) < max_levels
           and stagnated < 2):
        Al = levels[-1].A
        if coarsening.kind == "smoothed_aggregation":
            P_hat = sa_aggregate(Al, coarsening.strength_theta)
        else:
            P_hat = matching_aggregate(Al, coarsening.matching_sweeps)
        if coarsening.prolongator_smoothing:
            d = Al.diagonal()
            lam = estimate_lambda_max(Al, d)
            P = smooth_prolongator(Al, P_hat, 4.0 / (3.0 * lam))
        else:
            P = P_hat
        if P.ncols >= 0.95 * Al.nrows:
            stagnated += 1
        else:
            stagnated = 0
        if P.ncols >= Al.nrows:
            break
        Ac = galerkin_rap(Al, P)
        levels[-1].P = P
        levels[-1].n_aggregates = P.ncols
        levels.append(Level(A=Ac, M=l1_jacobi_diag(Ac), smoother=smoother))
    return AmgHierarchy(levels=levels, coarse_solver=coarse_solver, coarse_sweeps=coarse_sweeps,
                        stagnated=stagnated >= 2)
