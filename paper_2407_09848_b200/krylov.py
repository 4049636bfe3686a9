"""PCG / FCG on the GPU (reference krylov.py).

``solve`` keeps the reference signature and report (krylov.py:15-120); the
whole iteration -- SpMV, dots, axpys and the V-cycle preconditioner -- runs
in libamgp (csrc/pcg.cu) with deterministic reductions, and only the relative
residual crosses to the host once per iteration, when the preconditioner is
one of the package's device preconditioners (or None).

Any other callable r -> z (the reference accepts one, krylov.py:88) takes the
reference-exact path: the same iteration with the vectors on the device and
every operation a libamgp kernel carrying the reference's arithmetic -- the
dots in OpenBLAS ddot order (the reference's numpy dots, one BLAS thread),
the axpys rounded as numpy rounds them -- while the callable itself is called
with the residual in the container type of b (a numpy array for numpy input:
one host round trip per iteration).  Same iterates as the reference,
bit for bit, given a preconditioner that returns the same bits.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .amg import AmgHierarchy, DeviceHierarchy, Level, VcyclePreconditioner
from .smoothers import SmootherPreconditioner
from .sparse import device_of


@dataclass
class KrylovConfig:
    variant: str = "pcg"  # pcg | fcg
    tol: float = 1e-7
    itmax: int = 1000
    record_history: bool = True

    def __post_init__(self):
        if self.variant not in N.VARIANT_CODES:  # pcg | fcg | pcg1 (single reduction)
            raise ValueError(f"unknown Krylov variant {self.variant!r}")
        if self.tol <= 0.0 or self.itmax < 1:
            raise ValueError("tol must be positive and itmax >= 1")


@dataclass
class SolveReport:
    iterations: int
    converged: bool
    final_relres: float
    residual_history: list = field(default_factory=list)
    spmv_count: int = 0
    precond_count: int = 0
    breakdown: bool = False
    elapsed_s: float = 0.0


def _device_precond(precond):
    if precond is None:
        return None
    if isinstance(precond, VcyclePreconditioner):
        D = precond.h.device()
        D.sync_smoothers()
        return D
    if isinstance(precond, SmootherPreconditioner):
        # one-level hierarchy whose "coarse solve" is the smoother itself
        if getattr(precond, "_dev", None) is None:
            h = AmgHierarchy(levels=[Level(A=precond.A, M=precond.M, smoother=precond.config)])
            precond._dev = DeviceHierarchy(h, coarse_solver="smoother")
        precond._dev.sync_smoothers()
        return precond._dev
    return "callable"


def solve(A, b, precond=None, cfg=None, x0=None):
    """Solve SPD A x = b on the GPU; returns (x, SolveReport) (krylov.py:45-120)."""
    cfg = cfg or KrylovConfig()
    D = device_of(A)
    n = b.shape[0] if hasattr(b, "shape") else len(b)
    if D.nrows != n or D.ncols != n:
        raise ValueError("dimension mismatch")
    H = _device_precond(precond)
    if H == "callable":
        if not callable(precond):
            raise TypeError("solve: precond must be callable or None")
        return _solve_callable(D, b, precond, cfg, x0)
    c = D.ctx
    rep = N.SolveReportC()
    hist = np.empty(cfg.itmax + 1) if cfg.record_history else None
    with c.scope():
        bd = N.to_device(b, c)
        x = N.to_device(x0, c, copy=True) if x0 is not None else N.empty(n, c)
        N.check(N.lib().amgp_pcg_solve(
            c.handle, D.handle, H.handle if H is not None else None, N.ptr(bd), N.ptr(x),
            int(x0 is not None), N.VARIANT_CODES[cfg.variant], float(cfg.tol), int(cfg.itmax),
            hist.ctypes.data_as(N._PD) if hist is not None else None, C.byref(rep)))
    report = SolveReport(
        iterations=rep.iterations,
        converged=bool(rep.converged),
        final_relres=rep.final_relres,
        residual_history=hist[: rep.n_history].tolist() if hist is not None else [],
        spmv_count=rep.spmv_count,
        precond_count=rep.precond_count,
        breakdown=bool(rep.breakdown),
        elapsed_s=rep.elapsed_s,
    )
    return N.like(x, b), report


def _solve_callable(D, b, precond, cfg, x0):
    """Reference krylov.solve (krylov.py:45-120) step for step with a user
    preconditioner callable: device vectors, libamgp kernels (OpenBLAS-order
    dots amgp_ds_blas_dot3, numpy-rounded axpys amgp_vec_update, in-order
    SpMV), scalars as the reference's Python floats."""
    import math
    import time

    from .dsetup import blas_threads
    from .sparse import _count

    lib = N.lib()
    c = D.ctx
    n = D.nrows
    th = blas_threads()
    t0 = time.perf_counter()
    out3 = (C.c_double * 3)()

    def dot(u, v):  # float(u @ v)
        N.check(lib.amgp_ds_blas_dot3(c.handle, n, N.ptr(u), N.ptr(v), th, out3))
        return out3[0]

    def norm(u):  # np.linalg.norm(u) = sqrt(u @ u)
        N.check(lib.amgp_ds_blas_dot3(c.handle, n, N.ptr(u), N.ptr(u), th, out3))
        return math.sqrt(out3[0])

    def axpy(a, s, v, out, sign):  # out = a + s*v (sign +1) / a - s*v (sign -1)
        N.check(lib.amgp_vec_update(c.handle, n, float(s), N.ptr(a), N.ptr(v), N.ptr(out), sign))

    def matvec(v, out):
        N.check(lib.amgp_spmv(c.handle, D.handle, N.ptr(v), N.ptr(out)))
        _count()

    def prec(r):
        rin = N.like(r, b)
        z = precond(rin)
        return N.to_device(z, c, copy=True)

    spmv = pc = 0
    history = []

    def report(it, converged, relres, breakdown=False):
        return SolveReport(iterations=it, converged=converged, final_relres=relres, residual_history=history,
                           spmv_count=spmv, precond_count=pc, breakdown=breakdown,
                           elapsed_s=time.perf_counter() - t0)

    with c.scope():
        bd = N.to_device(b, c)
        x = N.to_device(x0, c, copy=True) if x0 is not None else c.torch.zeros(n, dtype=c.torch.float64,
                                                                               device=c.device)
        bnorm = norm(bd)
        if bnorm == 0.0:
            return N.like(x * 0.0, b), report(0, True, 0.0)
        r = N.empty(n, c)
        tmp = N.empty(n, c)
        matvec(x, tmp)
        axpy(bd, 1.0, tmp, r, -1)  # r = b - A x (1.0 * y == y exactly)
        spmv += 1
        relres = norm(r) / bnorm
        if cfg.record_history:
            history.append(relres)
        if relres <= cfg.tol:
            return N.like(x, b), report(0, True, relres)
        z = prec(r)
        pc += 1
        d = z.clone()
        rz = dot(r, z)
        Ad = N.empty(n, c)
        for it in range(1, cfg.itmax + 1):
            matvec(d, Ad)
            spmv += 1
            dAd = dot(d, Ad)
            if dAd <= 0.0:
                return N.like(x, b), report(it - 1, False, relres, breakdown=True)
            alpha = rz / dAd if cfg.variant != "fcg" else dot(r, d) / dAd
            axpy(x, alpha, d, x, +1)
            axpy(r, alpha, Ad, r, -1)
            relres = norm(r) / bnorm
            if cfg.record_history:
                history.append(relres)
            if relres <= cfg.tol:
                return N.like(x, b), report(it, True, relres)
            z = prec(r)
            pc += 1
            if cfg.variant != "fcg":
                rz_new = dot(r, z)
                beta = rz_new / rz
                rz = rz_new
                axpy(z, beta, d, d, +1)
            else:
                beta = dot(z, Ad) / dAd
                axpy(z, beta, d, d, -1)
        return N.like(x, b), report(cfg.itmax, False, relres)
