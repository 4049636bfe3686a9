"""PCG / FCG on the GPU (reference krylov.py).

``solve`` keeps the reference signature and report (krylov.py:15-120); the
whole iteration -- SpMV, dots, axpys and the V-cycle preconditioner -- runs
in libamgp (csrc/pcg.cu) with deterministic reductions, and only the relative
residual crosses to the host once per iteration.  The preconditioner must be
one of the package's device preconditioners (or None); an arbitrary Python
callable would force a host round trip per iteration and is rejected.
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
    raise TypeError("solve: precond must be None, as_vcycle_preconditioner(h) or "
                    "as_preconditioner(...) (device path; no host callback)")


def solve(A, b, precond=None, cfg=None, x0=None):
    """Solve SPD A x = b on the GPU; returns (x, SolveReport) (krylov.py:45-120)."""
    cfg = cfg or KrylovConfig()
    D = device_of(A)
    n = b.shape[0] if hasattr(b, "shape") else len(b)
    if D.nrows != n or D.ncols != n:
        raise ValueError("dimension mismatch")
    H = _device_precond(precond)
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
