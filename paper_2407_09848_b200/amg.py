"""AMG hierarchy and the device V-cycle (reference amg.py).

Setup (aggregation, prolongator smoothing, Galerkin products) runs on the
host, as the north star allows; ``build_hierarchy`` uses the native C++
restatement in csrc/setup.cpp, bit-exact with the reference (amg.py:97-287).
The V-cycle itself (amg.py:293-319) runs entirely on the GPU
(csrc/vcycle.cu) and is replayed from a CUDA graph.
"""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .smoothers import DeviceL1JacobiData, L1JacobiData, PolySmootherConfig, l1_jacobi_diag
from .sparse import CsrMatrix, device_of


@dataclass
class CoarseningConfig:
    kind: str = "smoothed_aggregation"  # or "pairwise_matching"
    strength_theta: float = 0.01
    matching_sweeps: int = 3
    prolongator_smoothing: bool = True

    def __post_init__(self):
        if self.kind not in ("smoothed_aggregation", "pairwise_matching"):
            raise ValueError(f"unknown coarsening kind {self.kind!r}")
        if not 0.0 <= self.strength_theta < 1.0:
            raise ValueError("strength_theta must lie in [0, 1)")
        if self.matching_sweeps < 1:
            raise ValueError("matching_sweeps must be >= 1")


@dataclass
class Level:
    A: CsrMatrix
    M: L1JacobiData
    smoother: PolySmootherConfig
    P: CsrMatrix | None = None
    n_aggregates: int = 0
    _Pt: CsrMatrix | None = field(default=None, repr=False)

    def restrict_op(self):
        """Explicit P^T (amg.py:56-59), cached."""
        if self._Pt is None:
            self._Pt = self.P.transpose()
        return self._Pt


def _smoother_key(cfg):
    beta = tuple(cfg.beta.beta.tolist()) if cfg.family == "opt_cheb4" else ()
    return (cfg.family, int(cfg.degree), cfg.a, float(cfg.rho_scale), beta)


class DeviceHierarchy:
    """libamgp hierarchy handle built from host levels; keeps device images alive."""

    def __init__(self, h, coarse_solver=None):
        c = N.ctx()
        self.ctx = c
        self.levels = h.levels
        L = len(h.levels)
        self._A = [device_of(lv.A) for lv in h.levels]
        from .smoothers import _m_device

        self._m = [_m_device(lv.M, c) for lv in h.levels]
        self._P = [device_of(lv.P) for lv in h.levels[:-1]]
        self._R = [device_of(lv.restrict_op()) for lv in h.levels[:-1]]
        Aa = (N._VP * L)(*[a.handle for a in self._A])
        Ma = (N._VP * L)(*[m.data_ptr() for m in self._m])
        Pa = (N._VP * max(L - 1, 1))(*[p.handle for p in self._P])
        Ra = (N._VP * max(L - 1, 1))(*[r.handle for r in self._R])
        solver = coarse_solver or h.coarse_solver
        handle = N._VP()
        with c.scope():
            N.check(N.lib().amgp_hier_create(c.handle, L, Aa, Ma, Pa, Ra, N.COARSE_CODES[solver],
                                             int(h.coarse_sweeps), C.byref(handle)))
        self.handle = handle
        self._keys = [None] * L
        if solver == "dense_direct":
            Ad = h.levels[-1].A.to_dense()
            try:
                Lf = np.linalg.cholesky(Ad)
            except np.linalg.LinAlgError as exc:
                raise ValueError("matrix is not positive definite") from exc
            Lc = np.ascontiguousarray(Lf.T)  # column-major L
            N.check(N.lib().amgp_hier_set_coarse_cholesky(handle, Lc.ctypes.data_as(N._PD)))

    def sync_smoothers(self):
        for l, lv in enumerate(self.levels):
            key = _smoother_key(lv.smoother)
            if key != self._keys[l]:
                cfg = N.smoother_cfg(lv.smoother)
                N.check(N.lib().amgp_hier_set_smoother(self.handle, l, C.byref(cfg)))
                self._keys[l] = key

    def apply(self, r, z):
        """z = V(r) for device tensors."""
        self.sync_smoothers()
        N.check(N.lib().amgp_vcycle_apply(self.handle, N.ptr(r), N.ptr(z)))

    def use_graph(self, enable=True):
        N.check(N.lib().amgp_hier_use_graph(self.handle, int(enable)))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and N._lib is not None:
            try:
                N.lib().amgp_hier_destroy(h)
            except Exception:
                pass
            self.handle = None


@dataclass
class AmgHierarchy:
    levels: list
    coarse_solver: str = "l1_jacobi"  # or "dense_direct"
    coarse_sweeps: int = 30
    stagnated: bool = False
    _dev: DeviceHierarchy | None = field(default=None, repr=False)

    def operator_complexity(self):
        return sum(l.A.nnz for l in self.levels) / self.levels[0].A.nnz

    def summary(self):
        return {
            "levels": [
                {
                    "size": l.A.nrows,
                    "nnz": l.A.nnz,
                    "aggregates": l.n_aggregates,
                    "smoother": l.smoother.family,
                    "degree": l.smoother.degree,
                }
                for l in self.levels
            ],
            "coarse_solver": self.coarse_solver,
            "operator_complexity": self.operator_complexity(),
            "stagnated": self.stagnated,
        }

    def summary_json(self):
        return json.dumps(self.summary(), indent=2)

    def device(self):
        """GPU image of the hierarchy (built once; smoothers re-synced per apply)."""
        if self._dev is None:
            self._dev = DeviceHierarchy(self)
        return self._dev


def hierarchy_from_levels(levels, smoother, coarse_solver="l1_jacobi", coarse_sweeps=30):
    """AmgHierarchy from explicit (A, P) level matrices (e.g. an exported hierarchy)."""
    out = []
    for l, (A, P) in enumerate(levels):
        lv = Level(A=A, M=l1_jacobi_diag(A), smoother=smoother, P=P,
                   n_aggregates=P.ncols if P is not None else 0)
        out.append(lv)
    return AmgHierarchy(levels=out, coarse_solver=coarse_solver, coarse_sweeps=coarse_sweeps)


def build_hierarchy(A, coarsening=None, smoother=None, max_levels=10, min_coarse_size=200,
                    coarse_solver="l1_jacobi", coarse_sweeps=30, setup=None):
    """Build levels until the coarse size or level cap is hit (amg.py:238-287).

    setup="device" (default when a GPU is present): the GPU setup of
    dsetup.py -- levels stay on the device (their host views download on
    demand).  setup="host": the native C++ host restatement (csrc/setup.cpp).
    Both are bitwise the reference's hierarchy.
    """
    coarsening = coarsening or CoarseningConfig()
    smoother = smoother or PolySmootherConfig(family="opt_cheb1", degree=4)
    if setup is None:
        setup = "device" if _gpu_present() else "host"
    if setup == "host":
        from . import setup as _setup

        return _setup.build_hierarchy(A, coarsening, smoother, max_levels, min_coarse_size,
                                      coarse_solver, coarse_sweeps)
    if setup != "device":
        raise ValueError(f"unknown setup {setup!r}")
    from . import dsetup

    dl, stagnated = dsetup.build_levels(A, coarsening, max_levels=max_levels,
                                        min_coarse_size=min_coarse_size)
    levels = []
    for L in dl:
        lv = Level(A=L.A, M=DeviceL1JacobiData(L.m), smoother=smoother, P=L.P,
                   n_aggregates=L.n_aggregates if L.P is not None else 0)
        lv._Pt = L.R
        levels.append(lv)
    return AmgHierarchy(levels=levels, coarse_solver=coarse_solver, coarse_sweeps=coarse_sweeps,
                        stagnated=stagnated)


def _gpu_present():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


class _TailView:
    """Levels _level.. of a hierarchy as a hierarchy of their own (a V-cycle
    started below the finest level, reference amg.py:303 with _level > 0)."""

    def __init__(self, h, level):
        self.levels = h.levels[level:]
        self.coarse_solver = h.coarse_solver
        self.coarse_sweeps = h.coarse_sweeps


def _device_hierarchy(h, level=0):
    """DeviceHierarchy of ours (h.device()) or of any object with the
    reference AmgHierarchy fields (levels of A, M, smoother, P and
    restrict_op(); coarse_solver, coarse_sweeps), built once and cached."""
    if level == 0 and isinstance(h, AmgHierarchy):
        return h.device()
    cache = getattr(h, "_b200_devs", None)
    if cache is None:
        cache = {}
        try:
            h._b200_devs = cache
        except AttributeError:
            pass
    if level not in cache:
        cache[level] = DeviceHierarchy(_TailView(h, level) if level else h)
    return cache[level]


def vcycle_spmv_count(h, level=0):
    """SpMVs one reference V-cycle performs from `level` (cost accounting of
    sparse.py:18-29): per level pre + post smoother degrees, residual,
    restriction, prolongation; coarse l1 sweeps (dense_direct: none)."""
    n = 0
    L = len(h.levels)
    for l in range(level, L - 1):
        n += 2 * h.levels[l].smoother.degree + 3
    if h.coarse_solver != "dense_direct":
        n += h.coarse_sweeps
    return n


def vcycle_apply(h, r, _level=0):
    """One symmetric V-cycle applied to a residual on the GPU; returns the
    correction (amg.py:303-315).  h: our hierarchy or the reference's."""
    n = r.shape[0] if hasattr(r, "shape") else len(r)
    if n != h.levels[_level].A.nrows:
        raise ValueError("dimension mismatch")
    D = _device_hierarchy(h, _level)
    c = D.ctx
    with c.scope():
        rd = N.to_device(r, c)
        z = N.empty(n, c)
        D.apply(rd, z)
    from .sparse import _count

    _count(vcycle_spmv_count(h, _level))
    return N.like(z, r)


class VcyclePreconditioner:
    """r -> V(r) (amg.py:318-319); ``krylov.solve`` runs it inside the device PCG."""

    def __init__(self, h):
        self.h = h

    def __call__(self, r):
        return vcycle_apply(self.h, r)


def as_vcycle_preconditioner(h):
    return VcyclePreconditioner(h)
