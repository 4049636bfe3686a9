"""Polynomial smoothers on the GPU (reference smoothers.py).

``smoother_apply`` keeps the reference signature (smoothers.py:92-137) and
returns bitwise the reference's iterate; the k degree steps run as k fused
sm_100a kernels (csrc/smoother.cu), each streaming the matrix once.

Error polynomial p of each family, M the l1-Jacobi diagonal:
  l1_jacobi   (1 - t)^k
  cheb4       W_k(1 - 2t)/(2k+1)
  opt_cheb4   sum_j (beta_j - beta_{j+1})/(2j+1) W_j(1 - 2t)
  opt_cheb1   tau_k^{[a,1]}(t)
"""

from __future__ import annotations

import logging
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .params import BetaTable, load_beta_tables, optimal_a
from .sparse import DeviceMatrix, _count, device_of

log = logging.getLogger(__name__)

FAMILIES = ("l1_jacobi", "cheb4", "opt_cheb4", "opt_cheb1")


@dataclass
class L1JacobiData:
    """Per-row diagonal M_i = a_ii + sum_{j != i} |a_ij| (host array or device tensor)."""

    m_diag: object
    _dev: object = None

    def device(self, c):
        if self._dev is None:
            self._dev = N.to_device(self.m_diag, c)
        return self._dev


class DeviceL1JacobiData(L1JacobiData):
    """l1 diagonal computed on the device (device setup levels): the device
    tensor is the working copy, ``m_diag`` a host view downloaded on demand
    (the reference's field is a numpy array)."""

    def __init__(self, dev):
        self._dev = dev
        self._host = None

    @property
    def m_diag(self):
        if self._host is None:
            self._host = N.to_host(self._dev)
        return self._host

    def device(self, c):
        return self._dev


def _reduceat_abs_rowsum(A):
    """scipy's |A|.sum(axis=1): numpy add.reduceat over each non-empty row."""
    out = np.zeros(A.nrows)
    lens = np.diff(A.row_ptr)
    nz = np.flatnonzero(lens)
    if len(nz):
        out[nz] = np.add.reduceat(np.abs(A.values), A.row_ptr[nz])
    return out


def l1_jacobi_diag(A):
    """l1-Jacobi diagonal of a square matrix with positive diagonal (smoothers.py:38-49).

    Host CSR: computed on the host with the reference's own reduction order
    (setup, not hot path).  DeviceMatrix: computed on the GPU in that order.
    """
    if hasattr(A, "l1_diag"):
        return L1JacobiData(m_diag=A.l1_diag())
    if A.nrows != A.ncols:
        raise ValueError("matrix must be square")
    diag = A.diagonal()
    if np.any(diag <= 0.0):
        raise ValueError("non-positive diagonal entry")
    abs_row = _reduceat_abs_rowsum(A)
    return L1JacobiData(m_diag=abs_row - np.abs(diag) + diag)


@dataclass
class PolySmootherConfig:
    """Family, degree, and the per-family parameters of a smoother (smoothers.py:52-85)."""

    family: str
    degree: int
    a: float | None = None
    beta: BetaTable | None = None
    rho_scale: float = 1.0

    def __post_init__(self):
        if self.family not in FAMILIES:
            raise ValueError(f"unknown smoother family {self.family!r}")
        if self.degree < 1:
            raise ValueError("degree must be >= 1")
        if self.rho_scale <= 0.0:
            raise ValueError("rho_scale must be positive")
        if self.family == "opt_cheb1":
            if self.a is None:
                self.a = optimal_a(self.degree)
            if not 0.0 < self.a < 1.0:
                raise ValueError("a must lie in (0, 1)")
        if self.family == "opt_cheb4" and self.beta is None:
            tables = load_beta_tables()
            if self.degree in tables:
                self.beta = tables[self.degree]
            else:
                log.warning("no beta table for degree %d; falling back to plain cheb4",
                            self.degree)
                self.family = "cheb4"
        if self.beta is not None and len(self.beta.beta) != self.degree:
            raise ValueError("beta table length must equal the degree")


def _m_device(M, c):
    """Device copy of an l1 diagonal: ours, or any object with an m_diag field
    (the reference's L1JacobiData), uploaded once and cached on it."""
    if hasattr(M, "device"):
        return M.device(c)
    d = getattr(M, "_b200_m", None)
    if d is None:
        d = N.to_device(M.m_diag, c)
        M._b200_m = d
    return d


def smoother_apply(config, A, M, b, x0):
    """One degree-k smoother application on the GPU; returns the updated iterate.

    Exactly k SpMVs are counted (the x0 == 0 SpMV is skipped on the device,
    which is bitwise-neutral).  b and x0 are not modified.  Inputs may be
    numpy arrays (result is numpy) or CUDA tensors (result is a tensor).
    """
    D = device_of(A)
    nb = b.shape[0] if hasattr(b, "shape") else len(b)
    nx = x0.shape[0] if hasattr(x0, "shape") else len(x0)
    if nb != nx or nb != D.nrows:
        raise ValueError("dimension mismatch")
    c = D.ctx
    cfg = N.smoother_cfg(config)
    zero_x0 = _is_zero_host(x0)
    with c.scope():
        bd = N.to_device(b, c)
        xd = None if zero_x0 else N.to_device(x0, c)
        md = _m_device(M, c)
        out = N.empty(D.nrows, c)
        N.check(N.lib().amgp_smoother_apply(c.handle, D.handle, N.ptr(md), C_byref(cfg),
                                            N.ptr(bd), N.ptr(xd) if xd is not None else None,
                                            N.ptr(out)))
    _count(config.degree)
    return N.like(out, b)


def _host_ptr(a):
    """(ctypes pointer, keep-alive) of a host float64 vector (numpy or CPU tensor)."""
    if N.is_torch(a):
        if a.is_cuda or a.dtype != _torch_f64() or not a.is_contiguous():
            raise TypeError("smoother_apply_batch: host float64 contiguous vectors expected")
        return N._VP(a.data_ptr()), a
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return N._VP(arr.ctypes.data), arr


def _torch_f64():
    import torch

    return torch.float64


def smoother_apply_batch(configs, A, M, bs, x0s, out=None):
    """``smoother_apply`` for a batch of independent host-side problems
    (configs[i], bs[i], x0s[i]) -> list of new host vectors, in one library
    call (amgp_smoother_apply_host): the uploads, kernels and downloads of
    consecutive applications overlap.  Each result equals
    ``smoother_apply(configs[i], A, M, bs[i], x0s[i])`` bit for bit.  Pinned
    torch inputs get pinned outputs (asynchronous DMA); numpy in, numpy out.
    ``out``: optional preallocated outputs (same container types)."""
    import ctypes

    D = device_of(A)
    k = len(configs)
    if not (len(bs) == len(x0s) == k) or (out is not None and len(out) != k):
        raise ValueError("smoother_apply_batch: configs, bs, x0s (and out) must have equal lengths")
    n = D.nrows
    keep, bp, xp, op = [], [], [], []
    outs = []
    for i in range(k):
        nb = bs[i].shape[0] if hasattr(bs[i], "shape") else len(bs[i])
        nx = x0s[i].shape[0] if hasattr(x0s[i], "shape") else len(x0s[i])
        if nb != nx or nb != n:
            raise ValueError("dimension mismatch")
        p, ref = _host_ptr(bs[i])
        keep.append(ref)
        bp.append(p)
        if _is_zero_host(x0s[i]):
            xp.append(None)
        else:
            p, ref = _host_ptr(x0s[i])
            keep.append(ref)
            xp.append(p)
        if out is not None:
            o = out[i]
        elif N.is_torch(bs[i]):
            import torch

            o = torch.empty(n, dtype=torch.float64, pin_memory=bs[i].is_pinned())
        else:
            o = np.empty(n)
        p, ref = _host_ptr(o)
        if ref is not o:
            raise TypeError("smoother_apply_batch: outputs must be contiguous float64 host vectors")
        op.append(p)
        outs.append(o)
    cfgs = [N.smoother_cfg(cfg) for cfg in configs]
    carr = (N.SmootherCfg * max(k, 1))(*cfgs)
    c = D.ctx
    with c.scope():
        md = _m_device(M, c)
        N.check(N.lib().amgp_smoother_apply_host(c.handle, D.handle, N.ptr(md), k, carr,
                                                 (N._VP * max(k, 1))(*bp), (N._VP * max(k, 1))(*xp),
                                                 (N._VP * max(k, 1))(*op)))
    _count(sum(int(cfg.degree) for cfg in configs))
    del keep, ctypes
    return outs


def C_byref(cfg):
    import ctypes

    return ctypes.byref(cfg)


def _is_zero_host(x0):
    """A host all-zero x0 is passed as NULL (skips the upload and one SpMV)."""
    if N.is_torch(x0):
        return False
    a = np.asarray(x0)
    return a.size == 0 or not np.any(a) and not np.any(np.signbit(a))


def smoother_error_apply(config, A, M, e0):
    """Error propagator action via the runtime kernel: G e0 with b = 0 (smoothers.py:188-190)."""
    if N.is_torch(e0):
        return smoother_apply(config, A, M, e0.new_zeros(e0.shape), e0)
    return smoother_apply(config, A, M, np.zeros_like(e0), e0)


class SmootherPreconditioner:
    """The smoother as a linear operator r -> S(r, 0) (smoothers.py:193-199).

    Callable like the reference's closure; ``krylov.solve`` recognises it and
    keeps the whole solve on the device.
    """

    def __init__(self, config, A, M):
        self.config, self.A, self.M = config, A, M

    def __call__(self, r):
        zeros = r.new_zeros(r.shape) if N.is_torch(r) else np.zeros_like(r)
        return smoother_apply(self.config, self.A, self.M, r, zeros)


def as_preconditioner(config, A, M):
    return SmootherPreconditioner(config, A, M)
