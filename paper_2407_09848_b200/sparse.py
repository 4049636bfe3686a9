"""Sparse storage and the device SpMV / fused update (reference sparse.py).

``CsrMatrix`` keeps the reference's host container and invariants
(sparse.py:32-115) so a hierarchy built on the host drops straight in; its
device image is a ``DeviceMatrix`` (SELL-32 on the GPU, created on first use
and cached on the object like the reference caches ``_scipy``,
sparse.py:41,87-92).  ``spmv`` and ``fused_update`` run on the GPU
(csrc/matrix.cu, csrc/smoother.cu) and return bitwise the reference's values.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse

from . import _native as N

# Global SpMV counter (reference sparse.py:18-29): one degree-k smoother
# application counts k, exactly as k plain sweeps do.
_spmv_calls = 0


def spmv_count():
    return _spmv_calls


def reset_spmv_count():
    global _spmv_calls
    _spmv_calls = 0


def _count(k=1):
    global _spmv_calls
    _spmv_calls += k


# ---------------------------------------------------------------- device matrix
class DeviceMatrix:
    """A matrix resident on the GPU in SELL-32 layout (owned by libamgp)."""

    def __init__(self, handle, c, nrows, ncols, nnz, row_offset=0):
        self.handle = handle
        self.ctx = c
        self.nrows = int(nrows)
        self.ncols = int(ncols)
        self.nnz = int(nnz)
        self.row_offset = int(row_offset)
        self._m = None
        self._host = None

    @classmethod
    def from_csr(cls, A, c=None):
        c = c or N.ctx()
        rp = np.ascontiguousarray(A.row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(A.col_idx, dtype=np.int64)
        v = np.ascontiguousarray(A.values, dtype=np.float64)
        h = N._VP()
        with c.scope():
            N.check(N.lib().amgp_mat_from_csr(
                c.handle, A.nrows, A.ncols, rp.ctypes.data_as(N._P64), ci.ctypes.data_as(N._P64),
                v.ctypes.data_as(N._PD), C.byref(h)))
        return cls(h, c, A.nrows, A.ncols, len(v))

    @classmethod
    def poisson3d(cls, m, stencil=7, row_begin=0, row_end=None, c=None):
        """Rows [row_begin, row_end) of the m^3 Poisson matrix, generated on the GPU
        (reference problems.py:32-60 conventions; 27-point: diagonal 26)."""
        c = c or N.ctx()
        n = m ** 3
        row_end = n if row_end is None else row_end
        h = N._VP()
        with c.scope():
            N.check(N.lib().amgp_mat_poisson3d(c.handle, int(m), int(stencil), int(row_begin),
                                               int(row_end), C.byref(h)))
        A = cls(h, c, row_end - row_begin, n, 0, row_offset=row_begin)
        A.nnz = A.info()["nnz"]
        return A

    def info(self):
        vals = [C.c_int64(0) for _ in range(5)]
        N.check(N.lib().amgp_mat_info(self.handle, *[C.byref(v) for v in vals]))
        keys = ("nrows", "ncols", "nnz", "stored", "bytes")
        return {k: v.value for k, v in zip(keys, vals)}

    def to_csr(self):
        rp = np.empty(self.nrows + 1, dtype=np.int64)
        ci = np.empty(self.nnz, dtype=np.int64)
        v = np.empty(self.nnz, dtype=np.float64)
        with self.ctx.scope():
            N.check(N.lib().amgp_mat_to_csr(self.handle, rp.ctypes.data_as(N._P64),
                                            ci.ctypes.data_as(N._P64), v.ctypes.data_as(N._PD)))
        return CsrMatrix(self.nrows, self.ncols, rp, ci, v)

    # -- host views (reference CsrMatrix fields; downloaded once, on demand)
    def host(self):
        """The matrix as a host CsrMatrix (local columns), cached."""
        if getattr(self, "_host", None) is None:
            self._host = self.to_csr()
        return self._host

    @property
    def row_ptr(self):
        return self.host().row_ptr

    @property
    def col_idx(self):
        return self.host().col_idx

    @property
    def values(self):
        return self.host().values

    def to_scipy(self):
        return self.host().to_scipy()

    def to_dense(self):
        return self.host().to_dense()

    def diagonal(self):
        return self.host().diagonal()

    def transpose(self):
        return self.host().transpose()

    def l1_diag(self):
        """Device l1-Jacobi diagonal (reference smoothers.py:38-49, same bits)."""
        if self._m is None:
            with self.ctx.scope():
                m = N.empty(self.nrows, self.ctx)
                N.check(N.lib().amgp_mat_l1_diag(self.handle, N.ptr(m)))
            self._m = m
        return self._m

    def matvec(self, x):
        return spmv(self, x)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and N._lib is not None:
            try:
                N.lib().amgp_mat_destroy(h)
            except Exception:
                pass
            self.handle = None


# ---------------------------------------------------------------- host container
@dataclass
class CsrMatrix:
    """Compressed sparse row matrix with sorted, duplicate-free columns.

    Host container of reference sparse.py:32-115 (same fields, constructors and
    validation); ``device()`` is its GPU image.
    """

    nrows: int
    ncols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray
    _dev: DeviceMatrix | None = field(default=None, repr=False, compare=False)
    _sp: object = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        self.row_ptr = np.asarray(self.row_ptr, dtype=np.int64)
        self.col_idx = np.asarray(self.col_idx, dtype=np.int64)
        self.values = np.asarray(self.values, dtype=np.float64)
        if self.row_ptr.shape != (self.nrows + 1,):
            raise ValueError("row_ptr must have length nrows+1")
        if self.row_ptr[0] != 0 or self.row_ptr[-1] != len(self.values):
            raise ValueError("row_ptr endpoints inconsistent with values")
        if np.any(self.row_ptr[1:] < self.row_ptr[:-1]):
            raise ValueError("row_ptr must be nondecreasing")
        if len(self.col_idx) != len(self.values):
            raise ValueError("col_idx and values length mismatch")

    # -- constructors (host assembly; scipy canonicalises exactly as the
    #    reference's from_coo / from_scipy do, sparse.py:58-75)
    @classmethod
    def from_scipy(cls, m):
        m = scipy.sparse.csr_matrix(m, copy=True)
        m.sum_duplicates()
        m.eliminate_zeros()
        m.sort_indices()
        return cls(m.shape[0], m.shape[1], m.indptr, m.indices, m.data)

    @classmethod
    def from_coo(cls, nrows, ncols, rows, cols, vals):
        m = scipy.sparse.coo_matrix(
            (np.asarray(vals, dtype=np.float64), (rows, cols)), shape=(nrows, ncols)).tocsr()
        return cls.from_scipy(m)

    @classmethod
    def from_dense(cls, a):
        return cls.from_scipy(scipy.sparse.csr_matrix(np.asarray(a, dtype=np.float64)))

    @classmethod
    def identity(cls, n):
        return cls(n, n, np.arange(n + 1), np.arange(n), np.ones(n))

    # -- views
    def to_scipy(self):
        if self._sp is None:
            self._sp = scipy.sparse.csr_matrix(
                (self.values, self.col_idx, self.row_ptr), shape=(self.nrows, self.ncols))
        return self._sp

    def to_dense(self):
        out = np.zeros((self.nrows, self.ncols))
        rows = np.repeat(np.arange(self.nrows), np.diff(self.row_ptr))
        out[rows, self.col_idx] = self.values
        return out

    def transpose(self):
        """Explicit CSR of A^T with sorted columns (reference sparse.py:97-98)."""
        order = np.lexsort((np.repeat(np.arange(self.nrows), np.diff(self.row_ptr)), self.col_idx))
        rows_t = self.col_idx[order]
        cols_t = np.repeat(np.arange(self.nrows), np.diff(self.row_ptr))[order]
        rp = np.zeros(self.ncols + 1, dtype=np.int64)
        np.add.at(rp, rows_t + 1, 1)
        return CsrMatrix(self.ncols, self.nrows, np.cumsum(rp), cols_t, self.values[order])

    def diagonal(self):
        d = np.zeros(min(self.nrows, self.ncols))
        rows = np.repeat(np.arange(self.nrows), np.diff(self.row_ptr))
        on = rows == self.col_idx
        d[rows[on]] = self.values[on]
        return d

    @property
    def nnz(self):
        return len(self.values)

    def device(self):
        """GPU image (uploaded once, cached)."""
        if self._dev is None:
            self._dev = DeviceMatrix.from_csr(self)
        return self._dev

    def matvec(self, x):
        return spmv(self, x)

    def is_symmetric(self, rtol=1e-13):
        if self.nrows != self.ncols:
            return False
        d = self.to_scipy() - self.to_scipy().T
        scale = max(np.max(np.abs(self.values)), 1.0) if self.nnz else 1.0
        return d.nnz == 0 or np.max(np.abs(d.data)) <= rtol * scale


def _csr_like(A):
    return all(hasattr(A, k) for k in ("nrows", "ncols", "row_ptr", "col_idx", "values"))


def device_of(A):
    """DeviceMatrix of a CsrMatrix / DeviceMatrix, or of any object with the
    reference CsrMatrix fields (nrows, ncols, row_ptr, col_idx, values -- e.g.
    the reference's own CsrMatrix, sparse.py:32-56), uploaded once and cached
    on the object as the reference caches its scipy view (sparse.py:87-92).
    TypeError otherwise (the dense spectral operators are out of scope)."""
    if isinstance(A, DeviceMatrix):
        return A
    if isinstance(A, CsrMatrix):
        return A.device()
    if _csr_like(A):
        D = getattr(A, "_b200_dev", None)
        if D is None:
            D = DeviceMatrix.from_csr(A)
            A._b200_dev = D
        return D
    raise TypeError(f"device operator must be CsrMatrix or DeviceMatrix, got {type(A).__name__}")


def spmv(A, x):
    """y = A @ x on the GPU, accumulated in stored-entry order (sparse.py:118-125)."""
    D = device_of(A)
    n = x.shape[0] if hasattr(x, "shape") else len(x)
    if D.ncols != n:
        raise ValueError(f"dimension mismatch: A is {D.nrows}x{D.ncols}, x has {n}")
    _count()
    c = D.ctx
    with c.scope():
        xd = N.to_device(x, c)
        y = N.empty(D.nrows, c)
        N.check(N.lib().amgp_spmv(c.handle, D.handle, N.ptr(xd), N.ptr(y)))
    return N.like(y, x)


def fused_update(rho, rho_prev, two_rho_over_delta, s, r, d, x):
    """In place: r -= s; d = rho*rho_prev*d + c*r; x += d (sparse.py:128-139)."""
    if not (len(s) == len(r) == len(d) == len(x)):
        raise ValueError("fused_update: vector length mismatch")
    c = N.ctx()
    with c.scope():
        sd, rd, dd, xd = (N.to_device(v, c) for v in (s, r, d, x))
        N.check(N.lib().amgp_fused_update(c.handle, len(r), float(rho), float(rho_prev),
                                          float(two_rho_over_delta), N.ptr(sd), N.ptr(rd),
                                          N.ptr(dd), N.ptr(xd)))
    for host, dev in ((r, rd), (d, dd), (x, xd)):
        if N.is_torch(host):
            if dev.data_ptr() != host.data_ptr():
                host.copy_(dev)
        else:
            host[...] = N.to_host(dev)
