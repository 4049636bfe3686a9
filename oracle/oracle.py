"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the C oracle.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module; the product package never
does.  Function-by-function correspondence with the reference is documented
in amgp_oracle.c; the restatement is pinned against the reference's own
outputs by tests/test_oracle.py (golden fixtures from tests/golden/).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

FAMILY_CODES = {"l1_jacobi": 0, "cheb4": 1, "opt_cheb4": 2, "opt_cheb1": 3}

_lib = None

_P64 = C.POINTER(C.c_int64)
_PD = C.POINTER(C.c_double)


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(
            os.path.join(HERE, "amgp_oracle.c")
        ):
            build()
        _lib = C.CDLL(LIB_PATH)
        _lib.oracle_pcg.restype = C.c_int
    return _lib


class _Hier(C.Structure):
    _fields_ = [
        ("nlev", C.c_int),
        ("n", _P64),
        ("A_rp", C.POINTER(_P64)), ("A_ci", C.POINTER(_P64)), ("A_v", C.POINTER(_PD)),
        ("m", C.POINTER(_PD)),
        ("P_rp", C.POINTER(_P64)), ("P_ci", C.POINTER(_P64)), ("P_v", C.POINTER(_PD)),
        ("R_rp", C.POINTER(_P64)), ("R_ci", C.POINTER(_P64)), ("R_v", C.POINTER(_PD)),
        ("family", C.c_int), ("k", C.c_int), ("a", C.c_double), ("rho", C.c_double),
        ("beta", _PD),
        ("coarse_sweeps", C.c_int),
    ]


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return a.ctypes.data_as(_PD if a.dtype == np.float64 else _P64)


def set_threads(t):
    lib().oracle_set_threads(C.c_int(int(t)))


def max_threads():
    return int(lib().oracle_max_threads())


def spmv(rp, ci, v, ncols, x):
    rp, ci, v, x = _i64(rp), _i64(ci), _f64(v), _f64(x)
    n = len(rp) - 1
    y = np.empty(n)
    lib().oracle_spmv(C.c_int64(n), C.c_int64(ncols), _p(rp), _p(ci), _p(v), _p(x), _p(y))
    return y


def fused_update(rho, rho_prev, c, s, r, d, x):
    for a in (s, r, d, x):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    lib().oracle_fused_update(C.c_int64(len(r)), C.c_double(rho), C.c_double(rho_prev),
                              C.c_double(c), _p(s), _p(r), _p(d), _p(x))


def smoother_apply(family, k, rp, ci, v, m, b, x0=None, a=0.0, rho=1.0, beta=None):
    rp, ci, v, m, b = _i64(rp), _i64(ci), _f64(v), _f64(m), _f64(b)
    n = len(b)
    out = np.empty(n)
    x0a = None if x0 is None else _f64(x0)
    beta_a = None if beta is None else _f64(beta)
    st = lib().oracle_smoother_apply(
        C.c_int(FAMILY_CODES[family]), C.c_int(k), C.c_double(a), C.c_double(rho),
        _p(beta_a) if beta_a is not None else None,
        C.c_int64(n), _p(rp), _p(ci), _p(v), _p(m), _p(b),
        _p(x0a) if x0a is not None else None, _p(out))
    if st != 0:
        raise RuntimeError(f"oracle_smoother_apply failed ({st})")
    return out


class Hierarchy:
    """Plain-array hierarchy for the oracle V-cycle.

    levels: list of dicts with A=(rp, ci, v), m, and (except the last)
    P=(rp, ci, v) and R=(rp, ci, v).
    """

    def __init__(self, levels, family, k, a=0.0, rho=1.0, beta=None, coarse_sweeps=30):
        self._keep = []
        L = len(levels)
        self.n = _i64([len(lv["m"]) for lv in levels])
        self.family, self.k, self.a, self.rho = family, k, a, rho
        self.beta = None if beta is None else _f64(beta)

        def arr(kind, key, idx):
            ptrs = []
            for lv in levels:
                if key in lv and lv[key] is not None:
                    val = lv[key][idx] if idx is not None else lv[key]
                    val = _f64(val) if kind == "f" else _i64(val)
                    self._keep.append(val)
                    ptrs.append(_p(val))
                else:
                    ptrs.append(None)
            T = _PD if kind == "f" else _P64
            out = (T * L)(*ptrs)
            self._keep.append(out)
            return out

        h = _Hier()
        h.nlev = L
        h.n = _p(self.n)
        h.A_rp, h.A_ci, h.A_v = arr("i", "A", 0), arr("i", "A", 1), arr("f", "A", 2)
        h.m = arr("f", "m", None)
        h.P_rp, h.P_ci, h.P_v = arr("i", "P", 0), arr("i", "P", 1), arr("f", "P", 2)
        h.R_rp, h.R_ci, h.R_v = arr("i", "R", 0), arr("i", "R", 1), arr("f", "R", 2)
        h.family = FAMILY_CODES[family]
        h.k, h.a, h.rho = k, a, rho
        h.beta = _p(self.beta) if self.beta is not None else None
        h.coarse_sweeps = coarse_sweeps
        self.h = h
        self.A0 = levels[0]["A"]

    def vcycle(self, r):
        r = _f64(r)
        z = np.empty_like(r)
        st = lib().oracle_vcycle_apply(C.byref(self.h), _p(r), _p(z))
        if st != 0:
            raise RuntimeError("oracle_vcycle_apply failed")
        return z


def pcg(A, b, hier=None, x0=None, fcg=False, tol=1e-7, itmax=1000):
    """Returns (x, iterations, final_relres, converged, breakdown, history)."""
    rp, ci, v = (_i64(A[0]), _i64(A[1]), _f64(A[2]))
    b = _f64(b)
    n = len(b)
    x = np.zeros(n) if x0 is None else _f64(x0).copy()
    hist = np.empty(itmax + 1)
    nh = C.c_int(0)
    fr = C.c_double(0.0)
    flags = C.c_int(0)
    it = lib().oracle_pcg(C.byref(hier.h) if hier is not None else None, C.c_int64(n),
                          _p(rp), _p(ci), _p(v), _p(b), _p(x), C.c_int(x0 is not None),
                          C.c_int(int(fcg)), C.c_double(tol), C.c_int(itmax), C.byref(fr),
                          C.byref(flags), _p(hist), C.byref(nh))
    return x, it, fr.value, bool(flags.value & 1), bool(flags.value & 2), hist[: nh.value]
