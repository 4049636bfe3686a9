"""Smoother parameter tables (host constants).

The optimal interval ends a*_k (k = 1..20) and the optimized fourth-kind
beta tables (k = 1..12) are the reference's shipped data assets
(pkg/src/amgpoly/data/{optimal_params,beta_tables}.csv, loaded by
optimize.py:278-318).  They are offline results, not hot-path work; this
module serves them from data/smoother_params.json (exported bit-exactly by
tests/golden/make_golden.py).
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np

_DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "smoother_params.json")
_cache = None


@dataclass
class BetaTable:
    """Optimized fourth-kind weights for one degree (reference optimize.py BetaTable)."""

    k: int
    beta: np.ndarray
    gamma_value: float


def _load():
    global _cache
    if _cache is None:
        with open(_DATA) as f:
            _cache = json.load(f)
    return _cache


def load_beta_tables():
    """BetaTable records keyed by degree (reference optimize.py:299-310)."""
    d = _load()
    return {
        int(k): BetaTable(k=int(k), beta=np.array(v, dtype=np.float64),
                          gamma_value=float(d["beta_gamma"][k]))
        for k, v in d["beta"].items()
    }


def _phi(k, x):
    """Root function of a*_k (reference optimize.py:50-57): the equi-oscillation
    condition 8k(1-x^2)^{2k} + x[(1-x)^{4k} - (1+x)^{4k}], divided through by
    (1+x)^{4k} so it stays in range for large k."""
    t = (1.0 - x) / (1.0 + x)
    return 8.0 * k * t ** (2 * k) + x * (t ** (4 * k) - 1.0)


_EPS = 2.220446049250313e-16  # binary64 machine epsilon (np.finfo(float).eps)


def _brent(f, lo, hi, xtol=1e-15, maxiter=200):
    """Brent's bracketed root finder (bisection / secant / inverse quadratic
    interpolation), stepping exactly as reference optimize.py:60-103 does so
    that a*_k comes out with the same bits."""
    fa, fb = f(lo), f(hi)
    if fa * fb > 0.0:
        raise ValueError("root is not bracketed")
    if fa == 0.0:
        return lo
    if fb == 0.0:
        return hi
    a, b = lo, hi
    c, fc = a, fa
    step = prev = b - a
    it = 0
    while it < maxiter:
        it += 1
        if fb * fc > 0.0:  # keep the root between b and c
            c, fc = a, fa
            step = prev = b - a
        if abs(fc) < abs(fb):  # b is the best estimate
            a, fa = b, fb
            b, fb = c, fc
            c, fc = a, fa
        tol = 2.0 * _EPS * abs(b) + 0.5 * xtol
        half = 0.5 * (c - b)
        if abs(half) <= tol or fb == 0.0:
            return b
        bisect = abs(prev) < tol or abs(fa) <= abs(fb)
        if not bisect:
            s = fb / fa
            if a == c:  # secant
                p, q = 2.0 * half * s, 1.0 - s
            else:  # inverse quadratic interpolation
                q, r = fa / fc, fb / fc
                p = s * (2.0 * half * q * (q - r) - (b - a) * (r - 1.0))
                q = (q - 1.0) * (r - 1.0) * (s - 1.0)
            if p > 0.0:
                q = -q
            p = abs(p)
            if 2.0 * p < min(3.0 * half * q - abs(tol * q), abs(prev * q)):
                prev, step = step, p / q
            else:
                bisect = True
        if bisect:
            step = prev = half
        a, fa = b, fb
        b = b + (step if abs(step) > tol else (tol if half > 0 else -tol))
        fb = f(b)
    return b


def solve_a_star(k):
    """a*_k = square of the unique root of phi_k in (0, 1) (reference
    optimize.py:106-111); reproduces the shipped table bit for bit."""
    if k < 1:
        raise ValueError("degree must be >= 1")
    x = _brent(lambda x: _phi(k, x), 1e-8, 1.0 - 1e-8)
    return x * x


def optimal_a(k):
    """a*_k from the shipped table when available, else solved on demand
    (reference optimize.py:313-318)."""
    d = _load()["a_star"]
    if str(k) in d:
        return float(d[str(k)])
    return solve_a_star(k)
