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


def optimal_a(k):
    """a*_k from the shipped table (reference optimize.py:313-318).

    Degrees beyond the table need the offline minimax solve, which is out of
    scope for this package: pass ``a`` explicitly for them.
    """
    d = _load()["a_star"]
    if str(k) in d:
        return float(d[str(k)])
    raise ValueError(f"no tabulated a*_k for degree {k}; pass PolySmootherConfig(a=...)")
