"""Benchmark matrices: 3D Poisson, 7- and 27-point (reference problems.py:32-60).

``poisson3d`` builds the reference's host CSR directly (no COO triplets, so
no O(7n) int64 temporaries beyond the result) and is array-equal to the
reference's.  ``poisson3d_device`` generates the SELL matrix on the GPU for
sizes where a host CSR is impractical (512^3: 938M entries).
The 27-point stencil is not in the reference; its convention here is the
7-point one extended: unscaled, Dirichlet rows eliminated, x-fastest,
diagonal 26 and -1 for each of the 26 neighbours, b = 1.
"""

from __future__ import annotations

import numpy as np

from .sparse import CsrMatrix, DeviceMatrix


def _stencil_csr(m, offsets, diag):
    n = m ** 3
    idx = np.arange(n, dtype=np.int64)
    ix, iy, iz = idx % m, (idx // m) % m, idx // (m * m)
    cols, vals, masks = [], [], []
    for dx, dy, dz in offsets:  # offsets sorted by column delta
        ok = np.ones(n, dtype=bool)
        for comp, dd in ((ix, dx), (iy, dy), (iz, dz)):
            if dd < 0:
                ok &= comp > 0
            elif dd > 0:
                ok &= comp < m - 1
        masks.append(ok)
        cols.append(idx + dx + dy * m + dz * m * m)
        vals.append(diag if (dx, dy, dz) == (0, 0, 0) else -1.0)
    mask = np.stack(masks, axis=1)                      # (n, s) row-major: row, then column order
    col = np.stack(cols, axis=1)[mask]
    val = np.broadcast_to(np.array(vals), mask.shape)[mask].astype(np.float64)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(mask.sum(axis=1), out=row_ptr[1:])
    return CsrMatrix(n, n, row_ptr, col, val)


def poisson3d(m):
    """7-point Poisson on the unit cube (diagonal 6, -1 per neighbour) and b = 1."""
    if m < 2:
        raise ValueError("m must be >= 2")
    offs = [(0, 0, -1), (0, -1, 0), (-1, 0, 0), (0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]
    return _stencil_csr(m, offs, 6.0), np.ones(m ** 3)


def poisson3d_27(m):
    """27-point Poisson (diagonal 26, -1 per neighbour) and b = 1."""
    if m < 2:
        raise ValueError("m must be >= 2")
    offs = [(dx, dy, dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
    return _stencil_csr(m, offs, 26.0), np.ones(m ** 3)


def poisson3d_device(m, stencil=7, row_begin=0, row_end=None):
    """Rows [row_begin, row_end) of the m^3 Poisson matrix generated on the GPU."""
    if m < 2:
        raise ValueError("m must be >= 2")
    return DeviceMatrix.poisson3d(m, stencil, row_begin, row_end)
