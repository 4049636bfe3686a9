#!/usr/bin/env python
"""Per-level SpMV timing of an AMG hierarchy (graph-captured loops).

    python tools/level_spmv.py --m 128 [--reps 200]

For every level's A, P and R: rows, nnz, widest row, the schedule the
library picks, microseconds per SpMV (CUDA graph of `reps` launches, timed
with events on the library stream) and the algorithmic bandwidth
12 nnz + 4 (rows+1) + 8 rows (y) + 8 cols (x read once).  Run it with
AMGP_LIB=<variant.so> to compare kernel variants on the same hierarchy.
"""

import argparse
import ctypes
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=128)
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--kind", default="smoothed_aggregation")
    args = ap.parse_args()
    import torch

    import paper_2407_09848_b200 as P
    from paper_2407_09848_b200 import _native as N
    from paper_2407_09848_b200.sparse import DeviceMatrix

    A, _ = P.poisson3d(args.m)
    h = P.build_hierarchy(A, coarsening=P.CoarseningConfig(kind=args.kind),
                          smoother=P.PolySmootherConfig(family="opt_cheb1", degree=4))
    c = N.ctx()
    lib = os.environ.get("AMGP_LIB", "default")
    total = 0.0
    for l, lv in enumerate(h.levels):
        mats = [("A", lv.A)]
        if lv.P is not None:
            mats += [("P", lv.P), ("R", lv.restrict_op())]
        for name, M in mats:
            D = DeviceMatrix.from_csr(M, c)
            x = torch.randn(M.ncols, dtype=torch.float64, device="cuda")
            y = torch.empty(M.nrows, dtype=torch.float64, device="cuda")
            ms = ctypes.c_double()
            with c.scope():
                N.check(N.lib().amgp_spmv_timed(c.handle, D.handle, N.ptr(x), N.ptr(y), args.reps, 1,
                                                ctypes.byref(ms)))
            us = ms.value * 1e3
            width = int(np.diff(M.row_ptr).max()) if M.nrows else 0
            nbytes = 12 * M.nnz + 4 * (M.nrows + 1) + 8 * M.nrows + 8 * M.ncols
            total += us
            print(json.dumps({"lib": os.path.basename(lib), "m": args.m, "level": l, "mat": name,
                              "rows": M.nrows, "nnz": M.nnz, "max_width": width,
                              "slices": (M.nrows + 31) // 32, "us": round(us, 2),
                              "GBps": round(nbytes / us / 1e3, 1)}), flush=True)
    print(json.dumps({"lib": os.path.basename(lib), "m": args.m, "sum_us": round(total, 1)}), flush=True)


if __name__ == "__main__":
    main()
