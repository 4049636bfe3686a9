#!/usr/bin/env python
"""Per-level SpMV rates of a device hierarchy + whole-solve time (GPU box).

    python tools/level_bench.py --m 128 [--reps 50]

Each SpMV (A_l, R_l = P_l^T, P_l) is launched REPS times back to back on
the library stream and timed with CUDA events (L2-warm, as inside a
V-cycle; launch gaps included); GB/s = (12 nnz + 4 (n+1) + 8 ncols + 8 nrows) / time.  Then the
PCG solve (opt_cheb1 k=4, rtol 1e-6), median of 5.  Schedule experiments:
library variants via AMGP_LIB (tools/ab_solve.py for A/B).
"""
import argparse
import json
import os
import statistics
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=128)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--kind", default="smoothed_aggregation")
    args = ap.parse_args()
    import torch

    import paper_2407_09848_b200 as P
    from paper_2407_09848_b200 import _native as N

    D0 = P.poisson3d_device(args.m)
    h = P.build_hierarchy(D0, coarsening=P.CoarseningConfig(kind=args.kind),
                          smoother=P.PolySmootherConfig(family="opt_cheb1", degree=4))
    c = D0.ctx
    out = {"m": args.m, "rows_variant": os.environ.get("AMGP_ROWS", "0"), "levels": []}

    def time_spmv(M):
        x = torch.randn(M.ncols, dtype=torch.float64, device="cuda")
        y = torch.empty(M.nrows, dtype=torch.float64, device="cuda")
        with c.scope():
            N.check(N.lib().amgp_spmv(c.handle, M.handle, N.ptr(x), N.ptr(y)))
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with c.scope():
                e0.record(c.stream)
                for _ in range(args.reps):
                    N.check(N.lib().amgp_spmv(c.handle, M.handle, N.ptr(x), N.ptr(y)))
                e1.record(c.stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / args.reps)
        t = min(ts)
        byts = 12 * M.nnz + 4 * (M.nrows + 1) + 8 * M.ncols + 8 * M.nrows
        info = M.info()
        return {"us": t * 1e3, "GBs": byts / (t * 1e-3) / 1e9, "nrows": M.nrows, "nnz": M.nnz,
                "slices": (M.nrows + 31) // 32, "stored": info["stored"]}

    for l, lv in enumerate(h.levels):
        ent = {"level": l, "A": time_spmv(lv.A)}
        if lv.P is not None:
            ent["R"] = time_spmv(lv.restrict_op())
            ent["P"] = time_spmv(lv.P)
        out["levels"].append(ent)
    b = torch.ones(D0.nrows, dtype=torch.float64, device="cuda")
    pre = P.as_vcycle_preconditioner(h)
    P.solve(D0, b, precond=pre, cfg=P.KrylovConfig(tol=1e-6))
    ts, its = [], None
    for _ in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(c.stream)
        _, rep = P.solve(D0, b, precond=pre, cfg=P.KrylovConfig(tol=1e-6))
        e1.record(c.stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
        its = rep.iterations
    out["solve_ms"] = statistics.median(ts)
    out["iterations"] = its
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
