#!/usr/bin/env python
"""One PCG + AMG solve on poisson3d(m) through the public API (profiling aid).

    python tools/run_solve.py --m 128 --kind smoothed_aggregation --family opt_cheb1 --k 4
"""

import argparse
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=64)
    ap.add_argument("--stencil", type=int, default=7, choices=[7, 27])
    ap.add_argument("--kind", default="smoothed_aggregation")
    ap.add_argument("--family", default="opt_cheb1")
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--repeat", type=int, default=2)
    ap.add_argument("--no-graph", action="store_true")
    args = ap.parse_args()
    import torch

    import paper_2407_09848_b200 as P
    from paper_2407_09848_b200 import _native as N

    A = P.poisson3d_device(args.m, args.stencil)
    t0 = time.perf_counter()
    h = P.build_hierarchy(A, coarsening=P.CoarseningConfig(kind=args.kind),
                          smoother=P.PolySmootherConfig(family=args.family, degree=args.k))
    setup = time.perf_counter() - t0
    D = h.device()
    if args.no_graph:
        D.use_graph(False)
    bd = torch.ones(A.nrows, dtype=torch.float64, device="cuda")
    for i in range(args.repeat):
        x, rep = P.solve(A, bd, precond=P.as_vcycle_preconditioner(h), cfg=P.KrylovConfig(tol=1e-6))
        torch.cuda.synchronize()
        print(f"m={args.m} {args.stencil}-pt {args.kind} {args.family} k={args.k}: setup {setup:.2f}s "
              f"iters {rep.iterations} relres {rep.final_relres:.3e} solve {rep.elapsed_s * 1e3:.2f} ms "
              f"levels {[lv.A.nrows for lv in h.levels]}", flush=True)


if __name__ == "__main__":
    main()
