#!/usr/bin/env python
"""Every libamgp kernel family at small sizes, for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per run):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_smoke.py

smoother steps of all families (thread-per-row and split schedules), SpMV
epilogues, V-cycle (graph and eager, l1 / dense coarse), device PCG/FCG/PCG1
and the callable-preconditioner path (OpenBLAS-order TMA dot, axpys), the
pipelined host-buffer smoother path, and the device setup (strength,
lambda_max, prolongator, hash SpGEMM incl. its larger-table stages,
symmetrisation, SELL packing) on 7-/27-point and an arrow matrix with one
dense row.  Checks results against the host/oracle where cheap; exit 0."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))


def main():
    import numpy as np
    import torch

    import paper_2407_09848_b200 as P

    rng = np.random.default_rng(0)
    fams = ("l1_jacobi", "cheb4", "opt_cheb4", "opt_cheb1")
    for A in (P.poisson3d(10)[0], P.poisson3d_27(8)[0]):
        M = P.l1_jacobi_diag(A)
        b, x0 = rng.standard_normal(A.nrows), rng.standard_normal(A.nrows)
        for f in fams:
            for k in (1, 3):
                cfg = P.PolySmootherConfig(family=f, degree=k)
                y = P.smoother_apply(cfg, A, M, b, x0)
                y0 = P.smoother_apply(cfg, A, M, b, np.zeros(A.nrows))
                assert np.all(np.isfinite(y)) and np.all(np.isfinite(y0))
        outs = P.smoother_apply_batch([P.PolySmootherConfig(family="cheb4", degree=2)] * 3, A, M, [b] * 3, [x0] * 3)
        assert all(np.array_equal(o, outs[0]) for o in outs)
    # hierarchies from the device setup (7-pt SA / matching, 27-pt SA), V-cycles and solves
    for A, kind in ((P.poisson3d(16)[0], "smoothed_aggregation"), (P.poisson3d(12)[0], "pairwise_matching"),
                    (P.poisson3d_27(12)[0], "smoothed_aggregation")):
        h = P.build_hierarchy(A, coarsening=P.CoarseningConfig(kind=kind), setup="device")
        hh = P.build_hierarchy(A, coarsening=P.CoarseningConfig(kind=kind), setup="host")
        for lv, lh in zip(h.levels, hh.levels):
            assert np.array_equal(lv.A.values, lh.A.values)
        r = rng.standard_normal(A.nrows)
        for f in fams:
            for lv in h.levels:
                lv.smoother = P.PolySmootherConfig(family=f, degree=2)
            z = P.vcycle_apply(h, r)
            assert np.all(np.isfinite(z))
        D = h.device()
        D.use_graph(False)
        assert np.array_equal(P.vcycle_apply(h, r), z)
        D.use_graph(True)
        for variant in ("pcg", "fcg", "pcg1"):
            _, rep = P.solve(A, np.ones(A.nrows), precond=P.as_vcycle_preconditioner(h),
                             cfg=P.KrylovConfig(tol=1e-8, variant=variant))
            assert rep.converged
        _, rep = P.solve(A, np.ones(A.nrows), precond=lambda v: P.vcycle_apply(h, v), cfg=P.KrylovConfig(tol=1e-8))
        assert rep.converged
    h = P.build_hierarchy(P.poisson3d(8)[0], coarse_solver="dense_direct", setup="device")
    assert np.all(np.isfinite(P.vcycle_apply(h, rng.standard_normal(512))))
    # arrow matrix: a dense first row/column pushes the SpGEMM into its big-table stages
    n = 3000
    Ad = np.diag(np.full(n, 4.0 * n)) + np.diag(np.full(n - 1, -1.0), 1) + np.diag(np.full(n - 1, -1.0), -1)
    Ad[0, 1:] = Ad[1:, 0] = -0.5
    A = P.CsrMatrix.from_dense(Ad)
    h = P.build_hierarchy(A, setup="device")
    hh = P.build_hierarchy(A, setup="host")
    assert len(h.levels) == len(hh.levels)
    for lv, lh in zip(h.levels, hh.levels):
        assert np.array_equal(lv.A.col_idx, lh.A.col_idx) and np.array_equal(lv.A.values, lh.A.values)
    torch.cuda.synchronize()
    print("sanitize smoke ok", flush=True)


if __name__ == "__main__":
    main()
