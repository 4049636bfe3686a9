#!/usr/bin/env python
"""Multi-GPU parity check (run under torchrun, one process per GPU).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/dist_check.py [--grid 32]

Compares on every rank, against the C oracle on the global problem:
  1. fine-level smoother apply on a generated row block (halo-exchanged
     SpMVs), all four families, k = 4: bitwise;
  2. the distributed V-cycle of a native hierarchy (distributed + replicated
     levels): bitwise;
  3. distributed PCG iterations: equal to the single-process count (+-1 bar).
Prints one JSON line per rank; exit code 1 on any mismatch.
"""

import argparse
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=32)
    ap.add_argument("--replicate-below", type=int, default=2000)
    ap.add_argument("--graph", action="store_true")
    args = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    import oracle
    import paper_2407_09848_b200 as P
    from paper_2407_09848_b200 import dist as D

    comm = D.Communicator(local)
    me, world = comm.rank, comm.size
    out = {"rank": me, "world": world, "ok": True, "checks": {}}
    m = args.grid
    fams = ("l1_jacobi", "cheb4", "opt_cheb4", "opt_cheb1")

    # 1. fine-level row block
    A, b = P.poisson3d(m)
    n = A.nrows
    Mg = P.l1_jacobi_diag(A).m_diag
    rhs = np.random.default_rng(0).standard_normal(n)
    x0 = np.random.default_rng(1).standard_normal(n)
    Db = D.poisson3d_block(m, comm)
    lo, hi = Db.global_rows
    mloc = Db.l1_diag()
    ok_m = np.array_equal(mloc.cpu().numpy(), Mg[lo:hi])
    res = {}
    for fam in fams:
        cfg = P.PolySmootherConfig(family=fam, degree=4)
        got = P.smoother_apply(cfg, Db, P.L1JacobiData(m_diag=mloc),
                               torch.tensor(rhs[lo:hi], device="cuda"),
                               torch.tensor(x0[lo:hi], device="cuda")).cpu().numpy()
        beta = cfg.beta.beta if cfg.family == "opt_cheb4" else None
        want = oracle.smoother_apply(cfg.family, 4, A.row_ptr, A.col_idx, A.values, Mg, rhs, x0,
                                     a=cfg.a or 0.0, beta=beta)
        res[fam] = bool(np.array_equal(got, want[lo:hi]))
    out["checks"]["block_l1diag"] = bool(ok_m)
    out["checks"]["block_smoother_bitwise"] = res

    # 2./3. distributed hierarchy
    def build():
        return P.build_hierarchy(A, smoother=P.PolySmootherConfig(family="opt_cheb1", degree=4), setup="host")

    d, path = D.share_hierarchy(build, me, dist.barrier)
    h = build() if me != 0 else None  # every rank needs the global levels for the oracle
    if h is None:
        h = build()
    dh = D.DistHierarchy(d, comm, P.PolySmootherConfig(family="opt_cheb1", degree=4),
                         replicate_below=args.replicate_below, use_graph=args.graph)
    out["partitions"] = [None if p is None else int(p[-1]) for p in dh.parts]
    lo0, hi0 = dh.row_range
    levels = [{"A": (lv.A.row_ptr, lv.A.col_idx, lv.A.values), "m": lv.M.m_diag,
               **({"P": (lv.P.row_ptr, lv.P.col_idx, lv.P.values),
                   "R": (lv.restrict_op().row_ptr, lv.restrict_op().col_idx, lv.restrict_op().values)}
                  if lv.P is not None else {})} for lv in h.levels]
    r = np.random.default_rng(5).standard_normal(n)
    vc = {}
    for fam in fams:
        cfg = P.PolySmootherConfig(family=fam, degree=4)
        dh.set_smoother(cfg)
        got = dh.vcycle(torch.tensor(r[lo0:hi0], device="cuda")).cpu().numpy()
        beta = cfg.beta.beta if cfg.family == "opt_cheb4" else None
        oh = oracle.Hierarchy(levels, cfg.family, 4, a=cfg.a or 0.0, beta=beta)
        want = oh.vcycle(r)
        vc[fam] = bool(np.array_equal(got, want[lo0:hi0]))
    out["checks"]["vcycle_bitwise"] = vc
    pcg = {}
    for fam in fams:
        cfg = P.PolySmootherConfig(family=fam, degree=4)
        dh.set_smoother(cfg)
        for variant in ("pcg", "fcg"):
            x, rep = dh.solve(torch.ones(hi0 - lo0, dtype=torch.float64, device="cuda"),
                              cfg=P.KrylovConfig(tol=1e-6, variant=variant))
            beta = cfg.beta.beta if cfg.family == "opt_cheb4" else None
            oh = oracle.Hierarchy(levels, cfg.family, 4, a=cfg.a or 0.0, beta=beta)
            _, it, rr, conv, brk, _ = oracle.pcg(levels[0]["A"], np.ones(n), oh, tol=1e-6,
                                                 fcg=variant == "fcg")
            pcg[f"{fam}_{variant}"] = {"iters": rep.iterations, "oracle": it,
                                       "ok": bool(rep.converged and abs(rep.iterations - it) <= 1)}
    out["checks"]["pcg"] = pcg
    flat = [out["checks"]["block_l1diag"]] + list(res.values()) + list(vc.values()) + \
           [v["ok"] for v in pcg.values()]
    out["ok"] = bool(all(flat))
    for r in range(comm.size):  # one rank at a time: whole lines on the shared stdout
        if r == me:
            print(json.dumps(out), flush=True)
        dist.barrier()
    if me == 0:
        try:
            D.release_shared(path)
        except OSError:
            pass
    dist.destroy_process_group()
    sys.exit(0 if out["ok"] else 1)


if __name__ == "__main__":
    main()
