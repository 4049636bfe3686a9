#!/usr/bin/env python
"""Distributed device setup parity (run under torchrun, one process per GPU).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/dsetup_dist_check.py --grid 32

Every rank builds its row blocks of the hierarchy with the device setup
(decoupled aggregation, dsetup.py).  Rank 0 gathers every level (global
indices) and recomputes the same hierarchy on the host from the reference's
formulas: per-block sa_aggregate / matching_aggregate of the diagonal blocks
(csrc/setup.cpp restatements), lambda_max with the per-rank OpenBLAS-order
dots folded in rank order, smooth_prolongator and galerkin_rap -- the device
levels must be bitwise equal.  Then the distributed V-cycle must be bitwise
the C oracle's on the gathered hierarchy, and PCG iterations within +-1 of
the oracle and of the single-GPU (reference) hierarchy.
Prints one JSON line (rank 0); exit code 1 on a mismatch.
"""

import argparse
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))


def main():
    if os.environ.get("AMGP_WATCHDOG"):
        import faulthandler

        faulthandler.dump_traceback_later(float(os.environ["AMGP_WATCHDOG"]), exit=True)
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=32)
    ap.add_argument("--stencil", type=int, default=7)
    ap.add_argument("--kind", default="smoothed_aggregation")
    ap.add_argument("--replicate-below", type=int, default=2000)
    ap.add_argument("--backend", default="nccl")
    args = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if args.backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group("gloo")
    import oracle
    import paper_2407_09848_b200 as P
    from paper_2407_09848_b200 import dist as D
    from paper_2407_09848_b200 import dsetup as DS
    from paper_2407_09848_b200 import setup as S

    comm = D.Communicator(local)
    me, world = comm.rank, comm.size
    m = args.grid
    cc = P.CoarseningConfig(kind=args.kind)
    D0 = D.poisson3d_block(m, comm, stencil=args.stencil)
    levels, stag = DS.build_levels(D0, cc, comm=comm, replicate_below=args.replicate_below)
    print(f"[rank {me}] setup done: {[L.n for L in levels]}", file=sys.stderr, flush=True)

    def global_csr(Dm, row_lo=None):
        H = Dm.to_csr()
        cm = getattr(Dm, "col_map", None)
        ci = H.col_idx if cm is None else cm.cpu().numpy()[H.col_idx]
        return (int(getattr(Dm, "row_lo", 0) if row_lo is None else row_lo), H.row_ptr, ci, H.values)

    mine = []
    for L in levels:
        ent = {"n": L.n, "off": None if L.off is None else [int(x) for x in L.off],
               "A": global_csr(L.A, L.lo) if (L.off is not None or me == 0) else None, "m": L.m.cpu().numpy()}
        if L.P is not None:
            ent["P"] = global_csr(L.P)
            ent["R"] = global_csr(L.R) if L.off is not None or me == 0 else None
            ent["R_repl"] = L.R.nrows == L.n_aggregates
        mine.append(ent)
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)

    # distributed V-cycle and PCG on the device hierarchy
    fams = ("l1_jacobi", "cheb4", "opt_cheb4", "opt_cheb1")
    cfg0 = P.PolySmootherConfig(family="opt_cheb1", degree=4)
    dh = D.DistHierarchy.from_levels(levels, comm, cfg0)
    lo0, hi0 = dh.row_range
    n0 = levels[0].n
    r = np.random.default_rng(5).standard_normal(n0)
    vres, pres = {}, {}
    for fam in fams:
        cfg = P.PolySmootherConfig(family=fam, degree=4)
        dh.set_smoother(cfg)
        vres[fam] = dh.vcycle(torch.tensor(r[lo0:hi0], device="cuda")).cpu().numpy()
        x, rep = dh.solve(torch.ones(hi0 - lo0, dtype=torch.float64, device="cuda"),
                          cfg=P.KrylovConfig(tol=1e-6))
        pres[fam] = (rep.iterations, rep.converged)
    print(f"[rank {me}] vcycle/pcg done {pres}", file=sys.stderr, flush=True)
    vall = [None] * world
    dist.all_gather_object(vall, {f: v for f, v in vres.items()})

    out = {"world": world, "grid": m, "stencil": args.stencil, "kind": args.kind,
           "levels": [L.n for L in levels], "distributed_levels": sum(L.off is not None for L in levels)}
    ok = True
    if me == 0:
        # ---- host recomputation of the decoupled hierarchy
        A, _ = (P.poisson3d if args.stencil == 7 else P.poisson3d_27)(m)

        def assemble(key, l, nrows, ncols):
            rows = {}
            for g in gathered:
                ent = g[l].get(key)
                if ent is None:
                    continue
                lo, rp, ci, v = ent
                for i in range(len(rp) - 1):
                    rows[lo + i] = (ci[rp[i]:rp[i + 1]], v[rp[i]:rp[i + 1]])
            rp = np.zeros(nrows + 1, dtype=np.int64)
            for i in range(nrows):
                rp[i + 1] = rp[i] + len(rows[i][0])
            ci = np.concatenate([rows[i][0] for i in range(nrows)]) if nrows else np.zeros(0, np.int64)
            v = np.concatenate([rows[i][1] for i in range(nrows)]) if nrows else np.zeros(0)
            return P.CsrMatrix(nrows, ncols, rp, ci.astype(np.int64), v)

        def block(A, lo, hi):
            rp, ci, v = A.row_ptr, A.col_idx, A.values
            rows, cols, vals = [], [], []
            sub_rp = [0]
            for i in range(lo, hi):
                seg = slice(rp[i], rp[i + 1])
                k = (ci[seg] >= lo) & (ci[seg] < hi)
                cols.append(ci[seg][k] - lo)
                vals.append(v[seg][k])
                sub_rp.append(sub_rp[-1] + int(k.sum()))
            return P.CsrMatrix(hi - lo, hi - lo, np.array(sub_rp), np.concatenate(cols), np.concatenate(vals))

        def lam_folded(Al, off):
            d = Al.diagonal()
            ds = np.sqrt(d)
            v = np.ones(Al.nrows) + np.random.default_rng(0).uniform(-0.5, 0.5, Al.nrows)
            lam = 1.0
            blocks = [(int(off[p]), int(off[p + 1])) for p in range(len(off) - 1)] if off is not None \
                else [(0, Al.nrows)]
            for _ in range(25):
                w = S.host_spmv(Al, v / ds) / ds
                dots = []
                for x, y in ((v, w), (v, v), (w, w)):
                    if off is None:
                        dots.append(S.blas_dot(x, y))
                    else:
                        s = 0.0
                        for lo, hi in blocks:
                            s = s + S.blas_dot(x[lo:hi], y[lo:hi])
                        dots.append(s)
                lam = dots[0] / dots[1]
                nrm = np.sqrt(dots[2])
                if nrm == 0.0:
                    return 0.0
                v = w / nrm
            return lam

        Al = A
        checks = []
        for l, L in enumerate(levels):
            off = gathered[0][l]["off"]
            got_A = assemble("A", l, Al.nrows, Al.ncols)
            if got_A is not None:
                checks.append((f"A{l}", np.array_equal(got_A.row_ptr, Al.row_ptr) and
                               np.array_equal(got_A.col_idx, Al.col_idx) and np.array_equal(got_A.values, Al.values)))
            if "P" not in gathered[0][l]:
                break
            # aggregation per block
            if off is not None:
                aggs, base = [], 0
                for p in range(world):
                    B = block(Al, off[p], off[p + 1])
                    Ph = S.sa_aggregate(B, cc.strength_theta) if args.kind == "smoothed_aggregation" \
                        else S.matching_aggregate(B, cc.matching_sweeps)
                    aggs.append(Ph.col_idx + base)
                    base += Ph.ncols
                agg = np.concatenate(aggs)
                nc = base
            else:
                Ph = S.sa_aggregate(Al, cc.strength_theta) if args.kind == "smoothed_aggregation" \
                    else S.matching_aggregate(Al, cc.matching_sweeps)
                agg, nc = Ph.col_idx, Ph.ncols
            P_hat = P.CsrMatrix(Al.nrows, nc, np.arange(Al.nrows + 1), agg, np.ones(Al.nrows))
            lam = lam_folded(Al, off)
            Pm = S.smooth_prolongator(Al, P_hat, 4.0 / (3.0 * lam))
            got_P = assemble("P", l, Al.nrows, nc)
            checks.append((f"P{l}", np.array_equal(got_P.row_ptr, Pm.row_ptr) and
                           np.array_equal(got_P.col_idx, Pm.col_idx) and np.array_equal(got_P.values, Pm.values)))
            Rm = Pm.transpose()
            got_R = assemble("R", l, nc, Al.nrows)
            checks.append((f"R{l}", np.array_equal(got_R.row_ptr, Rm.row_ptr) and
                           np.array_equal(got_R.col_idx, Rm.col_idx) and np.array_equal(got_R.values, Rm.values)))
            Ac = S.galerkin_rap(Al, Pm)
            Al = Ac
        if levels[-1].off is None:
            pass
        out["setup_checks"] = {k: bool(v) for k, v in checks}
        ok &= all(v for _, v in checks)
        # ---- V-cycle / PCG vs the oracle on the gathered hierarchy
        hl = []
        Al = None
        for l, L in enumerate(levels):
            ent0 = gathered[0][l]
            if ent0["off"] is not None:
                Ag = assemble("A", l, ent0["n"], ent0["n"])
                mg = np.concatenate([g[l]["m"] for g in gathered])
            else:
                lo_, rp_, ci_, v_ = ent0["A"]
                Ag = P.CsrMatrix(len(rp_) - 1, len(rp_) - 1, rp_, ci_.astype(np.int64), v_)
                mg = ent0["m"]
            lv = {"A": (Ag.row_ptr, Ag.col_idx, Ag.values), "m": mg}
            if "P" in ent0:
                nc = levels[l + 1].n if l + 1 < len(levels) else None
                Pg = assemble("P", l, ent0["n"], nc)
                Rg = Pg.transpose()
                lv["P"] = (Pg.row_ptr, Pg.col_idx, Pg.values)
                lv["R"] = (Rg.row_ptr, Rg.col_idx, Rg.values)
            hl.append(lv)
        vb, pc = {}, {}
        Aglob, _ = (P.poisson3d if args.stencil == 7 else P.poisson3d_27)(m)
        hg = P.build_hierarchy(Aglob, coarsening=cc, setup="device")
        for fam in fams:
            cfg = P.PolySmootherConfig(family=fam, degree=4)
            beta = cfg.beta.beta if cfg.family == "opt_cheb4" else None
            oh = oracle.Hierarchy(hl, cfg.family, 4, a=cfg.a or 0.0, beta=beta)
            want = oh.vcycle(r)
            got = np.concatenate([vall[p][fam] for p in range(world)])
            vb[fam] = bool(np.array_equal(got, want))
            _, it, rr, conv, brk, _ = oracle.pcg(hl[0]["A"], np.ones(n0), oh, tol=1e-6)
            for lv in hg.levels:
                lv.smoother = cfg
            _, rg = P.solve(Aglob, np.ones(n0), precond=P.as_vcycle_preconditioner(hg),
                            cfg=P.KrylovConfig(tol=1e-6))
            pc[fam] = {"dist": pres[fam][0], "oracle_same_hier": it, "global_hier": rg.iterations,
                       "ok": bool(pres[fam][1] and abs(pres[fam][0] - it) <= 1 and
                                  abs(pres[fam][0] - rg.iterations) <= 1)}
        out["vcycle_bitwise"] = vb
        out["pcg"] = pc
        ok &= all(vb.values()) and all(v["ok"] for v in pc.values())
        out["ok"] = bool(ok)
        print(json.dumps(out), flush=True)
    okt = torch.tensor([1 if ok else 0], device="cuda")
    dist.broadcast(okt, 0)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if okt.item() else 1)


if __name__ == "__main__":
    main()
