#!/usr/bin/env python
"""Per-level SpMV times of the distributed device hierarchy (GPU box).

    python bench.py-style launch:  torchrun --nproc-per-node 4 --master-addr 127.0.0.1 \
        tools/dist_levels.py --weak-grid 400        (also runs as one plain process: N = 1)

Same construction as bench.py's weak-scaled solve (global cube
round(m N^(1/3)), distributed device setup, levels under 20,000 rows
replicated).  For every level: A_l, R_l = P_l^T and P_l SpMVs launched REPS
times back to back on the library stream (eager, halo exchange included),
time = max over ranks of the CUDA-event time / REPS; then one V-cycle and the
PCG solve.  Rank 0 prints one JSON line.
"""
import argparse
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--weak-grid", type=int, default=400)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--family", default="opt_cheb4")
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--no-solve", action="store_true", help="skip the PCG solve (AMGP_HALO_NOSYNC experiments)")
    ap.add_argument("--per-rank", action="store_true",
                    help="also: per-rank rows / nnz of levels >= 1 and their SpMV time without the exchange")
    args = ap.parse_args()
    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_2407_09848_b200 as P
    from paper_2407_09848_b200 import _native as N

    ws = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    cfg = P.PolySmootherConfig(family=args.family, degree=args.k)
    m = int(round(args.weak_grid * ws ** (1.0 / 3.0)))
    if ws > 1:
        from paper_2407_09848_b200 import dist as Dist
        from paper_2407_09848_b200 import dsetup as DS

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = Dist.Communicator(local)
        rank = comm.rank
        D0 = Dist.poisson3d_block(m, comm)
        levels, _ = DS.build_levels(D0, P.CoarseningConfig(), comm=comm)
        dh = Dist.DistHierarchy.from_levels(levels, comm, cfg, use_graph=True)
        As, Ps, Rs, c = dh.As, dh.Ps, dh.Rs, dh.ctx
        parts = dh.parts
    else:
        rank = 0
        D0 = P.poisson3d_device(m)
        h = P.build_hierarchy(D0, smoother=cfg)
        As = [lv.A for lv in h.levels]
        Ps = [lv.P for lv in h.levels[:-1]]
        Rs = [lv.restrict_op() for lv in h.levels[:-1]]
        c = D0.ctx
        parts = [None] * len(As)

    def sync():
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()

    def maxr(v):
        if ws == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def halo(M):
        v = [C.c_int64(0) for _ in range(4)]
        N.check(N.lib().amgp_mat_halo_info(M.handle, *[C.byref(x) for x in v]))
        return [x.value for x in v]

    def time_spmv(M):
        x = torch.randn(M.ncols, dtype=torch.float64, device="cuda")
        y = torch.empty(M.nrows, dtype=torch.float64, device="cuda")
        with c.scope():
            N.check(N.lib().amgp_spmv(c.handle, M.handle, N.ptr(x), N.ptr(y)))
        best = None
        for _ in range(3):
            sync()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with c.scope():
                e0.record(c.stream)
                for _ in range(args.reps):
                    N.check(N.lib().amgp_spmv(c.handle, M.handle, N.ptr(x), N.ptr(y)))
                e1.record(c.stream)
            torch.cuda.synchronize()
            t = maxr(e0.elapsed_time(e1) / args.reps)
            best = t if best is None else min(best, t)
        byts = 12 * M.nnz + 4 * (M.nrows + 1) + 8 * M.ncols + 8 * M.nrows
        nown, nhalo, nint, nbnd = halo(M)
        return {"us": round(best * 1e3, 2), "GBs": round(byts / (best * 1e-3) / 1e9, 1), "nrows": M.nrows,
                "nnz": M.nnz, "nhalo": nhalo, "interior": nint, "boundary": nbnd}

    def gather(v):
        if ws == 1:
            return [v]
        objs = [None] * ws
        dist.all_gather_object(objs, v)
        return objs

    def time_local(M):
        # the rank's own block as a plain matrix (halo columns as extra local
        # columns, no exchange): each rank alone, all ranks concurrently
        L = P.DeviceMatrix.from_csr(M.to_csr(), c)
        x = torch.randn(L.ncols, dtype=torch.float64, device="cuda")
        y = torch.empty(L.nrows, dtype=torch.float64, device="cuda")
        best = None
        for _ in range(3):
            sync()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with c.scope():
                e0.record(c.stream)
                for _ in range(args.reps):
                    N.check(N.lib().amgp_spmv(c.handle, L.handle, N.ptr(x), N.ptr(y)))
                e1.record(c.stream)
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / args.reps
            best = t if best is None else min(best, t)
        return round(best * 1e3, 2)

    out = {"world": ws, "m": m, "levels": []}
    if args.per_rank:
        pr = []
        for l in range(1, len(As)):
            if parts[l] is None:
                break
            ent = {"level": l, "A_rows": gather(As[l].nrows), "A_nnz": gather(As[l].nnz),
                   "A_local_us": gather(time_local(As[l]))}
            if l < len(Ps):
                ent["R_nnz"] = gather(Rs[l].nnz)
                ent["R_local_us"] = gather(time_local(Rs[l]))
            pr.append(ent)
        out["per_rank"] = pr
        torch.cuda.empty_cache()
    for l in range(len(As)):
        ent = {"level": l, "distributed": parts[l] is not None, "A": time_spmv(As[l])}
        if l < len(Ps):
            ent["R"] = time_spmv(Rs[l])
            ent["P"] = time_spmv(Ps[l])
        out["levels"].append(ent)
    n0 = As[0].nrows
    b = torch.ones(n0, dtype=torch.float64, device="cuda")
    kc = P.KrylovConfig(tol=1e-6)

    def run():
        if ws > 1:
            return dh.solve(b, cfg=kc)
        return P.solve(D0, b, precond=P.as_vcycle_preconditioner(h), cfg=kc)

    if args.no_solve:
        if rank == 0:
            print(json.dumps(out), flush=True)
        if ws > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    run()
    ts = []
    for _ in range(3):
        sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(c.stream)
        _, rep = run()
        e1.record(c.stream)
        torch.cuda.synchronize()
        ts.append(maxr(e0.elapsed_time(e1)))
    out["solve_ms"] = sorted(ts)[1]
    out["iterations"] = rep.iterations
    if rank == 0:
        print(json.dumps(out), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
