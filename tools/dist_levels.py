#!/usr/bin/env python
"""Per-level cost of halo exchanges in the distributed hierarchy (torchrun).

For every distributed matrix of the rank (A_l, P_l, R_l) times amgp_spmv
with its halo plan (NCCL exchange overlapped with interior rows) against the
same local matrix without a plan (operand already extended: no
communication), and the exchange alone.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/dist_levels.py --grid 161
"""

import argparse
import ctypes
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=161)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--replicate-below", type=int, default=20000)
    ap.add_argument("--stencil", type=int, default=7, choices=[7, 27])
    ap.add_argument("--cache", default=None, help="hierarchy directory kept across runs")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    import paper_2407_09848_b200 as P
    from paper_2407_09848_b200 import _native as N
    from paper_2407_09848_b200 import dist as D
    from paper_2407_09848_b200.sparse import DeviceMatrix

    comm = D.Communicator(local)
    c = comm.ctx
    cfg = P.PolySmootherConfig(family="opt_cheb4", degree=4)

    def build():
        A, _ = (P.poisson3d if args.stencil == 7 else P.poisson3d_27)(args.grid)
        return P.build_hierarchy(A, smoother=cfg)

    d, path = D.share_hierarchy(build, comm.rank, dist.barrier, cache=args.cache)
    L = int(d["nlev"][0])
    A_glob = [D._mat(d, f"A{l}") for l in range(L)]

    class _H:
        levels = [type("Lv", (), {"A": a}) for a in A_glob]

    parts = D.level_partitions(_H, comm.size, args.replicate_below)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(c.stream)
        for _ in range(args.reps):
            fn()
        e1.record(c.stream)
        torch.cuda.synchronize()
        return round(e0.elapsed_time(e1) / args.reps * 1e3, 2)

    rows = []
    for l in range(L):
        mats = [("A", A_glob[l], parts[l], parts[l])]
        if l < L - 1:
            mats += [("P", D._mat(d, f"P{l}"), parts[l], parts[l + 1]),
                     ("R", D._mat(d, f"R{l}"), parts[l + 1], parts[l])]
        for name, M, roff, coff in mats:
            Ml, plan = D.localize(M, roff, coff, comm.rank)
            Dh = D.attach_halo(DeviceMatrix.from_csr(Ml, c), plan)
            Dn = DeviceMatrix.from_csr(Ml, c)
            nown = plan.nown if plan is not None else Ml.ncols
            x = torch.randn(Ml.ncols, dtype=torch.float64, device="cuda")
            y = torch.empty(Ml.nrows, dtype=torch.float64, device="cuda")

            def graph_us(Dm, flags=1):
                ms = ctypes.c_double()
                dist.barrier()
                with c.scope():
                    N.check(N.lib().amgp_spmv_timed(c.handle, Dm.handle, N.ptr(x), N.ptr(y),
                                                    args.reps, flags, ctypes.byref(ms)))
                return round(ms.value * 1e3, 2)

            hi = [ctypes.c_int64() for _ in range(4)]
            N.check(N.lib().amgp_mat_halo_info(Dh.handle, *[ctypes.byref(v) for v in hi]))
            rec = {"level": l, "mat": name, "rows": Ml.nrows, "nnz": Ml.nnz,
                   "slices_interior": hi[2].value, "slices_boundary": hi[3].value,
                   "halo": plan.nhalo if plan is not None else 0,
                   "peers": len(plan.peers) if plan is not None else 0,
                   "us_halo_graph": graph_us(Dh), "us_local_graph": graph_us(Dn),
                   "us_exchange_graph": graph_us(Dh, 3)}
            rows.append(rec)
    # every rank's numbers; report the slowest rank (interior ranks have two
    # neighbours) per matrix
    allrows = [None] * comm.size
    dist.all_gather_object(allrows, rows)
    if comm.rank == 0:
        for i, r in enumerate(rows):
            per = [a[i] for a in allrows]
            worst = max(per, key=lambda q: q["us_halo_graph"])
            out = dict(worst)
            out["rank_of_max"] = per.index(worst)
            out["us_halo_graph_per_rank"] = [q["us_halo_graph"] for q in per]
            print(json.dumps(out), flush=True)
        if args.cache is None:
            D.release_shared(path)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
