#!/usr/bin/env python
"""Multi-GPU micro-timings of the halo-exchanged SpMV / smoother step.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/dist_micro.py --grid 323
"""

import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=323)
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    import paper_2407_09848_b200 as P
    from paper_2407_09848_b200 import _native as N
    from paper_2407_09848_b200 import dist as D

    comm = D.Communicator(local)
    c = comm.ctx
    Db = D.poisson3d_block(args.grid, comm)
    n = Db.nrows
    # same-size local matrix without halo (cube rows of the block's size)
    Dl = P.poisson3d_device(int(round(n ** (1 / 3))))
    out = {"rank": comm.rank}

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(c.stream)
        for _ in range(reps):
            fn()
        e1.record(c.stream)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / reps
        return e0.elapsed_time(e1) / reps * 1e3, wall * 1e6

    x = torch.randn(n, dtype=torch.float64, device="cuda")
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    xl = torch.randn(Dl.nrows, dtype=torch.float64, device="cuda")
    yl = torch.empty(Dl.nrows, dtype=torch.float64, device="cuda")

    def spmv_dist():
        with c.scope():
            N.check(N.lib().amgp_spmv(c.handle, Db.handle, N.ptr(x), N.ptr(y)))

    def spmv_local():
        with c.scope():
            N.check(N.lib().amgp_spmv(c.handle, Dl.handle, N.ptr(xl), N.ptr(yl)))

    out["spmv_dist_us"] = timed(spmv_dist, args.reps)
    out["spmv_local_us"] = timed(spmv_local, args.reps)
    cfg = P.PolySmootherConfig(family="cheb4", degree=6)
    M = P.L1JacobiData(m_diag=Db.l1_diag())
    Ml = P.L1JacobiData(m_diag=Dl.l1_diag())
    out["cheb4_k6_dist_us"] = timed(lambda: P.smoother_apply(cfg, Db, M, x, y), 10)
    out["cheb4_k6_local_us"] = timed(lambda: P.smoother_apply(cfg, Dl, Ml, xl, yl), 10)
    nint = [C for C in [0, 0, 0, 0]]
    import ctypes

    vals = [ctypes.c_int64() for _ in range(4)]
    N.check(N.lib().amgp_mat_halo_info(Db.handle, *[ctypes.byref(v) for v in vals]))
    out["halo"] = [v.value for v in vals]
    print(json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
