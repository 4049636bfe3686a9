#!/usr/bin/env python
"""Stress of the p2p / NCCL halo protocols (run under torchrun, >= 2 GPUs).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/p2p_stress.py --iters 10000

Every rank repeats a halo-exchanging SpMV of its row block of the m^3
Poisson matrix ITERS times, each preceded by a random per-rank spin
(torch.cuda._sleep, 0..2^SPIN cycles) on the library stream, so ranks reach
every exchange at uncorrelated times (the epoch waits and the parity double
buffer get exercised in every interleaving); each result must equal the
single-GPU SpMV rows bitwise.  Also the V-cycle of a distributed hierarchy
ITERS/20 times.  Prints one JSON line per rank; exit 1 on any mismatch.
"""
import argparse
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=48)
    ap.add_argument("--iters", type=int, default=10000)
    ap.add_argument("--spin", type=int, default=14)
    args = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2407_09848_b200 as P
    from paper_2407_09848_b200 import _native as N
    from paper_2407_09848_b200 import dist as D
    from paper_2407_09848_b200 import dsetup as DS

    comm = D.Communicator(local)
    c = comm.ctx
    m = args.grid
    Db = D.poisson3d_block(m, comm)
    lo, hi = Db.global_rows
    A, _ = P.poisson3d(m)
    xg = np.random.default_rng(3).standard_normal(A.nrows)
    x = torch.as_tensor(xg[lo:hi], device="cuda")
    want = torch.as_tensor(A.to_scipy().dot(xg)[lo:hi], device="cuda")  # csr_matvec order == device order
    rng = np.random.default_rng(100 + comm.rank)
    y = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
    bad = 0
    for it in range(args.iters):
        with c.scope():
            torch.cuda._sleep(int(rng.integers(0, 1 << args.spin)))
            N.check(N.lib().amgp_spmv(c.handle, Db.handle, N.ptr(x), N.ptr(y)))
            if not torch.equal(y, want):
                bad += 1
    # distributed V-cycles vs the first one (bitwise repeatable under random skew)
    levels, _ = DS.build_levels(Db, P.CoarseningConfig(), comm=comm, replicate_below=2000)
    dh = D.DistHierarchy.from_levels(levels, comm, P.PolySmootherConfig(family="opt_cheb1", degree=4))
    r = torch.as_tensor(np.random.default_rng(5).standard_normal(hi - lo), device="cuda")
    z0 = dh.vcycle(r)
    vbad = 0
    for it in range(max(1, args.iters // 20)):
        with c.scope():
            torch.cuda._sleep(int(rng.integers(0, 1 << args.spin)))
        if not torch.equal(dh.vcycle(r), z0):
            vbad += 1
    out = {"rank": comm.rank, "world": comm.size, "transport": "p2p" if os.environ.get("AMGP_HALO", "p2p") == "p2p"
           else os.environ.get("AMGP_HALO"), "spmv_exchanges": args.iters, "spmv_mismatches": bad,
           "vcycles": max(1, args.iters // 20), "vcycle_mismatches": vbad, "ok": bad == 0 and vbad == 0}
    for q in range(comm.size):
        if q == comm.rank:
            print(json.dumps(out), flush=True)
        dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if out["ok"] else 1)


if __name__ == "__main__":
    main()
