#!/usr/bin/env python
"""Time the distributed PCG + AMG solve (run under torchrun).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/dist_solve.py \
        --grid 161 --replicate-below 20000 50000 200000 --graph 0 1
    (--stencil 27 --family opt_cheb1 --k 3: BASELINE configs[4] shape)
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
    ap.add_argument("--grid", type=int, default=161)
    ap.add_argument("--stencil", type=int, default=7, choices=[7, 27])
    ap.add_argument("--family", default="opt_cheb4")
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--replicate-below", type=int, nargs="+", default=[20000])
    ap.add_argument("--graph", type=int, nargs="+", default=[1])
    ap.add_argument("--repeat", type=int, default=3)
    ap.add_argument("--cache", default=None, help="hierarchy directory kept across runs (strong scaling)")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    import paper_2407_09848_b200 as P
    from paper_2407_09848_b200 import dist as D

    comm = D.Communicator(local)
    cfg = P.PolySmootherConfig(family=args.family, degree=args.k)

    def build():
        A, _ = (P.poisson3d if args.stencil == 7 else P.poisson3d_27)(args.grid)
        return P.build_hierarchy(A, smoother=cfg)

    t0 = time.perf_counter()
    d, path = D.share_hierarchy(build, comm.rank, dist.barrier, cache=args.cache)
    setup = time.perf_counter() - t0
    res = []
    for rb in args.replicate_below:
        for g in args.graph:
            dh = D.DistHierarchy(d, comm, cfg, replicate_below=rb, use_graph=bool(g))
            lo, hi = dh.row_range
            b = torch.ones(hi - lo, dtype=torch.float64, device="cuda")
            times = []
            for _ in range(args.repeat):
                dist.barrier()
                x, rep = dh.solve(b, cfg=P.KrylovConfig(tol=1e-6))
                t = torch.tensor([rep.elapsed_s], dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                times.append(float(t.item()))
            res.append({"replicate_below": rb, "graph": g, "iters": rep.iterations,
                        "dist_levels": sum(p is not None for p in dh.parts),
                        "solve_ms": [round(1e3 * t, 3) for t in times]})
            del dh
    if comm.rank == 0:
        print(json.dumps({"grid": args.grid, "stencil": args.stencil, "family": args.family, "k": args.k,
                          "world": comm.size, "setup_s": setup,
                          "levels": [int(d[f"A{l}_shape"][0]) for l in range(int(d["nlev"][0]))],
                          "runs": res}),
              flush=True)
        if args.cache is None:
            D.release_shared(path)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
