"""Host-side logic of the multi-GPU path (paper_2407_09848_b200/dist.py), on CPU.

* Partition + localization + halo plans: emulating every rank's SpMV
  (own entries + halo gathered through the plan) reproduces the global SpMV
  bit for bit, for every matrix of a hierarchy, 1-5 ranks, distributed and
  replicated levels.
* Plan consistency across ranks: what rank p sends to q is exactly what q
  receives from p -- checked by 2 real processes exchanging their plans over
  torch.distributed (gloo, world size 2).
"""

import os

import numpy as np
import pytest

import oracle
import paper_2407_09848_b200 as P
from paper_2407_09848_b200 import dist as D


def emulate_spmv(A_loc, plan, x_global, col_off, me):
    """Rank me's rows of A @ x using only its own x entries + the halo."""
    if plan is None:
        xe = x_global
    else:
        c_lo, c_hi = col_off[me], col_off[me + 1]
        own = x_global[c_lo:c_hi]
        # the halo arrives from the peers' packed send buffers
        halo = np.concatenate([x_global[cols] for cols in plan.recv_cols]) if plan.recv_cols else np.zeros(0)
        xe = np.concatenate([own, halo])
    return oracle.spmv(A_loc.row_ptr, A_loc.col_idx, A_loc.values, A_loc.ncols, xe)


def sends_as_global(plan, col_off, me):
    out, o = {}, 0
    for q, cnt in zip(plan.peers, plan.send_cnt):
        out[int(q)] = plan.send_idx[o:o + cnt] + col_off[me]
        o += cnt
    return out


@pytest.mark.parametrize("nranks", [1, 2, 3, 5])
@pytest.mark.parametrize("kind", ["smoothed_aggregation", "pairwise_matching"])
def test_localized_spmv_is_bitwise_global(nranks, kind):
    A, _ = P.poisson3d(12)
    h = P.build_hierarchy(A, coarsening=P.CoarseningConfig(kind=kind))

    class _H:
        levels = h.levels

    parts = D.level_partitions(_H, nranks, replicate_below=150)
    assert parts[0] is not None or nranks == 1
    rng = np.random.default_rng(nranks)
    mats = []
    for l, lv in enumerate(h.levels):
        mats.append((lv.A, parts[l], parts[l]))
        if lv.P is not None:
            mats.append((lv.P, parts[l], parts[l + 1]))
            mats.append((lv.restrict_op(), parts[l + 1], parts[l]))
    for M, roff, coff in mats:
        x = rng.standard_normal(M.ncols)
        y = oracle.spmv(M.row_ptr, M.col_idx, M.values, M.ncols, x)
        plans = []
        for me in range(nranks):
            Ml, plan = D.localize(M, roff, coff, me)
            plans.append(plan)
            lo, hi = (roff[me], roff[me + 1]) if roff is not None else (0, M.nrows)
            assert np.array_equal(emulate_spmv(Ml, plan, x, coff, me), y[lo:hi])
            if plan is not None:
                assert Ml.ncols == plan.nown + plan.nhalo
                for cols in plan.recv_cols:
                    assert np.all(np.diff(cols) > 0)
        # sends of p to q == receives of q from p
        if coff is not None:
            for p in range(nranks):
                for q, cols in sends_as_global(plans[p], coff, p).items():
                    k = list(plans[q].peers).index(p)
                    assert np.array_equal(plans[q].recv_cols[k], cols)


def test_level_partitions_replicate_coarse_levels():
    A, _ = P.poisson3d(16)
    h = P.build_hierarchy(A)

    class _H:
        levels = h.levels

    parts = D.level_partitions(_H, 4, replicate_below=500)
    sizes = [lv.A.nrows for lv in h.levels]
    seen_rep = False
    for n, p in zip(sizes, parts):
        if p is None:
            seen_rep = True
        else:
            assert not seen_rep and p[-1] == n and len(p) == 5
    assert parts[0] is not None and parts[-1] is None


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A, _ = P.poisson3d(10)
        h = P.build_hierarchy(A)

        class _H:
            levels = h.levels

        parts = D.level_partitions(_H, world, replicate_below=100)
        mine = []
        for l, lv in enumerate(h.levels):
            Ml, plan = D.localize(lv.A, parts[l], parts[l], rank)
            if plan is None:
                mine.append(None)
                continue
            sends = {int(k): v.tolist() for k, v in sends_as_global(plan, parts[l], rank).items()}
            recvs = {int(p): c.tolist() for p, c in zip(plan.peers, plan.recv_cols)}
            mine.append((sends, recvs))
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        ok = True
        for l in range(len(mine)):
            if allp[0][l] is None:
                continue
            for p in range(world):
                for qq, cols in allp[p][l][0].items():
                    ok &= allp[qq][l][1].get(p) == cols
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_gloo_two_process_plan_exchange():
    import multiprocessing as mp
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res
