"""Host-side / collective logic of the distributed device setup (dsetup.py)
on CPU tensors with gloo, world size 2 and 3 (the device kernels themselves
are covered by the GPU tests).

Every rank holds a contiguous row block of a global sparse matrix with
global column ids:
* make_halo localises the columns (own first, halo ascending) and its plan
  is consistent across ranks (what p sends q is what q receives from p);
* Exchanger.values / Exchanger.rows deliver exactly the neighbours' entries
  / rows of the halo, in halo order;
* _gather_rows reassembles the global matrix on every rank;
* _start_vector slices are the global reference start vector.
"""

import os

import numpy as np
import pytest

import paper_2407_09848_b200 as P


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2407_09848_b200 import dsetup as DS

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A, _ = P.poisson3d(7)
        n = A.nrows
        off = np.array([p * n // world for p in range(world + 1)], dtype=np.int64)
        lo, hi = int(off[rank]), int(off[rank + 1])
        rp = torch.as_tensor(A.row_ptr[lo:hi + 1] - A.row_ptr[lo])
        col = torch.as_tensor(A.col_idx[A.row_ptr[lo]:A.row_ptr[hi]])
        val = torch.as_tensor(A.values[A.row_ptr[lo]:A.row_ptr[hi]])
        local, halo_g, plan, ex = DS.make_halo(col, lo, hi, off, rank)
        ok = {}
        # localisation: own -> c - lo, halo -> nown + rank in halo_g
        back = torch.where(local < hi - lo, local + lo, halo_g[torch.clamp(local - (hi - lo), min=0)])
        ok["localise"] = bool(torch.equal(back, col))
        ok["halo_sorted"] = bool(torch.all(halo_g[1:] > halo_g[:-1])) if halo_g.numel() > 1 else True
        # values: each rank sends its own global ids; the halo must come back as halo_g
        gid = torch.arange(lo, hi, dtype=torch.int64)
        ok["values"] = bool(torch.equal(ex.values(gid), halo_g))
        # rows: the halo rows of A are A's global rows halo_g
        M = DS.DCsr(rp, col, val)
        Hr = ex.rows(M)
        good = Hr.nrows == halo_g.numel()
        for t, g in enumerate(halo_g.tolist()):
            a, b = A.row_ptr[g], A.row_ptr[g + 1]
            good &= np.array_equal(Hr.col[Hr.rp[t]:Hr.rp[t + 1]].numpy(), A.col_idx[a:b])
            good &= np.array_equal(Hr.val[Hr.rp[t]:Hr.rp[t + 1]].numpy(), A.values[a:b])
        ok["rows"] = bool(good)
        # gather: the whole matrix on every rank
        G = DS._gather_rows(M, world)
        ok["gather"] = bool(np.array_equal(G.rp.numpy(), A.row_ptr) and np.array_equal(G.col.numpy(), A.col_idx)
                            and np.array_equal(G.val.numpy(), A.values))
        # plan consistency across ranks
        sends, o = {}, 0
        for qq, cnt in zip(plan.peers, plan.send_cnt):
            sends[int(qq)] = (plan.send_idx[o:o + cnt] + lo).tolist()
            o += cnt
        mine = {"sends": sends, "halo": halo_g.tolist(), "off": off.tolist()}
        allp = [None] * world
        dist.all_gather_object(allp, mine)
        cons = True
        for p in range(world):
            for qq, ids in allp[p]["sends"].items():
                q_lo, q_hi = off[p], off[p + 1]
                want = [g for g in allp[qq]["halo"] if q_lo <= g < q_hi]
                cons &= ids == want
        ok["plan"] = bool(cons)
        # start vector slices
        v = DS._start_vector(n, lo, hi)
        ref = np.ones(n) + np.random.default_rng(0).uniform(-0.5, 0.5, n)
        ok["start_vector"] = bool(np.array_equal(v, ref[lo:hi]))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_setup_host_logic_gloo(world):
    import multiprocessing as mp
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok in res:
        assert all(ok.values()), (rank, ok)
