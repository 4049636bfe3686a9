"""AMG hierarchy setup on the GPU, one device or row blocks over several.

Mirrors reference amg.py:238-287 (``build_hierarchy``) level by level:

* aggregation (amg.py:102-191): strength lists on the device
  (``amgp_ds_strength``), the sequential greedy passes on the host
  (csrc/setup.cpp ``amgp_setup_sa_pass1/2``; matching: the host restatement
  of ``matching_aggregate``);
* lambda_max (amg.py:194-216): power iteration on the device with the dots in
  OpenBLAS order (``amgp_ds_lambda_max``);
* smoothed prolongator (amg.py:219-226), Galerkin product and symmetrisation
  (amg.py:229-235): ``amgp_ds_prolongator``, ``amgp_ds_spgemm``,
  ``amgp_ds_symmetrize`` -- every entry summed in scipy's order.

On one GPU the hierarchy is bitwise the reference's (tests/test_gpu_setup.py).
On P GPUs each rank owns a contiguous row block of every level; aggregation is
*decoupled* (the paper's VBM choice): each rank aggregates its
own block using only its own columns, so coarse rows inherit the block
partition.  lambda_max is global (per-rank OpenBLAS-order partial dots folded
in rank order), the prolongator and the Galerkin product are the reference's
formulas evaluated on the rank's rows with the halo rows of P and A*P
exchanged over NCCL (torch.distributed all-to-all).  With P = 1 the decoupled
hierarchy IS the reference's.  Levels below ``replicate_below`` rows are
gathered to every rank and the rest of the setup runs redundantly (coarse
agglomeration).  torch provides device memory, index bookkeeping (prefix
sums, sorts of index keys) and the collectives; every floating-point
operation of the setup is a libamgp kernel.
"""

from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .sparse import DeviceMatrix

_I32P = C.POINTER(C.c_int32)


def _lib():
    return N.lib()


def _p(t):
    return None if t is None else N._VP(t.data_ptr())


def blas_threads():
    """OpenBLAS thread count whose ddot order lambda_max reproduces
    (AMGP_BLAS_THREADS, default 1 -- the reference run single-threaded)."""
    return int(os.environ.get("AMGP_BLAS_THREADS", "1"))


# ---------------------------------------------------------------- device CSR helpers
@dataclass
class DCsr:
    """Device CSR: row_ptr int64[n+1], col int64 (global ids), val float64."""

    rp: object
    col: object
    val: object

    @property
    def nrows(self):
        return self.rp.numel() - 1

    @property
    def nnz(self):
        return self.col.numel()

    def lens(self):
        return self.rp[1:] - self.rp[:-1]


def _torch():
    import torch

    return torch


def _count_fill(n, dev, count, fill):
    """Run a count/fill pair of library calls; returns DCsr."""
    torch = _torch()
    cnt = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    if n:
        count(cnt)
    rp = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    if n:
        torch.cumsum(cnt[:n], 0, out=rp[1:])
    nnz = int(rp[-1].item())
    col = torch.empty(nnz, dtype=torch.int64, device=dev)
    val = torch.empty(nnz, dtype=torch.float64, device=dev)
    if n and nnz:
        fill(rp, col, val)
    return DCsr(rp, col, val)


def _ragged(starts, lens):
    """Concatenated ranges [starts[r], starts[r] + lens[r]) (device int64)."""
    torch = _torch()
    total = int(lens.sum().item()) if lens.numel() else 0
    if total == 0:
        return torch.zeros(0, dtype=torch.int64, device=starts.device)
    rid = torch.repeat_interleave(torch.arange(lens.numel(), device=starts.device), lens)
    first = torch.cumsum(lens, 0) - lens
    return starts[rid] + (torch.arange(total, device=starts.device) - first[rid])


def _rows_of(lens):
    torch = _torch()
    return torch.repeat_interleave(torch.arange(lens.numel(), device=lens.device), lens)


def _sell(c, csr, ncols):
    """SELL DeviceMatrix from a device CSR with local columns."""
    if csr.nnz > (1 << 27):  # the library allocates outside torch's cache: return cached blocks first
        _torch().cuda.empty_cache()
    h = N._VP()
    with c.scope():
        N.check(_lib().amgp_mat_from_dcsr(c.handle, csr.nrows, int(ncols), _p(csr.rp), _p(csr.col),
                                          _p(csr.val), 1, C.byref(h)))
    return DeviceMatrix(h, c, csr.nrows, int(ncols), csr.nnz)


def _nown(D):
    v = C.c_int64()
    N.check(_lib().amgp_mat_nown(D.handle, C.byref(v)))
    return v.value


# ---------------------------------------------------------------- halo exchange of setup data
class Exchanger:
    """Neighbour exchange of one row-distributed level over torch.distributed:
    rank p sends the own rows send_idx (grouped by destination, ascending)
    and receives its halo rows (grouped by source = ascending global order)."""

    def __init__(self, send_idx, send_counts, recv_counts):
        self.send_idx = send_idx          # device int64
        self.send_counts = list(map(int, send_counts))  # per rank
        self.recv_counts = list(map(int, recv_counts))

    @property
    def nhalo(self):
        return sum(self.recv_counts)

    def values(self, x):
        import torch.distributed as dist

        torch = _torch()
        out = torch.empty(self.nhalo, dtype=x.dtype, device=x.device)
        _a2a(out, x[self.send_idx].contiguous(), self.recv_counts, self.send_counts)
        return out

    def rows(self, m):
        """Halo rows of a row-distributed DCsr (own rows) -> DCsr (halo order)."""
        import torch.distributed as dist

        torch = _torch()
        dev = m.rp.device
        lens = m.lens()[self.send_idx]
        rl = torch.empty(self.nhalo, dtype=torch.int64, device=dev)
        _a2a(rl, lens.contiguous(), self.recv_counts, self.send_counts)
        ent_send = _split_sums(lens, self.send_counts)
        ent_recv = _split_sums(rl, self.recv_counts)
        idx = _ragged(m.rp[self.send_idx], lens)
        col = torch.empty(sum(ent_recv), dtype=torch.int64, device=dev)
        val = torch.empty(sum(ent_recv), dtype=torch.float64, device=dev)
        _a2a(col, m.col[idx].contiguous(), ent_recv, ent_send)
        _a2a(val, m.val[idx].contiguous(), ent_recv, ent_send)
        rp = torch.zeros(self.nhalo + 1, dtype=torch.int64, device=dev)
        if self.nhalo:
            torch.cumsum(rl, 0, out=rp[1:])
        return DCsr(rp, col, val)


def _a2a(out, inp, out_splits=None, in_splits=None):
    """all_to_all_single; gloo process groups get host copies."""
    import torch.distributed as dist

    if dist.get_backend() == "gloo" and out.is_cuda:
        o = out.cpu()
        dist.all_to_all_single(o, inp.cpu(), out_splits, in_splits)
        out.copy_(o)
    else:
        dist.all_to_all_single(out, inp, out_splits, in_splits)


def _all_gather(outs, t):
    import torch.distributed as dist

    if dist.get_backend() == "gloo" and t.is_cuda:
        oc = [o.cpu() for o in outs]
        dist.all_gather(oc, t.cpu())
        for o, h in zip(outs, oc):
            o.copy_(h)
    else:
        dist.all_gather(outs, t)


def _split_sums(x, counts):
    """Sums of consecutive segments of x of the given lengths (host ints)."""
    torch = _torch()
    if not counts:
        return []
    if x.numel() == 0:
        return [0] * len(counts)
    cs = torch.cumsum(x, 0)
    ends = np.cumsum(counts)
    out, prev = [], 0
    tot = cs[torch.as_tensor(np.maximum(ends - 1, 0), device=x.device)].tolist()
    for i, cnt in enumerate(counts):
        cur = tot[i] if cnt else prev
        out.append(int(cur - prev))
        prev = cur
    return out


def _all_gather_ints(vals, dev):
    import torch.distributed as dist

    torch = _torch()
    t = torch.as_tensor(np.asarray(vals, dtype=np.int64), device=dev)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    _all_gather(out, t)
    return np.stack([o.cpu().numpy() for o in out])


def _all_to_all_counts(counts, dev):
    import torch.distributed as dist

    torch = _torch()
    t = torch.as_tensor(np.asarray(counts, dtype=np.int64), device=dev)
    out = torch.empty_like(t)
    _a2a(out, t)
    return out.cpu().tolist()


def make_halo(cols, lo, hi, off, me):
    """Localise global columns of a rank's rows against the column partition
    `off` (own block [lo, hi)): returns (local cols, halo global ids, HaloPlan,
    Exchanger).  Own columns map to [0, nown), halo columns to nown + their
    rank in the sorted halo list (grouped by owner, ascending)."""
    import torch.distributed as dist

    from .dist import HaloPlan

    torch = _torch()
    dev = cols.device
    nranks = len(off) - 1
    nown = hi - lo
    own = (cols >= lo) & (cols < hi)
    halo_g = torch.unique(cols[~own])
    local = torch.where(own, cols - lo, nown + torch.searchsorted(halo_g, cols))
    off_t = torch.as_tensor(np.asarray(off, dtype=np.int64), device=dev)
    owner = torch.searchsorted(off_t, halo_g, right=True) - 1
    recv_counts = torch.bincount(owner, minlength=nranks).cpu().tolist() if halo_g.numel() else [0] * nranks
    send_counts = _all_to_all_counts(recv_counts, dev)
    need = torch.empty(sum(send_counts), dtype=torch.int64, device=dev)
    _a2a(need, halo_g.contiguous(), send_counts, recv_counts)
    send_idx = need - lo
    peers = [q for q in range(nranks) if q != me and (recv_counts[q] or send_counts[q])]
    plan = HaloPlan(
        nown=nown, peers=np.array(peers, dtype=np.int32),
        recv_cnt=np.array([recv_counts[q] for q in peers], dtype=np.int64),
        send_cnt=np.array([send_counts[q] for q in peers], dtype=np.int64),
        send_idx=send_idx.cpu().numpy(), recv_cols=[])
    return local, halo_g, plan, Exchanger(send_idx, send_counts, recv_counts)


def exchanger_of(plan, nranks, dev):
    """Exchanger for an existing HaloPlan (numpy)."""
    torch = _torch()
    sc, rc = [0] * nranks, [0] * nranks
    for q, s, r in zip(plan.peers, plan.send_cnt, plan.recv_cnt):
        sc[int(q)], rc[int(q)] = int(s), int(r)
    return Exchanger(torch.as_tensor(np.asarray(plan.send_idx, dtype=np.int64), device=dev), sc, rc)


# ---------------------------------------------------------------- one level
@dataclass
class DLevel:
    A: DeviceMatrix
    n: int                      # global rows
    off: object                 # row partition offsets (np) or None (one GPU / replicated)
    lo: int
    hi: int
    halo_g: object = None       # device int64: global ids of A's halo columns
    plan: object = None         # HaloPlan (numpy) of A
    exch: object = None         # Exchanger of A's halo
    m: object = None            # l1 diagonal (device)
    P: DeviceMatrix = None
    R: DeviceMatrix = None
    n_aggregates: int = 0

    @property
    def distributed(self):
        return self.off is not None


def _start_vector(n, lo, hi):
    """Rows [lo, hi) of the reference's power-iteration start vector
    ones + default_rng(0).uniform(-0.5, 0.5, n) (amg.py:207); PCG64 draws one
    64-bit word per double, so the slice is an exact advance."""
    rng = np.random.default_rng(0)
    if lo:
        rng.bit_generator.advance(int(lo))
    return np.ones(hi - lo) + rng.uniform(-0.5, 0.5, hi - lo)


def _aggregate_sa(L, d, theta, c):
    """Decoupled SA aggregation of the rank's block (amg.py:102-149)."""
    torch = _torch()
    A = L.A
    n = A.nrows
    nown = _nown(A)
    lib = _lib()
    dev = c.device
    cnt = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    N.check(lib.amgp_ds_strength(A.handle, _p(d), float(theta), nown, None, n, None, _p(cnt), None, None))
    srp = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(cnt[:n], 0, out=srp[1:])
    ns = int(srp[-1].item())
    scol = torch.empty(max(ns, 1), dtype=torch.int32, device=dev)
    N.check(lib.amgp_ds_strength(A.handle, _p(d), float(theta), nown, None, n, _p(srp), None, _p(scol), None))
    srp_h = srp.cpu().numpy()
    scol_h = scol[:ns].cpu().numpy()
    del scol, cnt
    agg = np.empty(n, dtype=np.int64)
    n_agg = C.c_int64()
    N.check(lib.amgp_setup_sa_pass1(n, srp_h.ctypes.data_as(N._P64), scol_h.ctypes.data_as(_I32P),
                                    agg.ctypes.data_as(N._P64), C.byref(n_agg)))
    del srp_h, scol_h
    left = np.flatnonzero(agg < 0).astype(np.int64)
    if left.size:
        rows = torch.as_tensor(left, device=dev)
        lc = torch.empty(left.size, dtype=torch.int64, device=dev)
        N.check(lib.amgp_ds_strength(A.handle, _p(d), float(theta), nown, _p(rows), left.size, None, _p(lc),
                                     None, None))
        lrp = torch.zeros(left.size + 1, dtype=torch.int64, device=dev)
        torch.cumsum(lc, 0, out=lrp[1:])
        nl = int(lrp[-1].item())
        lcol = torch.empty(max(nl, 1), dtype=torch.int32, device=dev)
        labs = torch.empty(max(nl, 1), dtype=torch.float64, device=dev)
        N.check(lib.amgp_ds_strength(A.handle, _p(d), float(theta), nown, _p(rows), left.size, _p(lrp), None,
                                     _p(lcol), _p(labs)))
        lrp_h, lcol_h, labs_h = lrp.cpu().numpy(), lcol.cpu().numpy(), labs.cpu().numpy()
        N.check(lib.amgp_setup_sa_pass2(left.size, left.ctypes.data_as(N._P64), lrp_h.ctypes.data_as(N._P64),
                                        lcol_h.ctypes.data_as(_I32P), labs_h.ctypes.data_as(N._PD),
                                        agg.ctypes.data_as(N._P64), C.byref(n_agg)))
    return agg, n_agg.value


def _aggregate_matching(L, sweeps):
    """Decoupled pairwise matching of the rank's block (amg.py:152-191, host)."""
    A = L.A
    nown = _nown(A)
    H = A.to_csr()
    rp, ci, v = H.row_ptr, H.col_idx, H.values
    keep = ci < nown
    rows = np.repeat(np.arange(H.nrows), np.diff(rp))
    ci, v, rows = ci[keep], v[keep], rows[keep]
    rp2 = np.zeros(H.nrows + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=H.nrows), out=rp2[1:])
    ci = np.ascontiguousarray(ci, dtype=np.int64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    agg = np.empty(H.nrows, dtype=np.int64)
    n_agg = C.c_int64()
    N.check(_lib().amgp_setup_matching_aggregate(H.nrows, rp2.ctypes.data_as(N._P64), ci.ctypes.data_as(N._P64),
                                                 v.ctypes.data_as(N._PD), int(sweeps), agg.ctypes.data_as(N._P64),
                                                 C.byref(n_agg)))
    return agg, n_agg.value


def _spgemm(c, n_out, b, a_sell=None, a_csr=None, a_rows=None, b_off=0):
    torch = _torch()
    lib = _lib()
    ah = a_sell.handle if a_sell is not None else None
    arp, acol, aval = (a_csr.rp, a_csr.col, a_csr.val) if a_csr is not None else (None, None, None)

    def count(cnt):
        N.check(lib.amgp_ds_spgemm(c.handle, ah, _p(arp), _p(acol), _p(aval), _p(a_rows), n_out, _p(b.rp),
                                   _p(b.col), _p(b.val), int(b_off), None, _p(cnt), None, None))

    def fill(rp, col, val):
        N.check(lib.amgp_ds_spgemm(c.handle, ah, _p(arp), _p(acol), _p(aval), _p(a_rows), n_out, _p(b.rp),
                                   _p(b.col), _p(b.val), int(b_off), _p(rp), None, _p(col), _p(val)))

    return _count_fill(n_out, c.device, count, fill)


def _concat(a, b):
    torch = _torch()
    rp = torch.cat([a.rp, b.rp[1:] + a.rp[-1]])
    return DCsr(rp, torch.cat([a.col, b.col]), torch.cat([a.val, b.val]))


def _csr_from_entries(nrows, rows, cols, vals, key):
    """CSR of entries (rows, cols, vals) ordered by `key` (unique per entry)."""
    torch = _torch()
    order = torch.argsort(key)
    rows, cols, vals = rows[order], cols[order], vals[order]
    rp = torch.zeros(nrows + 1, dtype=torch.int64, device=cols.device)
    if rows.numel():
        torch.cumsum(torch.bincount(rows, minlength=nrows), 0, out=rp[1:])
    return DCsr(rp, cols.contiguous(), vals.contiguous())


def _gather_rows(m, comm_size):
    """All-gather a row-distributed DCsr (rank order) onto every rank."""
    import torch.distributed as dist

    torch = _torch()
    sizes = _all_gather_ints([m.nrows, m.nnz], m.rp.device)
    nr, nz = sizes[:, 0], sizes[:, 1]
    dev = m.rp.device

    def gather(x, counts, dtype):
        mx = int(counts.max()) if len(counts) else 0
        buf = torch.zeros(max(mx, 1), dtype=dtype, device=dev)
        buf[: x.numel()] = x
        outs = [torch.empty_like(buf) for _ in range(comm_size)]
        _all_gather(outs, buf)
        return torch.cat([o[: int(cnt)] for o, cnt in zip(outs, counts)])

    lens = gather(m.lens(), nr, torch.int64)
    col = gather(m.col, nz, torch.int64)
    val = gather(m.val, nz, torch.float64)
    rp = torch.zeros(lens.numel() + 1, dtype=torch.int64, device=dev)
    torch.cumsum(lens, 0, out=rp[1:])
    return DCsr(rp, col, val)


def _attach(D, plan):
    from .dist import attach_halo

    return attach_halo(D, plan) if plan is not None else D


def _galerkin_chunks(c, L, P, R, R_csr, budget_entries):
    """One-GPU Galerkin G = R (A P) in coarse-row chunks, so that only a
    window of A P is ever resident: chunk [J0, J1) needs the rows of A P
    between the first and last fine row its restriction rows touch.  Two
    sweeps over the chunks (row counts, then rows written in place)."""
    torch = _torch()
    dev = c.device
    lib = _lib()
    n = L.A.nrows
    nc = R.nrows
    cnt = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    N.check(lib.amgp_ds_spgemm(c.handle, L.A.handle, None, None, None, None, n, _p(P.rp), _p(P.col), _p(P.val), 0,
                               None, _p(cnt), None, None))
    ccum = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(cnt[:n], 0, out=ccum[1:])
    del cnt
    total = int(ccum[-1].item())
    nchunks = max(1, math.ceil(total / budget_entries))
    lens = R_csr.lens()
    imin = torch.where(lens > 0, R_csr.col[torch.clamp(R_csr.rp[:-1], max=max(R_csr.nnz - 1, 0))],
                       torch.full_like(lens, n))
    imax = torch.where(lens > 0, R_csr.col[torch.clamp(R_csr.rp[1:] - 1, min=0)], torch.full_like(lens, -1))
    bounds = [nc * k // nchunks for k in range(nchunks + 1)]
    chunks = []
    for k in range(nchunks):
        J0, J1 = bounds[k], bounds[k + 1]
        if J1 > J0:
            w0 = int(imin[J0:J1].min().item())
            w1 = int(imax[J0:J1].max().item()) + 1
            chunks.append((J0, J1, min(w0, w1), max(w0, w1)))
    del imin, imax, lens

    def window(w0, w1):
        rows = torch.arange(w0, w1, dtype=torch.int64, device=dev)
        rp = ccum[w0:w1 + 1] - ccum[w0]
        nnz = int(rp[-1].item())
        Cw = DCsr(rp, torch.empty(nnz, dtype=torch.int64, device=dev),
                  torch.empty(nnz, dtype=torch.float64, device=dev))
        if nnz:
            N.check(lib.amgp_ds_spgemm(c.handle, L.A.handle, None, None, None, _p(rows), w1 - w0, _p(P.rp),
                                       _p(P.col), _p(P.val), 0, _p(Cw.rp), None, _p(Cw.col), _p(Cw.val)))
        return Cw

    gcnt = torch.empty(max(nc, 1), dtype=torch.int64, device=dev)
    for J0, J1, w0, w1 in chunks:  # sweep 1: row counts of G
        Cw = window(w0, w1)
        jr = torch.arange(J0, J1, dtype=torch.int64, device=dev)
        N.check(lib.amgp_ds_spgemm(c.handle, R.handle, None, None, None, _p(jr), J1 - J0, _p(Cw.rp), _p(Cw.col),
                                   _p(Cw.val), int(w0), None, _p(gcnt[J0:J1]), None, None))
        del Cw
    grp = torch.zeros(nc + 1, dtype=torch.int64, device=dev)
    torch.cumsum(gcnt[:nc], 0, out=grp[1:])
    del gcnt
    gnnz = int(grp[-1].item())
    G = DCsr(grp, torch.empty(gnnz, dtype=torch.int64, device=dev), torch.empty(gnnz, dtype=torch.float64, device=dev))
    for J0, J1, w0, w1 in chunks:  # sweep 2: rows written in place
        Cw = window(w0, w1)
        jr = torch.arange(J0, J1, dtype=torch.int64, device=dev)
        rp = grp[J0:J1 + 1] - grp[J0]
        o = int(grp[J0].item())
        N.check(lib.amgp_ds_spgemm(c.handle, R.handle, None, None, None, _p(jr), J1 - J0, _p(Cw.rp), _p(Cw.col),
                                   _p(Cw.val), int(w0), _p(rp), None, _p(G.col[o:]), _p(G.val[o:])))
        del Cw
    return G


# ---------------------------------------------------------------- the setup
def build_levels(A0, coarsening, max_levels=10, min_coarse_size=200, comm=None, replicate_below=20000,
                 galerkin_budget=None, trace=None):
    """Device setup of every level.  A0: a DeviceMatrix (one GPU: global
    columns; several GPUs: the rank's row block, localised, halo attached,
    with ``global_rows`` and ``halo_g`` set) or a CsrMatrix (one GPU).
    Returns (levels: list of DLevel, stagnated)."""
    import time

    from .sparse import CsrMatrix

    torch = _torch()
    c = comm.ctx if comm is not None else (A0.ctx if isinstance(A0, DeviceMatrix) else N.ctx())
    dev = c.device
    lib = _lib()
    size = comm.size if comm is not None else 1
    me = comm.rank if comm is not None else 0
    budget = galerkin_budget or int(os.environ.get("AMGP_GALERKIN_BUDGET", str(1 << 28)))
    t_start = time.perf_counter()

    if trace is None and os.environ.get("AMGP_SETUP_TRACE"):
        import sys

        trace = lambda s: print(f"[rank {me}] {s}", file=sys.stderr, flush=True)  # noqa: E731

    def log(msg):
        if trace:
            trace(f"[dsetup {time.perf_counter() - t_start:8.2f}s] {msg}")

    with c.scope():
        if isinstance(A0, CsrMatrix):
            D0 = DeviceMatrix.from_csr(A0, c)
            L = DLevel(A=D0, n=A0.nrows, off=None, lo=0, hi=A0.nrows)
        elif size > 1 and getattr(A0, "halo", None) is not None:
            lo, hi = A0.global_rows
            n = int(A0.n_global)
            L = DLevel(A=A0, n=n, off=np.asarray(A0.row_partition, dtype=np.int64), lo=lo, hi=hi,
                       halo_g=A0.halo_g, plan=A0.halo, exch=exchanger_of(A0.halo, size, dev))
        else:
            L = DLevel(A=A0, n=A0.nrows, off=None, lo=0, hi=A0.nrows)
        L.m = L.A.l1_diag()
        levels = [L]
        stagnated = 0
        while L.n > min_coarse_size and len(levels) < max_levels and stagnated < 2:
            A = L.A
            dist_l = L.distributed
            n_loc = A.nrows
            d = torch.empty(max(n_loc, 1), dtype=torch.float64, device=dev)
            N.check(lib.amgp_ds_diag(A.handle, _p(d)))
            # -- aggregation (host greedy over device strength lists)
            if coarsening.kind == "smoothed_aggregation":
                agg, na = _aggregate_sa(L, d, coarsening.strength_theta, c)
            else:
                agg, na = _aggregate_matching(L, coarsening.matching_sweeps)
            if dist_l:
                coff = np.concatenate([[0], np.cumsum(_all_gather_ints([na], dev)[:, 0])]).astype(np.int64)
            else:
                coff = np.array([0, na], dtype=np.int64)
            nc = int(coff[-1])
            clo = int(coff[me]) if dist_l else 0
            chi = clo + na
            log(f"level {len(levels) - 1}: n={L.n} aggregates={nc}")
            agg_g = torch.as_tensor(agg + clo, device=dev)
            del agg
            # -- smoothed prolongator
            if coarsening.prolongator_smoothing:
                v = torch.as_tensor(_start_vector(L.n, L.lo, L.hi), device=dev)
                lam = C.c_double()
                N.check(lib.amgp_ds_lambda_max(c.handle, A.handle, _p(d), _p(v), 25, blas_threads(),
                                               int(dist_l), C.byref(lam)))
                lam = lam.value
                omega = 4.0 / (3.0 * lam)
                del v
                agg_h = L.exch.values(agg_g) if dist_l else torch.zeros(1, dtype=torch.int64, device=dev)
            else:
                omega = 0.0
                agg_h = torch.zeros(1, dtype=torch.int64, device=dev)
            smooth = int(coarsening.prolongator_smoothing)

            def pcount(cnt):
                N.check(lib.amgp_ds_prolongator(A.handle, _p(d), _p(agg_g), _p(agg_h), float(omega), smooth,
                                                None, _p(cnt), None, None))

            def pfill(rp, col, val):
                N.check(lib.amgp_ds_prolongator(A.handle, _p(d), _p(agg_g), _p(agg_h), float(omega), smooth,
                                                _p(rp), None, _p(col), _p(val)))

            Prow = _count_fill(n_loc, dev, pcount, pfill)
            del agg_g, agg_h, d
            log(f"  P rows: nnz={Prow.nnz} omega={omega!r}")
            # amg.py:272-277 (global sizes)
            if nc >= 0.95 * L.n:
                stagnated += 1
            else:
                stagnated = 0
            if nc >= L.n:
                break
            replicate_next = dist_l and nc < replicate_below
            # -- restriction rows R = P^T for own coarse rows (ext = own + halo fine rows)
            Pext = _concat(Prow, L.exch.rows(Prow)) if dist_l else Prow
            n_ext = Pext.nrows
            if dist_l:
                ext_g = torch.cat([torch.arange(L.lo, L.hi, dtype=torch.int64, device=dev), L.halo_g])
            else:
                ext_g = torch.arange(n_ext, dtype=torch.int64, device=dev)
            erow = _rows_of(Pext.lens())
            keep = (Pext.col >= clo) & (Pext.col < chi)
            J = Pext.col[keep] - clo
            I = erow[keep]
            R_csr = _csr_from_entries(na, J, I, Pext.val[keep], J * max(L.n, 1) + ext_g[I])
            del erow, keep, J, I
            R = _attach(_sell(c, R_csr, A.ncols), L.plan if dist_l else None)
            R.col_map, R.row_lo = (ext_g if dist_l else None), clo
            # P as a device matrix (columns: coarse level, localised when it stays distributed)
            if dist_l and not replicate_next:
                pl, phg, pplan, _ = make_halo(Prow.col, clo, chi, coff, me)
                P = _attach(_sell(c, DCsr(Prow.rp, pl, Prow.val), pplan.nown + int(pplan.recv_cnt.sum())), pplan)
                P.col_map = torch.cat([torch.arange(clo, chi, dtype=torch.int64, device=dev), phg])
            else:
                P = _sell(c, Prow, nc)
                P.col_map = None
            P.row_lo = L.lo
            # -- Galerkin (amg.py:229-235)
            if dist_l:
                Cm = _spgemm(c, n_loc, Pext, a_sell=A)
                del Pext
                Cext = _concat(Cm, L.exch.rows(Cm))
                del Cm
                G = _spgemm(c, na, Cext, a_sell=R)
                del Cext
            else:
                G = _galerkin_chunks(c, L, Prow, R, R_csr, budget)
            del Prow
            R_g = DCsr(R_csr.rp, ext_g[R_csr.col], R_csr.val) if replicate_next else None
            del R_csr
            log(f"  G: nnz={G.nnz}")
            if dist_l:
                # G^T restricted to own rows: entries with a foreign column go to its owner
                import torch.distributed as dist

                Gr = _rows_of(G.lens()) + clo
                coff_t = torch.as_tensor(coff, device=dev)
                dest = torch.searchsorted(coff_t, G.col, right=True) - 1
                order = torch.argsort(dest, stable=True)
                send_counts = torch.bincount(dest, minlength=size).cpu().tolist()
                recv_counts = _all_to_all_counts(send_counts, dev)
                tr, tc, tv = (torch.empty(sum(recv_counts), dtype=dt, device=dev)
                              for dt in (torch.int64, torch.int64, torch.float64))
                _a2a(tr, G.col[order].contiguous(), recv_counts, send_counts)
                _a2a(tc, Gr[order].contiguous(), recv_counts, send_counts)
                _a2a(tv, G.val[order].contiguous(), recv_counts, send_counts)
                del dest, order, Gr
                Gt = _csr_from_entries(na, tr - clo, tc, tv, (tr - clo) * max(nc, 1) + tc)
                del tr, tc, tv

                def scount(cnt):
                    N.check(lib.amgp_ds_symmetrize(c.handle, na, _p(G.rp), _p(G.col), _p(G.val), _p(Gt.rp),
                                                   _p(Gt.col), _p(Gt.val), None, _p(cnt), None, None))

                def sfill(rp, col, val):
                    N.check(lib.amgp_ds_symmetrize(c.handle, na, _p(G.rp), _p(G.col), _p(G.val), _p(Gt.rp),
                                                   _p(Gt.col), _p(Gt.val), _p(rp), None, _p(col), _p(val)))
            else:
                # one GPU: G^T values looked up in G itself (no transposed copy)
                gt = torch.empty(max(G.nnz, 1), dtype=torch.float64, device=dev)
                cap = 1 << 16
                while True:
                    orow = torch.empty(cap, dtype=torch.int64, device=dev)
                    ocol = torch.empty(cap, dtype=torch.int64, device=dev)
                    oval = torch.empty(cap, dtype=torch.float64, device=dev)
                    no = C.c_int64()
                    N.check(lib.amgp_ds_sym_lookup(c.handle, na, _p(G.rp), _p(G.col), _p(G.val), _p(gt), _p(orow),
                                                   _p(ocol), _p(oval), cap, C.byref(no)))
                    if no.value <= cap:
                        break
                    cap = no.value
                no = no.value
                O = _csr_from_entries(na, orow[:no], ocol[:no], oval[:no], orow[:no] * max(nc, 1) + ocol[:no])
                del orow, ocol, oval
                Gt = None

                def scount(cnt):
                    N.check(lib.amgp_ds_symmetrize_lookup(c.handle, na, _p(G.rp), _p(G.col), _p(G.val), _p(gt),
                                                          _p(O.rp), _p(O.col), _p(O.val), None, _p(cnt), None, None))

                def sfill(rp, col, val):
                    N.check(lib.amgp_ds_symmetrize_lookup(c.handle, na, _p(G.rp), _p(G.col), _p(G.val), _p(gt),
                                                          _p(O.rp), _p(O.col), _p(O.val), _p(rp), None, _p(col),
                                                          _p(val)))

            Ac = _count_fill(na, dev, scount, sfill)
            del G, Gt
            if not dist_l:
                del gt, O
            log(f"  A_c: nnz={Ac.nnz}")
            # -- next level
            L.n_aggregates = nc
            L.P = P
            if replicate_next:
                # coarse agglomeration: every rank gets the whole coarse level,
                # and the restriction into it all rows of P^T
                Afull = _gather_rows(Ac, size)
                Rfull = _gather_rows(R_g, size)
                rl, rhg, rplan, _ = make_halo(Rfull.col, L.lo, L.hi, L.off, me)
                L.R = _attach(_sell(c, DCsr(Rfull.rp, rl, Rfull.val), rplan.nown + sum(rplan.recv_cnt)), rplan)
                L.R.col_map = torch.cat([torch.arange(L.lo, L.hi, dtype=torch.int64, device=dev), rhg])
                L.R.row_lo = 0
                del R, Rfull, R_g
                nxt = DLevel(A=_sell(c, Afull, nc), n=nc, off=None, lo=0, hi=nc)
                del Afull
            elif dist_l:
                L.R = R
                al, hg, aplan, aex = make_halo(Ac.col, clo, chi, coff, me)
                Aloc = DCsr(Ac.rp, al, Ac.val)
                nxt = DLevel(A=_attach(_sell(c, Aloc, na + int(hg.numel())), aplan), n=nc, off=coff, lo=clo,
                             hi=chi, halo_g=hg, plan=aplan, exch=aex)
                nxt.A.col_map = torch.cat([torch.arange(clo, chi, dtype=torch.int64, device=dev), hg])
                del Aloc, al
            else:
                L.R = R
                nxt = DLevel(A=_sell(c, Ac, nc), n=nc, off=None, lo=0, hi=nc)
            del Ac, ext_g
            torch.cuda.empty_cache()
            nxt.m = nxt.A.l1_diag()
            levels.append(nxt)
            L = nxt
    return levels, stagnated >= 2
