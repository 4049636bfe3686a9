"""Multi-GPU execution: one process per GPU, every AMG level row-partitioned.

The reference is a single process; the paper runs
the same algorithm over MPI ranks with descriptor-based halos (PAPER.md:
1018, 1067).  Here each torch.distributed rank drives one GPU:

* every level's rows are split into contiguous blocks (``block_partition``);
  columns are renumbered locally -- own entries first, then the halo grouped
  by owner rank in ascending global order (``localize``); the halo plan says
  which own entries each neighbour needs;
* the library exchanges halos with NCCL send/recv on a side stream while the
  interior rows compute (csrc/dist.cu, csrc/rows.cuh), so every SpMV, every
  smoother step and every V-cycle returns the single-GPU bits;
* levels below ``replicate_below`` global rows are replicated on every rank
  (coarse-level agglomeration): the restriction into the first replicated
  level all-gathers its operand through the same halo machinery, and all
  ranks then run the coarse levels redundantly;
* PCG dots are per-rank deterministic partials all-gathered and folded in
  rank order, identical on every rank.

The global hierarchy is built once on the host by the native setup (rank 0)
and shared through a file in /dev/shm; every rank cuts its blocks from it.
"""

from __future__ import annotations

import ctypes as C
import os
import tempfile
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .sparse import CsrMatrix, DeviceMatrix


# ---------------------------------------------------------------- partitions
def block_partition(n, nranks):
    """Offsets of a balanced contiguous row partition (len nranks + 1)."""
    return np.array([p * n // nranks for p in range(nranks + 1)], dtype=np.int64)


@dataclass
class HaloPlan:
    nown: int
    peers: np.ndarray        # int32, ascending
    recv_cnt: np.ndarray     # int64 per peer
    send_cnt: np.ndarray     # int64 per peer
    send_idx: np.ndarray     # int64 own (local) indices, concatenated per peer
    recv_cols: list          # per peer: global columns received (ascending)

    @property
    def nhalo(self):
        return int(self.recv_cnt.sum())


def _rows(A, lo, hi):
    a, b = A.row_ptr[lo], A.row_ptr[hi]
    return A.row_ptr[lo:hi + 1] - a, A.col_idx[a:b], A.values[a:b]


def halo_columns(A, row_lo, row_hi, col_off, me):
    """Global columns referenced by rows [row_lo, row_hi) outside rank me's
    column block, ascending (hence grouped by owner rank)."""
    _, ci, _ = _rows(A, row_lo, row_hi)
    c_lo, c_hi = col_off[me], col_off[me + 1]
    return np.unique(ci[(ci < c_lo) | (ci >= c_hi)])


def localize(A, row_off, col_off, me):
    """Rank me's rows of A with local columns, and the halo plan.

    row_off / col_off: partition offsets of the rows / columns, or None for a
    replicated dimension (every rank holds everything).
    """
    r_lo, r_hi = (int(row_off[me]), int(row_off[me + 1])) if row_off is not None else (0, A.nrows)
    rp, ci, v = _rows(A, r_lo, r_hi)
    if col_off is None:  # replicated operand: nothing to exchange
        return CsrMatrix(r_hi - r_lo, A.ncols, rp, ci.copy(), v.copy()), None
    nranks = len(col_off) - 1
    c_lo, c_hi = int(col_off[me]), int(col_off[me + 1])
    nown = c_hi - c_lo
    halo = halo_columns(A, r_lo, r_hi, col_off, me)
    own = (ci >= c_lo) & (ci < c_hi)
    local = np.empty_like(ci)
    local[own] = ci[own] - c_lo
    local[~own] = nown + np.searchsorted(halo, ci[~own])
    owner = np.searchsorted(col_off, halo, side="right") - 1
    peers, recv_cnt = np.unique(owner, return_counts=True)
    recv_cols = [halo[owner == q] for q in peers]
    # what the other ranks need from me: their halo columns owned by me
    send_cnt, send_idx = [], []
    for q in range(nranks):
        if q == me:
            continue
        q_lo, q_hi = (row_off[q], row_off[q + 1]) if row_off is not None else (0, A.nrows)
        need = halo_columns(A, q_lo, q_hi, col_off, q)
        mine = need[(need >= c_lo) & (need < c_hi)]
        if len(mine):
            send_cnt.append((q, len(mine)))
            send_idx.append(mine - c_lo)
    # peers of a symmetric exchange: union of senders and receivers
    all_peers = sorted(set(int(q) for q in peers) | {q for q, _ in send_cnt})
    rc = {int(q): int(c) for q, c in zip(peers, recv_cnt)}
    sc = dict(send_cnt)
    sidx = {q: idx for (q, _), idx in zip(send_cnt, send_idx)}
    plan = HaloPlan(
        nown=nown,
        peers=np.array(all_peers, dtype=np.int32),
        recv_cnt=np.array([rc.get(q, 0) for q in all_peers], dtype=np.int64),
        send_cnt=np.array([sc.get(q, 0) for q in all_peers], dtype=np.int64),
        send_idx=(np.concatenate([sidx[q] for q in all_peers if q in sidx]).astype(np.int64)
                  if sidx else np.zeros(0, dtype=np.int64)),
        recv_cols=[recv_cols[list(peers).index(q)] if q in rc else np.zeros(0, np.int64)
                   for q in all_peers],
    )
    return CsrMatrix(r_hi - r_lo, nown + len(halo), rp, local, v.copy()), plan


def level_partitions(h, nranks, replicate_below=20000):
    """Row partition per level: offsets, or None once the level is replicated."""
    parts = []
    replicated = False
    for l, lv in enumerate(h.levels):
        n = lv.A.nrows
        if l > 0 and (replicated or n < replicate_below or n < 4 * nranks):
            replicated = True
        parts.append(None if replicated or nranks == 1 else block_partition(n, nranks))
    return parts


# ---------------------------------------------------------------- communicator
class Communicator:
    """NCCL communicator inside libamgp, bootstrapped over torch.distributed."""

    def __init__(self, device=None):
        import torch
        import torch.distributed as dist

        self.rank = dist.get_rank()
        self.size = dist.get_world_size()
        dev = torch.cuda.current_device() if device is None else device
        self.ctx = N.ctx(dev)
        buf = C.create_string_buffer(128)
        if self.rank == 0:
            N.check(N.lib().amgp_comm_unique_id(buf))
        obj = [bytes(buf.raw) if self.rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        N.check(N.lib().amgp_ctx_init_comm(self.ctx.handle, self.size, self.rank, obj[0]))


def attach_halo(D, plan):
    """Give a DeviceMatrix its halo plan (libamgp amgp_mat_set_halo)."""
    if plan is None:
        return D
    peers = np.ascontiguousarray(plan.peers, dtype=np.int32)
    sc = np.ascontiguousarray(plan.send_cnt, dtype=np.int64)
    si = np.ascontiguousarray(plan.send_idx, dtype=np.int64)
    rc = np.ascontiguousarray(plan.recv_cnt, dtype=np.int64)
    N.check(N.lib().amgp_mat_set_halo(D.handle, int(plan.nown), len(peers),
                                      peers.ctypes.data_as(C.POINTER(C.c_int)),
                                      sc.ctypes.data_as(N._P64), si.ctypes.data_as(N._P64),
                                      rc.ctypes.data_as(N._P64)))
    D.halo = plan
    return D


# ---------------------------------------------------------------- fine-level block (bench)
def poisson3d_block(m, comm, stencil=7):
    """Rank's contiguous row block of the m^3 Poisson matrix generated on its
    GPU, localized, with the halo plan of the neighbouring planes."""
    n = m ** 3
    off = block_partition(n, comm.size)
    me = comm.rank
    lo, hi = int(off[me]), int(off[me + 1])
    D = DeviceMatrix.poisson3d(m, stencil, lo, hi)
    hw = m * m if stencil == 7 else m * m + m + 1
    # halo columns: [lo - hw, lo) and [hi, hi + hw), split by owner rank
    def segments(a, b):
        out = []
        for q in range(comm.size):
            s, e = max(a, int(off[q])), min(b, int(off[q + 1]))
            if s < e and q != me:
                out.append((q, s, e))
        return out

    segs = segments(max(lo - hw, 0), lo) + segments(hi, min(hi + hw, n))
    seg_lo = np.array([s for _, s, _ in segs], dtype=np.int64)
    seg_hi = np.array([e for _, _, e in segs], dtype=np.int64)
    D.l1_diag()  # global columns still in place: diagonal at row_offset + i
    N.check(N.lib().amgp_mat_localize(D.handle, lo, hi, len(segs), seg_lo.ctypes.data_as(N._P64),
                                      seg_hi.ctypes.data_as(N._P64)))
    D.ncols = D.info()["ncols"]
    # send lists: neighbour q's halo intersected with my block, ascending
    peers, rc, sc, sidx = [], [], [], []
    for q in range(comm.size):
        if q == me:
            continue
        qlo, qhi = int(off[q]), int(off[q + 1])
        recv = sum(e - s for p, s, e in segs if p == q)
        need = [(max(qlo - hw, 0), qlo), (qhi, min(qhi + hw, n))]
        mine = [np.arange(max(a, lo), min(b, hi), dtype=np.int64) for a, b in need if max(a, lo) < min(b, hi)]
        mine = np.concatenate(mine) if mine else np.zeros(0, np.int64)
        if recv or len(mine):
            peers.append(q)
            rc.append(recv)
            sc.append(len(mine))
            sidx.append(mine - lo)
    plan = HaloPlan(nown=hi - lo, peers=np.array(peers, dtype=np.int32),
                    recv_cnt=np.array(rc, dtype=np.int64), send_cnt=np.array(sc, dtype=np.int64),
                    send_idx=np.concatenate(sidx) if sidx else np.zeros(0, np.int64),
                    recv_cols=[])
    attach_halo(D, plan)
    D.global_rows = (lo, hi)
    D.n_global = n
    D.row_partition = off
    # global ids of the halo columns in local order (device setup, dsetup.py)
    import torch

    D.halo_g = torch.cat([torch.arange(a, b, dtype=torch.int64) for _, a, b in segs]).to(comm.ctx.device) \
        if segs else torch.zeros(0, dtype=torch.int64, device=comm.ctx.device)
    D.col_map = torch.cat([torch.arange(lo, hi, dtype=torch.int64, device=comm.ctx.device), D.halo_g])
    return D


# ---------------------------------------------------------------- hierarchy
class _SharedArrays:
    """Mapping key -> array over a directory of .npy files (memory-mapped, so
    every rank reads only the row blocks it cuts and the page cache is shared)."""

    def __init__(self, path):
        self.path = path
        self._cache = {}

    def __getitem__(self, key):
        if key not in self._cache:
            self._cache[key] = np.load(os.path.join(self.path, key + ".npy"), mmap_mode="r")
        return self._cache[key]

    def __contains__(self, key):
        return os.path.exists(os.path.join(self.path, key + ".npy"))


def share_hierarchy(h_or_builder, comm_rank, barrier, cache=None):
    """Rank 0 builds (callable) or holds the host hierarchy and writes its
    arrays as .npy files to /dev/shm (or the temp dir when /dev/shm is too
    small); every rank memory-maps them.  Returns (arrays, directory).
    cache: a directory kept across runs -- reused when it holds a complete
    hierarchy (e.g. one setup for a strong-scaling sweep over world sizes),
    else written there; the caller does not release it."""
    import shutil

    name = f"amgp_hier_{os.environ.get('MASTER_PORT', '0')}"
    where = os.path.join(tempfile.gettempdir(), name + ".where")
    if cache is not None and os.path.exists(os.path.join(cache, "complete")):
        barrier()
        return _SharedArrays(cache), cache
    if comm_rank == 0:
        h = h_or_builder() if callable(h_or_builder) else h_or_builder
        need = 2 * sum(lv.A.nnz * 16 + (lv.P.nnz * 32 if lv.P is not None else 0) for lv in h.levels)
        base = os.environ.get("AMGP_SHM")
        if base is None:  # /dev/shm when it has room (containers often cap it at 64 MB)
            base = tempfile.gettempdir()
            if os.path.isdir("/dev/shm") and shutil.disk_usage("/dev/shm").free > need:
                base = "/dev/shm"
        path = cache if cache is not None else os.path.join(base, name)
        shutil.rmtree(path, ignore_errors=True)
        os.makedirs(path)
        arrs = {"nlev": np.array([len(h.levels)]), "coarse_sweeps": np.array([h.coarse_sweeps]),
                "coarse_solver": np.array([h.coarse_solver])}
        for l, lv in enumerate(h.levels):
            for key, M in (("A", lv.A), ("P", lv.P), ("R", lv.restrict_op() if lv.P is not None else None)):
                if M is None:
                    continue
                arrs[f"{key}{l}_shape"] = np.array([M.nrows, M.ncols])
                arrs[f"{key}{l}_rp"], arrs[f"{key}{l}_ci"], arrs[f"{key}{l}_v"] = M.row_ptr, M.col_idx, M.values
            arrs[f"M{l}"] = N.to_host(lv.M.m_diag) if N.is_torch(lv.M.m_diag) else np.asarray(lv.M.m_diag)
        for k, a in arrs.items():
            np.save(os.path.join(path, k + ".npy"), a)
        open(os.path.join(path, "complete"), "w").close()
        with open(where, "w") as f:
            f.write(path)
    barrier()
    if comm_rank != 0:
        with open(where) as f:
            path = f.read().strip()
    return _SharedArrays(path), path


def release_shared(path):
    import shutil

    shutil.rmtree(path, ignore_errors=True)


def _mat(d, key):
    nr, nc = (int(v) for v in d[key + "_shape"])
    return CsrMatrix(nr, nc, np.asarray(d[key + "_rp"]), np.asarray(d[key + "_ci"]), np.asarray(d[key + "_v"]))


class DistHierarchy:
    """This rank's slice of an AMG hierarchy on its GPU (libamgp hierarchy
    with halo-exchanging matrices).  Vectors are the rank's fine-level rows."""

    def __init__(self, d, comm, smoother, replicate_below=20000, coarse_sweeps=None, use_graph=True,
                 coarse_solver=None):
        """Partition a shared global hierarchy (share_hierarchy) by rows."""
        c = comm.ctx
        L = int(d["nlev"][0])
        A_glob = [_mat(d, f"A{l}") for l in range(L)]

        class _H:  # minimal view for level_partitions
            levels = [type("Lv", (), {"A": a}) for a in A_glob]

        parts = level_partitions(_H, comm.size, replicate_below)
        me = comm.rank
        As, Ms, Ps, Rs = [], [], [], []
        plans = []
        for l in range(L):
            Al, plan = localize(A_glob[l], parts[l], parts[l], me)
            DA = attach_halo(DeviceMatrix.from_csr(Al, c), plan)
            lo, hi = (parts[l][me], parts[l][me + 1]) if parts[l] is not None else (0, A_glob[l].nrows)
            m = N.to_device(np.ascontiguousarray(d[f"M{l}"][lo:hi]), c)
            As.append(DA)
            Ms.append(m)
            plans.append(plan)
            if l < L - 1:
                Pl, pplan = localize(_mat(d, f"P{l}"), parts[l], parts[l + 1], me)
                Rl, rplan = localize(_mat(d, f"R{l}"), parts[l + 1], parts[l], me)
                Ps.append(attach_halo(DeviceMatrix.from_csr(Pl, c), pplan))
                Rs.append(attach_halo(DeviceMatrix.from_csr(Rl, c), rplan))
        # the coarse solve of the shared hierarchy (amg.py:65-66), unless overridden
        if coarse_solver is None:
            coarse_solver = str(d["coarse_solver"][0]) if "coarse_solver" in d else "l1_jacobi"
        if coarse_sweeps is None:
            coarse_sweeps = int(d["coarse_sweeps"][0]) if "coarse_sweeps" in d else 30
        row_range = (int(parts[0][me]), int(parts[0][me + 1])) if parts[0] is not None else (0, As[0].nrows)
        self._setup(comm, As, Ms, Ps, Rs, parts, row_range, smoother, coarse_solver, coarse_sweeps, use_graph,
                    coarse_A=A_glob[-1])
        self.plans = plans

    @classmethod
    def from_levels(cls, levels, comm, smoother, coarse_solver="l1_jacobi", coarse_sweeps=30, use_graph=True):
        """Hierarchy from the per-rank levels of the distributed device setup
        (dsetup.build_levels)."""
        self = cls.__new__(cls)
        As = [L.A for L in levels]
        Ms = [L.m for L in levels]
        Ps = [L.P for L in levels[:-1]]
        Rs = [L.R for L in levels[:-1]]
        parts = [L.off for L in levels]
        row_range = (levels[0].lo, levels[0].hi)
        self._setup(comm, As, Ms, Ps, Rs, parts, row_range, smoother, coarse_solver, coarse_sweeps, use_graph,
                    coarse_A=levels[-1].A if levels[-1].off is None else None)
        self.levels = levels
        return self

    def _setup(self, comm, As, Ms, Ps, Rs, parts, row_range, smoother, coarse_solver, coarse_sweeps, use_graph,
               coarse_A=None):
        self.comm = comm
        c = comm.ctx
        self.ctx = c
        L = len(As)
        self.parts = parts
        self.As, self.Ms, self.Ps, self.Rs = As, Ms, Ps, Rs
        self.n_local = As[0].nrows
        self.row_range = row_range
        Aa = (N._VP * L)(*[a.handle for a in As])
        Ma = (N._VP * L)(*[m.data_ptr() for m in Ms])
        Pa = (N._VP * max(L - 1, 1))(*[p.handle for p in Ps])
        Ra = (N._VP * max(L - 1, 1))(*[r.handle for r in Rs])
        if coarse_solver not in N.COARSE_CODES or coarse_solver == "smoother":
            raise ValueError(f"unknown coarse solver {coarse_solver!r}")
        if coarse_solver == "dense_direct" and (parts[-1] is not None and comm.size > 1):
            raise ValueError("dense_direct needs a replicated coarsest level")
        handle = N._VP()
        with c.scope():
            N.check(N.lib().amgp_hier_create(c.handle, L, Aa, Ma, Pa, Ra, N.COARSE_CODES[coarse_solver],
                                             int(coarse_sweeps), C.byref(handle)))
            N.check(N.lib().amgp_hier_use_graph(handle, int(use_graph)))
        self.handle = handle
        if coarse_solver == "dense_direct":
            Ad = coarse_A.to_dense()
            try:
                Lf = np.linalg.cholesky(Ad)
            except np.linalg.LinAlgError as exc:
                raise ValueError("matrix is not positive definite") from exc
            Lc = np.ascontiguousarray(Lf.T)
            N.check(N.lib().amgp_hier_set_coarse_cholesky(handle, Lc.ctypes.data_as(N._PD)))
        self.coarse_solver = coarse_solver
        self.coarse_sweeps = coarse_sweeps
        self.set_smoother(smoother)

    def set_smoother(self, cfg):
        self.smoother = cfg
        s = N.smoother_cfg(cfg)
        N.check(N.lib().amgp_hier_set_smoother(self.handle, -1, C.byref(s)))

    def vcycle(self, r):
        c = self.ctx
        with c.scope():
            rd = N.to_device(r, c)
            z = N.empty(self.n_local, c)
            N.check(N.lib().amgp_vcycle_apply(self.handle, N.ptr(rd), N.ptr(z)))
        return N.like(z, r)

    def solve(self, b, cfg=None, x0=None):
        """Distributed PCG/FCG preconditioned by the distributed V-cycle."""
        from .krylov import KrylovConfig, SolveReport

        cfg = cfg or KrylovConfig()
        c = self.ctx
        rep = N.SolveReportC()
        hist = np.empty(cfg.itmax + 1) if cfg.record_history else None
        with c.scope():
            bd = N.to_device(b, c)
            x = N.to_device(x0, c, copy=True) if x0 is not None else N.empty(self.n_local, c)
            N.check(N.lib().amgp_pcg_solve(
                c.handle, self.As[0].handle, self.handle, N.ptr(bd), N.ptr(x), int(x0 is not None),
                N.VARIANT_CODES[cfg.variant], float(cfg.tol), int(cfg.itmax),
                hist.ctypes.data_as(N._PD) if hist is not None else None, C.byref(rep)))
        report = SolveReport(iterations=rep.iterations, converged=bool(rep.converged),
                             final_relres=rep.final_relres,
                             residual_history=hist[: rep.n_history].tolist() if hist is not None else [],
                             spmv_count=rep.spmv_count, precond_count=rep.precond_count,
                             breakdown=bool(rep.breakdown), elapsed_s=rep.elapsed_s)
        return N.like(x, b), report

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and N._lib is not None:
            try:
                N.lib().amgp_hier_destroy(h)
            except Exception:
                pass
            self.handle = None


def dist_smoother_apply(config, D, m, b, x0):
    """smoother_apply on a rank's row block (own rows of b / x0 / m, device tensors)."""
    from .smoothers import smoother_apply, L1JacobiData

    return smoother_apply(config, D, L1JacobiData(m_diag=m), b, x0)
