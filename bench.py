#!/usr/bin/env python
"""Benchmark: fused polynomial-smoother apply on the 3D Poisson fine level.

Workload (BASELINE.json configs[1]): the 7-point Poisson fine level of a
256^3 grid (n = 16.8M rows, 117M nnz, generated on the GPU), one *step* =
the smoother sweep over opt_cheb1(a*), cheb4 and opt_cheb4 at degrees 1..6
(18 smoother applications, x0 != 0 so all k SpMVs run).  Metric: algorithmic
smoother-apply bytes / time (GB/s) -- SURVEY.md section 8d:
    A = 12 nnz + 4 (n+1);  k = 1: A + 32 n;  k >= 2: k A + (56 k - 24) n.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N > 1 (torchrun, one process per GPU): weak scaling -- the global cube has
m = round(256 N^(1/3)) (N = 8: 512^3), split into N contiguous row blocks of
~256^3 rows; every SpMV exchanges the neighbouring planes with NCCL
send/recv on a side stream while the interior rows compute.
"""

from __future__ import annotations

import argparse
import datetime
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
# the device setup frees and re-allocates large index arrays (BASELINE configs[4]
# on one GPU peaks near 120 GB): keep the caching allocator from fragmenting
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
sys.path.insert(0, REPO)

METRIC = "smoother-apply GB/s (% HBM peak); PCG+AMG solve s & iters, 3D Poisson 1–8 GPU"
SWEEP = [(fam, k) for fam in ("opt_cheb1", "cheb4", "opt_cheb4") for k in range(1, 7)]


def apply_bytes(n, nnz, k):
    A = 12 * nnz + 4 * (n + 1)
    return A + 32 * n if k == 1 else k * A + (56 * k - 24) * n


def mid_step_bytes(n, nnz):
    return 12 * nnz + 4 * (n + 1) + 56 * n


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks.mem,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.f = None

    def start(self):
        """Start sampling; returns once the first sample has been written."""
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return
        t0 = time.time()
        while time.time() - t0 < 10 and self.proc.poll() is None:
            if os.path.getsize(self.f.name) > 0:
                break
            time.sleep(0.05)

    def stop(self, t_begin=None, t_end=None):
        """Stop; summarise the samples taken in [t_begin, t_end] (wall clock),
        or all samples when the window caught none (a very short region)."""
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                p = [x.strip() for x in line.split(",")]
                if len(p) >= 10:
                    try:
                        p[0] = datetime.datetime.strptime(p[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                    except ValueError:
                        continue
                    rows.append(p)
        os.unlink(self.f.name)
        window = "timed region"
        if t_begin is not None:
            inside = [r for r in rows if t_begin <= r[0] <= t_end]
            if inside:
                rows = inside
            else:
                window = "whole run (timed region shorter than the sampling period)"
        if not rows:
            return None

        def num(v):
            try:
                return float(v)
            except ValueError:
                return None

        sm = [num(r[1]) for r in rows if num(r[1]) is not None]
        mx = [num(r[2]) for r in rows if num(r[2]) is not None]
        mem = [num(r[3]) for r in rows if num(r[3]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[6 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "mem_mhz": statistics.median(mem) if mem else None, "reasons": reasons,
                "samples": len(rows), "window": window}


# ---------------------------------------------------------------- distributed
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def traffic_per_launch():
    p = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return None


# ---------------------------------------------------------------- reference arm
def run_reference(args):
    """The reference's algorithm on the host (C oracle port, all host threads)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle
    from paper_2407_09848_b200.params import load_beta_tables, optimal_a
    from paper_2407_09848_b200.problems import poisson3d

    m = args.grid
    from paper_2407_09848_b200.smoothers import l1_jacobi_diag

    A, _ = poisson3d(m)
    n, nnz = A.nrows, A.nnz
    mdiag = l1_jacobi_diag(A).m_diag
    rng = np.random.default_rng(0)
    b = rng.standard_normal(n)
    x0 = np.random.default_rng(1).standard_normal(n)
    threads = oracle.max_threads()
    oracle.set_threads(threads)
    betas = load_beta_tables()

    def one(i):
        fam, k = SWEEP[i % len(SWEEP)]
        a = optimal_a(k) if fam == "opt_cheb1" else 0.0
        beta = betas[k].beta if fam == "opt_cheb4" else None
        t0 = time.perf_counter()
        oracle.smoother_apply(fam, k, A.row_ptr, A.col_idx, A.values, mdiag, b, x0, a=a, beta=beta)
        return time.perf_counter() - t0, apply_bytes(n, nnz, k)

    for i in range(args.warmup):
        one(i)
    tot_t = tot_b = 0.0
    for i in range(args.steps):
        t, by = one(args.warmup + i)
        tot_t += t
        tot_b += by
    value = tot_b / tot_t / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"poisson3d 7-pt {m}^3 fine level, smoother sweep",
                   "m": m, "n": n, "nnz": nnz,
                   "sample": "one smoother_apply per step cycling the 18-case sweep"},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} applies of the {m}^3 sweep (C oracle, "
                                   f"{threads} threads)"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- b200 arm
def cpu_baseline(m):
    """C oracle (port) on a bounded sample of the same workload, all host threads."""
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle
    from paper_2407_09848_b200.params import load_beta_tables, optimal_a
    from paper_2407_09848_b200.problems import poisson3d

    from paper_2407_09848_b200.smoothers import l1_jacobi_diag

    A, _ = poisson3d(m)
    n, nnz = A.nrows, A.nnz
    mdiag = l1_jacobi_diag(A).m_diag
    b = np.random.default_rng(0).standard_normal(n)
    x0 = np.random.default_rng(1).standard_normal(n)
    threads = oracle.max_threads()
    oracle.set_threads(threads)
    betas = load_beta_tables()
    tot_t = tot_b = 0.0
    for fam in ("opt_cheb1", "cheb4", "opt_cheb4"):
        k = 4
        a = optimal_a(k) if fam == "opt_cheb1" else 0.0
        beta = betas[k].beta if fam == "opt_cheb4" else None
        t0 = time.perf_counter()
        oracle.smoother_apply(fam, k, A.row_ptr, A.col_idx, A.values, mdiag, b, x0, a=a, beta=beta)
        tot_t += time.perf_counter() - t0
        tot_b += apply_bytes(n, nnz, k)
    oracle.set_threads(1)
    return {"value": tot_b / tot_t / 1e9, "unit": "GB/s", "cores": threads, "kind": "port",
            "sample": f"{m}^3 fine level, opt_cheb1/cheb4/opt_cheb4 k=4, one apply each "
                      f"({tot_t:.1f} s); the C restatement of the reference's smoother_apply "
                      f"(oracle/amgp_oracle.c, pthreads row split), not the reference's "
                      f"single-core Python, which cannot run on the GPU box"}


def mat_bytes(nrows, nnz):
    return 12 * nnz + 4 * (nrows + 1)


def vcycle_bytes(levels, k, family):
    """Algorithmic HBM bytes of one V-cycle:
    per level pre-smoother (x0 = 0: the first SpMV skipped), residual,
    restriction, prolongation, post-smoother; coarsest: one pass of its
    sweeps' data (the single-CTA solve keeps the level on chip).
    levels: [(n, nnz_A, nnz_P, nnz_R, n_coarse)]"""
    tot = 0
    for i, (n, nnz, pnnz, rnnz, nc) in enumerate(levels):
        A = mat_bytes(n, nnz)
        if nc is None:
            tot += A + 32 * n
            continue
        post = (A + 32 * n) * k if family == "l1_jacobi" else apply_bytes(n, nnz, k)
        pre = post - (A + 8 * n)
        tot += pre + post + (A + 24 * n) + (mat_bytes(nc, rnnz) + 8 * n + 8 * nc) + (mat_bytes(n, pnnz) + 16 * n + 8 * nc)
    return tot


def pcg_iter_bytes(n0, nnz0):
    """PCG vector kernels + the SpMV of one iteration (pcg.cu K7 table)."""
    return mat_bytes(n0, nnz0) + 104 * n0


def _level_shapes(As, Ps, Rs):
    out = []
    for i, A in enumerate(As):
        if i < len(Ps):
            out.append((A.nrows, A.nnz, Ps[i].nnz, Rs[i].nnz, Rs[i].nrows))
        else:
            out.append((A.nrows, A.nnz, 0, 0, None))
    return out


def solve_roofline(shapes, k, family, iters, seconds, peak):
    """Algorithmic GB/s of a whole solve: (iters + 1) V-cycles + iters PCG
    iterations (+ the initial residual) over the measured solve time."""
    n0, nnz0 = shapes[0][0], shapes[0][1]
    byts = (iters + 1) * vcycle_bytes(shapes, k, family) + (iters + 1) * pcg_iter_bytes(n0, nnz0)
    gbs = byts / seconds / 1e9
    return {"bound": "hbm", "bytes": byts, "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
            "note": "per-level algorithmic bytes (12 nnz + 4 (n+1) per matrix + vector streams) over the "
                    "device-timed solve; every rank's own rows at N > 1"}


def solve_bench(m, kind="smoothed_aggregation", cpu=True, stencil=7, k=4, cpu_family="opt_cheb1",
                families=("opt_cheb1", "cheb4", "opt_cheb4", "l1_jacobi")):
    """PCG + AMG V-cycle solve (BASELINE metric part 2) on the m^3 7-point
    (or 27-point) Poisson matrix generated on the GPU: device setup
    (dsetup.py, bitwise the reference's hierarchy), then per smoother family
    (degree k) one device solve at rtol 1e-6 timed with CUDA events on the
    library stream; the C oracle solves the same hierarchy on the host (all
    cores) for the CPU column."""
    import torch

    import paper_2407_09848_b200 as P

    D0 = P.poisson3d_device(m, stencil)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = P.build_hierarchy(D0, coarsening=P.CoarseningConfig(kind=kind),
                          smoother=P.PolySmootherConfig(family="opt_cheb1", degree=k))
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    D = h.device()
    c = D.ctx
    n = D0.nrows
    bd = torch.ones(n, dtype=torch.float64, device="cuda")
    cfg_k = P.KrylovConfig(tol=1e-6, itmax=1000)
    shapes = _level_shapes([lv.A for lv in h.levels], [lv.P for lv in h.levels[:-1]],
                           [lv.restrict_op() for lv in h.levels[:-1]])
    peak, _ = peaks()
    out = {"m": m, "n": n, "stencil": stencil, "degree": k, "coarsening": kind,
           "levels": [lv.A.nrows for lv in h.levels], "nnz": [lv.A.nnz for lv in h.levels],
           "operator_complexity": h.operator_complexity(), "setup_s": setup_s,
           "setup": "device (dsetup.py; bitwise the reference hierarchy)", "tol": 1e-6, "results": {}}
    for fam in families:
        cfg = P.PolySmootherConfig(family=fam, degree=k)
        for lv in h.levels:
            lv.smoother = cfg
        pre = P.as_vcycle_preconditioner(h)
        P.solve(D0, bd, precond=pre, cfg=cfg_k)  # warm-up (graph capture)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(c.stream)
        x, rep = P.solve(D0, bd, precond=pre, cfg=cfg_k)
        e1.record(c.stream)
        torch.cuda.synchronize()
        sec = e0.elapsed_time(e1) / 1e3
        out["results"][fam] = {"iterations": rep.iterations, "final_relres": rep.final_relres,
                               "solve_s": sec, "wall_s": rep.elapsed_s,
                               "roofline": solve_roofline(shapes, k, fam, rep.iterations, sec, peak)}
    if cpu:
        sys.path.insert(0, os.path.join(REPO, "oracle"))
        import oracle

        lv = []
        for l in h.levels:
            Ah = l.A.host()
            ent = {"A": (Ah.row_ptr, Ah.col_idx, Ah.values), "m": np.asarray(l.M.m_diag)}
            if l.P is not None:
                Ph, Rh = l.P.host(), l.restrict_op().host()
                ent["P"] = (Ph.row_ptr, Ph.col_idx, Ph.values)
                ent["R"] = (Rh.row_ptr, Rh.col_idx, Rh.values)
            lv.append(ent)
        cfg = P.PolySmootherConfig(family=cpu_family, degree=k)
        beta = cfg.beta.beta if cfg.family == "opt_cheb4" else None
        oh = oracle.Hierarchy(lv, cpu_family, k, a=cfg.a or 0.0, beta=beta)
        threads = oracle.max_threads()
        oracle.set_threads(threads)
        t0 = time.perf_counter()
        _, it, rr, conv, brk, _ = oracle.pcg(lv[0]["A"], np.ones(n), oh, tol=1e-6)
        out["cpu_" + cpu_family] = {"iterations": it, "final_relres": rr,
                                    "solve_s": time.perf_counter() - t0, "cores": threads,
                                    "kind": "port (C oracle, same hierarchy)"}
        oracle.set_threads(1)
    return out


def dist_solve_bench(comm, m_base, ws, family="opt_cheb4", k=4, stencil=7, strong=False, replicate_below=20000,
                     variant="pcg", graph=True):
    """PCG + AMG solve over all ranks (also N = 1): weak-scaled (BASELINE
    configs[3]: global cube round(m_base N^(1/3)), ~m_base^3 rows per GPU) or
    strong-scaled (configs[4]: global cube m_base).  Each rank generates its
    row block on its GPU and the hierarchy is built by the distributed device
    setup (decoupled aggregation, halo rows over NCCL); coarse levels under
    replicate_below rows are replicated.  Returns iterations and the
    max-over-ranks device time."""
    import torch
    import torch.distributed as dist

    import paper_2407_09848_b200 as P
    from paper_2407_09848_b200 import dist as Dist
    from paper_2407_09848_b200 import dsetup as DS

    m = m_base if strong else int(round(m_base * ws ** (1.0 / 3.0)))
    cfg = P.PolySmootherConfig(family=family, degree=k)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if comm is not None:
        D0 = Dist.poisson3d_block(m, comm, stencil=stencil)
        levels, _ = DS.build_levels(D0, P.CoarseningConfig(), comm=comm, replicate_below=replicate_below)
        dh = Dist.DistHierarchy.from_levels(levels, comm, cfg, use_graph=graph)
        c = dh.ctx
        lo, hi = dh.row_range
        As, Ps, Rs = dh.As, dh.Ps, dh.Rs
    else:
        D0 = P.poisson3d_device(m, stencil)
        h = P.build_hierarchy(D0, smoother=cfg)
        lo, hi = 0, D0.nrows
        dh = None
        As = [lv.A for lv in h.levels]
        Ps = [lv.P for lv in h.levels[:-1]]
        Rs = [lv.restrict_op() for lv in h.levels[:-1]]
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    if comm is not None:
        t = torch.tensor([setup_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        setup_s = float(t.item())
    bd = torch.ones(hi - lo, dtype=torch.float64, device="cuda")
    kc = P.KrylovConfig(tol=1e-6, itmax=1000, variant=variant)

    def run():
        if dh is not None:
            return dh.solve(bd, cfg=kc)
        return P.solve(D0, bd, precond=P.as_vcycle_preconditioner(h), cfg=kc)

    run()  # warm-up (graph capture)
    torch.cuda.synchronize()
    if comm is not None:
        dist.barrier()
    c = As[0].ctx
    sampler = ClockSampler(torch.cuda.current_device())
    sampler.start()
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wall0 = time.time()
    e0.record(c.stream)
    x, rep = run()
    e1.record(c.stream)
    torch.cuda.synchronize()
    clocks = sampler.stop(wall0 - 0.5, time.time())
    t = torch.tensor([e0.elapsed_time(e1) / 1e3, rep.elapsed_s], device="cuda", dtype=torch.float64)
    if comm is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    sec = float(t[0].item())
    peak, _ = peaks()
    shapes = _level_shapes(As, Ps, Rs)
    levels_n = [L.n for L in levels] if comm is not None else [a.nrows for a in As]
    return {"m": m, "n": int(m ** 3), "stencil": stencil, "scaling": "strong" if strong else "weak",
            "rows_per_gpu": hi - lo, "family": family, "degree": k, "levels": levels_n,
            "distributed_levels": sum(p is not None for p in dh.parts) if dh is not None else 0,
            "setup": "device" + (", distributed (decoupled aggregation)" if comm is not None else ""),
            "setup_s": setup_s, "iterations": rep.iterations, "final_relres": rep.final_relres,
            "solve_s": sec, "wall_s": float(t[1].item()), "tol": 1e-6, "krylov": variant,
            "replicate_below": replicate_below, "vcycle_graph": bool(graph) if comm is not None else True,
            "roofline_rank0": solve_roofline(shapes, k, family, rep.iterations, sec, peak),
            "clocks_rank0": clocks}


def run_b200(args):
    import torch
    import torch.distributed as dist

    import paper_2407_09848_b200 as P
    from paper_2407_09848_b200 import _native as N

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.cuda.current_device()
    c = N.ctx(dev)
    halo_info = None
    if args.solve_only:
        # diagnostic runs of the PCG+AMG solves alone (BASELINE configs[3] / [4] at
        # their configured sizes); not the driver's bench line
        comm = None
        if ws > 1:
            from paper_2407_09848_b200 import dist as Dist

            comm = Dist.Communicator(local)
        res = dist_solve_bench(comm, args.weak_grid, ws, family=args.solve_family or "opt_cheb4",
                               k=args.solve_k, stencil=args.solve_stencil, strong=args.solve_scaling == "strong",
                               replicate_below=args.replicate_below, variant=args.krylov,
                               graph=bool(args.dist_graph))
        if rank == 0:
            res["peak_mem_gb_rank0"] = torch.cuda.max_memory_allocated() / 1e9
            print(json.dumps({"solve_only": True, "n_gpus": ws, "solve": res}), flush=True)
        if ws > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0
    if ws == 1:
        m = args.grid
        D = P.poisson3d_device(m)
    else:
        # weak scaling: a global cube with ~m^3 rows per GPU, contiguous row
        # blocks, NCCL halo exchange of the neighbouring planes per SpMV
        from paper_2407_09848_b200 import dist as Dist

        comm = Dist.Communicator(local)
        m = int(round(args.grid * ws ** (1.0 / 3.0)))
        D = Dist.poisson3d_block(m, comm)
        halo_info = {"peers": len(D.halo.peers), "halo_rows": int(D.halo.recv_cnt.sum()),
                     "rows": D.nrows}
    n, nnz = D.nrows, D.nnz
    M = P.L1JacobiData(m_diag=D.l1_diag())
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    b = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    x0 = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    cfgs = [P.PolySmootherConfig(family=f, degree=k) for f, k in SWEEP]
    step_bytes = sum(apply_bytes(n, nnz, k) for _, k in SWEEP)
    job_step_bytes = step_bytes
    if ws > 1:
        t = torch.tensor([float(step_bytes)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t)
        job_step_bytes = float(t.item())

    def step(evs=None):
        for i, cfg in enumerate(cfgs):
            if evs is not None:
                evs[i][0].record(c.stream)
            P.smoother_apply(cfg, D, M, b, x0)
            if evs is not None:
                evs[i][1].record(c.stream)

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    sampler = ClockSampler(dev)
    sampler.start()
    for _ in range(args.warmup):
        step()
    barrier()
    per = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in cfgs] for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    launches0 = c.launches()
    wall0 = time.time()
    t_start.record(c.stream)
    for s in range(args.steps):
        step(per[s])
    t_end.record(c.stream)
    torch.cuda.synchronize()
    wall1 = time.time()
    launches = c.launches() - launches0
    clocks = sampler.stop(wall0, wall1)
    ms = t_start.elapsed_time(t_end)
    if ws > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = job_step_bytes / (ms_step * 1e-3) / 1e9

    # per-(family, degree) apply times -> middle-step kernel time per family
    t_apply = {}
    for i, (f, k) in enumerate(SWEEP):
        t_apply[(f, k)] = statistics.mean(per[s][i][0].elapsed_time(per[s][i][1])
                                          for s in range(args.steps))
    mids = {f: (t_apply[(f, 6)] - t_apply[(f, 2)]) / 4.0 for f in ("opt_cheb1", "cheb4", "opt_cheb4")}
    peak, peak_kind = peaks()
    mb = mid_step_bytes(n, nnz)
    t_mid = mids["cheb4"]
    achieved = mb / (t_mid * 1e-3) / 1e9
    traffic = traffic_per_launch()

    # end-to-end through the public API from pinned host memory: every
    # application uploads its own b and x0 and downloads its result
    # (smoother_apply_batch -> amgp_smoother_apply_host: consecutive
    # applications overlap their copies with each other's kernels)
    bh = b.cpu().pin_memory()
    xh = x0.cpu().pin_memory()
    outs = [torch.empty(n, dtype=torch.float64, pin_memory=True) for _ in cfgs]
    P.smoother_apply_batch(cfgs[:3], D, M, [bh] * 3, [xh] * 3, out=outs[:3])
    barrier()
    e2e_steps = max(1, min(args.steps, 3))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        P.smoother_apply_batch(cfgs, D, M, [bh] * len(cfgs), [xh] * len(cfgs), out=outs)
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    # the batched host path is the per-apply call's arithmetic: spot-check it
    e2e_bitwise = bool(torch.equal(outs[-1].cuda(), P.smoother_apply(cfgs[-1], D, M, b, x0)))
    if ws > 1:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    # the e2e bound: this box's pinned host -> device copy rate (the H2D
    # stream carries 2/3 of the copied bytes and is never idle in the pipeline)
    h2d_bytes = len(cfgs) * 2 * n * 8
    hb = torch.empty(n, dtype=torch.float64, pin_memory=True)
    db = torch.empty(n, dtype=torch.float64, device="cuda")
    db.copy_(hb, non_blocking=True)
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record()
    for _ in range(8):
        db.copy_(hb, non_blocking=True)
    c1.record()
    torch.cuda.synchronize()
    h2d_gbs = 8 * n * 8 / (c0.elapsed_time(c1) * 1e-3) / 1e9
    # the same uploads while a download stream runs (the pipeline's duplex case)
    hd = torch.empty(n, dtype=torch.float64, pin_memory=True)
    dd = torch.empty(n, dtype=torch.float64, device="cuda")
    sd = torch.cuda.Stream()
    torch.cuda.synchronize()
    c0.record()
    with torch.cuda.stream(sd):
        for _ in range(4):
            hd.copy_(dd, non_blocking=True)
    for _ in range(8):
        db.copy_(hb, non_blocking=True)
    torch.cuda.current_stream().wait_stream(sd)
    c1.record()
    torch.cuda.synchronize()
    h2d_duplex_gbs = 8 * n * 8 / (c0.elapsed_time(c1) * 1e-3) / 1e9
    del hb, db, hd, dd
    e2e_bound = job_step_bytes / (h2d_bytes / (h2d_gbs * 1e9)) / 1e9
    e2e = {"value": job_step_bytes / e2e_s / 1e9, "unit": "GB/s",
           "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": len(cfgs) * n * 8,
           "h2d_GBs_measured": h2d_gbs, "h2d_GBs_with_concurrent_d2h": h2d_duplex_gbs, "bound_GBs": e2e_bound,
           "frac_of_bound": job_step_bytes / e2e_s / 1e9 / e2e_bound,
           "frac_of_duplex_bound": job_step_bytes / e2e_s / 1e9 / (e2e_bound * h2d_duplex_gbs / h2d_gbs),
           "bound": "pinned H2D copy rate of this GPU (measured here): h2d_bytes_per_step / rate",
           "api": "smoother_apply_batch (amgp_smoother_apply_host): per-apply H2D of b, x0 and D2H of x, "
                  "pipelined across the 18 applies", "bitwise_vs_device_call": e2e_bitwise}

    # free the sweep's fine level before the solves
    del D, M, b, x0, bh, xh, outs
    torch.cuda.empty_cache()
    dsolve = None
    if ws > 1 and args.weak_grid > 0:
        dsolve = dist_solve_bench(comm, args.weak_grid, ws, family=args.solve_family or "opt_cheb4",
                                  k=args.solve_k, stencil=args.solve_stencil,
                                  strong=args.solve_scaling == "strong", replicate_below=args.replicate_below,
                                  variant=args.krylov, graph=bool(args.dist_graph))

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"poisson3d 7-pt {m}^3 fine level "
                                   + (f"row-partitioned over {ws} GPUs " if ws > 1 else "")
                                   + "smoother sweep opt_cheb1/cheb4/opt_cheb4 x k=1..6 (18 applies/step)",
                       "m": m, "n_per_gpu": n, "nnz_per_gpu": nnz, "bytes_per_step": job_step_bytes,
                       "l2": "inputs larger than L2 (A = %.2f GB per GPU)" % ((12 * nnz + 4 * n) / 1e9),
                       "parallelism": (f"row blocks x{ws}, NCCL halo exchange per SpMV overlapped "
                                       "with interior rows" if ws > 1 else "single GPU"),
                       "halo": halo_info},
            "hbm_frac": value / ws / peak,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_kind": peak_kind,
                         "kernel": "k_thread_rows<Cheb4Step<0,0,0>,0> (cheb4 middle degree step)",
                         "bytes_per_launch": mb, "ms_per_launch": t_mid,
                         # the static capture is of the 256^3 single-GPU kernel: other sizes get null
                         "traffic": (traffic or {}).get("bytes_per_launch") if (m == 256 and ws == 1) else None,
                         "traffic_source": "static: ncu --set full capture of this kernel at 256^3, "
                                           "profiles/ncu_traffic.json (not measured in this run)"
                                           if (m == 256 and ws == 1) else
                                           "none: the static ncu capture is of the 256^3 single-GPU kernel"},
            "mid_step_ms": mids,
            "apply_ms": {f"{f}_k{k}": v for (f, k), v in t_apply.items()},
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(args.cpu_grid)
        if ws == 1 and args.solve_grid > 0:
            line["solve"] = solve_bench(args.solve_grid, cpu=not args.no_cpu_baseline,
                                        stencil=args.solve_stencil, k=args.solve_k,
                                        cpu_family=args.solve_family or "opt_cheb1")
            torch.cuda.empty_cache()
        if ws == 1 and args.weak_grid > 0:
            # BASELINE configs[3] at N = 1: the weak-scaling reference point
            line["solve_weak"] = dist_solve_bench(None, args.weak_grid, 1, family=args.solve_family or "opt_cheb4",
                                                  k=args.solve_k, stencil=args.solve_stencil)
        if dsolve is not None:
            line["solve_weak" if args.solve_scaling == "weak" else "solve_strong"] = dsolve
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    if os.environ.get("AMGP_WATCHDOG"):  # diagnostics: Python stacks of a stuck run, then exit
        import faulthandler

        faulthandler.dump_traceback_later(float(os.environ["AMGP_WATCHDOG"]), exit=True)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    # (--grid, not --m: torchrun's parser would take --m for its own options)
    ap.add_argument("--grid", type=int, default=256, help="fine-level cube edge per GPU (weak-scaled for N > 1)")
    ap.add_argument("--cpu-grid", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--solve-grid", type=int, default=256,
                    help="N = 1: grid of the PCG+AMG solve section, all families (BASELINE configs[1]; 0: skip)")
    ap.add_argument("--weak-grid", type=int, default=400,
                    help="rows per GPU (cube edge) of the weak-scaled PCG+AMG solve (BASELINE configs[3]; "
                         "with --solve-scaling strong: the global cube edge; 0: skip)")
    ap.add_argument("--solve-stencil", type=int, default=7, choices=[7, 27])
    ap.add_argument("--solve-k", type=int, default=4, help="smoother degree of the solve section")
    ap.add_argument("--solve-family", default=None,
                    help="smoother family of the multi-GPU solve / the CPU oracle solve "
                         "(default opt_cheb4 / opt_cheb1)")
    ap.add_argument("--replicate-below", type=int, default=20000,
                    help="N > 1: AMG levels with fewer global rows are replicated on every rank")
    ap.add_argument("--krylov", default="pcg", choices=["pcg", "fcg", "pcg1"],
                    help="Krylov variant of the multi-GPU / weak-scaling solves")
    ap.add_argument("--dist-graph", type=int, default=1, choices=[0, 1],
                    help="N > 1: replay the distributed V-cycle from a CUDA graph (0: eager launches)")
    ap.add_argument("--solve-only", action="store_true",
                    help="run only the --weak-grid solve (diagnostics for BASELINE configs[3]/[4])")
    ap.add_argument("--solve-scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak (solve-grid^3 rows per GPU) or strong (solve-grid^3 in total)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (the driver's own launch line)
        import socket

        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; using {ws}", file=sys.stderr)
        args.gpus = ws
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
