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
                      f"({tot_t:.1f} s)"}


def solve_bench(m, kind="smoothed_aggregation", cpu=True, stencil=7, k=4, cpu_family="opt_cheb1"):
    """PCG + AMG V-cycle solve (BASELINE metric part 2) on poisson3d(m)
    (7-point) or the 27-point stencil: native host setup, then per smoother
    family (degree k) one device solve at rtol 1e-6 timed with CUDA events on
    the library stream; the C oracle solves the same hierarchy on the host
    (all cores) for the CPU column."""
    import torch

    import paper_2407_09848_b200 as P
    from paper_2407_09848_b200 import _native as N

    A, b = (P.poisson3d if stencil == 7 else P.poisson3d_27)(m)
    t0 = time.perf_counter()
    h = P.build_hierarchy(A, coarsening=P.CoarseningConfig(kind=kind),
                          smoother=P.PolySmootherConfig(family="opt_cheb1", degree=4))
    setup_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    D = h.device()
    upload_s = time.perf_counter() - t0
    c = D.ctx
    bd = torch.ones(A.nrows, dtype=torch.float64, device="cuda")
    cfg_k = P.KrylovConfig(tol=1e-6, itmax=1000)
    out = {"m": m, "n": A.nrows, "stencil": stencil, "degree": k, "coarsening": kind,
           "levels": [lv.A.nrows for lv in h.levels],
           "operator_complexity": h.operator_complexity(), "setup_s": setup_s,
           "upload_s": upload_s, "tol": 1e-6, "results": {}}
    for fam in ("opt_cheb1", "cheb4", "opt_cheb4", "l1_jacobi"):
        cfg = P.PolySmootherConfig(family=fam, degree=k)
        for lv in h.levels:
            lv.smoother = cfg
        pre = P.as_vcycle_preconditioner(h)
        P.solve(A, bd, precond=pre, cfg=cfg_k)  # warm-up (graph capture)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(c.stream)
        x, rep = P.solve(A, bd, precond=pre, cfg=cfg_k)
        e1.record(c.stream)
        torch.cuda.synchronize()
        out["results"][fam] = {"iterations": rep.iterations, "final_relres": rep.final_relres,
                               "solve_s": e0.elapsed_time(e1) / 1e3, "wall_s": rep.elapsed_s}
    if cpu:
        sys.path.insert(0, os.path.join(REPO, "oracle"))
        import oracle

        lv = [{"A": (l.A.row_ptr, l.A.col_idx, l.A.values), "m": l.M.m_diag,
               **({"P": (l.P.row_ptr, l.P.col_idx, l.P.values),
                   "R": (l.restrict_op().row_ptr, l.restrict_op().col_idx, l.restrict_op().values)}
                  if l.P is not None else {})} for l in h.levels]
        cfg = P.PolySmootherConfig(family=cpu_family, degree=k)
        beta = cfg.beta.beta if cfg.family == "opt_cheb4" else None
        oh = oracle.Hierarchy(lv, cpu_family, k, a=cfg.a or 0.0, beta=beta)
        threads = oracle.max_threads()
        oracle.set_threads(threads)
        t0 = time.perf_counter()
        _, it, rr, conv, brk, _ = oracle.pcg(lv[0]["A"], np.ones(A.nrows), oh, tol=1e-6)
        out["cpu_" + cpu_family] = {"iterations": it, "final_relres": rr,
                                "solve_s": time.perf_counter() - t0, "cores": threads,
                                "kind": "port"}
        oracle.set_threads(1)
    return out


def dist_solve_bench(comm, m_base, ws, family="opt_cheb4", k=4, stencil=7, strong=False):
    """PCG + AMG solve over all ranks: weak-scaled (BASELINE configs[3]
    shape: global cube round(m_base N^(1/3))) or strong-scaled (configs[4]
    shape: global cube m_base), hierarchy built once on rank 0 (native
    setup) and shared, every level row-partitioned (coarse levels
    replicated).  Returns (on every rank) iterations and max-over-ranks time."""
    import torch
    import torch.distributed as dist

    import paper_2407_09848_b200 as P
    from paper_2407_09848_b200 import dist as Dist

    m = m_base if strong else int(round(m_base * ws ** (1.0 / 3.0)))
    cfg = P.PolySmootherConfig(family=family, degree=k)
    t0 = time.perf_counter()

    def build():
        A, _ = (P.poisson3d if stencil == 7 else P.poisson3d_27)(m)
        return P.build_hierarchy(A, smoother=cfg)

    d, path = Dist.share_hierarchy(build, comm.rank, dist.barrier)
    setup_s = time.perf_counter() - t0
    dh = Dist.DistHierarchy(d, comm, cfg)
    lo, hi = dh.row_range
    bd = torch.ones(hi - lo, dtype=torch.float64, device="cuda")
    kc = P.KrylovConfig(tol=1e-6, itmax=1000)
    dh.solve(bd, cfg=kc)  # warm-up
    torch.cuda.synchronize()
    dist.barrier()
    c = dh.ctx
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(c.stream)
    x, rep = dh.solve(bd, cfg=kc)
    e1.record(c.stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / 1e3, rep.elapsed_s], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.barrier()
    if comm.rank == 0:
        try:
            Dist.release_shared(path)
        except OSError:
            pass
    return {"m": m, "n": int(m ** 3), "stencil": stencil, "scaling": "strong" if strong else "weak",
            "rows_per_gpu": hi - lo, "family": family, "degree": k,
            "levels": [int(d[f"A{l}_shape"][0]) for l in range(int(d["nlev"][0]))],
            "distributed_levels": sum(p is not None for p in dh.parts),
            "setup_s": setup_s, "iterations": rep.iterations, "final_relres": rep.final_relres,
            "solve_s": float(t[0].item()), "wall_s": float(t[1].item()), "tol": 1e-6}


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

    # end-to-end through the public API from pinned host memory (inputs
    # uploaded and result downloaded every application)
    bh = b.cpu().pin_memory()
    xh = x0.cpu().pin_memory()
    for cfg in cfgs[:3]:
        P.smoother_apply(cfg, D, M, bh, xh)
    barrier()
    e2e_steps = max(1, min(args.steps, 3))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        for cfg in cfgs:
            out = P.smoother_apply(cfg, D, M, bh, xh)
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if ws > 1:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": job_step_bytes / e2e_s / 1e9, "unit": "GB/s",
           "h2d_bytes_per_step": len(cfgs) * 2 * n * 8, "d2h_bytes_per_step": len(cfgs) * n * 8}

    dsolve = None
    if ws > 1 and args.solve_grid > 0:
        dsolve = dist_solve_bench(comm, args.solve_grid, ws, family=args.solve_family or "opt_cheb4",
                                  k=args.solve_k, stencil=args.solve_stencil,
                                  strong=args.solve_scaling == "strong")

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
                         "traffic": (traffic or {}).get("bytes_per_launch")},
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
        if dsolve is not None:
            line["solve"] = dsolve
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    # (--grid, not --m: torchrun's parser would take --m for its own options)
    ap.add_argument("--grid", type=int, default=256, help="fine-level cube edge per GPU (weak-scaled for N > 1)")
    ap.add_argument("--cpu-grid", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--solve-grid", type=int, default=128,
                    help="grid size of the PCG+AMG solve section (0: skip)")
    ap.add_argument("--solve-stencil", type=int, default=7, choices=[7, 27])
    ap.add_argument("--solve-k", type=int, default=4, help="smoother degree of the solve section")
    ap.add_argument("--solve-family", default=None,
                    help="smoother family of the multi-GPU solve / the CPU oracle solve "
                         "(default opt_cheb4 / opt_cheb1)")
    ap.add_argument("--solve-scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak (solve-grid^3 rows per GPU) or strong (solve-grid^3 in total)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
