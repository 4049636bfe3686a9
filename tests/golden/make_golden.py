"""Generate the golden fixtures by importing the reference package read-only.

Run ONLY in the development container (the reference is not present on the
GPU box):

    python tests/golden/make_golden.py

It imports ``amgpoly`` from /root/reference/pkg/src and writes

* ``paper_2407_09848_b200/data/smoother_params.json`` -- the a*_k table
  (``optimize.py:278-296`` / ``data/optimal_params.csv``) and the beta tables
  (``optimize.py:299-310`` / ``data/beta_tables.csv``), parsed exactly as the
  reference parses them, re-serialised with Python's round-trip float repr;
* ``tests/golden/smoother_small.npz`` -- smoother_apply outputs
  (``smoothers.py:92-137``) for 4 families x k=1..8 on small matrices, x0 = 0
  and x0 != 0, plus closed-form cases;
* ``tests/golden/hier_small.npz`` -- full hierarchies (``amg.py:238-287``) for
  poisson3d(16) SA and poisson3d(8) matching, with vcycle_apply outputs
  (``amg.py:303-315``) and PCG reports (``krylov.py:45-120``);
* ``tests/golden/hashes.json`` -- SHA-256 digests of the 32^3 / 64^3
  hierarchies, fine-level smoother outputs and V-cycle outputs, plus the PCG
  iteration tables (rtol 1e-6) at 32^3.

Digests are over little-endian bytes of int64 (indices) / float64 (values).

The reference runs with OPENBLAS_NUM_THREADS=1 (set below): its lambda_max
power iteration takes dot products through OpenBLAS, whose thread split
changes the last bits of lambda (and thus every coarse level) with the core
count.  One BLAS thread is the convention of SURVEY.md section 8d.
"""

from __future__ import annotations

import os

os.environ["OPENBLAS_NUM_THREADS"] = "1"
os.environ["OMP_NUM_THREADS"] = "1"

import hashlib  # noqa: E402
import json  # noqa: E402
import sys  # noqa: E402
import time  # noqa: E402

import numpy as np

REF = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, REF)
sys.path.insert(0, REF_TESTS)

from amgpoly.amg import (  # noqa: E402
    CoarseningConfig,
    as_vcycle_preconditioner,
    build_hierarchy,
    vcycle_apply,
)
from amgpoly.krylov import KrylovConfig, solve  # noqa: E402
from amgpoly.optimize import load_beta_tables, load_params_table  # noqa: E402
from amgpoly.problems import poisson3d  # noqa: E402
from amgpoly.smoothers import (  # noqa: E402
    FAMILIES,
    L1JacobiData,
    PolySmootherConfig,
    l1_jacobi_diag,
    smoother_apply,
)
from amgpoly.sparse import CsrMatrix  # noqa: E402
from conftest import random_spd, tridiag  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))


def sha(a, kind):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int64 if kind == "i" else np.float64))
    return hashlib.sha256(a.tobytes()).hexdigest()


def mat_digest(A):
    return {
        "nrows": int(A.nrows),
        "ncols": int(A.ncols),
        "nnz": int(A.nnz),
        "row_ptr": sha(A.row_ptr, "i"),
        "col_idx": sha(A.col_idx, "i"),
        "values": sha(A.values, "f"),
    }


def put_mat(out, prefix, A):
    out[prefix + "_shape"] = np.array([A.nrows, A.ncols], dtype=np.int64)
    out[prefix + "_rp"] = A.row_ptr.astype(np.int64)
    out[prefix + "_ci"] = A.col_idx.astype(np.int64)
    out[prefix + "_v"] = A.values.astype(np.float64)


def export_params():
    params = load_params_table()
    betas = load_beta_tables()
    doc = {
        "source": "reference pkg/src/amgpoly/data/{optimal_params,beta_tables}.csv "
        "parsed by optimize.py:278-310; re-serialised by tests/golden/make_golden.py",
        "a_star": {str(k): float(params[k].a_star) for k in sorted(params)},
        "beta": {str(k): [float(v) for v in betas[k].beta] for k in sorted(betas)},
        "beta_gamma": {str(k): float(betas[k].gamma_value) for k in sorted(betas)},
    }
    path = os.path.join(REPO, "paper_2407_09848_b200", "data", "smoother_params.json")
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
    print("wrote", path)


def smoother_small():
    out = {}
    mats = {
        "tridiag20": tridiag(20),
        "p3d6": poisson3d(6)[0],
        "p3d8": poisson3d(8)[0],
        "spd30": random_spd(30, seed=3),
    }
    for name, A in mats.items():
        put_mat(out, name, A)
        M = l1_jacobi_diag(A)
        out[name + "_m"] = M.m_diag
        n = A.nrows
        b = np.random.default_rng(0).standard_normal(n)
        x0 = np.random.default_rng(1).standard_normal(n)
        out[name + "_b"] = b
        out[name + "_x0"] = x0
        for fam in FAMILIES:
            for k in range(1, 9):
                cfg = PolySmootherConfig(family=fam, degree=k)
                out[f"{name}_{fam}_k{k}_x0"] = smoother_apply(cfg, A, M, b, x0)
                out[f"{name}_{fam}_k{k}_zero"] = smoother_apply(cfg, A, M, b, np.zeros(n))
        # rho_scale != 1 exercises the /rho divisions of smoothers.py:118,128,133
        for fam in FAMILIES:
            cfg = PolySmootherConfig(family=fam, degree=3, rho_scale=1.3)
            out[f"{name}_{fam}_rho1.3_k3_x0"] = smoother_apply(cfg, A, M, b, x0)
        # opt_cheb1 with a user-supplied interval end
        cfg = PolySmootherConfig(family="opt_cheb1", degree=5, a=0.1)
        out[f"{name}_opt_cheb1_a0.1_k5_x0"] = smoother_apply(cfg, A, M, b, x0)
    # opt_cheb1 diagonal decoupling case (tests/test_smoothers.py:92-105)
    lam = np.array([0.05, 0.2, 0.5, 0.9, 1.0])
    A = CsrMatrix.from_dense(np.diag(lam))
    put_mat(out, "diag5", A)
    M = L1JacobiData(m_diag=np.ones(5))
    e0 = np.array([1.0, -1.0, 2.0, 0.5, -0.25])
    for k in (1, 2, 4, 6):
        cfg = PolySmootherConfig(family="opt_cheb1", degree=k, a=0.1)
        out[f"diag5_opt_cheb1_a0.1_k{k}_err"] = smoother_apply(cfg, A, M, np.zeros(5), e0)
    path = os.path.join(HERE, "smoother_small.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


def hier_record(out, prefix, h):
    out[prefix + "_nlev"] = np.array([len(h.levels)], dtype=np.int64)
    for l, lev in enumerate(h.levels):
        put_mat(out, f"{prefix}_A{l}", lev.A)
        out[f"{prefix}_M{l}"] = lev.M.m_diag
        if lev.P is not None:
            put_mat(out, f"{prefix}_P{l}", lev.P)
            put_mat(out, f"{prefix}_R{l}", lev.restrict_op())


def set_smoother(h, cfg):
    for lev in h.levels:
        lev.smoother = cfg


def hier_small():
    out = {}
    cases = [
        ("sa16", poisson3d(16), CoarseningConfig()),
        ("mt8", poisson3d(8), CoarseningConfig(kind="pairwise_matching")),
        ("mt16", poisson3d(16), CoarseningConfig(kind="pairwise_matching")),
    ]
    for prefix, (A, b), coarsening in cases:
        h = build_hierarchy(A, coarsening=coarsening,
                            smoother=PolySmootherConfig(family="cheb4", degree=4))
        hier_record(out, prefix, h)
        n = A.nrows
        r = np.random.default_rng(5).standard_normal(n)
        out[prefix + "_r"] = r
        for fam in FAMILIES:
            for k in (1, 2, 4, 6):
                set_smoother(h, PolySmootherConfig(family=fam, degree=k))
                out[f"{prefix}_vc_{fam}_k{k}"] = vcycle_apply(h, r)
                x, rep = solve(A, b, precond=as_vcycle_preconditioner(h),
                               cfg=KrylovConfig(tol=1e-6, itmax=1000))
                out[f"{prefix}_pcg_{fam}_k{k}_iters"] = np.array([rep.iterations], dtype=np.int64)
                out[f"{prefix}_pcg_{fam}_k{k}_hist"] = np.array(rep.residual_history)
                out[f"{prefix}_pcg_{fam}_k{k}_x"] = x
    path = os.path.join(HERE, "hier_small.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


def hashes():
    doc = {"note": "sha256 over little-endian int64 indices / float64 values"}
    for m in (32, 64):
        for kind in ("smoothed_aggregation", "pairwise_matching"):
            A, b = poisson3d(m)
            t0 = time.perf_counter()
            h = build_hierarchy(A, coarsening=CoarseningConfig(kind=kind),
                                smoother=PolySmootherConfig(family="cheb4", degree=4))
            t_setup = time.perf_counter() - t0
            key = f"p3d{m}_{kind}"
            rec = {"setup_s": t_setup, "levels": []}
            for lev in h.levels:
                lr = {"A": mat_digest(lev.A), "M": sha(lev.M.m_diag, "f")}
                if lev.P is not None:
                    lr["P"] = mat_digest(lev.P)
                    lr["R"] = mat_digest(lev.restrict_op())
                rec["levels"].append(lr)
            n = A.nrows
            r = np.random.default_rng(5).standard_normal(n)
            rec["vcycle"] = {}
            for fam in FAMILIES:
                set_smoother(h, PolySmootherConfig(family=fam, degree=4))
                rec["vcycle"][fam] = sha(vcycle_apply(h, r), "f")
            if m == 32:
                # PCG iteration table, rtol 1e-6
                rec["pcg"] = {}
                for fam in FAMILIES:
                    for k in range(1, 7):
                        set_smoother(h, PolySmootherConfig(family=fam, degree=k))
                        _, rep = solve(A, b, precond=as_vcycle_preconditioner(h),
                                       cfg=KrylovConfig(tol=1e-6, itmax=1000))
                        rec["pcg"][f"{fam}_k{k}"] = {
                            "iterations": rep.iterations,
                            "final_relres": rep.final_relres,
                            "spmv_count": rep.spmv_count,
                            "converged": rep.converged,
                        }
                # fine-level smoother outputs (bitwise targets)
                M = h.levels[0].M
                bb = np.random.default_rng(0).standard_normal(n)
                x0 = np.random.default_rng(1).standard_normal(n)
                rec["smoother"] = {}
                for fam in FAMILIES:
                    for k in range(1, 7):
                        cfg = PolySmootherConfig(family=fam, degree=k)
                        rec["smoother"][f"{fam}_k{k}_x0"] = sha(smoother_apply(cfg, A, M, bb, x0), "f")
                        rec["smoother"][f"{fam}_k{k}_zero"] = sha(
                            smoother_apply(cfg, A, M, bb, np.zeros(n)), "f")
                # coarse-level smoother outputs on level 1 and 2
                for l in (1, 2):
                    Al, Ml = h.levels[l].A, h.levels[l].M
                    nl = Al.nrows
                    bl = np.random.default_rng(0).standard_normal(nl)
                    xl = np.random.default_rng(1).standard_normal(nl)
                    for fam in FAMILIES:
                        cfg = PolySmootherConfig(family=fam, degree=4)
                        rec["smoother"][f"L{l}_{fam}_k4_x0"] = sha(smoother_apply(cfg, Al, Ml, bl, xl), "f")
            doc[key] = rec
            print(key, "levels", len(h.levels), f"setup {t_setup:.1f}s", flush=True)
    path = os.path.join(HERE, "hashes.json")
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
    print("wrote", path)


def stencil27():
    """27-point Poisson (BASELINE configs[4]; not in the reference): the input
    matrix comes from this repo's numpy generator (problems.poisson3d_27, a
    pure data generator), everything else -- hierarchy, V-cycle, PCG -- from
    the reference."""
    sys.path.insert(0, REPO)
    from paper_2407_09848_b200.problems import poisson3d_27

    doc = {}
    for m in (12, 20):
        B, b = poisson3d_27(m)
        A = CsrMatrix(B.nrows, B.ncols, B.row_ptr, B.col_idx, B.values)
        rec = {}
        for kind in ("smoothed_aggregation", "pairwise_matching"):
            h = build_hierarchy(A, coarsening=CoarseningConfig(kind=kind),
                                smoother=PolySmootherConfig(family="opt_cheb1", degree=3))
            r = {"levels": []}
            for lev in h.levels:
                lr = {"A": mat_digest(lev.A), "M": sha(lev.M.m_diag, "f")}
                if lev.P is not None:
                    lr["P"] = mat_digest(lev.P)
                    lr["R"] = mat_digest(lev.restrict_op())
                r["levels"].append(lr)
            rr = np.random.default_rng(5).standard_normal(A.nrows)
            r["vcycle_opt_cheb1_k3"] = sha(vcycle_apply(h, rr), "f")
            r["pcg"] = {}
            for fam in FAMILIES:
                set_smoother(h, PolySmootherConfig(family=fam, degree=3))
                _, rep = solve(A, b, precond=as_vcycle_preconditioner(h),
                               cfg=KrylovConfig(tol=1e-6, itmax=1000))
                r["pcg"][f"{fam}_k3"] = {"iterations": rep.iterations,
                                         "final_relres": rep.final_relres}
            rec[kind] = r
        doc[f"p27_{m}"] = rec
        print("27-point", m, {k: v["pcg"]["opt_cheb1_k3"]["iterations"] for k, v in rec.items()})
    path = os.path.join(HERE, "hashes27.json")
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
    print("wrote", path)


def hier_digest_record(h):
    rec = {"levels": []}
    for lev in h.levels:
        lr = {"A": mat_digest(lev.A), "M": sha(lev.M.m_diag, "f")}
        if lev.P is not None:
            lr["P"] = mat_digest(lev.P)
            lr["R"] = mat_digest(lev.restrict_op())
        rec["levels"].append(lr)
    return rec


def big():
    """Benched sizes (Missing #2): 128^3 hierarchies of both
    coarsenings (digests), V-cycle digests and the PCG iteration tables
    (4 families x k = 1..6, rtol 1e-6); 256^3 SA (BASELINE configs[1])
    hierarchy digests and PCG iterations of every family at k = 4.
    Long: ~40 min and ~20 GB on one core."""
    doc = {"note": "sha256 over little-endian int64 indices / float64 values; OPENBLAS_NUM_THREADS=1"}
    path = os.path.join(HERE, "hashes_big.json")
    jobs = [(128, "smoothed_aggregation", range(1, 7)), (128, "pairwise_matching", range(1, 7)),
            (256, "smoothed_aggregation", (4,))]
    for m, kind, degrees in jobs:
        A, b = poisson3d(m)
        t0 = time.perf_counter()
        h = build_hierarchy(A, coarsening=CoarseningConfig(kind=kind),
                            smoother=PolySmootherConfig(family="cheb4", degree=4))
        rec = hier_digest_record(h)
        rec["setup_s"] = time.perf_counter() - t0
        print(m, kind, "setup", rec["setup_s"], flush=True)
        r = np.random.default_rng(5).standard_normal(A.nrows)
        rec["vcycle"] = {}
        for fam in FAMILIES:
            set_smoother(h, PolySmootherConfig(family=fam, degree=4))
            rec["vcycle"][fam] = sha(vcycle_apply(h, r), "f")
        rec["pcg"] = {}
        for fam in FAMILIES:
            for k in degrees:
                set_smoother(h, PolySmootherConfig(family=fam, degree=k))
                t0 = time.perf_counter()
                _, rep = solve(A, b, precond=as_vcycle_preconditioner(h), cfg=KrylovConfig(tol=1e-6, itmax=1000))
                rec["pcg"][f"{fam}_k{k}"] = {"iterations": rep.iterations, "final_relres": rep.final_relres,
                                             "spmv_count": rep.spmv_count, "converged": rep.converged,
                                             "solve_s": time.perf_counter() - t0}
                print(m, kind, fam, k, rep.iterations, flush=True)
        doc[f"p3d{m}_{kind}"] = rec
        with open(path, "w") as f:
            json.dump(doc, f, indent=1)
    print("wrote", path)


def a_star_beyond_table():
    """a*_k solved by the reference for degrees past its table (optimize.py:313-318)."""
    from amgpoly.optimize import solve_a_star

    doc = {str(k): solve_a_star(k) for k in range(21, 41)}
    with open(os.path.join(HERE, "a_star_k21_40.json"), "w") as f:
        json.dump(doc, f, indent=1)
    print("wrote a_star_k21_40.json")


def cli_reports():
    """Reference `amgpoly solve` JSON reports (cli.py:193-255) for small runs."""
    from amgpoly.cli import main as cli_main

    for name, overrides in {
        "cli_solve_m8_matching.json": ["m=8", "coarsening=pairwise_matching"],
        "cli_solve_m12_sa.json": ["m=12", "smoother=cheb4", "tol=1e-6"],
        "cli_solve_m6_itmax1.json": ["m=6", "itmax=1"],
    }.items():
        args = ["solve"] + [x for o in overrides for x in ("--override", o)]
        cli_main(args + ["-o", os.path.join(HERE, name)])
        print("wrote", name)


if __name__ == "__main__":
    if sys.argv[1:] == ["big"]:
        big()
        sys.exit(0)
    if sys.argv[1:] == ["a_star"]:
        a_star_beyond_table()
        sys.exit(0)
    export_params()
    smoother_small()
    hier_small()
    hashes()
    stencil27()
    cli_reports()
