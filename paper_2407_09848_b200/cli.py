"""Command line: the reference's ``amgpoly solve`` on the device path.

    python -m paper_2407_09848_b200.cli solve [--config FILE] [--override KEY=VAL ...] [-o OUT]

Mirrors reference cli.py:119-255 (flat ``key = value`` config with ``#``
comments, overrides win, the same keys and defaults, JSON report with the
config, the solve report and the hierarchy summary, elapsed time on stderr,
exit codes 0 / 2 config error / 3 breakdown).  The solve runs on the GPU;
its reductions are deterministic, so reruns are byte-identical (reference
tests/test_cli.py:109-122).  Problem kinds: ``poisson3d`` (reference) and
``poisson3d_27`` (the 27-point variant of BASELINE configs[4]); the dense
``spectral`` operator and the FE ``aniso2d`` generator are out of scope for the
device path and rejected as configuration errors.
"""

from __future__ import annotations

import argparse
import json
import sys
import time

EXIT_OK = 0
EXIT_CONFIG = 2
EXIT_BREAKDOWN = 3


class ConfigError(Exception):
    pass


SOLVE_DEFAULTS = {
    "problem": "poisson3d",
    "m": "8",
    "epsilon": "1.0",
    "angle": "0.0",
    "n": "64",
    "distribution": "equispaced",
    "coarsening": "smoothed_aggregation",
    "strength_theta": "0.01",
    "matching_sweeps": "3",
    "prolongator_smoothing": "true",
    "smoother": "opt_cheb1",
    "degree": "4",
    "variant": "pcg",
    "tol": "1e-7",
    "itmax": "1000",
    "coarse_solver": "l1_jacobi",
    "coarse_sweeps": "30",
    "min_coarse_size": "200",
    "max_levels": "10",
}


def parse_config(path, overrides):
    """Defaults, then the file, then --override KEY=VAL (last wins)."""
    cfg = dict(SOLVE_DEFAULTS)
    given = {}
    if path is not None:
        try:
            with open(path) as fh:
                lines = fh.read().splitlines()
        except OSError as exc:
            raise ConfigError(f"cannot read config {path}: {exc}") from exc
        for lineno, raw in enumerate(lines, 1):
            text = raw.strip()
            if not text or text.startswith("#"):
                continue
            key, sep, val = text.partition("=")
            if not sep:
                raise ConfigError(f"{path}:{lineno}: expected key = value")
            given[key.strip()] = val.strip()
    for item in overrides or []:
        key, sep, val = item.partition("=")
        if not sep:
            raise ConfigError(f"override {item!r}: expected key=value")
        given[key.strip()] = val.strip()
    unknown = [k for k in given if k not in cfg]
    if unknown:
        raise ConfigError(f"unknown config key {unknown[0]!r}")
    cfg.update(given)
    return cfg


def _bool(s):
    low = s.lower()
    if low in ("true", "1", "yes"):
        return True
    if low in ("false", "0", "no"):
        return False
    raise ConfigError(f"expected a boolean, got {s!r}")


def build_problem(cfg):
    from .problems import poisson3d, poisson3d_27

    kind = cfg["problem"]
    try:
        if kind == "poisson3d":
            return poisson3d(int(cfg["m"]))
        if kind == "poisson3d_27":
            return poisson3d_27(int(cfg["m"]))
    except ValueError as exc:
        raise ConfigError(f"bad problem config: {exc}") from exc
    if kind in ("aniso2d", "spectral"):
        raise ConfigError(f"problem kind {kind!r} is not supported on the device path")
    raise ConfigError(f"unknown problem kind {kind!r}")


def run_solve(cfg):
    from .amg import CoarseningConfig, as_vcycle_preconditioner, build_hierarchy
    from .krylov import KrylovConfig, solve
    from .smoothers import PolySmootherConfig

    A, b = build_problem(cfg)
    try:
        smoother = PolySmootherConfig(family=cfg["smoother"], degree=int(cfg["degree"]))
        coarsening = CoarseningConfig(kind=cfg["coarsening"],
                                      strength_theta=float(cfg["strength_theta"]),
                                      matching_sweeps=int(cfg["matching_sweeps"]),
                                      prolongator_smoothing=_bool(cfg["prolongator_smoothing"]))
        kcfg = KrylovConfig(variant=cfg["variant"], tol=float(cfg["tol"]), itmax=int(cfg["itmax"]))
        if cfg["coarse_solver"] not in ("l1_jacobi", "dense_direct"):
            raise ValueError(f"unknown coarse solver {cfg['coarse_solver']!r}")
        h = build_hierarchy(A, coarsening=coarsening, smoother=smoother,
                            max_levels=int(cfg["max_levels"]),
                            min_coarse_size=int(cfg["min_coarse_size"]),
                            coarse_solver=cfg["coarse_solver"],
                            coarse_sweeps=int(cfg["coarse_sweeps"]))
    except ValueError as exc:
        raise ConfigError(str(exc)) from exc
    _, rep = solve(A, b, precond=as_vcycle_preconditioner(h), cfg=kcfg)
    report = {
        "config": cfg,
        "solve": {
            "iterations": rep.iterations,
            "converged": rep.converged,
            "final_relres": rep.final_relres,
            "residual_history": rep.residual_history,
            "spmv_count": rep.spmv_count,
            "precond_count": rep.precond_count,
            "breakdown": rep.breakdown,
        },
        "hierarchy": h.summary(),
    }
    return report, rep


def cmd_solve(args):
    cfg = parse_config(args.config, args.override)
    t0 = time.perf_counter()
    report, rep = run_solve(cfg)
    elapsed = time.perf_counter() - t0
    text = json.dumps(report, indent=2) + "\n"
    if args.output in (None, "-"):
        sys.stdout.write(text)
    else:
        with open(args.output, "w") as fh:
            fh.write(text)
    print(f"elapsed_s={elapsed:.3f} solve_s={rep.elapsed_s:.6f}", file=sys.stderr)
    return EXIT_BREAKDOWN if rep.breakdown else EXIT_OK


def make_parser():
    p = argparse.ArgumentParser(prog="paper_2407_09848_b200", description=__doc__,
                                formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = p.add_subparsers(dest="command", required=True)
    ps = sub.add_parser("solve", help="AMG-PCG run from a key=value config (GPU)")
    ps.add_argument("--config", default=None)
    ps.add_argument("--override", action="append", metavar="KEY=VAL")
    ps.add_argument("--output", "-o", default=None)
    ps.set_defaults(func=cmd_solve)
    return p


def main(argv=None):
    args = make_parser().parse_args(argv)
    try:
        return args.func(args)
    except ConfigError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_CONFIG


if __name__ == "__main__":
    sys.exit(main())
