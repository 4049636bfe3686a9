"""The bench's algorithmic byte counts (the roofline numerators) against the
figures SURVEY.md section 8(d) states, and its command line (CPU only)."""

import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import bench  # noqa: E402


def _poisson(m):
    return m ** 3, 7 * m ** 3 - 6 * m ** 2  # tests/test_problems.py:31-34 of the reference


def test_apply_bytes_match_survey():
    # 256^3, k = 4: 9.242 GB per apply; 512^3, k = 4: 74.01 GB
    n, nnz = _poisson(256)
    assert abs(bench.apply_bytes(n, nnz, 4) / 1e9 - 9.242) < 5e-4
    n, nnz = _poisson(512)
    assert abs(bench.apply_bytes(n, nnz, 4) / 1e9 - 74.01) < 5e-3


def test_step_bytes_of_the_bench_line():
    # the 256^3 sweep: 18 applies (3 families x k = 1..6) -> bytes_per_step,
    # and the middle step's bytes_per_launch, as printed in the BENCH lines
    n, nnz = _poisson(256)
    assert nnz == 117047296
    assert sum(bench.apply_bytes(n, nnz, k) for _, k in bench.SWEEP) == 144657875196
    assert bench.mid_step_bytes(n, nnz) == 2411200516


def test_apply_bytes_per_step_structure():
    # k >= 2: first step A + 48 n, k - 2 middle steps A + 56 n, last A + 40 n
    n, nnz = 1000, 6000
    A = 12 * nnz + 4 * (n + 1)
    for k in range(2, 9):
        assert bench.apply_bytes(n, nnz, k) == (A + 48 * n) + (k - 2) * (A + 56 * n) + (A + 40 * n)
    assert bench.apply_bytes(n, nnz, 1) == A + 32 * n


def test_vcycle_bytes_pre_smoother_skips_first_spmv():
    n, nnz, pnnz, rnnz, nc = 1000, 7000, 3000, 3000, 100
    levels = [(n, nnz, pnnz, rnnz, nc), (nc, 900, 0, 0, None)]
    A = bench.mat_bytes(n, nnz)
    post = bench.apply_bytes(n, nnz, 4)
    want = (post - (A + 8 * n)) + post + (A + 24 * n) + (bench.mat_bytes(nc, rnnz) + 8 * n + 8 * nc) \
        + (bench.mat_bytes(n, pnnz) + 16 * n + 8 * nc) + bench.mat_bytes(nc, 900) + 32 * nc
    assert bench.vcycle_bytes(levels, 4, "cheb4") == want


def test_bench_command_line():
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--help"], capture_output=True,
                         text=True, timeout=120)
    assert out.returncode == 0
    for flag in ("--gpus", "--steps", "--warmup", "--impl", "--dist-graph", "--solve-only"):
        assert flag in out.stdout


def test_metric_matches_baseline():
    import json

    with open(os.path.join(REPO, "BASELINE.json")) as f:
        base = json.load(f)
    assert bench.METRIC == base["metric"]
