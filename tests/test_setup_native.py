"""Native host setup (csrc/setup.cpp) against the reference's hierarchies.

Bit-exact: every level's A, P, P^T and l1 diagonal must be np.array_equal
to the reference's (full arrays for the 8^3/16^3 fixtures, SHA-256 digests
for 32^3 and 64^3, both coarsenings).
"""

import hashlib

import numpy as np
import pytest

from conftest import golden, golden_mat

import paper_2407_09848_b200 as P
from paper_2407_09848_b200 import setup as S


def sha(a, kind):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int64 if kind == "i" else np.float64))
    return hashlib.sha256(a.tobytes()).hexdigest()


def mat_digest(A):
    return {"nrows": int(A.nrows), "ncols": int(A.ncols), "nnz": int(A.nnz),
            "row_ptr": sha(A.row_ptr, "i"), "col_idx": sha(A.col_idx, "i"),
            "values": sha(A.values, "f")}


def assert_mat_equal(A, d, key):
    nr, nc, rp, ci, v = golden_mat(d, key)
    assert (A.nrows, A.ncols) == (nr, nc), key
    assert np.array_equal(A.row_ptr, rp), key
    assert np.array_equal(A.col_idx, ci), key
    assert np.array_equal(A.values, v), key


KINDS = {"sa": "smoothed_aggregation", "mt": "pairwise_matching"}


@pytest.mark.parametrize("prefix,m", [("sa16", 16), ("mt8", 8), ("mt16", 16)])
def test_hierarchy_arrays_bitwise(prefix, m):
    d = golden("hier_small.npz")
    A, _ = P.poisson3d(m)
    h = P.build_hierarchy(A, coarsening=P.CoarseningConfig(kind=KINDS[prefix[:2]]), setup="host",
                          smoother=P.PolySmootherConfig(family="cheb4", degree=4))
    L = int(d[prefix + "_nlev"][0])
    assert len(h.levels) == L
    for l, lv in enumerate(h.levels):
        assert_mat_equal(lv.A, d, f"{prefix}_A{l}")
        assert np.array_equal(lv.M.m_diag, d[f"{prefix}_M{l}"])
        if l < L - 1:
            assert_mat_equal(lv.P, d, f"{prefix}_P{l}")
            assert_mat_equal(lv.restrict_op(), d, f"{prefix}_R{l}")


@pytest.mark.parametrize("m", [32, 64])
@pytest.mark.parametrize("kind", ["smoothed_aggregation", "pairwise_matching"])
def test_hierarchy_digests(m, kind):
    ref = golden("hashes.json")[f"p3d{m}_{kind}"]
    A, _ = P.poisson3d(m)
    h = P.build_hierarchy(A, coarsening=P.CoarseningConfig(kind=kind), setup="host",
                          smoother=P.PolySmootherConfig(family="cheb4", degree=4))
    assert len(h.levels) == len(ref["levels"])
    for l, (lv, lr) in enumerate(zip(h.levels, ref["levels"])):
        assert mat_digest(lv.A) == lr["A"], (m, kind, l, "A")
        assert sha(lv.M.m_diag, "f") == lr["M"], (m, kind, l, "M")
        if "P" in lr:
            assert mat_digest(lv.P) == lr["P"], (m, kind, l, "P")
            assert mat_digest(lv.restrict_op()) == lr["R"], (m, kind, l, "R")


@pytest.mark.parametrize("m", [12, 20])
@pytest.mark.parametrize("kind", ["smoothed_aggregation", "pairwise_matching"])
def test_hierarchy_digests_27point(m, kind):
    """27-point stencil (BASELINE configs[4]): native setup == reference setup."""
    ref = golden("hashes27.json")[f"p27_{m}"][kind]
    A, _ = P.poisson3d_27(m)
    h = P.build_hierarchy(A, coarsening=P.CoarseningConfig(kind=kind), setup="host",
                          smoother=P.PolySmootherConfig(family="opt_cheb1", degree=3))
    assert len(h.levels) == len(ref["levels"])
    for l, (lv, lr) in enumerate(zip(h.levels, ref["levels"])):
        assert mat_digest(lv.A) == lr["A"], (m, kind, l, "A")
        assert sha(lv.M.m_diag, "f") == lr["M"], (m, kind, l, "M")
        if "P" in lr:
            assert mat_digest(lv.P) == lr["P"], (m, kind, l, "P")
            assert mat_digest(lv.restrict_op()) == lr["R"], (m, kind, l, "R")


def test_aggregation_unit_cases():
    # tests/test_amg.py:25-68 of the reference
    Pm = S.sa_aggregate(P.CsrMatrix.identity(5))
    assert np.array_equal(Pm.to_dense(), np.eye(5))
    from conftest import GOLDEN  # noqa: F401

    T = P.CsrMatrix.from_dense(np.diag([2.0] * 6) + np.diag([-1.0] * 5, 1) + np.diag([-1.0] * 5, -1))
    agg = S.sa_aggregate(T).to_dense().argmax(axis=1)
    assert np.array_equal(agg, [0, 0, 0, 1, 1, 1])
    Pm = S.matching_aggregate(P.CsrMatrix.identity(4), sweeps=3)
    assert np.array_equal(Pm.to_dense(), np.eye(4))
    Pm = S.matching_aggregate(P.CsrMatrix.from_dense([[2.0, -1.0], [-1.0, 2.0]]), sweeps=1)
    assert Pm.ncols == 1
    A, _ = P.poisson3d(4)
    for sweeps in (1, 2, 3):
        Pm = S.matching_aggregate(A, sweeps=sweeps)
        assert np.max(Pm.to_dense().sum(axis=0)) <= 2 ** sweeps


def test_lambda_and_smoothing_unit_cases():
    A = P.CsrMatrix.from_dense(np.diag([2.0, 3.0, 4.0]))
    assert S.estimate_lambda_max(A, A.diagonal()) == pytest.approx(1.0)
    eye = P.CsrMatrix.identity(3)
    Pm = S.smooth_prolongator(eye, eye, 2.0 / 3.0)
    assert np.allclose(Pm.to_dense(), np.eye(3) / 3.0)
    n = 50
    T = P.CsrMatrix.from_dense(2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1))
    lam = S.estimate_lambda_max(T, T.diagonal())
    exact = 1.0 + np.cos(np.pi / (n + 1))
    assert abs(lam - exact) <= 0.05 * exact


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_blas_dot_emulation_matches_numpy(threads):
    """amgp_setup_blas_dot reproduces numpy's OpenBLAS ddot bit for bit
    (only checkable on a host whose OpenBLAS dispatches the SkylakeX kernel)."""
    from threadpoolctl import threadpool_info, threadpool_limits

    arch = [i.get("architecture") for i in threadpool_info() if i.get("internal_api") == "openblas"]
    if "SkylakeX" not in arch:
        pytest.skip(f"host OpenBLAS kernel {arch} is not SkylakeX")
    rng = np.random.default_rng(threads)
    with threadpool_limits(threads, user_api="blas"):
        for n in [1, 15, 16, 17, 32, 48, 100, 9999, 10001, 65535, 262144, 300001]:
            x = rng.standard_normal(n) * 10 ** rng.uniform(-3, 3, n)
            y = rng.standard_normal(n)
            assert S.blas_dot(x, y, threads) == x @ y, n
            assert np.sqrt(S.blas_dot(y, y, threads)) == np.linalg.norm(y), n


def test_operator_complexity_and_summary():
    A, _ = P.poisson3d(8)
    h = P.build_hierarchy(A, coarsening=P.CoarseningConfig(kind="pairwise_matching"), setup="host")
    assert h.operator_complexity() <= 3.0
    s = h.summary()
    assert s["levels"][0]["size"] == 512
