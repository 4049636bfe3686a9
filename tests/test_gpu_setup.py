"""Device hierarchy setup (dsetup.py / csrc/dsetup.cu) against the reference.

The device setup must build exactly the reference's hierarchy (amg.py:97-287):
every level's A, P, P^T and l1 diagonal np.array_equal to the reference's --
full arrays for the 8^3/16^3 fixtures, SHA-256 digests at 32^3, 64^3 (both
coarsenings), 27-point 12^3/20^3, and at the benched sizes 128^3 (both
coarsenings) and 256^3 (SA, BASELINE configs[1]) from tests/golden/
hashes_big.json (made by importing the reference, make_golden.py big).
Its building blocks are checked alone too: the OpenBLAS-order device dot and
the power iteration bitwise against the host restatements (setup.cpp), and
a >2^31-entry matrix against the C oracle on sampled rows.
"""

import hashlib
import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, golden, golden_mat, gpu_available

pytestmark = pytest.mark.gpu

KINDS = {"sa": "smoothed_aggregation", "mt": "pairwise_matching"}


@pytest.fixture(scope="module")
def P():
    if not gpu_available():
        pytest.skip("no CUDA device")
    import paper_2407_09848_b200 as pkg

    return pkg


def sha(a, kind):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int64 if kind == "i" else np.float64))
    return hashlib.sha256(a.tobytes()).hexdigest()


def mat_digest(A):
    return {"nrows": int(A.nrows), "ncols": int(A.ncols), "nnz": int(A.nnz),
            "row_ptr": sha(A.row_ptr, "i"), "col_idx": sha(A.col_idx, "i"), "values": sha(A.values, "f")}


def host_m(lv):
    m = lv.M.m_diag
    return m.cpu().numpy() if hasattr(m, "cpu") else np.asarray(m)


def check_digests(h, ref, tag):
    assert len(h.levels) == len(ref["levels"]), tag
    for l, (lv, lr) in enumerate(zip(h.levels, ref["levels"])):
        assert mat_digest(lv.A) == lr["A"], (tag, l, "A")
        assert sha(host_m(lv), "f") == lr["M"], (tag, l, "M")
        if "P" in lr:
            assert mat_digest(lv.P) == lr["P"], (tag, l, "P")
            assert mat_digest(lv.restrict_op()) == lr["R"], (tag, l, "R")


@pytest.mark.parametrize("prefix,m", [("sa16", 16), ("mt8", 8), ("mt16", 16)])
def test_device_hierarchy_arrays_bitwise(P, prefix, m):
    d = golden("hier_small.npz")
    A, _ = P.poisson3d(m)
    h = P.build_hierarchy(A, coarsening=P.CoarseningConfig(kind=KINDS[prefix[:2]]), setup="device",
                          smoother=P.PolySmootherConfig(family="cheb4", degree=4))
    L = int(d[prefix + "_nlev"][0])
    assert len(h.levels) == L
    for l, lv in enumerate(h.levels):
        for key, M in (("A", lv.A),) + ((("P", lv.P), ("R", lv.restrict_op())) if l < L - 1 else ()):
            nr, nc, rp, ci, v = golden_mat(d, f"{prefix}_{key}{l}")
            assert (M.nrows, M.ncols) == (nr, nc)
            assert np.array_equal(M.row_ptr, rp) and np.array_equal(M.col_idx, ci) and np.array_equal(M.values, v)
        assert np.array_equal(host_m(lv), d[f"{prefix}_M{l}"])


@pytest.mark.parametrize("m", [32, 64])
@pytest.mark.parametrize("kind", ["smoothed_aggregation", "pairwise_matching"])
def test_device_hierarchy_digests(P, m, kind):
    A, _ = P.poisson3d(m)
    h = P.build_hierarchy(A, coarsening=P.CoarseningConfig(kind=kind), setup="device",
                          smoother=P.PolySmootherConfig(family="cheb4", degree=4))
    check_digests(h, golden("hashes.json")[f"p3d{m}_{kind}"], (m, kind))


@pytest.mark.parametrize("m", [12, 20])
@pytest.mark.parametrize("kind", ["smoothed_aggregation", "pairwise_matching"])
def test_device_hierarchy_digests_27point(P, m, kind):
    A, _ = P.poisson3d_27(m)
    h = P.build_hierarchy(A, coarsening=P.CoarseningConfig(kind=kind), setup="device",
                          smoother=P.PolySmootherConfig(family="opt_cheb1", degree=3))
    check_digests(h, golden("hashes27.json")[f"p27_{m}"][kind], (m, kind))


def big_golden(key):
    if not os.path.exists(os.path.join(GOLDEN, "hashes_big.json")):
        pytest.skip("hashes_big.json not generated")
    d = golden("hashes_big.json")
    if key not in d:
        pytest.skip(f"{key} not in hashes_big.json")
    return d[key]


@pytest.mark.parametrize("m,kind", [(128, "smoothed_aggregation"), (128, "pairwise_matching"),
                                    (256, "smoothed_aggregation")])
def test_benched_size_hierarchy_vcycle_and_iterations(P, m, kind):
    """Bitwise hierarchy and V-cycle at the benched sizes; PCG iterations
    equal the reference's (only the dot order differs: +-1 bar)."""
    ref = big_golden(f"p3d{m}_{kind}")
    D = P.poisson3d_device(m)
    h = P.build_hierarchy(D, coarsening=P.CoarseningConfig(kind=kind), setup="device",
                          smoother=P.PolySmootherConfig(family="cheb4", degree=4))
    check_digests(h, ref, (m, kind))
    import torch

    r = torch.as_tensor(np.random.default_rng(5).standard_normal(D.nrows), device="cuda")
    for fam, dig in ref["vcycle"].items():
        for lv in h.levels:
            lv.smoother = P.PolySmootherConfig(family=fam, degree=4)
        assert sha(P.vcycle_apply(h, r).cpu().numpy(), "f") == dig, fam
    b = torch.ones(D.nrows, dtype=torch.float64, device="cuda")
    for key, rec in ref["pcg"].items():
        fam, k = key.rsplit("_k", 1)
        for lv in h.levels:
            lv.smoother = P.PolySmootherConfig(family=fam, degree=int(k))
        _, rep = P.solve(D, b, precond=P.as_vcycle_preconditioner(h), cfg=P.KrylovConfig(tol=1e-6))
        assert rep.converged and abs(rep.iterations - rec["iterations"]) <= 1, (key, rep.iterations, rec)


def test_device_blas_dot_is_the_host_openblas_restatement(P):
    import ctypes as C

    import torch

    from paper_2407_09848_b200 import _native as N
    from paper_2407_09848_b200 import setup as S

    c = N.ctx()
    for n in [1, 15, 16, 17, 31, 32, 33, 48, 100, 9999, 10001, 65535, 262144, 300001, 2000003]:
        rng = np.random.default_rng(n)
        x = rng.standard_normal(n) * 10 ** rng.uniform(-3, 3, n)
        y = rng.standard_normal(n)
        xd, yd = torch.as_tensor(x, device="cuda"), torch.as_tensor(y, device="cuda")
        for th in (1, 3, 8):
            out = (C.c_double * 3)()
            N.check(N.lib().amgp_ds_blas_dot3(c.handle, n, N.ptr(xd), N.ptr(yd), th, out))
            assert tuple(out) == (S.blas_dot(x, y, th), S.blas_dot(x, x, th), S.blas_dot(y, y, th)), (n, th)
        # misaligned start: the plain-load path
        out = (C.c_double * 3)()
        if n > 1:
            N.check(N.lib().amgp_ds_blas_dot3(c.handle, n - 1, N._VP(xd.data_ptr() + 8), N._VP(yd.data_ptr() + 8),
                                              1, out))
            assert out[0] == S.blas_dot(x[1:], y[1:], 1)


@pytest.mark.parametrize("m", [6, 24])
def test_device_lambda_max_bitwise(P, m):
    import ctypes as C

    import torch

    from paper_2407_09848_b200 import _native as N
    from paper_2407_09848_b200 import dsetup as DS
    from paper_2407_09848_b200 import setup as S

    A, _ = P.poisson3d(m)
    d = A.diagonal()
    want = S.estimate_lambda_max(A, d)
    D = A.device()
    v = torch.as_tensor(DS._start_vector(A.nrows, 0, A.nrows), device="cuda")
    lam = C.c_double()
    N.check(N.lib().amgp_ds_lambda_max(D.ctx.handle, D.handle, N.ptr(torch.as_tensor(d, device="cuda")),
                                       N.ptr(v), 25, 1, 0, C.byref(lam)))
    assert lam.value == want


def test_hierarchy_api_of_device_levels(P):
    A, _ = P.poisson3d(12)
    h = P.build_hierarchy(A, setup="device")
    hh = P.build_hierarchy(A, setup="host")
    assert h.summary() == hh.summary()
    assert h.operator_complexity() == hh.operator_complexity()
    assert h.levels[-1].P is None and h.levels[0].n_aggregates == hh.levels[0].n_aggregates
    np.testing.assert_array_equal(h.levels[1].A.to_dense(), hh.levels[1].A.to_dense())


def test_more_than_2_31_stored_entries_sampled_rows(P):
    """27-point 512^3 (BASELINE configs[4]: 3.61e9 stored entries, int64
    slice offsets): device SpMV and l1 diagonal against the C oracle on
    sampled rows (rows beyond entry 2^31 included)."""
    import torch

    m = 512
    D = P.poisson3d_device(m, 27)
    assert D.nnz == (3 * m - 2) ** 3 and D.nnz > 2 ** 31
    n = D.nrows
    x = torch.empty(n, dtype=torch.float64, device="cuda").uniform_(-1.0, 1.0)
    y = P.spmv(D, x)
    md = D.l1_diag()
    rng = np.random.default_rng(3)
    rows = np.unique(np.concatenate([rng.integers(0, n, 4000), np.arange(n - 2000, n),
                                     rng.integers(n // 2, n, 4000)]))
    # rows of the 27-point stencil (problems.poisson3d_27 conventions) for the samples
    rp, ci, va = [0], [], []
    for i in rows:
        iz, iy, ix = i // (m * m), (i // m) % m, i % m
        for dz in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    if 0 <= ix + dx < m and 0 <= iy + dy < m and 0 <= iz + dz < m:
                        ci.append(i + dx + dy * m + dz * m * m)
                        va.append(26.0 if (dx, dy, dz) == (0, 0, 0) else -1.0)
        rp.append(len(ci))
    rp, ci, va = np.array(rp, dtype=np.int64), np.array(ci, dtype=np.int64), np.array(va)
    xh = x.cpu().numpy()
    want = oracle.spmv(rp, ci, va, n, xh)
    assert np.array_equal(y[torch.as_tensor(rows, device="cuda")].cpu().numpy(), want)
    absrow = np.add.reduceat(np.abs(va), rp[:-1])
    assert np.array_equal(md[torch.as_tensor(rows, device="cuda")].cpu().numpy(), absrow - 26.0 + 26.0)
    del D, x, y
    torch.cuda.empty_cache()
