"""CPU-side checks of the native library and the host-side mirror of the API.

No kernel is launched here (no GPU in the development container): these
tests cover the C-ABI surface (every symbol of include/amgp.h is exported and
bound), the host-side helpers of libamgp (SELL packing, smoother step
scalars), and the Python host logic (configs, generators, l1 diagonal,
transpose) against the reference's golden data.
"""

import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import REPO, golden, golden_mat, smoother_params

import paper_2407_09848_b200 as P
from paper_2407_09848_b200 import _native as N


def header_symbols():
    text = open(os.path.join(REPO, "include", "amgp.h")).read()
    decl = r"^\s*(?:int|double|const char \*)\s*(amgp_[a-z0-9_]+)\s*\("
    return sorted(set(re.findall(decl, text, flags=re.M)))


def test_library_exports_every_header_symbol():
    lib = N.lib()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    # and the Python binding declares every one of them
    assert set(syms) == set(N.exported_symbols())


def test_error_reporting_without_device():
    lib = N.lib()
    st = lib.amgp_smoother_coefficients(None, None)
    assert st == N.AMGP_EINVAL
    assert b"null" in lib.amgp_last_error()
    with pytest.raises(ValueError):
        N.check(st)


def _pack(A):
    ns, st = C.c_int64(0), C.c_int64(0)
    rp = np.ascontiguousarray(A.row_ptr, np.int64)
    ci = np.ascontiguousarray(A.col_idx, np.int64)
    v = np.ascontiguousarray(A.values, np.float64)
    N.check(N.lib().amgp_sell_pack_host(A.nrows, rp.ctypes.data_as(N._P64), ci.ctypes.data_as(N._P64),
                                        v.ctypes.data_as(N._PD), C.byref(ns), C.byref(st),
                                        None, None, None))
    sp = np.empty(ns.value + 1, np.int64)
    col = np.empty(max(st.value, 1), np.int32)
    val = np.empty(max(st.value, 1), np.float64)
    N.check(N.lib().amgp_sell_pack_host(A.nrows, rp.ctypes.data_as(N._P64), ci.ctypes.data_as(N._P64),
                                        v.ctypes.data_as(N._PD), C.byref(ns), C.byref(st),
                                        sp.ctypes.data_as(N._P64),
                                        col.ctypes.data_as(C.POINTER(C.c_int32)),
                                        val.ctypes.data_as(N._PD)))
    return sp, col[: st.value], val[: st.value]


@pytest.mark.parametrize("name", ["tridiag20", "p3d6", "p3d8", "spd30"])
def test_sell_pack_roundtrip(name):
    d = golden("smoother_small.npz")
    nr, nc, rp, ci, v = golden_mat(d, name)
    A = P.CsrMatrix(nr, nc, rp, ci, v)
    sp, col, val = _pack(A)
    assert sp[0] == 0 and np.all(np.diff(sp) % 32 == 0)
    # unpack: slot j of row i at sp[i//32] + 32 j + i%32, stored order kept
    for i in range(nr):
        s, t = divmod(i, 32)
        w = (sp[s + 1] - sp[s]) // 32
        slots = sp[s] + 32 * np.arange(w) + t
        c = col[slots]
        got_c = c[c >= 0]
        assert np.array_equal(got_c, ci[rp[i]:rp[i + 1]])
        assert np.array_equal(val[slots][c >= 0], v[rp[i]:rp[i + 1]])
        assert np.all(c[len(got_c):] == -1)  # padding only at the end
        # slice width is the max row length of the slice
    for s in range(len(sp) - 1):
        rows = range(32 * s, min(nr, 32 * s + 32))
        assert (sp[s + 1] - sp[s]) // 32 == max(rp[i + 1] - rp[i] for i in rows)


def _py_coefficients(cfg):
    """The reference's Python scalar expressions (smoothers.py:112-135)."""
    k, rho = cfg.degree, cfg.rho_scale
    coef = np.zeros(3 * k)
    if cfg.family in ("cheb4", "opt_cheb4"):
        for j in range(1, k + 1):
            coef[3 * (j - 1)] = (2 * j - 3) / (2 * j + 1)
            coef[3 * (j - 1) + 1] = (8 * j - 4) / (2 * j + 1) / rho
            coef[3 * (j - 1) + 2] = cfg.beta.beta[j - 1] if cfg.family == "opt_cheb4" else 1.0
    elif cfg.family == "opt_cheb1":
        theta, delta = (1.0 + cfg.a) / 2.0, (1.0 - cfg.a) / 2.0
        sigma1 = theta / delta
        coef[0] = theta
        rho_prev = 1.0 / sigma1
        for j in range(1, k):
            rho_cur = 1.0 / (2.0 * sigma1 - rho_prev)
            coef[1 + 2 * (j - 1)] = rho_cur * rho_prev
            coef[2 + 2 * (j - 1)] = 2.0 * rho_cur / delta
            rho_prev = rho_cur
    return coef


@pytest.mark.parametrize("family", ["l1_jacobi", "cheb4", "opt_cheb4", "opt_cheb1"])
@pytest.mark.parametrize("rho", [1.0, 1.3])
def test_step_scalars_match_python(family, rho):
    for k in range(1, 13):
        cfg = P.PolySmootherConfig(family=family, degree=k, rho_scale=rho)
        c = N.smoother_cfg(cfg)
        out = np.zeros(3 * k)
        N.check(N.lib().amgp_smoother_coefficients(C.byref(c), out.ctypes.data_as(N._PD)))
        assert np.array_equal(out, _py_coefficients(cfg)), (family, k)


def test_config_validation_mirrors_reference(caplog):
    with pytest.raises(ValueError):
        P.PolySmootherConfig(family="sor", degree=2)
    with pytest.raises(ValueError):
        P.PolySmootherConfig(family="cheb4", degree=0)
    with pytest.raises(ValueError):
        P.PolySmootherConfig(family="cheb4", degree=2, rho_scale=0.0)
    with pytest.raises(ValueError):
        P.PolySmootherConfig(family="opt_cheb1", degree=3, a=1.5)
    cfg = P.PolySmootherConfig(family="opt_cheb1", degree=4)
    assert cfg.a == pytest.approx(0.0820780659590383, abs=1e-12)
    assert len(P.PolySmootherConfig(family="opt_cheb4", degree=3).beta.beta) == 3
    with caplog.at_level("WARNING"):
        assert P.PolySmootherConfig(family="opt_cheb4", degree=15).family == "cheb4"


def test_params_match_reference_tables():
    params = smoother_params()
    for k in range(1, 21):
        assert P.optimal_a(k) == params["a_star"][str(k)]
    tabs = P.load_beta_tables()
    assert sorted(tabs) == list(range(1, 13))
    assert tabs[4].beta[0] == 1.0039139269396271


@pytest.mark.parametrize("m", [2, 3, 6, 8])
def test_poisson3d_host_generator_is_reference(m):
    A, b = P.poisson3d(m)
    assert A.nnz == 7 * m ** 3 - 6 * m ** 2
    assert np.array_equal(b, np.ones(m ** 3))
    if m in (6, 8):
        d = golden("smoother_small.npz")
        nr, nc, rp, ci, v = golden_mat(d, f"p3d{m}")
        assert np.array_equal(A.row_ptr, rp)
        assert np.array_equal(A.col_idx, ci)
        assert np.array_equal(A.values, v)


def test_poisson27_generator():
    m = 5
    A, _ = P.poisson3d_27(m)
    assert A.nnz == (3 * m - 2) ** 3
    D = A.to_dense()
    assert np.allclose(D, D.T)
    assert np.all(np.diag(D) == 26.0)
    assert np.all(np.diff(A.col_idx)[np.diff(A.col_idx) != 0] != 0)
    for i in range(A.nrows):
        assert np.all(np.diff(A.col_idx[A.row_ptr[i]:A.row_ptr[i + 1]]) > 0)


@pytest.mark.parametrize("name", ["tridiag20", "p3d6", "p3d8", "spd30"])
def test_l1_diag_host_bitwise(name):
    d = golden("smoother_small.npz")
    nr, nc, rp, ci, v = golden_mat(d, name)
    A = P.CsrMatrix(nr, nc, rp, ci, v)
    assert np.array_equal(P.l1_jacobi_diag(A).m_diag, d[name + "_m"])


@pytest.mark.parametrize("prefix", ["sa16", "mt8", "mt16"])
def test_transpose_and_l1_of_golden_hierarchy(prefix):
    d = golden("hier_small.npz")
    L = int(d[prefix + "_nlev"][0])
    for l in range(L):
        A = P.CsrMatrix(*golden_mat(d, f"{prefix}_A{l}"))
        assert np.array_equal(P.l1_jacobi_diag(A).m_diag, d[f"{prefix}_M{l}"])
        if l < L - 1:
            Pm = P.CsrMatrix(*golden_mat(d, f"{prefix}_P{l}"))
            R = Pm.transpose()
            nr, nc, rp, ci, v = golden_mat(d, f"{prefix}_R{l}")
            assert (R.nrows, R.ncols) == (nr, nc)
            assert np.array_equal(R.row_ptr, rp)
            assert np.array_equal(R.col_idx, ci)
            assert np.array_equal(R.values, v)


def test_csr_validation():
    with pytest.raises(ValueError):
        P.CsrMatrix(2, 2, np.array([0, 1]), np.array([0]), np.array([1.0]))
    A = P.CsrMatrix.from_coo(2, 2, [0, 0, 1], [0, 0, 1], [1.0, 2.0, 0.0])
    assert A.nnz == 1 and A.to_dense()[0, 0] == 3.0


def test_device_ops_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    A, b = P.poisson3d(3)
    cfg = P.PolySmootherConfig(family="cheb4", degree=2)
    with pytest.raises(RuntimeError, match="CUDA device"):
        P.smoother_apply(cfg, A, P.l1_jacobi_diag(A), b, np.zeros_like(b))


def test_optimal_a_beyond_the_table_matches_reference():
    """optimal_a(k) for k > 20 solves for a*_k (reference optimize.py:106-111,
    313-318) with the same bits as the reference's solver; the restated Brent
    iteration also reproduces the shipped k <= 20 table exactly."""
    import json

    from paper_2407_09848_b200 import params as Pm

    ref = golden("a_star_k21_40.json")
    for k, v in ref.items():
        assert Pm.optimal_a(int(k)) == v, k
    table = json.load(open(os.path.join(REPO, "paper_2407_09848_b200", "data", "smoother_params.json")))["a_star"]
    for k, v in table.items():
        assert Pm.solve_a_star(int(k)) == float(v), k
    with pytest.raises(ValueError):
        Pm.solve_a_star(0)
