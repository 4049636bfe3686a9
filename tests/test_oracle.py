"""Pin the C oracle (oracle/amgp_oracle.c) to the reference's own outputs.

The golden fixtures were produced by importing the reference package
(tests/golden/make_golden.py).  Everything here is bitwise (np.array_equal)
except PCG, where the dot-product summation order differs from OpenBLAS and
the bar is the reference's: iterations equal (we observe exactly equal).
"""

import hashlib

import numpy as np
import pytest

import oracle
from conftest import golden, golden_levels, golden_mat, smoother_params

FAMILIES = ("l1_jacobi", "cheb4", "opt_cheb4", "opt_cheb1")
SMALL = ("tridiag20", "p3d6", "p3d8", "spd30")


def family_args(fam, k, params):
    """(family, a, beta) as PolySmootherConfig resolves them (smoothers.py:69-83)."""
    if fam == "opt_cheb1":
        return fam, params["a_star"][str(k)], None
    if fam == "opt_cheb4":
        if str(k) in params["beta"]:
            return fam, 0.0, np.array(params["beta"][str(k)])
        return "cheb4", 0.0, None
    return fam, 0.0, None


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


@pytest.mark.parametrize("name", SMALL)
def test_spmv_bitwise_vs_reference_smoother_k1(name):
    d = golden("smoother_small.npz")
    nr, nc, rp, ci, v = golden_mat(d, name)
    x = d[name + "_x0"]
    y = oracle.spmv(rp, ci, v, nc, x)
    dense = np.zeros((nr, nc))
    for i in range(nr):
        for jj in range(rp[i], rp[i + 1]):
            dense[i, ci[jj]] = v[jj]
    assert np.allclose(y, dense @ x, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("name", SMALL)
@pytest.mark.parametrize("fam", FAMILIES)
def test_smoother_apply_bitwise(name, fam):
    d = golden("smoother_small.npz")
    params = smoother_params()
    nr, nc, rp, ci, v = golden_mat(d, name)
    m, b, x0 = d[name + "_m"], d[name + "_b"], d[name + "_x0"]
    for k in range(1, 9):
        f, a, beta = family_args(fam, k, params)
        got = oracle.smoother_apply(f, k, rp, ci, v, m, b, x0, a=a, beta=beta)
        assert np.array_equal(got, d[f"{name}_{fam}_k{k}_x0"]), (fam, k)
        got = oracle.smoother_apply(f, k, rp, ci, v, m, b, None, a=a, beta=beta)
        assert np.array_equal(got, d[f"{name}_{fam}_k{k}_zero"]), (fam, k)
    f, a, beta = family_args(fam, 3, params)
    got = oracle.smoother_apply(f, 3, rp, ci, v, m, b, x0, a=a, beta=beta, rho=1.3)
    assert np.array_equal(got, d[f"{name}_{fam}_rho1.3_k3_x0"])


def test_opt_cheb1_custom_a_and_diag():
    d = golden("smoother_small.npz")
    for name in SMALL:
        nr, nc, rp, ci, v = golden_mat(d, name)
        got = oracle.smoother_apply("opt_cheb1", 5, rp, ci, v, d[name + "_m"], d[name + "_b"],
                                    d[name + "_x0"], a=0.1)
        assert np.array_equal(got, d[f"{name}_opt_cheb1_a0.1_k5_x0"])
    nr, nc, rp, ci, v = golden_mat(d, "diag5")
    e0 = np.array([1.0, -1.0, 2.0, 0.5, -0.25])
    for k in (1, 2, 4, 6):
        got = oracle.smoother_apply("opt_cheb1", k, rp, ci, v, np.ones(5), np.zeros(5), e0, a=0.1)
        assert np.array_equal(got, d[f"diag5_opt_cheb1_a0.1_k{k}_err"])


def test_fused_update_bitwise_vs_unfused(rng):
    n = 1000
    s, r, d, x = (rng.standard_normal(n) for _ in range(4))
    rho, rho_prev, c = rng.standard_normal(3)
    r2, d2, x2 = r.copy(), d.copy(), x.copy()
    oracle.fused_update(rho, rho_prev, c, s, r, d, x)
    r2 -= s
    d2 = rho * rho_prev * d2 + c * r2
    x2 += d2
    assert np.array_equal(r, r2) and np.array_equal(d, d2) and np.array_equal(x, x2)


@pytest.mark.parametrize("prefix", ["sa16", "mt8", "mt16"])
def test_vcycle_bitwise(prefix):
    d = golden("hier_small.npz")
    params = smoother_params()
    levels = golden_levels(d, prefix)
    r = d[prefix + "_r"]
    for fam in FAMILIES:
        for k in (1, 2, 4, 6):
            f, a, beta = family_args(fam, k, params)
            h = oracle.Hierarchy(levels, f, k, a=a, beta=beta)
            assert np.array_equal(h.vcycle(r), d[f"{prefix}_vc_{fam}_k{k}"]), (fam, k)


@pytest.mark.parametrize("prefix", ["sa16", "mt8", "mt16"])
def test_pcg_iterations(prefix):
    d = golden("hier_small.npz")
    params = smoother_params()
    levels = golden_levels(d, prefix)
    n = len(levels[0]["m"])
    b = np.ones(n)
    for fam in FAMILIES:
        for k in (1, 2, 4, 6):
            f, a, beta = family_args(fam, k, params)
            h = oracle.Hierarchy(levels, f, k, a=a, beta=beta)
            x, it, relres, conv, brk, hist = oracle.pcg(levels[0]["A"], b, h, tol=1e-6)
            want_it = int(d[f"{prefix}_pcg_{fam}_k{k}_iters"][0])
            assert conv and not brk
            assert it == want_it, (fam, k, it, want_it)
            want_hist = d[f"{prefix}_pcg_{fam}_k{k}_hist"]
            assert np.allclose(hist, want_hist, rtol=1e-9, atol=0)
            assert np.allclose(x, d[f"{prefix}_pcg_{fam}_k{k}_x"], rtol=1e-9, atol=1e-12)


def test_oracle_threads_do_not_change_bits():
    d = golden("smoother_small.npz")
    nr, nc, rp, ci, v = golden_mat(d, "p3d8")
    m, b, x0 = d["p3d8_m"], d["p3d8_b"], d["p3d8_x0"]
    try:
        oracle.set_threads(4)
        got = oracle.smoother_apply("cheb4", 4, rp, ci, v, m, b, x0)
    finally:
        oracle.set_threads(1)
    assert np.array_equal(got, d["p3d8_cheb4_k4_x0"])
