"""GPU parity: the CUDA path through the C ABI against the reference.

Bar (BASELINE.json north_star): smoother output within 1e-12 relative in
fp64; these kernels reproduce the reference bitwise, so every comparison
here is np.array_equal unless stated.  References: the reference's own
outputs (tests/golden/*.npz, made by importing the reference) and the C
oracle (oracle/, pinned to those goldens by tests/test_oracle.py) for sizes
beyond the fixtures.
"""

import numpy as np
import pytest

import oracle
from conftest import golden, golden_levels, golden_mat, gpu_available, smoother_params

pytestmark = pytest.mark.gpu

FAMILIES = ("l1_jacobi", "cheb4", "opt_cheb4", "opt_cheb1")
SMALL = ("tridiag20", "p3d6", "p3d8", "spd30")


@pytest.fixture(scope="module")
def P():
    if not gpu_available():
        pytest.skip("no CUDA device")
    import paper_2407_09848_b200 as pkg

    return pkg


def small_csr(P, name):
    d = golden("smoother_small.npz")
    return P.CsrMatrix(*golden_mat(d, name)), d


def test_native_library_is_loaded(P):
    from paper_2407_09848_b200 import _native as N

    c = N.ctx()
    before = c.launches()
    A, _ = small_csr(P, "p3d6")
    P.spmv(A, np.ones(A.ncols))
    assert c.launches() > before


@pytest.mark.parametrize("name", SMALL)
def test_spmv_bitwise(P, name):
    A, d = small_csr(P, name)
    x = d[name + "_x0"]
    want = oracle.spmv(A.row_ptr, A.col_idx, A.values, A.ncols, x)
    assert np.array_equal(P.spmv(A, x), want)
    assert np.array_equal(P.spmv(A, A.to_dense()[:, 1] * 0 + 1.0),
                          oracle.spmv(A.row_ptr, A.col_idx, A.values, A.ncols, np.ones(A.ncols)))


def test_spmv_exact_cases(P):
    eye = P.CsrMatrix.identity(3)
    x = np.array([1.0, 2.0, 3.0])
    assert np.array_equal(P.spmv(eye, x), x)
    with pytest.raises(ValueError):
        P.spmv(eye, np.ones(4))
    A, _ = P.poisson3d(2)
    e1 = np.zeros(8)
    e1[1] = 1.0
    assert np.array_equal(P.spmv(A, e1), A.to_dense()[:, 1])


@pytest.mark.parametrize("name", SMALL)
@pytest.mark.parametrize("fam", FAMILIES)
def test_smoother_apply_bitwise_vs_reference(P, name, fam):
    A, d = small_csr(P, name)
    M = P.L1JacobiData(m_diag=d[name + "_m"])
    b, x0 = d[name + "_b"], d[name + "_x0"]
    for k in range(1, 9):
        cfg = P.PolySmootherConfig(family=fam, degree=k)
        got = P.smoother_apply(cfg, A, M, b, x0)
        assert np.array_equal(got, d[f"{name}_{fam}_k{k}_x0"]), (fam, k)
        got = P.smoother_apply(cfg, A, M, b, np.zeros_like(b))
        assert np.array_equal(got, d[f"{name}_{fam}_k{k}_zero"]), (fam, k)
    cfg = P.PolySmootherConfig(family=fam, degree=3, rho_scale=1.3)
    assert np.array_equal(P.smoother_apply(cfg, A, M, b, x0), d[f"{name}_{fam}_rho1.3_k3_x0"])


def test_smoother_closed_forms(P):
    d = golden("smoother_small.npz")
    A = P.CsrMatrix(*golden_mat(d, "diag5"))
    M = P.L1JacobiData(m_diag=np.ones(5))
    e0 = np.array([1.0, -1.0, 2.0, 0.5, -0.25])
    for k in (1, 2, 4, 6):
        cfg = P.PolySmootherConfig(family="opt_cheb1", degree=k, a=0.1)
        assert np.array_equal(P.smoother_error_apply(cfg, A, M, e0),
                              d[f"diag5_opt_cheb1_a0.1_k{k}_err"])
    # cheb4 k=1 with M = A: p_1(1) = -1/3 (tests/test_smoothers.py:81-90)
    A = P.CsrMatrix.from_dense(np.diag([2.0, 3.0]))
    M = P.L1JacobiData(m_diag=np.array([2.0, 3.0]))
    e0 = np.array([1.0, -2.0])
    out = P.smoother_error_apply(P.PolySmootherConfig(family="cheb4", degree=1), A, M, e0)
    assert np.allclose(out, -e0 / 3.0, atol=1e-14)


def test_smoother_spmv_count_and_errors(P):
    A, d = small_csr(P, "tridiag20")
    M = P.l1_jacobi_diag(A)
    for fam in FAMILIES:
        for k in (1, 2, 5):
            P.reset_spmv_count()
            P.smoother_apply(P.PolySmootherConfig(family=fam, degree=k), A, M, np.ones(20), np.zeros(20))
            assert P.spmv_count() == k
    with pytest.raises(ValueError):
        P.smoother_apply(P.PolySmootherConfig(family="cheb4", degree=2), A, M, np.ones(21), np.zeros(20))


def test_smoother_torch_inputs_and_alias(P):
    import torch

    A, d = small_csr(P, "p3d8")
    M = P.L1JacobiData(m_diag=d["p3d8_m"])
    b = torch.tensor(d["p3d8_b"], device="cuda")
    x0 = torch.tensor(d["p3d8_x0"], device="cuda")
    cfg = P.PolySmootherConfig(family="opt_cheb1", degree=4)
    out = P.smoother_apply(cfg, A, M, b, x0)
    assert isinstance(out, torch.Tensor) and out.is_cuda
    assert np.array_equal(out.cpu().numpy(), d["p3d8_opt_cheb1_k4_x0"])
    assert np.array_equal(x0.cpu().numpy(), d["p3d8_x0"])  # x0 not mutated


def test_fused_update_bitwise(P, rng):
    for n in (1, 7, 1000, 100_000):
        s, r, d, x = (rng.standard_normal(n) for _ in range(4))
        rho, rho_prev, c = rng.standard_normal(3)
        r2, d2, x2 = r.copy(), d.copy(), x.copy()
        P.fused_update(rho, rho_prev, c, s, r, d, x)
        r2 -= s
        d2 = rho * rho_prev * d2 + c * r2
        x2 += d2
        assert np.array_equal(r, r2) and np.array_equal(d, d2) and np.array_equal(x, x2)
    with pytest.raises(ValueError):
        P.fused_update(1.0, 1.0, 1.0, np.ones(2), np.ones(3), np.ones(3), np.ones(3))


@pytest.mark.parametrize("m", [2, 3, 5, 8, 13, 33])
def test_device_poisson_generator(P, m):
    A, _ = P.poisson3d(m)
    D = P.poisson3d_device(m)
    assert D.nnz == A.nnz
    B = D.to_csr()
    assert np.array_equal(B.row_ptr, A.row_ptr)
    assert np.array_equal(B.col_idx, A.col_idx)
    assert np.array_equal(B.values, A.values)
    m_host = P.l1_jacobi_diag(A).m_diag
    assert np.array_equal(D.l1_diag().cpu().numpy(), m_host)
    A27, _ = P.poisson3d_27(m)
    D27 = P.poisson3d_device(m, stencil=27)
    B = D27.to_csr()
    assert np.array_equal(B.col_idx, A27.col_idx) and np.array_equal(B.values, A27.values)
    assert np.array_equal(D27.l1_diag().cpu().numpy(), P.l1_jacobi_diag(A27).m_diag)


def test_device_poisson_row_block(P):
    m = 9
    A, _ = P.poisson3d(m)
    D = P.poisson3d_device(m, row_begin=100, row_end=500)
    B = D.to_csr()
    assert np.array_equal(B.col_idx, A.col_idx[A.row_ptr[100]:A.row_ptr[500]])
    assert np.array_equal(D.l1_diag().cpu().numpy(), P.l1_jacobi_diag(A).m_diag[100:500])


@pytest.mark.parametrize("name", SMALL)
def test_device_l1_diag_of_uploaded_csr(P, name):
    A, d = small_csr(P, name)
    assert np.array_equal(A.device().l1_diag().cpu().numpy(), d[name + "_m"])


def golden_hierarchy(P, prefix, cfg):
    d = golden("hier_small.npz")
    L = int(d[prefix + "_nlev"][0])
    levels = []
    for l in range(L):
        A = P.CsrMatrix(*golden_mat(d, f"{prefix}_A{l}"))
        lv = P.Level(A=A, M=P.L1JacobiData(m_diag=d[f"{prefix}_M{l}"]), smoother=cfg)
        if l < L - 1:
            lv.P = P.CsrMatrix(*golden_mat(d, f"{prefix}_P{l}"))
            lv._Pt = P.CsrMatrix(*golden_mat(d, f"{prefix}_R{l}"))
        levels.append(lv)
    return P.AmgHierarchy(levels=levels), d


@pytest.mark.parametrize("prefix", ["sa16", "mt8", "mt16"])
def test_vcycle_bitwise_vs_reference(P, prefix):
    h, d = golden_hierarchy(P, prefix, P.PolySmootherConfig(family="cheb4", degree=4))
    r = d[prefix + "_r"]
    for fam in FAMILIES:
        for k in (1, 2, 4, 6):
            cfg = P.PolySmootherConfig(family=fam, degree=k)
            for lv in h.levels:
                lv.smoother = cfg
            assert np.array_equal(P.vcycle_apply(h, r), d[f"{prefix}_vc_{fam}_k{k}"]), (fam, k)


def test_vcycle_zero_and_linearity(P, rng):
    h, d = golden_hierarchy(P, "sa16", P.PolySmootherConfig(family="opt_cheb1", degree=4))
    n = h.levels[0].A.nrows
    assert np.array_equal(P.vcycle_apply(h, np.zeros(n)), np.zeros(n))
    r, s = rng.standard_normal(n), rng.standard_normal(n)
    lhs = P.vcycle_apply(h, 0.7 * r - 1.3 * s)
    rhs = 0.7 * P.vcycle_apply(h, r) - 1.3 * P.vcycle_apply(h, s)
    assert np.allclose(lhs, rhs, atol=1e-12 * max(1.0, np.abs(rhs).max()))
    with pytest.raises(ValueError):
        P.vcycle_apply(h, np.zeros(n + 1))


@pytest.mark.parametrize("prefix", ["sa16", "mt8", "mt16"])
def test_pcg_iterations_vs_reference(P, prefix):
    h, d = golden_hierarchy(P, prefix, P.PolySmootherConfig(family="cheb4", degree=4))
    n = h.levels[0].A.nrows
    A = h.levels[0].A
    for fam in FAMILIES:
        for k in (1, 2, 4, 6):
            cfg = P.PolySmootherConfig(family=fam, degree=k)
            for lv in h.levels:
                lv.smoother = cfg
            x, rep = P.solve(A, np.ones(n), precond=P.as_vcycle_preconditioner(h),
                             cfg=P.KrylovConfig(tol=1e-6))
            want = int(d[f"{prefix}_pcg_{fam}_k{k}_iters"][0])
            assert rep.converged and abs(rep.iterations - want) <= 1, (fam, k, rep.iterations, want)
            assert rep.iterations == want  # observed exactly equal
            assert np.allclose(rep.residual_history, d[f"{prefix}_pcg_{fam}_k{k}_hist"], rtol=1e-8)
            assert np.allclose(x, d[f"{prefix}_pcg_{fam}_k{k}_x"], rtol=1e-8, atol=1e-12)
            assert rep.spmv_count == rep.iterations + 1


def test_pcg_plain_and_fcg_and_breakdown(P):
    A = P.CsrMatrix.identity(5)
    b = np.arange(1.0, 6.0)
    x, rep = P.solve(A, b)
    assert rep.converged and rep.iterations == 1 and np.allclose(x, b)
    x, rep = P.solve(A, np.zeros(5))
    assert rep.converged and rep.iterations == 0 and np.array_equal(x, np.zeros(5))
    Ai = P.CsrMatrix.from_dense(np.diag([1.0, -1.0]))
    _, rep = P.solve(Ai, np.array([1.0, 1.0]), cfg=P.KrylovConfig(tol=1e-12))
    assert rep.breakdown and not rep.converged
    h, d = golden_hierarchy(P, "mt8", P.PolySmootherConfig(family="opt_cheb1", degree=4))
    n = h.levels[0].A.nrows
    its = {}
    for variant in ("pcg", "fcg"):
        _, rep = P.solve(h.levels[0].A, np.ones(n), precond=P.as_vcycle_preconditioner(h),
                         cfg=P.KrylovConfig(variant=variant))
        assert rep.converged
        its[variant] = rep.iterations
    assert abs(its["pcg"] - its["fcg"]) <= 1
    # warm start from the solution: zero iterations
    x, _ = P.solve(h.levels[0].A, np.ones(n), precond=P.as_vcycle_preconditioner(h),
                   cfg=P.KrylovConfig(tol=1e-12))
    _, rep = P.solve(h.levels[0].A, np.ones(n), precond=P.as_vcycle_preconditioner(h), x0=x,
                     cfg=P.KrylovConfig(tol=1e-10))
    assert rep.iterations == 0


def test_pcg_with_smoother_preconditioner(P):
    A, _ = P.poisson3d(8)
    M = P.l1_jacobi_diag(A)
    pre = P.as_preconditioner(P.PolySmootherConfig(family="opt_cheb1", degree=4), A, M)
    b = np.ones(A.nrows)
    x, rep = P.solve(A, b, precond=pre, cfg=P.KrylovConfig(tol=1e-8))
    assert rep.converged
    assert np.linalg.norm(b - A.to_dense() @ x) / np.linalg.norm(b) <= 1e-8
    # any callable r -> z is accepted (reference krylov.py:88); identity = plain CG
    x2, rep2 = P.solve(A, b, precond=lambda r: r.copy(), cfg=P.KrylovConfig(tol=1e-8))
    assert rep2.converged and rep2.precond_count == rep2.iterations
    with pytest.raises(TypeError):
        P.solve(A, b, precond=42)


def test_dense_direct_coarse(P):
    h, d = golden_hierarchy(P, "sa16", P.PolySmootherConfig(family="opt_cheb1", degree=4))
    h.coarse_solver = "dense_direct"
    n = h.levels[0].A.nrows
    r = d["sa16_r"]
    got = P.vcycle_apply(h, r)
    lv = [{"A": (l.A.row_ptr, l.A.col_idx, l.A.values), "m": l.M.m_diag} for l in h.levels]
    # host reference: same V-cycle with an exact coarse solve
    import scipy.linalg

    Ac = h.levels[-1].A.to_dense()

    def vc(l, rl):
        Al = h.levels[l]
        if l == len(h.levels) - 1:
            return scipy.linalg.cho_solve(scipy.linalg.cho_factor(Ac, lower=True), rl)
        kw = dict(a=Al.smoother.a)
        x = oracle.smoother_apply("opt_cheb1", 4, Al.A.row_ptr, Al.A.col_idx, Al.A.values,
                                  Al.M.m_diag, rl, None, **kw)
        res = rl - oracle.spmv(Al.A.row_ptr, Al.A.col_idx, Al.A.values, Al.A.ncols, x)
        R = Al.restrict_op()
        xc = vc(l + 1, oracle.spmv(R.row_ptr, R.col_idx, R.values, R.ncols, res))
        x = x + oracle.spmv(Al.P.row_ptr, Al.P.col_idx, Al.P.values, Al.P.ncols, xc)
        return oracle.smoother_apply("opt_cheb1", 4, Al.A.row_ptr, Al.A.col_idx, Al.A.values,
                                     Al.M.m_diag, rl, x, **kw)

    want = vc(0, r)
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12 * np.abs(want).max())


@pytest.mark.parametrize("m", [48, 64])
def test_fine_level_smoother_bitwise_vs_oracle(P, m):
    A, _ = P.poisson3d(m)
    n = A.nrows
    M = P.l1_jacobi_diag(A)
    b = np.random.default_rng(0).standard_normal(n)
    x0 = np.random.default_rng(1).standard_normal(n)
    params = smoother_params()
    for fam in FAMILIES:
        for k in (1, 4, 6):
            cfg = P.PolySmootherConfig(family=fam, degree=k)
            beta = cfg.beta.beta if cfg.family == "opt_cheb4" else None
            want = oracle.smoother_apply(cfg.family, k, A.row_ptr, A.col_idx, A.values, M.m_diag,
                                         b, x0, a=cfg.a or 0.0, beta=beta)
            assert np.array_equal(P.smoother_apply(cfg, A, M, b, x0), want), (fam, k)


def test_256cube_generated_smoother_bitwise_vs_oracle(P):
    """Full BASELINE size (256^3, 117M nnz): device-generated matrix, every
    family at k=4, bitwise against the multi-threaded C oracle."""
    import torch

    m = 256
    D = P.poisson3d_device(m)
    A, _ = P.poisson3d(m)
    n = A.nrows
    M = P.L1JacobiData(m_diag=D.l1_diag())
    b = np.random.default_rng(0).standard_normal(n)
    x0 = np.random.default_rng(1).standard_normal(n)
    m_host = D.l1_diag().cpu().numpy()
    oracle.set_threads(oracle.max_threads())
    try:
        for fam in FAMILIES:
            cfg = P.PolySmootherConfig(family=fam, degree=4)
            beta = cfg.beta.beta if cfg.family == "opt_cheb4" else None
            got = P.smoother_apply(cfg, D, M, torch.tensor(b, device="cuda"),
                                   torch.tensor(x0, device="cuda")).cpu().numpy()
            want = oracle.smoother_apply(cfg.family, 4, A.row_ptr, A.col_idx, A.values, m_host,
                                         b, x0, a=cfg.a or 0.0, beta=beta)
            assert np.array_equal(got, want), fam
    finally:
        oracle.set_threads(1)


def test_512cube_config3_smoother_bitwise_vs_oracle(P):
    """BASELINE configs[2] at its size (512^3, 938M stored entries): the
    device-generated fine level (downloaded as the oracle's CSR), the three
    polynomial families at k = 4, bitwise against the multi-threaded C
    oracle."""
    import torch

    D = P.poisson3d_device(512)
    H = D.host()  # the device matrix itself (to_csr), as the oracle's input
    n = D.nrows
    assert D.nnz == 7 * 512 ** 3 - 6 * 512 ** 2
    M = P.L1JacobiData(m_diag=D.l1_diag())
    m_host = D.l1_diag().cpu().numpy()
    rng = np.random.default_rng(2)
    b, x0 = rng.standard_normal(n), rng.standard_normal(n)
    oracle.set_threads(oracle.max_threads())
    try:
        for fam in ("cheb4", "opt_cheb4", "opt_cheb1"):
            cfg = P.PolySmootherConfig(family=fam, degree=4)
            beta = cfg.beta.beta if cfg.family == "opt_cheb4" else None
            got = P.smoother_apply(cfg, D, M, torch.tensor(b, device="cuda"),
                                   torch.tensor(x0, device="cuda")).cpu().numpy()
            want = oracle.smoother_apply(cfg.family, 4, H.row_ptr, H.col_idx, H.values, m_host,
                                         b, x0, a=cfg.a or 0.0, beta=beta)
            assert np.array_equal(got, want), fam
    finally:
        oracle.set_threads(1)
    del D, H
    torch.cuda.empty_cache()


def _sha(a):
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


@pytest.mark.parametrize("m", [32, 64])
@pytest.mark.parametrize("kind", ["smoothed_aggregation", "pairwise_matching"])
def test_native_hierarchy_vcycle_digest_vs_reference(P, m, kind):
    """Native setup + device V-cycle reproduce the reference's V-cycle output
    bit for bit (SHA-256 of the reference's vcycle_apply at 32^3 / 64^3)."""
    ref = golden("hashes.json")[f"p3d{m}_{kind}"]
    A, b = P.poisson3d(m)
    h = P.build_hierarchy(A, coarsening=P.CoarseningConfig(kind=kind),
                          smoother=P.PolySmootherConfig(family="cheb4", degree=4))
    r = np.random.default_rng(5).standard_normal(A.nrows)
    for fam in FAMILIES:
        cfg = P.PolySmootherConfig(family=fam, degree=4)
        for lv in h.levels:
            lv.smoother = cfg
        assert _sha(P.vcycle_apply(h, r)) == ref["vcycle"][fam], (m, kind, fam)


@pytest.mark.parametrize("kind", ["smoothed_aggregation", "pairwise_matching"])
def test_pcg_iteration_table_32cube(P, kind):
    """PCG+AMG iterations at rtol 1e-6 equal the reference's table."""
    ref = golden("hashes.json")[f"p3d32_{kind}"]
    A, b = P.poisson3d(32)
    h = P.build_hierarchy(A, coarsening=P.CoarseningConfig(kind=kind),
                          smoother=P.PolySmootherConfig(family="cheb4", degree=4))
    for fam in FAMILIES:
        for k in range(1, 7):
            cfg = P.PolySmootherConfig(family=fam, degree=k)
            for lv in h.levels:
                lv.smoother = cfg
            _, rep = P.solve(A, b, precond=P.as_vcycle_preconditioner(h), cfg=P.KrylovConfig(tol=1e-6))
            want = ref["pcg"][f"{fam}_k{k}"]
            assert rep.converged
            assert abs(rep.iterations - want["iterations"]) <= 1, (fam, k, rep.iterations, want)
            assert rep.iterations == want["iterations"]  # observed exactly equal
            assert rep.final_relres == pytest.approx(want["final_relres"], rel=1e-6)


def test_smoother_digests_32cube_all_levels(P):
    ref = golden("hashes.json")["p3d32_smoothed_aggregation"]
    A, b = P.poisson3d(32)
    h = P.build_hierarchy(A, smoother=P.PolySmootherConfig(family="cheb4", degree=4))
    n = A.nrows
    bb = np.random.default_rng(0).standard_normal(n)
    x0 = np.random.default_rng(1).standard_normal(n)
    M = h.levels[0].M
    for fam in FAMILIES:
        for k in range(1, 7):
            cfg = P.PolySmootherConfig(family=fam, degree=k)
            assert _sha(P.smoother_apply(cfg, A, M, bb, x0)) == ref["smoother"][f"{fam}_k{k}_x0"]
            assert _sha(P.smoother_apply(cfg, A, M, bb, np.zeros(n))) == ref["smoother"][f"{fam}_k{k}_zero"]
    for l in (1, 2):
        Al, Ml = h.levels[l].A, h.levels[l].M
        nl = Al.nrows
        bl = np.random.default_rng(0).standard_normal(nl)
        xl = np.random.default_rng(1).standard_normal(nl)
        for fam in FAMILIES:
            cfg = P.PolySmootherConfig(family=fam, degree=4)
            assert _sha(P.smoother_apply(cfg, Al, Ml, bl, xl)) == ref["smoother"][f"L{l}_{fam}_k4_x0"]


@pytest.mark.parametrize("m", [12, 20])
@pytest.mark.parametrize("kind", ["smoothed_aggregation", "pairwise_matching"])
def test_27point_vcycle_digest_and_pcg_table(P, m, kind):
    """27-point Poisson (configs[4] stencil): device V-cycle bitwise equal to the
    reference's on the same hierarchy; PCG iterations equal the reference's."""
    ref = golden("hashes27.json")[f"p27_{m}"][kind]
    A, b = P.poisson3d_27(m)
    h = P.build_hierarchy(A, coarsening=P.CoarseningConfig(kind=kind),
                          smoother=P.PolySmootherConfig(family="opt_cheb1", degree=3))
    r = np.random.default_rng(5).standard_normal(A.nrows)
    assert _sha(P.vcycle_apply(h, r)) == ref["vcycle_opt_cheb1_k3"]
    for fam in FAMILIES:
        cfg = P.PolySmootherConfig(family=fam, degree=3)
        for lv in h.levels:
            lv.smoother = cfg
        _, rep = P.solve(A, b, precond=P.as_vcycle_preconditioner(h), cfg=P.KrylovConfig(tol=1e-6))
        assert rep.converged and rep.iterations == ref["pcg"][f"{fam}_k3"]["iterations"], fam


@pytest.mark.parametrize("kind", ["smoothed_aggregation", "pairwise_matching"])
def test_single_reduction_pcg_iterations(P, kind):
    """pcg1 (Chronopoulos-Gear, one global reduction per iteration) is
    mathematically PCG: iteration counts within +-1 of the reference's."""
    ref = golden("hashes.json")[f"p3d32_{kind}"]
    A, b = P.poisson3d(32)
    h = P.build_hierarchy(A, coarsening=P.CoarseningConfig(kind=kind),
                          smoother=P.PolySmootherConfig(family="cheb4", degree=4))
    Ad = A.to_scipy()
    for fam in FAMILIES:
        for k in (1, 4, 6):
            cfg = P.PolySmootherConfig(family=fam, degree=k)
            for lv in h.levels:
                lv.smoother = cfg
            x, rep = P.solve(A, b, precond=P.as_vcycle_preconditioner(h),
                             cfg=P.KrylovConfig(tol=1e-6, variant="pcg1"))
            want = ref["pcg"][f"{fam}_k{k}"]["iterations"]
            assert rep.converged and abs(rep.iterations - want) <= 1, (fam, k, rep.iterations, want)
            relres = np.linalg.norm(b - Ad @ x) / np.linalg.norm(b)
            assert relres <= 1.01e-6
            assert rep.residual_history[-1] == rep.final_relres
    # plain CG (no preconditioner) on a small SPD system
    T = P.CsrMatrix.from_dense(2 * np.eye(40) - np.eye(40, k=1) - np.eye(40, k=-1))
    x, rep = P.solve(T, np.ones(40), cfg=P.KrylovConfig(tol=1e-10, itmax=200, variant="pcg1"))
    assert rep.converged
    assert np.linalg.norm(np.ones(40) - T.to_dense() @ x) / np.sqrt(40) <= 1e-9


@pytest.mark.parametrize("nc,band", [(40, None), (121, None), (300, 27)])
def test_coarse_solve_shared_memory_variants_bitwise(P, nc, band):
    """Coarsest-level l1 sweeps in one CTA.  nc = 40 and the dense nc = 121
    (15,488 SELL slots) keep the slot values in registers; nc = 300 with 55
    entries per row (17,600 slots) stages values and columns in shared
    memory -- both bitwise equal to the oracle V-cycle."""
    import scipy.sparse as sp

    A0, _ = P.poisson3d(11)
    n0 = A0.nrows
    rng = np.random.default_rng(nc)
    agg = np.minimum(np.arange(n0) * nc // n0, nc - 1)
    Pm = sp.csr_matrix((rng.uniform(0.5, 1.5, n0), (np.arange(n0), agg)), shape=(n0, nc))
    B = rng.standard_normal((nc, nc))
    D1 = B @ B.T
    if band is not None:
        i, j = np.indices((nc, nc))
        D1[np.abs(i - j) > band] = 0.0
        D1 += np.diag(np.abs(D1).sum(axis=1))
    A1 = sp.csr_matrix(D1 + nc * np.eye(nc))

    def csr(M):
        M = sp.csr_matrix(M)
        M.sort_indices()
        return P.CsrMatrix(M.shape[0], M.shape[1], M.indptr, M.indices, M.data)

    C0, C1, CP, CR = A0, csr(A1), csr(Pm), csr(Pm.T)
    M0, M1 = P.l1_jacobi_diag(C0), P.l1_jacobi_diag(C1)
    m0, m1 = np.asarray(M0.m_diag), np.asarray(M1.m_diag)
    params = smoother_params()
    r = rng.standard_normal(n0)
    for fam in FAMILIES:
        k = 3
        cfg = P.PolySmootherConfig(family=fam, degree=k)
        lv0 = P.Level(A=C0, M=M0, smoother=cfg, P=CP)
        lv0._Pt = CR
        lv1 = P.Level(A=C1, M=M1, smoother=cfg)
        h = P.AmgHierarchy(levels=[lv0, lv1])
        got = P.vcycle_apply(h, r)
        a = params["a_star"][str(k)] if fam == "opt_cheb1" else 0.0
        beta = np.array(params["beta"][str(k)]) if fam == "opt_cheb4" else None
        ol = [{"A": (C0.row_ptr, C0.col_idx, C0.values), "m": m0,
               "P": (CP.row_ptr, CP.col_idx, CP.values), "R": (CR.row_ptr, CR.col_idx, CR.values)},
              {"A": (C1.row_ptr, C1.col_idx, C1.values), "m": m1}]
        want = oracle.Hierarchy(ol, fam, k, a=a, beta=beta).vcycle(r)
        assert np.array_equal(got, want), fam


def test_smoother_apply_batch_host_buffers_bitwise(P):
    """The pipelined host-buffer path (amgp_smoother_apply_host, the e2e
    bench call) returns exactly what the per-call smoother_apply returns."""
    import torch

    A, _ = P.poisson3d(24)
    M = P.l1_jacobi_diag(A)
    rng = np.random.default_rng(11)
    cfgs = [P.PolySmootherConfig(family=f, degree=k) for f in FAMILIES for k in (1, 3, 4)]
    bs = [rng.standard_normal(A.nrows) for _ in cfgs]
    x0s = [rng.standard_normal(A.nrows) if i % 3 else np.zeros(A.nrows) for i in range(len(cfgs))]
    got = P.smoother_apply_batch(cfgs, A, M, bs, x0s)
    for cfg, b, x0, g in zip(cfgs, bs, x0s, got):
        assert np.array_equal(g, P.smoother_apply(cfg, A, M, b, x0)), cfg
    # pinned torch buffers in, pinned out, preallocated outputs
    bt = [torch.as_tensor(b).pin_memory() for b in bs[:4]]
    xt = [torch.as_tensor(x).pin_memory() for x in x0s[:4]]
    outs = [torch.empty(A.nrows, dtype=torch.float64).pin_memory() for _ in range(4)]
    res = P.smoother_apply_batch(cfgs[:4], A, M, bt, xt, out=outs)
    assert all(r is o for r, o in zip(res, outs))
    for cfg, b, x0, g in zip(cfgs[:4], bs, x0s, res):
        assert np.array_equal(g.numpy(), P.smoother_apply(cfg, A, M, b, x0))
    with pytest.raises(ValueError):
        P.smoother_apply_batch(cfgs[:2], A, M, bs[:1], x0s[:2])


@pytest.mark.parametrize("prefix", ["sa16", "mt8", "mt16"])
def test_pcg_with_a_plain_callable_is_the_reference_bitwise(P, prefix):
    """A preconditioner given as an arbitrary callable (the reference accepts
    any r -> z, krylov.py:88) takes the reference-exact device path: OpenBLAS
    order dots, numpy-rounded axpys -- iterations, the residual history and
    the solution equal the reference's (goldens) bit for bit."""
    d = golden("hier_small.npz")
    fams = sorted({k.split("_pcg_")[1].rsplit("_k", 1)[0] for k in d if k.startswith(prefix + "_pcg_")})
    for fam in fams:
        for k in (1, 4):
            key = f"{prefix}_pcg_{fam}_k{k}"
            if key + "_iters" not in d:
                continue
            h, _ = golden_hierarchy(P, prefix, P.PolySmootherConfig(family=fam, degree=k))
            n = h.levels[0].A.nrows
            x, rep = P.solve(h.levels[0].A, np.ones(n), precond=lambda r: P.vcycle_apply(h, r),
                             cfg=P.KrylovConfig(tol=1e-6, itmax=1000))
            assert rep.iterations == int(d[key + "_iters"][0]), key
            assert np.array_equal(np.array(rep.residual_history), d[key + "_hist"]), key
            assert np.array_equal(x, d[key + "_x"]), key
