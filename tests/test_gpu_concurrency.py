"""Reentrancy (the reference fans out with threads,
cli.py:289-294): smoother_apply, vcycle_apply and solve called concurrently
from a thread pool on shared matrices / hierarchies return exactly the
serial results.  ctypes releases the GIL, so the library calls really run
in parallel; libamgp serialises the work it enqueues on a context's stream
(amgp_ctx::mu) so a V-cycle graph capture never sees another thread's
launches."""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not gpu_available():
        pytest.skip("no CUDA device")
    import paper_2407_09848_b200 as pkg

    return pkg


def test_thread_pool_of_api_calls_is_bitwise_serial(P):
    A, b = P.poisson3d(20)
    M = P.l1_jacobi_diag(A)
    h = P.build_hierarchy(A, smoother=P.PolySmootherConfig(family="opt_cheb4", degree=3))
    n = A.nrows
    rng = np.random.default_rng(99)
    fams = ("l1_jacobi", "cheb4", "opt_cheb4", "opt_cheb1")
    jobs = []
    for i in range(96):
        kind = ("smooth", "vcycle", "solve", "solve_callable")[i % 4]
        jobs.append((kind, P.PolySmootherConfig(family=fams[i % 4], degree=1 + i % 5),
                     rng.standard_normal(n), rng.standard_normal(n)))

    def run(job):
        kind, cfg, u, v = job
        if kind == "smooth":
            return P.smoother_apply(cfg, A, M, u, v)
        if kind == "vcycle":
            return P.vcycle_apply(h, u)
        if kind == "solve":
            x, rep = P.solve(A, u, precond=P.as_vcycle_preconditioner(h), cfg=P.KrylovConfig(tol=1e-8))
            return np.concatenate([x, [rep.iterations]])
        x, rep = P.solve(A, u, precond=lambda r: P.vcycle_apply(h, r), cfg=P.KrylovConfig(tol=1e-8))
        return np.concatenate([x, [rep.iterations]])

    want = [run(j) for j in jobs]
    for workers in (4, 16):
        with ThreadPoolExecutor(workers) as ex:
            got = list(ex.map(run, jobs))
        for j, (g, w) in enumerate(zip(got, want)):
            assert np.array_equal(g, w), (workers, j, jobs[j][0])
