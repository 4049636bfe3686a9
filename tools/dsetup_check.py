"""Device setup vs host native setup (bitwise), plus timings (GPU box)."""
import sys, time, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_09848_b200 as P
from paper_2407_09848_b200 import setup as S, dsetup as DS

def cmp(a, b, name):
    ok = (a.nrows, a.ncols, a.nnz) == (b.nrows, b.ncols, b.nnz)
    if ok:
        ok = np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx) and np.array_equal(a.values, b.values)
    if not ok:
        print("  MISMATCH", name, (a.nrows, a.ncols, a.nnz), (b.nrows, b.ncols, b.nnz))
        if a.nnz == b.nnz and a.nrows == b.nrows:
            print("    rp eq", np.array_equal(a.row_ptr, b.row_ptr), "ci eq", np.array_equal(a.col_idx, b.col_idx),
                  "maxdiff", np.max(np.abs(a.values - b.values)))
    return ok

c = P._native.ctx()
# dot emulation
for n in [1, 15, 16, 17, 31, 32, 33, 48, 100, 9999, 10001, 65535, 262144, 300001, 5000017]:
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n) * 10 ** rng.uniform(-3, 3, n); y = rng.standard_normal(n)
    for th in (1, 3, 8):
        xd, yd = torch.as_tensor(x, device="cuda"), torch.as_tensor(y, device="cuda")
        out = (P._native.C.c_double * 3)()
        P._native.check(P._native.lib().amgp_ds_blas_dot3(c.handle, n, DS._p(xd), DS._p(yd), th, out))
        ref = (S.blas_dot(x, y, th), S.blas_dot(x, x, th), S.blas_dot(y, y, th))
        if tuple(out) != ref:
            print("DOT MISMATCH", n, th, tuple(out), ref)
print("dots checked", flush=True)
for m, kind in [(16, "smoothed_aggregation"), (16, "pairwise_matching"), (32, "smoothed_aggregation"),
                (32, "pairwise_matching"), (12, "smoothed_aggregation")]:
    for st in (7, 27):
        if st == 27 and m > 12: continue
        A, _ = (P.poisson3d if st == 7 else P.poisson3d_27)(m)
        cc = P.CoarseningConfig(kind=kind)
        t0 = time.perf_counter(); hh = P.build_hierarchy(A, coarsening=cc, setup="host"); th_ = time.perf_counter() - t0
        t0 = time.perf_counter(); hd = P.build_hierarchy(A, coarsening=cc, setup="device"); td = time.perf_counter() - t0
        ok = len(hh.levels) == len(hd.levels)
        print(f"{st}-pt {m}^3 {kind}: levels host {len(hh.levels)} dev {len(hd.levels)}  t host {th_:.2f} dev {td:.2f}", flush=True)
        for l, (a, b) in enumerate(zip(hh.levels, hd.levels)):
            ok &= cmp(a.A, b.A, f"A{l}")
            ok &= np.array_equal(a.M.m_diag, np.asarray(b.M.m_diag))
            if a.P is not None:
                ok &= cmp(a.P, b.P, f"P{l}")
                ok &= cmp(a.restrict_op(), b.restrict_op(), f"R{l}")
        print("   bitwise:", ok, flush=True)
for m in [int(x) for x in sys.argv[1:]]:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    D = P.poisson3d_device(m)
    levels, st = DS.build_levels(D, P.CoarseningConfig(), trace=lambda s: print(s, flush=True))
    torch.cuda.synchronize()
    print(f"device setup {m}^3: {time.perf_counter() - t0:.2f} s levels {[L.n for L in levels]} nnz {[L.A.nnz for L in levels]}", flush=True)
    print("mem GB", torch.cuda.max_memory_allocated() / 1e9)
