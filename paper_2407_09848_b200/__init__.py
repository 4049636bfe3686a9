"""B200-native polynomial smoothers inside AMG-preconditioned PCG.

Drop-in for the hot path of the reference package ``amgpoly``
(arXiv 2407.09848): the public names below keep the reference's signatures
(smoothers.py, amg.py, krylov.py, sparse.py, problems.py) while every
numeric operation of the solve phase runs in hand-written sm_100a kernels
(libamgp.so, C ABI in include/amgp.h).  There is no CPU fallback.
"""

from .amg import (
    AmgHierarchy,
    CoarseningConfig,
    DeviceHierarchy,
    Level,
    as_vcycle_preconditioner,
    build_hierarchy,
    hierarchy_from_levels,
    vcycle_apply,
)
from .krylov import KrylovConfig, SolveReport, solve
from .params import BetaTable, load_beta_tables, optimal_a
from .problems import poisson3d, poisson3d_27, poisson3d_device
from .smoothers import (
    FAMILIES,
    L1JacobiData,
    PolySmootherConfig,
    as_preconditioner,
    l1_jacobi_diag,
    smoother_apply,
    smoother_apply_batch,
    smoother_error_apply,
)
from .sparse import CsrMatrix, DeviceMatrix, fused_update, reset_spmv_count, spmv, spmv_count

__version__ = "0.1.0"
