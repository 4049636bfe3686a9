"""ctypes binding of libamgp.so (include/amgp.h) and device-memory plumbing.

The shared library is the product: every numeric operation of the hot path
runs in its sm_100a kernels.  There is no CPU fallback -- if the library is
missing or no CUDA device is present, every device operation raises.

Device vectors are torch CUDA float64 tensors (torch is plumbing: allocation,
streams); the library runs on its own CUDA stream, which is made to wait for
the caller's current stream on entry and vice versa on exit.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import os
import threading
import warnings

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AMGP_LIB", os.path.join(PKG, "libamgp.so"))  # override: tuning variants

AMGP_OK = 0
AMGP_EINVAL = -1

FAMILY_CODES = {"l1_jacobi": 0, "cheb4": 1, "opt_cheb4": 2, "opt_cheb1": 3}
COARSE_CODES = {"l1_jacobi": 0, "dense_direct": 1, "smoother": 2}
VARIANT_CODES = {"pcg": 0, "fcg": 1, "pcg1": 2}

_P64 = C.POINTER(C.c_int64)
_PD = C.POINTER(C.c_double)
_VP = C.c_void_p


class SmootherCfg(C.Structure):
    _fields_ = [
        ("family", C.c_int32),
        ("degree", C.c_int32),
        ("a", C.c_double),
        ("rho_scale", C.c_double),
        ("beta", _PD),
    ]


class SolveReportC(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32),
        ("converged", C.c_int32),
        ("breakdown", C.c_int32),
        ("spmv_count", C.c_int32),
        ("precond_count", C.c_int32),
        ("n_history", C.c_int32),
        ("final_relres", C.c_double),
        ("elapsed_s", C.c_double),
    ]


# name -> (restype, argtypes); mirrors include/amgp.h
_SIGS = {
    "amgp_last_error": (C.c_char_p, []),
    "amgp_version": (C.c_int, []),
    "amgp_ctx_create": (C.c_int, [C.c_int, _VP, C.POINTER(_VP)]),
    "amgp_ctx_destroy": (C.c_int, [_VP]),
    "amgp_ctx_set_stream": (C.c_int, [_VP, _VP]),
    "amgp_ctx_sync": (C.c_int, [_VP]),
    "amgp_ctx_launch_count": (C.c_int, [_VP, _P64]),
    "amgp_malloc": (C.c_int, [_VP, C.c_int64, C.POINTER(_VP)]),
    "amgp_free": (C.c_int, [_VP, _VP]),
    "amgp_memcpy_h2d": (C.c_int, [_VP, _VP, _VP, C.c_int64]),
    "amgp_memcpy_d2h": (C.c_int, [_VP, _VP, _VP, C.c_int64]),
    "amgp_mat_from_csr": (C.c_int, [_VP, C.c_int64, C.c_int64, _P64, _P64, _PD, C.POINTER(_VP)]),
    "amgp_mat_poisson3d": (C.c_int, [_VP, C.c_int64, C.c_int, C.c_int64, C.c_int64, C.POINTER(_VP)]),
    "amgp_mat_destroy": (C.c_int, [_VP]),
    "amgp_mat_info": (C.c_int, [_VP, _P64, _P64, _P64, _P64, _P64]),
    "amgp_mat_to_csr": (C.c_int, [_VP, _P64, _P64, _PD]),
    "amgp_mat_l1_diag": (C.c_int, [_VP, _VP]),
    "amgp_spmv": (C.c_int, [_VP, _VP, _VP, _VP]),
    "amgp_fused_update": (C.c_int, [_VP, C.c_int64, C.c_double, C.c_double, C.c_double,
                                     _VP, _VP, _VP, _VP]),
    "amgp_smoother_apply": (C.c_int, [_VP, _VP, _VP, C.POINTER(SmootherCfg), _VP, _VP, _VP]),
    "amgp_vec_update": (C.c_int, [_VP, C.c_int64, C.c_double, _VP, _VP, _VP, C.c_int]),
    "amgp_smoother_apply_host": (C.c_int, [_VP, _VP, _VP, C.c_int, C.POINTER(SmootherCfg), C.POINTER(_VP),
                                           C.POINTER(_VP), C.POINTER(_VP)]),
    "amgp_hier_create": (C.c_int, [_VP, C.c_int, C.POINTER(_VP), C.POINTER(_VP), C.POINTER(_VP),
                                    C.POINTER(_VP), C.c_int, C.c_int, C.POINTER(_VP)]),
    "amgp_hier_set_smoother": (C.c_int, [_VP, C.c_int, C.POINTER(SmootherCfg)]),
    "amgp_hier_set_coarse_cholesky": (C.c_int, [_VP, _PD]),
    "amgp_hier_use_graph": (C.c_int, [_VP, C.c_int]),
    "amgp_hier_info": (C.c_int, [_VP, C.POINTER(C.c_int)]),
    "amgp_hier_destroy": (C.c_int, [_VP]),
    "amgp_vcycle_apply": (C.c_int, [_VP, _VP, _VP]),
    "amgp_pcg_solve": (C.c_int, [_VP, _VP, _VP, _VP, _VP, C.c_int, C.c_int, C.c_double, C.c_int,
                                  _PD, C.POINTER(SolveReportC)]),
    "amgp_sell_pack_host": (C.c_int, [C.c_int64, _P64, _P64, _PD, _P64, _P64, _P64,
                                       C.POINTER(C.c_int32), _PD]),
    "amgp_smoother_coefficients": (C.c_int, [C.POINTER(SmootherCfg), _PD]),
    "amgp_setup_set_threads": (C.c_int, [C.c_int]),
    "amgp_hcsr_info": (C.c_int, [_VP, _P64, _P64, _P64]),
    "amgp_hcsr_copy": (C.c_int, [_VP, _P64, _P64, _PD]),
    "amgp_hcsr_free": (C.c_int, [_VP]),
    "amgp_setup_sa_aggregate": (C.c_int, [C.c_int64, _P64, _P64, _PD, C.c_double, _P64, _P64]),
    "amgp_setup_matching_aggregate": (C.c_int, [C.c_int64, _P64, _P64, _PD, C.c_int, _P64, _P64]),
    "amgp_setup_smooth_prolongator": (C.c_int, [C.c_int64, _P64, _P64, _PD, _P64, C.c_int64,
                                                 C.c_double, C.POINTER(_VP)]),
    "amgp_setup_galerkin": (C.c_int, [C.c_int64, _P64, _P64, _PD, C.c_int64, _P64, _P64, _PD,
                                       C.POINTER(_VP)]),
    "amgp_setup_spmv": (C.c_int, [C.c_int64, _P64, _P64, _PD, _PD, _PD]),
    "amgp_setup_blas_dot": (C.c_double, [C.c_int64, _PD, _PD, C.c_int]),
    "amgp_ds_diag": (C.c_int, [_VP, _VP]),
    "amgp_ds_strength": (C.c_int, [_VP, _VP, C.c_double, C.c_int64, _VP, C.c_int64, _VP, _VP, _VP, _VP]),
    "amgp_ds_blas_dot3": (C.c_int, [_VP, C.c_int64, _VP, _VP, C.c_int, _PD]),
    "amgp_ds_lambda_max": (C.c_int, [_VP, _VP, _VP, _VP, C.c_int, C.c_int, C.c_int, _PD]),
    "amgp_ds_prolongator": (C.c_int, [_VP, _VP, _VP, _VP, C.c_double, C.c_int, _VP, _VP, _VP, _VP]),
    "amgp_ds_spgemm": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP, C.c_int64, _VP, _VP, _VP, C.c_int64,
                                  _VP, _VP, _VP, _VP]),
    "amgp_ds_symmetrize": (C.c_int, [_VP, C.c_int64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "amgp_ds_sym_lookup": (C.c_int, [_VP, C.c_int64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, C.c_int64, _P64]),
    "amgp_ds_symmetrize_lookup": (C.c_int, [_VP, C.c_int64, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP,
                                             _VP]),
    "amgp_mat_from_dcsr": (C.c_int, [_VP, C.c_int64, C.c_int64, _VP, _VP, _VP, C.c_int, C.POINTER(_VP)]),
    "amgp_mat_nown": (C.c_int, [_VP, _P64]),
    "amgp_setup_sa_pass1": (C.c_int, [C.c_int64, _P64, C.POINTER(C.c_int32), _P64, _P64]),
    "amgp_setup_sa_pass2": (C.c_int, [C.c_int64, _P64, _P64, C.POINTER(C.c_int32), _PD, _P64, _P64]),
    "amgp_comm_unique_id": (C.c_int, [C.c_char_p]),
    "amgp_ctx_init_comm": (C.c_int, [_VP, C.c_int, C.c_int, C.c_char_p]),
    "amgp_ctx_comm_info": (C.c_int, [_VP, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "amgp_mat_set_halo": (C.c_int, [_VP, C.c_int64, C.c_int, C.POINTER(C.c_int), _P64, _P64, _P64]),
    "amgp_mat_halo_info": (C.c_int, [_VP, _P64, _P64, _P64, _P64]),
    "amgp_mat_localize": (C.c_int, [_VP, C.c_int64, C.c_int64, C.c_int, _P64, _P64]),
}

_lib = None
_lib_lock = threading.Lock()


def lib():
    """The loaded libamgp.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        with _lib_lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"{LIB_PATH} not found: build it with "
                        "`python -m paper_2407_09848_b200._build` (no CPU fallback exists)")
                handle = C.CDLL(LIB_PATH)
                for name, (res, args) in _SIGS.items():
                    fn = getattr(handle, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = handle
    return _lib


def exported_symbols():
    return list(_SIGS)


def check(status):
    if status == AMGP_OK:
        return
    msg = lib().amgp_last_error().decode(errors="replace")
    if status == AMGP_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"libamgp error {status}: {msg}")


# ---------------------------------------------------------------- context
class Context:
    """One library context per CUDA device, running on a private torch stream."""

    def __init__(self, device):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("paper_2407_09848_b200 needs a CUDA device (no CPU fallback)")
        self.torch = torch
        self.device = torch.device("cuda", device)
        with torch.cuda.device(self.device):
            self.stream = torch.cuda.Stream(device=self.device)
        h = _VP()
        check(lib().amgp_ctx_create(device, _VP(self.stream.cuda_stream), C.byref(h)))
        self.handle = h

    def launches(self):
        c = C.c_int64(0)
        check(lib().amgp_ctx_launch_count(self.handle, C.byref(c)))
        return c.value

    def sync(self):
        check(lib().amgp_ctx_sync(self.handle))

    @contextlib.contextmanager
    def scope(self):
        """Run library work on the private stream, ordered against the caller's."""
        torch = self.torch
        with torch.cuda.device(self.device):
            caller = torch.cuda.current_stream(self.device)
            if caller.cuda_stream == self.stream.cuda_stream:
                yield self
                return
            self.stream.wait_stream(caller)
            with torch.cuda.stream(self.stream):
                yield self
            caller.wait_stream(self.stream)


_ctxs = {}
_ctx_lock = threading.Lock()


def current_device():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2407_09848_b200 needs a CUDA device (no CPU fallback)")
    return torch.cuda.current_device()


def ctx(device=None):
    dev = current_device() if device is None else int(device)
    with _ctx_lock:
        if dev not in _ctxs:
            _ctxs[dev] = Context(dev)
        return _ctxs[dev]


# ---------------------------------------------------------------- vectors
def is_torch(a):
    try:
        import torch

        return isinstance(a, torch.Tensor)
    except ImportError:
        return False


def to_device(a, c=None, copy=False):
    """numpy / torch -> contiguous float64 CUDA tensor on the context device.

    Host arrays go through pinned memory.  Device tensors are used in place
    unless ``copy`` (or a dtype/contiguity/device change forces a copy).
    """
    c = c or ctx()
    torch = c.torch
    if is_torch(a):
        t = a
        if not t.is_cuda:  # host tensor (pinned: asynchronous upload)
            t = t.to(dtype=torch.float64).contiguous()
            return t.to(c.device, non_blocking=t.is_pinned())
        if t.device != c.device or t.dtype != torch.float64 or not t.is_contiguous():
            t = t.to(device=c.device, dtype=torch.float64).contiguous()
        elif copy:
            t = t.clone()
        t.record_stream(c.stream)
        return t
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    with warnings.catch_warnings():
        # read-only arrays are only read (pinned copy / H2D upload)
        warnings.simplefilter("ignore", UserWarning)
        host = torch.from_numpy(arr)
    if host.numel() * 8 >= (1 << 16):
        host = host.pin_memory()
    return host.to(c.device, non_blocking=True)


def empty(n, c=None):
    c = c or ctx()
    return c.torch.empty(int(n), dtype=c.torch.float64, device=c.device)


def ptr(t):
    return _VP(t.data_ptr()) if t is not None else None


def to_host(t):
    """CUDA tensor -> numpy (synchronous)."""
    return t.cpu().numpy()


def like(t, ref):
    """Return device result t in the container type of the input ref:
    CUDA tensor -> as is; host tensor -> host tensor; else numpy."""
    if is_torch(ref):
        if ref.is_cuda:
            return t
        if ref.is_pinned():  # pinned in -> pinned out (cached pinned allocator, DMA copy)
            out = t.new_empty(t.shape, device="cpu", pin_memory=True)
            out.copy_(t)
            return out
        return t.cpu()
    return to_host(t)


def smoother_cfg(config):
    """Build the C struct from a PolySmootherConfig (keeps beta alive)."""
    beta = None
    if config.family == "opt_cheb4":
        beta = np.ascontiguousarray(config.beta.beta, dtype=np.float64)
    cfg = SmootherCfg(
        FAMILY_CODES[config.family],
        int(config.degree),
        float(config.a) if config.a is not None else 0.0,
        float(config.rho_scale),
        beta.ctypes.data_as(_PD) if beta is not None else None,
    )
    cfg._keep = beta
    return cfg
