"""Binding of the C ABI in ``include/fastpoisson_b200.h``.

This is the only place the Python host mirror touches native code.  The
library is loaded lazily; a missing or unloadable library raises immediately
(there is no CPU fallback for the solve path).

Two layers: ctypes for plan management and the cold entry points, and the
PyTorch extension ``lib/fastpoisson_b200_torch.so`` (csrc/fp_torch_ext.cpp) for
the solve itself -- ``torch.ops.fastpoisson_b200.solve`` takes the tensors,
reads the current stream and calls ``fp_solve`` of this same library instance.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import POINTER, Structure, c_double, c_float, c_int, c_int32, c_int64, c_size_t, c_void_p, c_char_p

from ._build import LIB_PATH, TORCH_EXT_PATH

FP_OK = 0
FP_ERR_CONFIG = 1
FP_ERR_VALUE = 2
FP_ERR_UNSUPPORTED = 3
FP_ERR_CUDA = 4
FP_ERR_NONFINITE = 5
FP_ERR_ALLOC = 6

FP_BC_PERIODIC, FP_BC_DIRICHLET, FP_BC_NEUMANN = 0, 1, 2
FP_GRID_REGULAR, FP_GRID_STAGGERED = 0, 1
FP_APPROX_SPECTRAL, FP_APPROX_FD2 = 0, 1
FP_F64, FP_F32, FP_C128, FP_C64 = 0, 1, 2, 3
FP_DFT, FP_IDFT, FP_DST1, FP_DST2, FP_DST3, FP_DCT1, FP_DCT2, FP_DCT3 = range(8)


class FpConfig(Structure):
    _fields_ = [
        ("ndim", c_int),
        ("n", c_int64 * 3),
        ("length", c_double * 3),
        ("bc", c_int * 3),
        ("kind", c_int * 3),
        ("approx", c_int),
        ("precision", c_int),
        ("eig", POINTER(c_double) * 3),
    ]


class FpPlanInfo(Structure):
    _fields_ = [
        ("ndim", c_int),
        ("mode_mixed", c_int),
        ("singular", c_int),
        ("periodic_mask", c_int),
        ("null_scale", c_double),
        ("num_passes", c_int),
        ("middle_axis", c_int),
        ("fft_axes_mask", c_int),
        ("exact_mean", c_int),
    ]


class FpSolveInfo(Structure):
    _fields_ = [("dc", c_double), ("nonfinite", c_int32), ("reserved", c_int32)]


class FpDistInfo(Structure):
    _fields_ = [
        ("nranks", c_int), ("rank", c_int),
        ("local_n0", c_int64), ("offset0", c_int64),
        ("exch_n1", c_int64), ("true_n1", c_int64), ("exch_n2", c_int64), ("block_n1", c_int64),
        ("exch_complex", c_int), ("r_axis", c_int), ("elem_bytes", c_int),
        ("exchange_bytes", c_size_t),
        ("pitch_n0", c_int64),
    ]


class FpSolveResult(Structure):
    _fields_ = [("removed_mean", c_double), ("timing", c_double * 3), ("total_seconds", c_double)]


# symbol -> (restype, argtypes); the CPU test tier checks every one is exported
SIGNATURES = {
    "fp_abi_version": (c_int, []),
    "fp_last_error": (c_char_p, []),
    "fp_plan_create": (c_int, [POINTER(FpConfig), c_int, POINTER(c_void_p)]),
    "fp_plan_destroy": (c_int, [c_void_p]),
    "fp_plan_info_get": (c_int, [c_void_p, POINTER(FpPlanInfo)]),
    "fp_plan_workspace_bytes": (c_int, [c_void_p, c_int, POINTER(c_size_t)]),
    "fp_solve": (
        c_int,
        [c_void_p, c_void_p, c_int, POINTER(c_int64), c_void_p, POINTER(c_int64), c_void_p, c_size_t,
         c_void_p, c_void_p, POINTER(c_void_p)],
    ),
    "fp_solve_ex": (
        c_int,
        [c_void_p, c_void_p, c_int, POINTER(c_int64), c_void_p, POINTER(c_int64), c_void_p, c_size_t,
         c_void_p, c_void_p, POINTER(c_void_p), POINTER(c_void_p)],
    ),
    "fp_solve_override": (
        c_int,
        [c_void_p, c_void_p, c_int, POINTER(c_int64), c_void_p, POINTER(c_int64), c_void_p, c_size_t,
         c_void_p, c_void_p, POINTER(c_void_p), c_void_p],
    ),
    "fp_plan_workspace_bytes_ex": (c_int, [c_void_p, c_int, c_int, POINTER(c_size_t)]),
    "fp_plan_spectrum": (c_int, [c_void_p, POINTER(c_int64), POINTER(c_int)]),
    "fp_solve_host": (
        c_int,
        [c_void_p, c_void_p, c_int, POINTER(c_int64), c_void_p, POINTER(c_int64), POINTER(FpSolveResult)],
    ),
    "fp_removed_mean": (c_int, [c_void_p, POINTER(FpSolveInfo), POINTER(c_double)]),
    "fp_transform_create": (c_int, [c_int, c_int64, c_int, c_int, POINTER(c_void_p)]),
    "fp_transform_destroy": (c_int, [c_void_p]),
    "fp_transform_execute": (
        c_int,
        [c_void_p, c_int, POINTER(c_int64), c_int, c_void_p, c_int, POINTER(c_int64), c_void_p, c_int,
         POINTER(c_int64), c_void_p],
    ),
    "fp_solve_divergence": (
        c_int,
        [c_void_p, c_void_p, POINTER(c_int64), c_void_p, POINTER(c_int64), c_double, c_void_p, POINTER(c_int64),
         c_void_p, c_size_t, c_void_p, c_void_p],
    ),
    "fp_project_correct": (
        c_int,
        [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_void_p],
    ),
    "fp_dist_layout": (c_int, [POINTER(FpConfig), c_int, c_int, POINTER(FpDistInfo)]),
    "fp_plan_create_dist": (c_int, [POINTER(FpConfig), c_int, c_int, c_int, POINTER(c_void_p)]),
    "fp_solve_phase": (
        c_int,
        [c_void_p, c_int, c_void_p, c_int, POINTER(c_int64), c_void_p, POINTER(c_int64), c_void_p, c_void_p,
         c_size_t, c_void_p, c_void_p],
    ),
    "fp_dist_mean_partial": (
        c_int, [c_void_p, c_void_p, POINTER(c_int64), c_void_p, c_size_t, c_void_p, c_void_p],
    ),
    "fp_dist_mean_subtract": (c_int, [c_void_p, c_void_p, POINTER(c_int64), c_void_p, c_void_p]),
    "fp_solve_mid_rows": (
        c_int, [c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_size_t, c_void_p, c_void_p],
    ),
    "fp_event_create": (c_int, [POINTER(c_void_p)]),
    "fp_event_create_on": (c_int, [c_int, POINTER(c_void_p)]),
    "fp_event_destroy": (c_int, [c_void_p]),
    "fp_event_elapsed_ms": (c_int, [c_void_p, c_void_p, POINTER(c_float)]),
}

_lib = None
_lock = threading.Lock()


def load(path=None):
    """Load (once) and return the native library; raises if it is missing."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        # FP_NATIVE_LIB: a variant build of the same library (A/B benchmarks only)
        p = str(path or os.environ.get("FP_NATIVE_LIB") or LIB_PATH)
        try:
            lib = ctypes.CDLL(p)
        except OSError as exc:
            raise RuntimeError(
                f"native library {p} is not loadable ({exc}); build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` -- the solve path has no CPU fallback"
            ) from None
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


_ext_ops = None


def torch_ext():
    """``torch.ops.fastpoisson_b200`` bound to the loaded kernel library (raises if the
    extension is missing: build it with ``__graft_entry__.build()``).  ``FP_BINDING=ctypes``
    selects the plain ctypes call instead (A/B and debugging)."""
    global _ext_ops
    if _ext_ops is not None:
        return _ext_ops
    lib = load()
    with _lock:
        if _ext_ops is not None:
            return _ext_ops
        import torch

        try:
            torch.ops.load_library(str(TORCH_EXT_PATH))
        except (OSError, RuntimeError) as exc:
            raise RuntimeError(
                f"PyTorch extension {TORCH_EXT_PATH} is not loadable ({exc}); build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'`"
            ) from None
        ops = torch.ops.fastpoisson_b200
        ops.bind(ctypes.cast(lib.fp_solve, c_void_p).value, ctypes.cast(lib.fp_solve_override, c_void_p).value)
        _ext_ops = ops
        return ops


_ext_missing_warned = False


def use_torch_ext() -> bool:
    """The solve goes through the PyTorch extension unless ``FP_BINDING=ctypes`` -- or the
    extension was never built, in which case the same C ABI entry point is called through
    ctypes (same kernels, same library; a warning says so once)."""
    global _ext_missing_warned
    if os.environ.get("FP_BINDING", "torch") == "ctypes":
        return False
    if _ext_ops is None and not TORCH_EXT_PATH.exists():
        if not _ext_missing_warned:
            import warnings

            warnings.warn(f"{TORCH_EXT_PATH} not built: calling fp_solve through ctypes "
                          "(build it with `python -c 'import __graft_entry__ as g; g.build()'`)", RuntimeWarning)
            _ext_missing_warned = True
        return False
    return True


def last_error() -> str:
    msg = load().fp_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = ""):
    """Map an fp_status to the reference's exception types."""
    if status == FP_OK:
        return
    from .grid import ConfigurationError

    msg = last_error() or what
    if status == FP_ERR_CONFIG:
        raise ConfigurationError(msg)
    if status in (FP_ERR_VALUE, FP_ERR_NONFINITE):
        raise ValueError(msg)
    if status == FP_ERR_ALLOC:
        raise MemoryError(msg)
    if status == FP_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


def strides_array(strides):
    arr = (c_int64 * 3)()
    for i, s in enumerate(strides):
        arr[i] = int(s)
    return arr
