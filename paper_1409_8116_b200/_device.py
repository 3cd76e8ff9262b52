"""Device plumbing shared by the solver and transform front ends.

PyTorch provides HBM allocations (caching allocator), streams and host<->device
copies; every arithmetic operation on the solve path is a kernel of the native
library.  Nothing here computes on the CPU.
"""

from __future__ import annotations

import numpy as np

from . import _native as nat

_NP_TO_FP = {np.dtype(np.float64): nat.FP_F64, np.dtype(np.float32): nat.FP_F32,
             np.dtype(np.complex128): nat.FP_C128, np.dtype(np.complex64): nat.FP_C64}


def torch():
    import torch as _t

    return _t


def is_tensor(obj) -> bool:
    return type(obj).__module__.startswith("torch") and hasattr(obj, "data_ptr")


def require_cuda(device=None):
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError(
            "no CUDA device available: the fastpoisson B200 solve path runs only on the GPU (no CPU fallback)"
        )
    if device is None:
        return t.device("cuda", t.cuda.current_device())
    dev = t.device(device)
    if dev.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {dev}")
    if dev.index is None:
        dev = t.device("cuda", t.cuda.current_device())
    return dev


def fp_dtype_of_torch(dt) -> int:
    t = torch()
    table = {t.float64: nat.FP_F64, t.float32: nat.FP_F32, t.complex128: nat.FP_C128, t.complex64: nat.FP_C64}
    if dt not in table:
        raise TypeError(f"unsupported dtype {dt}")
    return table[dt]


def torch_dtype(np_dtype):
    t = torch()
    return {np.dtype(np.float64): t.float64, np.dtype(np.float32): t.float32,
            np.dtype(np.complex128): t.complex128, np.dtype(np.complex64): t.complex64}[np.dtype(np_dtype)]


def stream_handle(device) -> int:
    return torch().cuda.current_stream(device).cuda_stream


def to_device(arr: np.ndarray, device):
    """Host array -> device tensor (dense C order); async when ``arr`` is pinned."""
    t = torch()
    a = np.ascontiguousarray(arr)
    host = t.from_numpy(a)
    return host.to(device, non_blocking=True)


def overlaps(x, y) -> bool:
    """Do two device tensors share any bytes?"""
    if x.numel() == 0 or y.numel() == 0:
        return False
    xs, xe = _span(x)
    ys, ye = _span(y)
    return xs < ye and ys < xe


def _span(x):
    start = x.data_ptr()
    extent = sum((s - 1) * st for s, st in zip(x.shape, x.stride())) + 1
    return start, start + extent * x.element_size()


def same_view(x, y) -> bool:
    return (x.data_ptr() == y.data_ptr() and tuple(x.shape) == tuple(y.shape)
            and tuple(x.stride()) == tuple(y.stride()) and x.dtype == y.dtype)
