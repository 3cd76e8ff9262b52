"""Fourier-family line transforms with the solver's conventions (reference: transforms.py).

Definitions (unnormalized forward sums; DFT carries 1/n on the forward leg),
`/root/reference/pkg/src/fastpoisson/transforms.py:3-28`:

    DST-I    2 sum f_j sin(pi (j+1)(k+1)/(n+1))
    DST-II   2 sum f_j sin(pi (j+1/2)(k+1)/n)
    DST-III  (-1)^k f_{n-1} + 2 sum_{j<n-1} f_j sin(pi (j+1)(k+1/2)/n)
    DCT-I    f_0 + (-1)^k f_{n-1} + 2 sum_{0<j<n-1} f_j cos(pi j k/(n-1))
    DCT-II   2 sum f_j cos(pi (j+1/2) k/n)
    DCT-III  f_0 + 2 sum_{j>0} f_j cos(pi j (k+1/2)/n)
    DFT      (1/n) sum f_j e^{-2 pi i k j/n};  IDFT  sum f^_k e^{+2 pi i k j/n}

Execution is on the GPU through the native library, one engine per (kind, n):
power-of-two lengths on the FFT line engine (half-length complex FFT + pre/post
twiddles); lengths whose FFT length factors into primes <= 61 on the mixed-radix
engine (csrc/fp_mr.cu); any other length on the Bluestein (chirp-z) engine
(csrc/fp_blue.cu: a zero-padded power-of-two convolution on the FFT engine,
four-step beyond 8192 points), except short lines (n < 128), which stay on the
dense direct-summation engine with correctly rounded coefficients.  Every n is
supported, as in the reference (scipy.fft).  ``naive_transform`` is the literal
O(n^2) host evaluation kept as part of the public API (transforms.py:188-229).
"""

from __future__ import annotations

import threading
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _device as dv
from . import _native as nat
from .grid import BoundaryCondition, ConfigurationError, GridKind


class TransformKind(Enum):
    DFT = "dft"
    IDFT = "idft"
    DST1 = "dst1"
    DST2 = "dst2"
    DST3 = "dst3"
    DCT1 = "dct1"
    DCT2 = "dct2"
    DCT3 = "dct3"

    @property
    def is_complex(self) -> bool:
        return self in (TransformKind.DFT, TransformKind.IDFT)


_TK = TransformKind
_KIND_ID = {_TK.DFT: nat.FP_DFT, _TK.IDFT: nat.FP_IDFT, _TK.DST1: nat.FP_DST1, _TK.DST2: nat.FP_DST2,
            _TK.DST3: nat.FP_DST3, _TK.DCT1: nat.FP_DCT1, _TK.DCT2: nat.FP_DCT2, _TK.DCT3: nat.FP_DCT3}
_MIN_LENGTH = {_TK.DCT1: 2}


@dataclass(frozen=True)
class TransformPair:
    """Forward/backward kinds of one boundary row and the backward scale."""

    forward: TransformKind
    backward: TransformKind

    def backward_scale(self, n: int) -> float:
        # backward(forward(f)) == f  (transforms.py:88-96)
        if self.forward is _TK.DFT:
            return 1.0
        if self.forward is _TK.DST1:
            return 1.0 / (2.0 * (n + 1))
        if self.forward is _TK.DCT1:
            return 1.0 / (2.0 * (n - 1))
        return 1.0 / (2.0 * n)


_PAIRS = {
    (BoundaryCondition.PERIODIC, GridKind.REGULAR): TransformPair(_TK.DFT, _TK.IDFT),
    (BoundaryCondition.DIRICHLET, GridKind.REGULAR): TransformPair(_TK.DST1, _TK.DST1),
    (BoundaryCondition.DIRICHLET, GridKind.STAGGERED): TransformPair(_TK.DST2, _TK.DST3),
    (BoundaryCondition.NEUMANN, GridKind.REGULAR): TransformPair(_TK.DCT1, _TK.DCT1),
    (BoundaryCondition.NEUMANN, GridKind.STAGGERED): TransformPair(_TK.DCT2, _TK.DCT3),
}


def transform_pair_for(bc: BoundaryCondition, grid: GridKind) -> TransformPair:
    pair = _PAIRS.get((bc, grid))
    if pair is None:
        raise ConfigurationError(
            f"no discrete transform for boundary condition {bc.value!r} on a {grid.value} grid"
        )
    return pair


# native transform objects, shared by all plans of one (kind, n, precision, device)
_native_cache: dict = {}
_cache_lock = threading.Lock()


class _NativeTransform:
    def __init__(self, kind: TransformKind, n: int, precision: int, device: int):
        import ctypes

        lib = nat.load()
        h = ctypes.c_void_p()
        nat.check(lib.fp_transform_create(_KIND_ID[kind], int(n), precision, device, ctypes.byref(h)))
        self.handle = h
        self._lib = lib

    def __del__(self):
        try:
            self._lib.fp_transform_destroy(self.handle)
        except Exception:  # pragma: no cover - interpreter shutdown
            pass


def _native_for(kind, n, precision, device_index):
    key = (kind, n, precision, device_index)
    with _cache_lock:
        obj = _native_cache.get(key)
        if obj is None:
            obj = _NativeTransform(kind, n, precision, device_index)
            _native_cache[key] = obj
        return obj


@dataclass(frozen=True)
class TransformPlan:
    """1D transform of one kind and length along ``axis`` (transforms.py:128-177).

    Accepts numpy arrays (copied to the GPU and back) or CUDA tensors (computed
    in place in HBM, result returned as a tensor).  ``workers`` is accepted for
    signature compatibility; parallelism is the GPU's.
    """

    kind: TransformKind
    n: int
    axis: int = -1
    workers: int = 1

    def __post_init__(self):
        if self.n < _MIN_LENGTH.get(self.kind, 1):
            raise ConfigurationError(f"{self.kind.value} requires n >= {_MIN_LENGTH[self.kind]}, got n={self.n}")

    def _check(self, line):
        if not dv.is_tensor(line):
            line = np.asarray(line)
        if line.ndim == 0 or line.shape[self.axis] != self.n:
            raise ValueError(f"plan expects length {self.n} along axis {self.axis}, got shape {tuple(line.shape)}")
        return line

    def execute_real(self, line):
        if self.kind.is_complex:
            raise ValueError(f"{self.kind.value} is a complex transform; use execute_complex")
        line = self._check(line)
        return self._run(line)

    def execute_complex(self, line):
        if not self.kind.is_complex:
            raise ValueError(f"{self.kind.value} is a real transform; use execute_real")
        line = self._check(line)
        return self._run(line)

    def execute(self, line):
        return self.execute_complex(line) if self.kind.is_complex else self.execute_real(line)

    # -- device execution -------------------------------------------------
    def _run(self, line):
        t = dv.torch()
        host = not dv.is_tensor(line)
        if host:
            arr = line
            if self.kind.is_complex:
                if arr.dtype in (np.float32, np.complex64):
                    work_np = np.complex64 if arr.dtype == np.complex64 else np.float32
                elif np.iscomplexobj(arr):
                    work_np = np.complex128
                else:
                    work_np = np.float64
                arr = np.asarray(arr, dtype=work_np)
            else:
                if np.iscomplexobj(arr):
                    raise TypeError("real transforms take real input")
                arr = np.asarray(arr, dtype=np.float32 if arr.dtype == np.float32 else np.float64)
            device = dv.require_cuda()
            x = dv.to_device(arr, device)
        else:
            x = line
            device = x.device
            if self.kind.is_complex:
                if x.dtype not in (t.float32, t.float64, t.complex64, t.complex128):
                    x = x.to(t.float64)
            else:
                if x.is_complex():
                    raise TypeError("real transforms take real input")
                if x.dtype not in (t.float32, t.float64):
                    x = x.to(t.float64)
        single = x.dtype in (t.float32, t.complex64)
        precision = nat.FP_F32 if single else nat.FP_F64
        out_dtype = (t.complex64 if single else t.complex128) if self.kind.is_complex else x.dtype
        if self.kind.is_complex and not x.is_complex():
            x = x.to(out_dtype)   # the ABI takes complex operands for DFT/IDFT
        nd = x.ndim
        ax = self.axis % nd
        # collapse to (pre, n, post) so any rank maps onto the 3D ABI
        pre = int(np.prod(x.shape[:ax], dtype=np.int64))
        post = int(np.prod(x.shape[ax + 1:], dtype=np.int64))
        if nd > 3 or not _collapsible(x, ax):
            x = x.contiguous()
        x3 = x.reshape(pre, self.n, post)
        y3 = t.empty((pre, self.n, post), dtype=out_dtype, device=device)
        if pre * post > 0:
            nt = _native_for(self.kind, self.n, precision, device.index)
            shape = nat.strides_array((pre, self.n, post))
            rc = nt._lib.fp_transform_execute(
                nt.handle, 3, shape, 1,
                x3.data_ptr(), dv.fp_dtype_of_torch(x3.dtype), nat.strides_array(x3.stride()),
                y3.data_ptr(), dv.fp_dtype_of_torch(y3.dtype), nat.strides_array(y3.stride()),
                dv.stream_handle(device))
            nat.check(rc)
        y = y3.reshape(x.shape)
        if host:
            return y.cpu().numpy()
        return y


def _collapsible(x, ax) -> bool:
    try:
        x.view(int(np.prod(x.shape[:ax], dtype=np.int64)), x.shape[ax], -1)
        return True
    except Exception:
        return False


def execute_real(plan: TransformPlan, line):
    return plan.execute_real(line)


def execute_complex(plan: TransformPlan, line):
    return plan.execute_complex(line)


def naive_transform(kind: TransformKind, line) -> np.ndarray:
    """Direct O(n^2) evaluation of the defining sums on the host (API compat)."""
    x = np.asarray(line)
    n = x.shape[-1]
    if n < _MIN_LENGTH.get(kind, 1):
        raise ValueError(f"{kind.value} requires n >= {_MIN_LENGTH[kind]}, got n={n}")
    jj = np.arange(n)[None, :]
    kk = np.arange(n)[:, None]
    if kind.is_complex:
        sign = -1.0 if kind is _TK.DFT else 1.0
        basis = np.exp(sign * 2j * np.pi * kk * jj / n)
        if kind is _TK.DFT:
            basis = basis / n
        return basis @ x.astype(np.complex128)
    if kind is _TK.DST1:
        basis = 2.0 * np.sin(np.pi * (jj + 1) * (kk + 1) / (n + 1))
    elif kind is _TK.DST2:
        basis = 2.0 * np.sin(np.pi * (jj + 0.5) * (kk + 1) / n)
    elif kind is _TK.DST3:
        basis = 2.0 * np.sin(np.pi * (jj + 1) * (kk + 0.5) / n)
        basis[:, n - 1] = (-1.0) ** np.arange(n)
    elif kind is _TK.DCT1:
        basis = 2.0 * np.cos(np.pi * jj * kk / (n - 1))
        basis[:, 0] = 1.0
        basis[:, n - 1] = (-1.0) ** np.arange(n)
    elif kind is _TK.DCT2:
        basis = 2.0 * np.cos(np.pi * (jj + 0.5) * kk / n)
    else:
        basis = 2.0 * np.cos(np.pi * jj * (kk + 0.5) / n)
        basis[:, 0] = 1.0
    dtype = np.complex128 if np.iscomplexobj(x) else np.float64
    return basis @ x.astype(dtype)
