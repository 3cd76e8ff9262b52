"""Plan/execute Poisson solver on B200 (reference: solver.py).

Drop-in for `/root/reference/pkg/src/fastpoisson/solver.py`: the same
``SolverConfig`` / ``SolverPlan(config, threads).solve(rhs, out)`` /
``SolveReport`` / ``plan_create`` / ``solve`` / ``solve_mixed`` surface, the
same validation errors, the same null-mode policy.  The solve itself runs in
HBM through the native library (include/fastpoisson_b200.h): a handful of
passes, each reading and writing the field once, with the eigenvalue division
fused into the middle pass.

Inputs
  numpy arrays / Fields over numpy: copied to the GPU, solved, copied back
      (`out` is only written after the device reports a finite rhs, so the
      reference's "ValueError before any output is written" holds).
  torch CUDA tensors / Fields over them: solved in place in HBM through their
      strides (ghost-cell sub-blocks included), no host round trip.

Deviations (documented in DESIGN.md): the final `work -= work.mean()` of the
reference (solver.py:224-225) is not a separate pass -- the null coefficient is
zeroed exactly, so the output mean is zero to roundoff; for device tensors a
non-finite rhs is reported after the solve, with `out` undefined.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field as dataclass_field

import numpy as np

from . import _device as dv
from . import _native as nat
from .eigenvalues import combine_eigenvalues, eigenvalue_table, null_modes_of
from .field import as_array
from .grid import Approximation, BoundaryCondition, ConfigurationError, GridKind, GridSpec
from .transforms import TransformKind, transform_pair_for

_PRECISIONS = {"double": np.float64, "single": np.float32}
_BC_ID = {BoundaryCondition.PERIODIC: nat.FP_BC_PERIODIC, BoundaryCondition.DIRICHLET: nat.FP_BC_DIRICHLET,
          BoundaryCondition.NEUMANN: nat.FP_BC_NEUMANN}
_KIND_ID = {GridKind.REGULAR: nat.FP_GRID_REGULAR, GridKind.STAGGERED: nat.FP_GRID_STAGGERED}
_APPROX_ID = {Approximation.PSEUDO_SPECTRAL: nat.FP_APPROX_SPECTRAL, Approximation.FINITE_DIFFERENCE_2: nat.FP_APPROX_FD2}

# forward transform of the all-ones line at the null index (solver.py:56-62)
_ONES_NULL_COEFF = {
    TransformKind.DFT: lambda n: 1.0,
    TransformKind.DCT1: lambda n: 2.0 * (n - 1),
    TransformKind.DCT2: lambda n: 2.0 * n,
}


def _config_struct(config, tables=None):
    """fp_config for a SolverConfig, carrying the host mirror's numpy eigenvalue
    tables (bit-identical to the reference's, eigenvalues.py:51-83)."""
    if tables is None:
        tables = [eigenvalue_table(g, config.approximation) for g in config.grids]
    cfg = nat.FpConfig()
    cfg.ndim = config.dims
    keep = []
    for a, g in enumerate(config.grids):
        cfg.n[a] = g.n
        cfg.length[a] = float(g.length)
        cfg.bc[a] = _BC_ID[g.bc]
        cfg.kind[a] = _KIND_ID[g.kind]
        tab = np.ascontiguousarray(tables[a].values, dtype=np.float64)
        keep.append(tab)
        cfg.eig[a] = tab.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    cfg.approx = _APPROX_ID[config.approximation]
    cfg.precision = nat.FP_F32 if config.precision == "single" else nat.FP_F64
    return cfg, keep


@dataclass(frozen=True)
class SolverConfig:
    """Grid specification per axis plus the approximation to diagonalize (solver.py:65-119)."""

    grids: tuple
    approximation: Approximation
    precision: str = "double"

    def __post_init__(self):
        grids = tuple(self.grids)
        object.__setattr__(self, "grids", grids)
        if not 1 <= len(grids) <= 3:
            raise ConfigurationError(f"1 to 3 dimensions supported, got {len(grids)}")
        if any(not isinstance(g, GridSpec) for g in grids):
            raise ConfigurationError("grids must be GridSpec instances")
        if self.precision not in _PRECISIONS:
            raise ConfigurationError(f"precision must be one of {sorted(_PRECISIONS)}, got {self.precision!r}")
        walls = {(g.bc, g.kind) for g in grids if g.bc is not BoundaryCondition.PERIODIC}
        if len(walls) > 1:
            rows = sorted((b.value, k.value) for b, k in walls)
            raise ConfigurationError(
                "unsupported boundary pattern: non-periodic axes must all carry the same condition and "
                f"grid kind, got {rows}"
            )

    @property
    def dims(self) -> int:
        return len(self.grids)

    @property
    def shape(self) -> tuple:
        return tuple(g.n for g in self.grids)

    @property
    def dtype(self):
        return np.dtype(_PRECISIONS[self.precision])

    @property
    def periodic_axes(self) -> tuple:
        return tuple(i for i, g in enumerate(self.grids) if g.bc is BoundaryCondition.PERIODIC)

    @property
    def mode(self) -> str:
        return "uniform" if len({(g.bc, g.kind) for g in self.grids}) == 1 else "mixed"

    @property
    def singular(self) -> bool:
        return not any(g.bc is BoundaryCondition.DIRICHLET for g in self.grids)


@dataclass
class SolveReport:
    """Outcome bookkeeping for one solve (solver.py:122-129)."""

    removed_mean: float = 0.0
    mode: str = "uniform"
    periodic_axes: tuple = ()
    timing: dict = dataclass_field(default_factory=dict)


class _Events:
    """Four CUDA events (start / after forward / after diagonal / end), created on
    the plan's device (an event must share the device of the stream it is
    recorded on, whatever device is current)."""

    def __init__(self, lib, device_index: int):
        self._lib = lib
        self.ev = (ctypes.c_void_p * 4)()
        for i in range(4):
            h = ctypes.c_void_p()
            nat.check(lib.fp_event_create_on(int(device_index), ctypes.byref(h)))
            self.ev[i] = h

    def timing(self) -> dict:
        ms = ctypes.c_float()
        out = []
        for a, b in ((0, 1), (1, 2), (2, 3)):
            nat.check(self._lib.fp_event_elapsed_ms(self.ev[a], self.ev[b], ctypes.byref(ms)))
            out.append(ms.value * 1e-3)
        return {"forward": out[0], "diagonal": out[1], "backward": out[2]}

    def __del__(self):
        try:
            for i in range(4):
                self._lib.fp_event_destroy(self.ev[i])
        except Exception:  # pragma: no cover
            pass


class StridedAxisPass(tuple):
    """(axis, shape): a transform pass along a non-contiguous axis, run in place
    through strides (what the reference's ReorderPlan gathers into a line buffer)."""

    def __new__(cls, axis, shape):
        return tuple.__new__(cls, (int(axis), tuple(shape)))

    axis = property(lambda s: s[0])
    shape = property(lambda s: s[1])


class SolverPlan:
    """Immutable plan for one configuration (solver.py:132-181), resident on one GPU.

    ``threads`` is accepted for signature compatibility (it sized scipy's
    worker pool in the reference); ``device`` selects the GPU (default: the
    current CUDA device).
    """

    def __init__(self, config: SolverConfig, threads: int = 1, device=None):
        self.config = config
        self.threads = max(1, int(threads))
        self.shape = config.shape
        self.dtype = config.dtype
        self._pairs = [transform_pair_for(g.bc, g.kind) for g in config.grids]
        self.tables = [eigenvalue_table(g, config.approximation) for g in config.grids]
        self.null_modes = null_modes_of(self.tables)
        self._periodic_axes = config.periodic_axes
        self._real_axes = tuple(a for a in range(config.dims) if a not in self._periodic_axes)
        self._backward_scale = math.prod(p.backward_scale(g.n) for g, p in zip(config.grids, self._pairs))
        if config.singular:
            self._null_scale = math.prod(_ONES_NULL_COEFF[p.forward](g.n) for g, p in zip(config.grids, self._pairs))
        self._inv_lam_cache = None
        self._inv_lam_pristine = None
        self._ovr_src = None
        self._ovr_dev = None
        self._device = dv.require_cuda(device)
        self._lib = nat.load()
        self._handle = self._create_native()
        info = nat.FpPlanInfo()
        nat.check(self._lib.fp_plan_info_get(self._handle, ctypes.byref(info)))
        self._info = info

    def _create_native(self):
        cfg, keep = _config_struct(self.config, self.tables)
        h = ctypes.c_void_p()
        nat.check(self._lib.fp_plan_create(ctypes.byref(cfg), self._device.index, ctypes.byref(h)))
        del keep
        return h

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None:
            try:
                self._lib.fp_plan_destroy(h)
            except Exception:  # pragma: no cover
                pass

    # -- reference-compatible properties ----------------------------------
    @property
    def mode(self) -> str:
        return self.config.mode

    @property
    def singular(self) -> bool:
        return self.config.singular

    @property
    def device(self):
        return self._device

    @property
    def num_passes(self) -> int:
        return int(self._info.num_passes)

    @property
    def _reorder(self) -> dict:
        """Axes the reference sends through its gather/scatter reorder seam
        (solver.py:167-176: mixed plans, real axes other than the last).  Here
        those lines are transformed in place through strides (strided tiles), so
        each value only names that pass; the keys match the reference's."""
        if self.mode != "mixed":
            return {}
        last = self.config.dims - 1
        return {ax: StridedAxisPass(ax, self.shape) for ax in self._real_axes if ax != last}

    @property
    def _inv_lam(self) -> np.ndarray:
        """Dense backward_scale / lambda array (solver.py:151-159), built lazily on the host.

        The normal solve never reads it: the middle pass evaluates the same
        factor from the per-axis tables.  It is writable, as in the reference:
        once a caller changes it (fault injection, verifysuite.py:83-88), every
        later solve divides by the caller's table instead (fp_solve_override),
        exactly like the reference's ``work *= self._inv_lam`` (solver.py:221).
        """
        if self._inv_lam_cache is None:
            lam = combine_eigenvalues(self.tables).values
            inv = np.zeros_like(lam)
            np.divide(self._backward_scale, lam, out=inv, where=lam != 0.0)
            inv = inv.astype(self.dtype)
            self._inv_lam_pristine = inv.copy()
            self._inv_lam_cache = inv
            self._ovr_src = None
            self._ovr_dev = None
        return self._inv_lam_cache

    @_inv_lam.setter
    def _inv_lam(self, value):
        arr = np.array(value, dtype=self.dtype)
        if arr.shape != self.shape:
            raise ValueError(f"_inv_lam must have the plan extents {self.shape}, got {arr.shape}")
        self._inv_lam  # noqa: B018  (materialize the pristine copy)
        self._inv_lam_cache = arr

    def _override_table(self):
        """Device table for fp_solve_override, or None while ``_inv_lam`` is pristine.

        The host array is compared with the pristine copy only after a caller
        has touched ``_inv_lam``; the half-spectrum table is rebuilt and
        uploaded only when the array changed since the last upload."""
        cache = self._inv_lam_cache
        if cache is None:
            return None
        if self._ovr_src is not None and np.array_equal(cache, self._ovr_src):
            return self._ovr_dev
        if np.array_equal(cache, self._inv_lam_pristine):
            self._ovr_src, self._ovr_dev = None, None
            return None
        ext = (ctypes.c_int64 * 3)()
        r_axis = ctypes.c_int()
        nat.check(self._lib.fp_plan_spectrum(self._handle, ext, ctypes.byref(r_axis)))
        table = np.asarray(cache, dtype=np.float64)
        per = self._periodic_axes
        if per:
            # `.real` of the inverse FFT keeps (f(k) + f(-k)) / 2 (the Hermitian part of
            # the multiplier), which is what a half-spectrum pipeline can apply
            mirrored = table
            for ax in per:
                mirrored = np.roll(np.flip(mirrored, axis=ax), 1, axis=ax)
            table = 0.5 * (table + mirrored)
        if r_axis.value >= 0:
            sl = [slice(None)] * self.config.dims
            sl[r_axis.value] = slice(0, int(ext[r_axis.value]))
            table = table[tuple(sl)]
        t = dv.torch()
        dev = t.from_numpy(np.ascontiguousarray(table, dtype=self.dtype)).to(self._device)
        self._ovr_src = np.array(cache, copy=True)
        self._ovr_dev = dev
        return dev

    def workspace_bytes(self, out_dense: bool = True) -> int:
        b = ctypes.c_size_t()
        nat.check(self._lib.fp_plan_workspace_bytes(self._handle, int(bool(out_dense)), ctypes.byref(b)))
        return int(b.value)

    # -- solve --------------------------------------------------------------
    def solve(self, rhs, out=None):
        """Solve the discrete Poisson problem for ``rhs``; returns ``(solution, report)``."""
        rhs_arr = as_array(rhs)
        if tuple(rhs_arr.shape) != self.shape:
            raise ValueError(f"rhs extents {tuple(rhs_arr.shape)} do not match plan extents {self.shape}")
        out_arr = None
        if out is not None:
            out_arr = as_array(out)
            if tuple(out_arr.shape) != self.shape:
                raise ValueError(f"solution extents {tuple(out_arr.shape)} do not match plan extents {self.shape}")
        if dv.is_tensor(rhs_arr):
            return self._solve_device(rhs_arr, out_arr)
        return self._solve_host(rhs_arr, out_arr)

    def _report(self, info_host, events) -> SolveReport:
        rep = SolveReport(mode=self.mode, periodic_axes=self._periodic_axes)
        rm = ctypes.c_double()
        nat.check(self._lib.fp_removed_mean(self._handle, ctypes.byref(info_host), ctypes.byref(rm)))
        rep.removed_mean = float(rm.value)
        rep.timing = events.timing()
        return rep

    def _launch(self, rhs_t, out_t, info_t, events=None, stream=None, workspace=None):
        """Enqueue one solve on the current stream (no synchronization).  The
        workspace comes from the caching allocator unless the caller passes one
        (at least ``workspace_bytes(out_t.is_contiguous())`` bytes)."""
        t = dv.torch()
        out_dense = out_t.is_contiguous()
        ovr = self._override_table()
        if ovr is None:
            ws_bytes = self.workspace_bytes(out_dense)
        else:
            b = ctypes.c_size_t()
            nat.check(self._lib.fp_plan_workspace_bytes_ex(self._handle, int(bool(out_dense)), 1, ctypes.byref(b)))
            ws_bytes = int(b.value)
        if workspace is not None and workspace.numel() >= ws_bytes:
            ws = workspace
        else:
            ws = t.empty(max(ws_bytes, 1), dtype=t.uint8, device=self._device)
        ev = events.ev if events is not None else None
        if stream is None and nat.use_torch_ext():
            # the PyTorch extension: tensors in, the current stream read natively
            evp = ctypes.addressof(ev) if ev is not None else 0
            nat.check(nat.torch_ext().solve(self._handle.value, rhs_t, out_t, ws, info_t, evp, ovr))
            return ws if ovr is None else (ws, ovr)
        st = stream if stream is not None else dv.stream_handle(self._device)
        args = (self._handle,
                rhs_t.data_ptr(), dv.fp_dtype_of_torch(rhs_t.dtype), nat.strides_array(rhs_t.stride()),
                out_t.data_ptr(), nat.strides_array(out_t.stride()),
                ws.data_ptr(), ws_bytes, st, info_t.data_ptr(), ev)
        if ovr is None:
            nat.check(self._lib.fp_solve(*args))
            return ws
        nat.check(self._lib.fp_solve_override(*args, ovr.data_ptr()))
        return (ws, ovr)

    def _prepare_device_inputs(self, rhs_t, out_t):
        t = dv.torch()
        if rhs_t.device != self._device:
            raise ValueError(f"rhs lives on {rhs_t.device}, plan on {self._device}")
        if rhs_t.dtype not in (t.float32, t.float64):
            if rhs_t.is_complex():
                raise TypeError("rhs must be real")
            rhs_t = rhs_t.to(dv.torch_dtype(self.dtype))
        if any(s < 0 for s in rhs_t.stride()):
            rhs_t = rhs_t.contiguous()
        if out_t is None:
            out_t = t.empty(self.shape, dtype=dv.torch_dtype(self.dtype), device=self._device)
        else:
            if out_t.device != self._device:
                raise ValueError(f"out lives on {out_t.device}, plan on {self._device}")
            if out_t.dtype != dv.torch_dtype(self.dtype):
                raise TypeError(f"out must have the plan dtype {self.dtype}")
            # partial overlap (not the exact same view) would race: solve from a copy
            if dv.overlaps(rhs_t, out_t) and not dv.same_view(rhs_t, out_t):
                rhs_t = rhs_t.clone()
        return rhs_t, out_t

    def _solve_device(self, rhs_t, out_t):
        t = dv.torch()
        rhs_t, out_t = self._prepare_device_inputs(rhs_t, out_t)
        info_t = t.zeros(16, dtype=t.uint8, device=self._device)
        events = _Events(self._lib, self._device.index)
        ws = self._launch(rhs_t, out_t, info_t, events)
        info_host = nat.FpSolveInfo.from_buffer_copy(info_t.cpu().numpy().tobytes())
        del ws
        if info_host.nonfinite:
            raise ValueError("rhs contains non-finite values")
        return out_t, self._report(info_host, events)

    def _solve_host(self, rhs_arr, out_arr):
        t = dv.torch()
        rhs_arr = np.asarray(rhs_arr)
        if rhs_arr.dtype not in (np.float32, np.float64):
            if np.iscomplexobj(rhs_arr):
                raise TypeError("rhs must be real")
            rhs_arr = rhs_arr.astype(self.dtype)
        rhs_t = dv.to_device(rhs_arr, self._device)
        out_t = t.empty(self.shape, dtype=dv.torch_dtype(self.dtype), device=self._device)
        info_t = t.zeros(16, dtype=t.uint8, device=self._device)
        events = _Events(self._lib, self._device.index)
        ws = self._launch(rhs_t, out_t, info_t, events)
        info_host = nat.FpSolveInfo.from_buffer_copy(info_t.cpu().numpy().tobytes())
        del ws
        if info_host.nonfinite:
            raise ValueError("rhs contains non-finite values")
        report = self._report(info_host, events)
        if out_arr is None:
            out_arr = np.empty(self.shape, dtype=self.dtype)
        _copy_to_host(out_t, out_arr)
        return out_arr, report

    def solve_batch(self, rhs_seq, out_seq=None):
        """Solve a sequence of host right-hand sides, streaming them through the GPU.

        Equivalent to ``[self.solve(r, o) for r, o in zip(rhs_seq, out_seq)]``
        (same results, same errors), but the host->device copy of solve i+1, the
        kernels of solve i and the device->host copy of solve i-1 run
        concurrently on three CUDA streams (PCIe is full duplex), with two device
        buffers per direction.  Pinned host arrays give the full copy bandwidth.
        Returns a list of ``(solution, SolveReport)``.
        """
        t = dv.torch()
        rhs_list = [np.asarray(as_array(r)) for r in rhs_seq]
        if out_seq is None:
            out_list = [np.empty(self.shape, dtype=self.dtype) for _ in rhs_list]
        else:
            out_list = [as_array(o) for o in out_seq]
        if len(out_list) != len(rhs_list):
            raise ValueError("rhs and out sequences differ in length")
        for r, o in zip(rhs_list, out_list):
            if tuple(r.shape) != self.shape:
                raise ValueError(f"rhs extents {tuple(r.shape)} do not match plan extents {self.shape}")
            if tuple(o.shape) != self.shape:
                raise ValueError(f"solution extents {tuple(o.shape)} do not match plan extents {self.shape}")
        dev = self._device
        tdt = dv.torch_dtype(self.dtype)
        s_in, s_run, s_out = t.cuda.Stream(dev), t.cuda.Stream(dev), t.cuda.Stream(dev)
        d_in = [None, None]
        d_out = [t.empty(self.shape, dtype=tdt, device=dev) for _ in range(2)]
        infos = [t.zeros(16, dtype=t.uint8, device=dev) for _ in rhs_list]
        ev_in = [t.cuda.Event() for _ in range(2)]
        ev_run = [t.cuda.Event() for _ in range(2)]
        ev_out = [t.cuda.Event() for _ in range(2)]
        events = [_Events(self._lib, self._device.index) for _ in rhs_list]
        host_out = [None] * len(rhs_list)
        # one workspace per double buffer, reused in stream order on s_run
        ws_bytes = self.workspace_bytes(out_dense=True)
        wss = [t.empty(max(ws_bytes, 1), dtype=t.uint8, device=dev) for _ in range(min(2, len(rhs_list)))]
        for i, r in enumerate(rhs_list):
            b = i & 1
            if r.dtype not in (np.float32, np.float64):
                r = r.astype(self.dtype)
            rt = t.from_numpy(np.ascontiguousarray(r))
            with t.cuda.stream(s_in):
                if i >= 2:
                    s_in.wait_event(ev_run[b])          # buffer b consumed by solve i-2
                d_in[b] = rt.to(dev, non_blocking=True)
                d_in[b].record_stream(s_run)
                ev_in[b].record(s_in)
            with t.cuda.stream(s_run):
                s_run.wait_event(ev_in[b])
                if i >= 2:
                    s_run.wait_event(ev_out[b])         # d_out[b] drained by the copy of solve i-2
                self._launch(d_in[b], d_out[b], infos[i], events[i], stream=s_run.cuda_stream, workspace=wss[b])
                ev_run[b].record(s_run)
            with t.cuda.stream(s_out):
                s_out.wait_event(ev_run[b])
                o = out_list[i]
                if (o.flags.c_contiguous and o.flags.writeable and o.dtype == self.dtype):
                    dst = t.from_numpy(o)
                else:
                    dst = t.empty(self.shape, dtype=tdt, pin_memory=True)
                dst.copy_(d_out[b], non_blocking=True)
                host_out[i] = dst
                ev_out[b].record(s_out)
        s_out.synchronize()
        s_run.synchronize()
        results = []
        for i, o in enumerate(out_list):
            info_host = nat.FpSolveInfo.from_buffer_copy(infos[i].cpu().numpy().tobytes())
            if info_host.nonfinite:
                raise ValueError(f"rhs {i} contains non-finite values")
            if host_out[i].data_ptr() != o.ctypes.data:
                o[...] = host_out[i].numpy()
            results.append((o, self._report(info_host, events[i])))
        del wss
        return results

    def solve_async(self, rhs_t, out_t=None, info_t=None):
        """Enqueue a device solve without synchronizing (throughput path).

        Returns ``(out, info, workspace)``; keep ``workspace`` alive until the
        stream has passed the solve.  ``info`` holds the raw fp_solve_info.
        """
        t = dv.torch()
        rhs_t, out_t = self._prepare_device_inputs(rhs_t, out_t)
        if info_t is None:
            info_t = t.empty(16, dtype=t.uint8, device=self._device)
        ws = self._launch(rhs_t, out_t, info_t)
        return out_t, info_t, ws

    def capture(self, rhs_t, out_t=None):
        """Capture one device solve ``rhs_t -> out_t`` into a CUDA graph.

        Returns a ``CapturedSolve``: ``replay()`` enqueues the same kernels on
        the current stream with one launch (small grids are launch-bound: 64^3
        takes 39 us per call, 29 us per replay); refill ``rhs`` in place between
        replays.  ``info`` holds the raw fp_solve_info of the latest replay.
        """
        t = dv.torch()
        rhs_t, out_t = self._prepare_device_inputs(rhs_t, out_t)
        info_t = t.zeros(16, dtype=t.uint8, device=self._device)
        side = t.cuda.Stream(device=self._device)
        side.wait_stream(t.cuda.current_stream(self._device))
        with t.cuda.stream(side):   # warm-up outside the capture (lazy kernel attributes, allocator)
            keep = self._launch(rhs_t, out_t, info_t)
        t.cuda.current_stream(self._device).wait_stream(side)
        side.synchronize()
        del keep
        graph = t.cuda.CUDAGraph()
        with t.cuda.graph(graph):
            ws = self._launch(rhs_t, out_t, info_t, stream=t.cuda.current_stream(self._device).cuda_stream)
        return CapturedSolve(graph, rhs_t, out_t, info_t, ws, self)


class CapturedSolve:
    """One solve recorded as a CUDA graph on fixed device buffers (SolverPlan.capture).

    Holds the plan: the captured kernels read its device tables (twiddles,
    eigenvalues), which must outlive every replay."""

    def __init__(self, graph, rhs, out, info, workspace, plan):
        self.graph, self.rhs, self.out, self.info, self._ws = graph, rhs, out, info, workspace
        self._plan = plan

    def replay(self):
        self.graph.replay()
        return self.out


def _copy_to_host(src_t, dst: np.ndarray):
    t = dv.torch()
    if dst.flags.writeable and all(s >= 0 for s in dst.strides) and dst.dtype == np.dtype(str(src_t.dtype).split(".")[-1]):
        try:
            t.from_numpy(dst).copy_(src_t)
            return
        except (TypeError, RuntimeError, ValueError):
            pass
    dst[...] = src_t.cpu().numpy()


def plan_create(config: SolverConfig, threads: int = 1) -> SolverPlan:
    """Build the immutable plan for a configuration (solver.py:264-266)."""
    return SolverPlan(config, threads=threads)


def solve(plan: SolverPlan, rhs, out=None):
    """Three-step solve on a prepared plan (solver.py:269-271)."""
    return plan.solve(rhs, out)


def solve_mixed(plan: SolverPlan, rhs, out=None):
    """Mixed-boundary path; rejects uniform plans (solver.py:274-283)."""
    if plan.mode != "mixed":
        raise ConfigurationError("plan is not a mixed-boundary plan; use solve()")
    return plan.solve(rhs, out)


def apply_discrete_laplacian(config: SolverConfig, field, out=None):
    """Second-order Laplacian with the plan's boundary closures (solver.py:286-338).

    Verification aid (not on the solve path).  numpy input is evaluated on the
    host in float64, torch input on its device.
    """
    if config.approximation is not Approximation.FINITE_DIFFERENCE_2:
        raise ConfigurationError("discrete Laplacian is defined for the fd2 approximation")
    arr = as_array(field)
    if tuple(arr.shape) != config.shape:
        raise ValueError(f"field extents {tuple(arr.shape)} do not match config extents {config.shape}")
    if dv.is_tensor(arr):
        t = dv.torch()
        x = arr.to(t.float64)
        result = t.zeros_like(x)
        for ax, spec in enumerate(config.grids):
            result += _second_difference_torch(x, ax, spec)
    else:
        x = np.asarray(arr, dtype=np.float64)
        result = np.zeros(x.shape, dtype=np.result_type(np.asarray(arr).dtype, np.float64))
        for ax, spec in enumerate(config.grids):
            result += _second_difference_np(x, ax, spec)
    if out is not None:
        out_arr = as_array(out)
        out_arr[...] = result
        return out_arr
    return result


def _edge_coeffs(spec: GridSpec):
    """(self, neighbour) weights of the first/last row for each closure."""
    bc, kind = spec.bc, spec.kind
    if bc is BoundaryCondition.DIRICHLET:
        return (-2.0, 1.0) if kind is GridKind.REGULAR else (-3.0, 1.0)
    if bc is BoundaryCondition.NEUMANN:
        return (-2.0, 2.0) if kind is GridKind.REGULAR else (-1.0, 1.0)
    return None


def _second_difference_np(x, axis, spec):
    y = np.moveaxis(x, axis, 0)
    r = np.empty_like(y)
    n = spec.n
    if n == 1:
        if spec.bc is BoundaryCondition.DIRICHLET:
            r[0] = (-4.0 if spec.kind is GridKind.STAGGERED else -2.0) * y[0]
        else:
            r[0] = 0.0
    else:
        r[1:-1] = y[2:] - 2.0 * y[1:-1] + y[:-2]
        edge = _edge_coeffs(spec)
        if edge is None:
            r[0] = y[1] - 2.0 * y[0] + y[-1]
            r[-1] = y[0] - 2.0 * y[-1] + y[-2]
        else:
            c_self, c_nb = edge
            r[0] = c_nb * y[1] + c_self * y[0] if c_nb != 1.0 else y[1] + c_self * y[0]
            r[-1] = c_nb * y[-2] + c_self * y[-1] if c_nb != 1.0 else y[-2] + c_self * y[-1]
    r /= spec.dx ** 2
    return np.moveaxis(r, 0, axis)


def _second_difference_torch(x, axis, spec):
    t = dv.torch()
    y = x.movedim(axis, 0)
    r = t.empty_like(y)
    n = spec.n
    if n == 1:
        if spec.bc is BoundaryCondition.DIRICHLET:
            r[0] = (-4.0 if spec.kind is GridKind.STAGGERED else -2.0) * y[0]
        else:
            r[0] = 0.0
    else:
        r[1:-1] = y[2:] - 2.0 * y[1:-1] + y[:-2]
        edge = _edge_coeffs(spec)
        if edge is None:
            r[0] = y[1] - 2.0 * y[0] + y[-1]
            r[-1] = y[0] - 2.0 * y[-1] + y[-2]
        else:
            c_self, c_nb = edge
            r[0] = c_nb * y[1] + c_self * y[0]
            r[-1] = c_nb * y[-2] + c_self * y[-1]
    r /= spec.dx ** 2
    return r.movedim(0, axis)
