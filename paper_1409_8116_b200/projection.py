"""The pressure-projection step of the 2D staggered-grid flow, fused around the solve.

Reference: ``ProjectionFlow.rk3_step`` (flow.py:284-295), per RK stage::

    rhs = divergence(star) / (alpha_k dt)            # flow.py:114-122, 290
    phi, _ = self.poisson.solve(rhs)                  # the hot path
    gfx, gfz = gradient(vel, phi)                     # flow.py:125-139
    vel.u = ustar - alpha_k dt gfx;  vel.w = wstar - alpha_k dt gfz;  pres.p += phi

Here the divergence is formed by the solve's first pass while it loads its
lines (no rhs array is written or read: ``fp_solve_divergence``), and one
corrector kernel applies both gradient updates and the pressure increment
(``fp_project_correct``).  Geometry as in flow.py:1-20: axis 0 = x periodic,
axis 1 = z periodic or closed by walls (staggered Neumann pressure), u on
x-faces (nx, nz), w on z-faces (nx, nz) periodic / (nx, nz + 1) with walls.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _device as dv
from . import _native as nat
from .grid import Approximation, BoundaryCondition, GridKind, GridSpec
from .solver import SolveReport, SolverConfig, SolverPlan


class ProjectionStep:
    """``project(ustar, wstar, scale)`` = one projection of flow.py:290-295 with
    ``scale = alpha_k * dt``; returns ``(u, w, phi, report)``."""

    def __init__(self, cells, lengths, z_walls: bool = False, precision: str = "double", device=None):
        nx, nz = (int(c) for c in cells)
        lx, lz = (float(x) for x in lengths)
        zspec = (GridSpec(nz, lz, BoundaryCondition.NEUMANN, GridKind.STAGGERED) if z_walls
                 else GridSpec(nz, lz, BoundaryCondition.PERIODIC, GridKind.REGULAR))
        config = SolverConfig((GridSpec(nx, lx, BoundaryCondition.PERIODIC, GridKind.REGULAR), zspec),
                              Approximation.FINITE_DIFFERENCE_2, precision)
        self.plan = SolverPlan(config, device=device)   # the flow's own plan (flow.py:241-250)
        self.cells = (nx, nz)
        self.z_walls = bool(z_walls)
        self.w_shape = (nx, nz + 1) if z_walls else (nx, nz)

    def _dev(self, a, shape, name):
        t = dv.torch()
        tdt = dv.torch_dtype(self.plan.dtype)
        if isinstance(a, np.ndarray):
            a = t.from_numpy(np.ascontiguousarray(a, dtype=self.plan.dtype)).to(self.plan._device)
        if tuple(a.shape) != tuple(shape):
            raise ValueError(f"{name} extents {tuple(a.shape)} do not match {tuple(shape)}")
        if a.dtype != tdt:
            a = a.to(tdt)
        return a.contiguous()

    def project(self, ustar, wstar, scale: float, p=None, u_out=None, w_out=None, phi_out=None):
        """Divergence -> solve -> gradient correction on the GPU (device tensors in and
        out; numpy arrays are copied in).  ``p`` (device tensor, optional) gets
        ``p += phi`` in place.  ``u_out``/``w_out`` may alias ``ustar``/``wstar``."""
        t = dv.torch()
        plan = self.plan
        u = self._dev(ustar, self.cells, "ustar")
        w = self._dev(wstar, self.w_shape, "wstar")
        if p is not None and (tuple(p.shape) != self.cells or not p.is_contiguous() or p.dtype != u.dtype):
            raise ValueError("p must be a contiguous device tensor of the cell extents and plan dtype")
        phi = phi_out if phi_out is not None else t.empty(self.cells, dtype=u.dtype, device=u.device)
        uo = u_out if u_out is not None else t.empty_like(u)
        wo = w_out if w_out is not None else t.empty_like(w)
        info = t.zeros(16, dtype=t.uint8, device=u.device)
        ws_bytes = plan.workspace_bytes(phi.is_contiguous())
        ws = t.empty(max(ws_bytes, 1), dtype=t.uint8, device=u.device)
        st = dv.stream_handle(plan._device)
        lib = plan._lib
        nat.check(lib.fp_solve_divergence(plan._handle, u.data_ptr(), None, w.data_ptr(), None, float(scale),
                                          phi.data_ptr(), nat.strides_array(phi.stride()), ws.data_ptr(), ws_bytes,
                                          st, info.data_ptr()))
        nat.check(lib.fp_project_correct(plan._handle, phi.data_ptr(), u.data_ptr(), w.data_ptr(), uo.data_ptr(),
                                         wo.data_ptr(), p.data_ptr() if p is not None else None, float(scale), st))
        info_host = nat.FpSolveInfo.from_buffer_copy(info.cpu().numpy().tobytes())
        del ws
        if info_host.nonfinite:
            raise ValueError("non-finite predictor velocity")
        rep = SolveReport(mode=plan.mode, periodic_axes=plan._periodic_axes)
        rm = ctypes.c_double()
        nat.check(lib.fp_removed_mean(plan._handle, ctypes.byref(info_host), ctypes.byref(rm)))
        rep.removed_mean = float(rm.value)
        return uo, wo, phi, rep
