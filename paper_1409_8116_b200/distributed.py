"""Slab-decomposed Poisson solve over a torch.distributed process group.

The reference package runs in one process (SPEC.md:11 drops distribution); the
paper's library decomposed the grid over MPI ranks with global transposes
(PAPER.md:409-447), and the reference keeps "the seam where a distributed
exchange would slot in" (reorder.py:7-8).  This module is that exchange on
B200s: one process per GPU, axis 0 split into slabs, and per solve

    phase 0  local transforms along axes d-1..1, packed into the send buffer
             (axis 1 outermost, so every peer's block is contiguous; any rank
             count: axis 0 is split evenly up to one plane, every block padded
             to the largest slab)
    all-to-all (NCCL over NVLink / NVSwitch)
    phase 1  fused forward / eigenvalue divide / inverse along the global axis 0
             (the kernel reads the receive layout directly: no unpack pass)
    all-to-all back
    phase 2  local inverse transforms into the caller's output slab

Phases are kernels of the native library (``fp_solve_phase``); the exchanges
are ``torch.distributed.all_to_all_single`` on byte tensors.  ``backend`` is
pluggable so the orchestration (layout contract, exchange pattern, reductions)
can be exercised on CPU with gloo in the test tier.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _device as dv
from . import _native as nat
from .solver import SolveReport, SolverConfig, _config_struct


def dist_layout(config: SolverConfig, nranks: int, rank: int) -> nat.FpDistInfo:
    """Layout of the decomposition (device-free; the native planner's own rules)."""
    lib = nat.load()
    cfg, keep = _config_struct(config)
    info = nat.FpDistInfo()
    nat.check(lib.fp_dist_layout(ctypes.byref(cfg), int(nranks), int(rank), ctypes.byref(info)))
    del keep
    return info


class NativeBackend:
    """The three solve phases on the local GPU through the C ABI."""

    def __init__(self, config: SolverConfig, nranks: int, rank: int, device=None):
        t = dv.torch()
        self.config = config
        self.device = dv.require_cuda(device)
        self._lib = nat.load()
        cfg, keep = _config_struct(config)
        h = ctypes.c_void_p()
        nat.check(self._lib.fp_plan_create_dist(ctypes.byref(cfg), self.device.index, int(nranks), int(rank),
                                                ctypes.byref(h)))
        del keep
        self._handle = h
        self.info = dist_layout(config, nranks, rank)
        self.local_shape = (int(self.info.local_n0),) + tuple(config.shape[1:])
        self.dtype = dv.torch_dtype(config.dtype)
        nbytes = int(self.info.exchange_bytes)
        self.send = t.empty(nbytes, dtype=t.uint8, device=self.device)
        self.recv = t.empty(nbytes, dtype=t.uint8, device=self.device)
        ws = ctypes.c_size_t()
        nat.check(self._lib.fp_plan_workspace_bytes(self._handle, 1, ctypes.byref(ws)))
        self._ws_dense = int(ws.value)
        nat.check(self._lib.fp_plan_workspace_bytes(self._handle, 0, ctypes.byref(ws)))
        self._ws_strided = int(ws.value)
        self.status = t.zeros(16, dtype=t.uint8, device=self.device)
        pinfo = nat.FpPlanInfo()
        nat.check(self._lib.fp_plan_info_get(self._handle, ctypes.byref(pinfo)))
        # DCT-I plans: the arithmetic mean is removed over the GLOBAL grid (solver.py:224-225)
        self.exact_mean = bool(pinfo.exact_mean)
        self._npts = float(np.prod(config.shape))

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None:
            try:
                self._lib.fp_plan_destroy(h)
            except Exception:  # pragma: no cover
                pass

    def _workspace(self, out_dense):
        t = dv.torch()
        n = self._ws_dense if out_dense else self._ws_strided
        return t.empty(max(n, 1), dtype=t.uint8, device=self.device), n

    def _call(self, phase, rhs, out, xbuf):
        t = dv.torch()
        out_dense = out is None or out.is_contiguous()
        ws, nws = self._workspace(out_dense)
        rhs_ptr = rhs.data_ptr() if rhs is not None else None
        rhs_dt = dv.fp_dtype_of_torch(rhs.dtype) if rhs is not None else 0
        rhs_st = nat.strides_array(rhs.stride()) if rhs is not None else None
        out_ptr = out.data_ptr() if out is not None else None
        out_st = nat.strides_array(out.stride()) if out is not None else None
        rc = self._lib.fp_solve_phase(self._handle, phase, rhs_ptr, rhs_dt, rhs_st, out_ptr, out_st,
                                      xbuf.data_ptr(), ws.data_ptr(), nws, dv.stream_handle(self.device),
                                      self.status.data_ptr())
        nat.check(rc)
        return ws

    def forward(self, rhs_local, out_local):
        # the real scratch of phase 0 may live in `out_local` (dense outputs)
        self._ws0 = self._call(0, rhs_local, out_local, self.send)

    def middle(self):
        self._ws1 = self._call(1, None, None, self.recv)

    def middle_rows(self, row0, nrows):
        """Phase 1 on axis-1 rows [row0, row0 + nrows) of this rank's block (pipelined exchange)."""
        ws, nws = self._workspace(True)
        nat.check(self._lib.fp_solve_mid_rows(self._handle, int(row0), int(nrows), self.recv.data_ptr(), ws.data_ptr(),
                                              nws, dv.stream_handle(self.device), self.status.data_ptr()))
        self._ws_rows = ws

    def backward(self, out_local):
        self._ws2 = self._call(2, None, out_local, self.send)

    def local_sum(self, out_local):
        """Sum of this rank's output slab (float64, shape (1,), on the device)."""
        t = dv.torch()
        s = t.zeros(1, dtype=t.float64, device=self.device)
        ws, nws = self._workspace(True)
        nat.check(self._lib.fp_dist_mean_partial(self._handle, out_local.data_ptr(), nat.strides_array(out_local.stride()),
                                                 ws.data_ptr(), nws, dv.stream_handle(self.device), s.data_ptr()))
        self._ws_mean = ws
        return s

    def subtract_mean(self, out_local, total):
        """out_local -= total / (global point count); `total` is the all-reduced sum (device tensor)."""
        nat.check(self._lib.fp_dist_mean_subtract(self._handle, out_local.data_ptr(), nat.strides_array(out_local.stride()),
                                                  total.data_ptr(), dv.stream_handle(self.device)))
        self._keep_total = total

    def read_status(self):
        """(raw null coefficient, non-finite flag) of this rank, as float64 tensor on the device."""
        t = dv.torch()
        dc = self.status[:8].view(t.float64)
        nf = self.status[8:12].view(t.int32).to(t.float64)
        return t.cat([dc, nf])

    def new_output(self):
        t = dv.torch()
        return t.empty(self.local_shape, dtype=self.dtype, device=self.device)


class DistributedSolverPlan:
    """Drop-in ``SolverPlan`` semantics for one global grid split over the ranks.

    ``solve(rhs_local, out_local=None)`` takes this rank's slab (planes
    ``local_slice`` of axis 0) and returns this rank's slab of the solution plus
    the global ``SolveReport`` (identical on every rank).
    """

    def __init__(self, config: SolverConfig, group=None, device=None, backend=None, chunks=None):
        import os

        import torch.distributed as dist

        self.config = config
        self.group = group
        # pipelined exchange: the MID of axis-1 row chunk c runs while chunk c+1 is in flight
        # (FP_DIST_CHUNKS, default 4; 1 = the two whole all-to-alls)
        self.chunks = int(chunks if chunks is not None else os.environ.get("FP_DIST_CHUNKS", "4"))
        self.nranks = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self._single = None
        if self.nranks == 1 and backend is None:
            # one rank: the whole grid is the slab; the single-GPU plan (fused MID, no exchange)
            from .solver import SolverPlan

            self._single = SolverPlan(config, device=device)
            self.local_shape = tuple(config.shape)
            self.local_slice = slice(0, config.shape[0])
            return
        self.backend = backend if backend is not None else NativeBackend(config, self.nranks, self.rank, device)
        self.info = self.backend.info
        self.local_shape = tuple(self.backend.local_shape)
        off = int(self.info.offset0)
        self.local_slice = slice(off, off + int(self.info.local_n0))
        # removed_mean = dc / (prod n_periodic * null_scale) (solver.py:218-220)
        from .solver import _ONES_NULL_COEFF
        from .transforms import transform_pair_for
        import math

        pairs = [transform_pair_for(g.bc, g.kind) for g in config.grids]
        self._np = math.prod(g.n for g in config.grids if g.bc.value == "periodic")
        self._null = math.prod(_ONES_NULL_COEFF[p.forward](g.n) for g, p in zip(config.grids, pairs)) if config.singular else 1.0

    def solve_async(self, rhs_local, out_local=None, events=None):
        """Enqueue one distributed solve (kernels + NCCL all-to-alls) without synchronizing.
        `events`: six CUDA events recorded on the current stream around phase 0, the
        first exchange, the MID, the second exchange and phase 2 (per-phase timing)."""
        import torch.distributed as dist

        def mark(k):
            if events is not None:
                events[k].record()

        if tuple(rhs_local.shape) != self.local_shape:
            raise ValueError(f"local rhs extents {tuple(rhs_local.shape)} do not match {self.local_shape}")
        if self._single is not None:
            out_local, _, self._keep = self._single.solve_async(rhs_local, out_local)
            return out_local
        if out_local is None:
            out_local = self.backend.new_output()
        be = self.backend
        mark(0)
        be.forward(rhs_local, out_local)
        mark(1)
        B = int(self.info.block_n1)
        C = max(1, min(self.chunks, B))
        if C == 1 or events is not None:
            dist.all_to_all_single(be.recv, be.send, group=self.group)
            mark(2)
            be.middle()
            mark(3)
            dist.all_to_all_single(be.send, be.recv, group=self.group)
        else:
            self._pipelined_exchange(be, B, C)
        mark(4)
        be.backward(out_local)
        mark(5)
        if getattr(be, "exact_mean", False):
            total = be.local_sum(out_local)
            dist.all_reduce(total, op=dist.ReduceOp.SUM, group=self.group)
            be.subtract_mean(out_local, total)
        return out_local

    def _pipelined_exchange(self, be, B, C):
        """Both exchanges and the MID in C chunks of axis-1 rows: chunk c is row range
        [c B/C, (c+1) B/C) of every peer's block -- one contiguous piece per peer -- so
        each chunk is a batch of point-to-point sends / receives (NCCL group) issued
        asynchronously; the MID of chunk c waits only for chunk c's receives, and chunk
        c's return exchange overlaps the MID of chunk c + 1."""
        import torch.distributed as dist

        P, r = self.nranks, self.rank
        blk = be.send.numel() // P                 # bytes per peer block
        row = blk // B                              # bytes per axis-1 row of a block
        bounds = [(c * B // C, (c + 1) * B // C) for c in range(C)]

        def exchange(src, dst, c):
            a, b = bounds[c]
            ops = []
            for q in range(P):
                s_view = src[q * blk + a * row: q * blk + b * row]
                d_view = dst[q * blk + a * row: q * blk + b * row]
                if q == r:
                    d_view.copy_(s_view)   # own block
                else:
                    ops.append(dist.P2POp(dist.isend, s_view, q, group=self.group))
                    ops.append(dist.P2POp(dist.irecv, d_view, q, group=self.group))
            return dist.batch_isend_irecv(ops) if ops else []

        fwd = [exchange(be.send, be.recv, c) for c in range(C)]
        back = []
        for c in range(C):
            for w in fwd[c]:
                w.wait()
            a, b = bounds[c]
            be.middle_rows(a, b - a)
            back.append(exchange(be.recv, be.send, c))
        for ws_ in back:
            for w in ws_:
                w.wait()

    def solve(self, rhs_local, out_local=None):
        import torch.distributed as dist

        if self._single is not None:
            return self._single.solve(rhs_local, out_local)
        out_local = self.solve_async(rhs_local, out_local)
        be = self.backend
        status = be.read_status()
        dist.all_reduce(status, op=dist.ReduceOp.SUM, group=self.group)
        dc, nonfinite = float(status[0]), float(status[1])
        if nonfinite > 0:
            raise ValueError("rhs contains non-finite values")
        rep = SolveReport(mode=self.config.mode, periodic_axes=self.config.periodic_axes)
        rep.removed_mean = (dc / self._np) / self._null if self.config.singular else 0.0
        return out_local, rep


class MultiDeviceSolverPlan:
    """Single-process multi-device solve of one global grid ("a
    single-process multi-device wrapper").

    One ``NativeBackend`` per device (rank r = ``devices[r]``, slab r of axis 0);
    the two exchanges are device-to-device copies of the per-peer blocks (peer
    copies over NVLink / NVSwitch when the devices differ) instead of NCCL.
    ``solve(rhs)`` takes the whole field (numpy, or a tensor on any device) and
    returns ``(solution, SolveReport)`` like ``SolverPlan.solve``: numpy in ->
    numpy out, tensor in -> tensor on ``devices[0]``.  The same device may
    appear several times (the ranks then share it; used by the tests).
    """

    def __init__(self, config: SolverConfig, devices):
        t = dv.torch()
        self.config = config
        self.devices = [dv.require_cuda(d) for d in devices]
        P = len(self.devices)
        self.backends = [NativeBackend(config, P, r, self.devices[r]) for r in range(P)]
        self.info = self.backends[0].info
        # balanced split of axis 0 (ranks may differ by one plane)
        self.slices = [slice(int(be.info.offset0), int(be.info.offset0) + int(be.info.local_n0)) for be in self.backends]
        from .solver import _ONES_NULL_COEFF
        from .transforms import transform_pair_for
        import math

        pairs = [transform_pair_for(g.bc, g.kind) for g in config.grids]
        self._np = math.prod(g.n for g in config.grids if g.bc.value == "periodic")
        self._null = math.prod(_ONES_NULL_COEFF[p.forward](g.n) for g, p in zip(config.grids, pairs)) if config.singular else 1.0
        self._t = t

    def _sync(self):
        for d in {(d.type, d.index): d for d in self.devices}.values():
            self._t.cuda.synchronize(d)

    def _exchange(self, src_attr, dst_attr):
        """dst_r[s-th block] <- src_s[r-th block] for every rank pair (all-to-all by copies)."""
        bes = self.backends
        P = len(bes)
        blk = getattr(bes[0], src_attr).numel() // P
        self._sync()
        for r in range(P):
            dst = getattr(bes[r], dst_attr)
            for s_ in range(P):
                dst[s_ * blk:(s_ + 1) * blk].copy_(getattr(bes[s_], src_attr)[r * blk:(r + 1) * blk], non_blocking=True)
        self._sync()

    def solve(self, rhs):
        t = self._t
        host = not dv.is_tensor(rhs)
        x = t.from_numpy(np.ascontiguousarray(rhs)) if host else rhs
        if tuple(x.shape) != self.config.shape:
            raise ValueError(f"rhs extents {tuple(x.shape)} do not match config extents {self.config.shape}")
        bes = self.backends
        outs = []
        for r, be in enumerate(bes):
            slab = x[self.slices[r]].to(be.device, non_blocking=False).contiguous()
            out = be.new_output()
            with t.cuda.device(be.device):
                be.forward(slab, out)
            outs.append(out)
        self._exchange("send", "recv")
        for be in bes:
            with t.cuda.device(be.device):
                be.middle()
        self._exchange("recv", "send")
        for r, be in enumerate(bes):
            with t.cuda.device(be.device):
                be.backward(outs[r])
        if bes[0].exact_mean:
            sums = []
            for r, be in enumerate(bes):
                with t.cuda.device(be.device):
                    sums.append(be.local_sum(outs[r]))
            self._sync()
            total = sum(float(s_.item()) for s_ in sums)
            for r, be in enumerate(bes):
                with t.cuda.device(be.device):
                    be.subtract_mean(outs[r], t.tensor([total], dtype=t.float64, device=be.device))
        self._sync()
        status = [be.read_status().cpu() for be in bes]
        dc = sum(float(s_[0]) for s_ in status)
        if sum(float(s_[1]) for s_ in status) > 0:
            raise ValueError("rhs contains non-finite values")
        rep = SolveReport(mode=self.config.mode, periodic_axes=self.config.periodic_axes)
        rep.removed_mean = (dc / self._np) / self._null if self.config.singular else 0.0
        sol = t.cat([o.to(self.devices[0]) for o in outs], dim=0)
        return (sol.cpu().numpy() if host else sol), rep

