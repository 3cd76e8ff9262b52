"""TEST INFRASTRUCTURE -- numpy stand-in for the native phases of the
distributed solve, following the exchange-layout contract of fp_dist_layout:

  send/recv buffers: the exchanged state (local_n0, exch_n1, exch_n2) stored
  with axis 1 outermost, axis 1 padded to exch_n1 (a multiple of P); peer q's
  block = axis-1 rows [q*block_n1, (q+1)*block_n1).  After the all-to-all the
  receive buffer is [source rank][block_n1][local_n0][exch_n2].

The transforms are the oracle's scipy restatement of the reference; only the
orchestration (paper_1409_8116_b200.distributed) and the layout are under test.
"""

from __future__ import annotations

import numpy as np
import torch

from oracle import fastpoisson_oracle as orc


class NumpyBackend:
    def __init__(self, case: orc.Case, info, nranks: int, rank: int):
        self.case = case
        self.info = info
        self.P = nranks
        self.rank = rank
        self.d = len(case.shape)
        self.a0 = int(info.local_n0)
        self.A = int(info.pitch_n0)          # planes per exchange block (balanced split, padded)
        n0 = case.axes[0].n
        q, r = divmod(n0, nranks)
        self.a0s = [q + (k < r) for k in range(nranks)]
        self.offs = [k * q + min(k, r) for k in range(nranks)]
        self.E1, self.e1, self.e2, self.B = int(info.exch_n1), int(info.true_n1), int(info.exch_n2), int(info.block_n1)
        self.cpx = bool(info.exch_complex)
        self.r_axis = int(info.r_axis)
        self.local_shape = (self.a0,) + tuple(case.shape[1:])
        nbytes = int(info.exchange_bytes)
        self.send = torch.zeros(nbytes, dtype=torch.uint8)
        self.recv = torch.zeros(nbytes, dtype=torch.uint8)
        self.dtype = np.complex128 if self.cpx else np.float64
        self.status = np.zeros(2)
        self.exact_mean = any(a.bc == orc.NEUMANN and a.kind == orc.REGULAR for a in case.axes)
        # forward order of the local axes: real descending, then periodic descending
        axes = [a for a in range(self.d - 1, 0, -1) if case.axes[a].bc != orc.PERIODIC]
        axes += [a for a in range(self.d - 1, 0, -1) if case.axes[a].bc == orc.PERIODIC]
        self.order = axes

    # exchange-buffer views
    def _view(self, buf):
        arr = buf.numpy().view(self.dtype)
        if self.d == 3:
            return arr.reshape(self.E1, self.A, self.e2)
        return arr.reshape(self.E1, self.A)

    def _fwd(self, x, ax):
        a = self.case.axes[ax]
        if a.bc == orc.PERIODIC:
            if ax == self.r_axis:
                return np.fft.rfft(x, axis=ax)
            return np.fft.fft(x, axis=ax)
        return orc.forward_1d(orc.pair(a)[0], x, axis=ax)

    def _inv(self, x, ax):
        a = self.case.axes[ax]
        if a.bc == orc.PERIODIC:
            if ax == self.r_axis:
                return np.fft.irfft(x, n=a.n, axis=ax) * a.n
            return np.fft.ifft(x, axis=ax) * a.n
        return orc.backward_1d(orc.pair(a)[1], x, axis=ax)

    def forward(self, rhs_local, out_local):
        x = np.asarray(rhs_local, dtype=np.float64)
        self.status[:] = 0.0
        self.status[1] = 0.0 if np.isfinite(x).all() else 1.0
        for ax in self.order:
            x = self._fwd(x, ax)
        s = self._view(self.send)
        s[...] = 0
        s[: self.e1, : self.a0] = np.swapaxes(x, 0, 1)

    def middle(self):
        case, d = self.case, self.d
        r = self._view(self.recv)
        # [src][B][A][e2] -> global axis 0 first: G[off(src) + i0, i1', i2], i0 < a0(src)
        blocks = r.reshape((self.P, self.B) + r.shape[1:])
        g = np.concatenate([np.swapaxes(blocks[s][:, : self.a0s[s]], 0, 1) for s in range(self.P)], axis=0)
        k1 = self.rank * self.B + np.arange(self.B)
        valid = k1 < self.e1
        lam1 = np.zeros(self.B)
        lam1[valid] = orc.eigenvalues(case.axes[1], case.approx)[k1[valid]]
        lam0 = orc.eigenvalues(case.axes[0], case.approx)
        lam2 = orc.eigenvalues(case.axes[2], case.approx)[: self.e2] if d == 3 else np.zeros(1)
        a0 = case.axes[0]
        # forward along axis 0 (unnormalized), scale, inverse
        if a0.bc == orc.PERIODIC:
            if self.r_axis == 0:
                spec = np.fft.rfft(g.real, axis=0)
            else:
                spec = np.fft.fft(g, axis=0)
        else:
            spec = orc.forward_1d(orc.pair(a0)[0], g, axis=0)
        k0 = np.arange(spec.shape[0])
        if d == 3:
            lam = (lam0[k0][:, None, None] + lam1[None, :, None]) + lam2[None, None, :]
        else:
            lam = lam0[k0][:, None] + lam1[None, :]
        bscale = np.prod([orc.backward_scale(a) for a in case.axes])
        np_prod = np.prod([a.n for a in case.axes if a.bc == orc.PERIODIC]) if case.periodic_axes else 1.0
        fac = np.zeros_like(lam)
        np.divide(bscale, lam, out=fac, where=lam != 0.0)
        fac = fac / np_prod
        if case.singular and self.rank == 0:
            self.status[0] = float(np.real(spec[(0,) * d]))
        spec = spec * fac
        if d == 3:
            spec[:, ~valid, :] = 0
        else:
            spec[:, ~valid] = 0
        if a0.bc == orc.PERIODIC:
            if self.r_axis == 0:
                g = np.fft.irfft(spec, n=a0.n, axis=0) * a0.n
            else:
                g = np.fft.ifft(spec, axis=0) * a0.n
        else:
            g = orc.backward_1d(orc.pair(a0)[1], spec, axis=0)
        for s in range(self.P):
            blocks[s][:, : self.a0s[s]] = np.swapaxes(g[self.offs[s]:self.offs[s] + self.a0s[s]], 0, 1)

    def middle_rows(self, row0, nrows):
        """Phase 1 on a chunk of axis-1 rows: the whole MID on a private copy of the receive
        buffer (lines are independent), then only rows [row0, row0 + nrows) of every source
        block written back -- the other chunks' rows may still be arriving."""
        live = self.recv
        self.recv = live.clone()
        status = self.status.copy()
        try:
            self.middle()
            done = self._view(self.recv)
        finally:
            self.recv = live
        if row0 > 0:   # only the chunk holding row 0 carries the null coefficient
            self.status[:] = status
        r = self._view(live)
        blocks = r.reshape((self.P, self.B) + r.shape[1:])
        dblocks = done.reshape((self.P, self.B) + done.shape[1:])
        blocks[:, row0:row0 + nrows] = dblocks[:, row0:row0 + nrows]

    def backward(self, out_local):
        s = self._view(self.send)
        x = np.swapaxes(s[: self.e1, : self.a0], 0, 1)
        for ax in reversed(self.order):
            x = self._inv(x, ax)
        out_local.numpy()[...] = np.real(x)

    def local_sum(self, out_local):
        return torch.tensor([float(out_local.numpy().sum())], dtype=torch.float64)

    def subtract_mean(self, out_local, total):
        out_local.numpy()[...] -= float(total[0]) / float(np.prod(self.case.shape))

    def read_status(self):
        return torch.tensor(self.status.copy(), dtype=torch.float64)

    def new_output(self):
        return torch.zeros(self.local_shape, dtype=torch.float64)
