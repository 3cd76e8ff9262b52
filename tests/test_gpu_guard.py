"""GPU tier: memory-safety and race checks without compute-sanitizer (closed on this
pool -- see profiles/r02/sanitize_*.txt): every kernel family runs through the C ABI
on buffers that sit inside guard bands, with a NaN-poisoned workspace and output.

  * memcheck stand-in: the guard bands around rhs, out and the workspace hold a
    sentinel pattern that must be bit-identical after the solve (any out-of-bounds
    store lands there), and the rhs must be unchanged (unless solved in place);
  * initcheck stand-in: workspace and out start as NaN -- a read of an element the
    solve did not write first propagates NaN into the result, which must match the
    oracle (solver.py:191-249) at the usual bar;
  * racecheck stand-in: the same solve repeated (and interleaved with other plans on
    the same stream) must be bit-identical -- shared-memory races between the
    Stockham stages, the in-place tiles and the mirrored-pair exchanges show up as
    run-to-run differences.
"""

import ctypes

import numpy as np
import pytest

from paper_1409_8116_b200 import _native as nat
from oracle import fastpoisson_oracle as orc

pytestmark = pytest.mark.gpu

PI2 = orc.TWO_PI
N_, D_, P_ = orc.NEUMANN, orc.DIRICHLET, orc.PERIODIC
R_, S_ = orc.REGULAR, orc.STAGGERED
CASES = {
    # FFT engine: contiguous + strided passes, register-path MID (M <= 512)
    "dct3d": orc.Case([(32, 1.0, N_, S_), (64, 1.0, N_, S_), (32, 2.0, N_, S_)], orc.FD2),
    "per3d": orc.Case([(32, PI2, P_), (16, PI2, P_), (64, PI2, P_)], orc.SPECTRAL),
    # shared-memory MID (M = 1024 / 2048 real lines), long strided lines
    "dst2d_long": orc.Case([(2048, 1.0, D_, S_), (48, 1.0, D_, S_)], orc.FD2),
    "rfft_long": orc.Case([(4096, PI2, P_), (16, PI2, P_)], orc.SPECTRAL),
    "mixed3d": orc.Case([(64, PI2, P_), (32, PI2, P_), (32, 2.0, N_, S_)], orc.FD2),
    # type-I placements (DCT-I / DST-I) and the exact mean removal
    "dct1": orc.Case([(33, 1.0, N_, R_), (65, 1.0, N_, R_)], orc.FD2),
    "dst1": orc.Case([(63, 1.0, D_, R_), (31, 1.0, D_, R_), (15, 1.0, D_, R_)], orc.FD2),
    # mixed-radix, dense and Bluestein engines
    "mr": orc.Case([(60, 1.0, N_, S_), (45, 1.0, N_, S_), (100, 1.0, N_, S_)], orc.FD2),
    "dense": orc.Case([(67, 1.0, D_, S_), (40, 1.0, D_, S_)], orc.FD2),
    "blue": orc.Case([(131, 1.0, N_, S_), (64, PI2, P_)], orc.FD2),
    # fp32 paths
    "f32_per": orc.Case([(64, PI2, P_)] * 3, orc.SPECTRAL, "single"),
    "f32_dct": orc.Case([(128, 1.0, N_, S_), (64, 1.0, N_, S_)], orc.FD2, "single"),
}
GUARD = 4096   # elements of sentinel on each side


def _plan(lib, case):
    from test_gpu_abi import make_cfg

    cfg = make_cfg(case)
    h = ctypes.c_void_p()
    assert lib.fp_plan_create(ctypes.byref(cfg), 0, ctypes.byref(h)) == nat.FP_OK, lib.fp_last_error()
    return h


def _guarded(torch, n, dtype, fill):
    """(whole buffer, inner view of n elements); the guards hold a bit pattern."""
    buf = torch.empty(n + 2 * GUARD, dtype=dtype, device="cuda")
    buf.fill_(fill)
    sentinel = torch.full((GUARD,), -7.25e3, dtype=dtype, device="cuda")
    buf[:GUARD] = sentinel
    buf[-GUARD:] = sentinel
    return buf, buf[GUARD:GUARD + n]


def _guards_intact(buf):
    g = buf[:GUARD].cpu().numpy(), buf[-GUARD:].cpu().numpy()
    return all((x == np.float32(-7.25e3) if x.dtype == np.float32 else x == -7.25e3).all() for x in g)


def _solve(lib, h, torch, case, rhs_np, in_place=False):
    dt = torch.float32 if case.precision == "single" else torch.float64
    n = int(np.prod(case.shape))
    rbuf, rhs = _guarded(torch, n, dt, 0.0)
    rhs.copy_(torch.from_numpy(rhs_np.ravel()).to(dt))
    if in_place:
        obuf, out = rbuf, rhs
    else:
        obuf, out = _guarded(torch, n, dt, float("nan"))
    ws_n = ctypes.c_size_t()
    assert lib.fp_plan_workspace_bytes(h, 1, ctypes.byref(ws_n)) == nat.FP_OK
    wbuf, ws = _guarded(torch, max(int(ws_n.value) // 8 + 1, 1), torch.float64, float("nan"))
    info = torch.zeros(16, dtype=torch.uint8, device="cuda")
    strides = nat.strides_array(tuple(int(np.prod(case.shape[a + 1:])) for a in range(len(case.shape))))
    rc = lib.fp_solve(h, rhs.data_ptr(), nat.FP_F32 if dt == torch.float32 else nat.FP_F64, strides,
                      out.data_ptr(), strides, ws.data_ptr(), int(ws_n.value), None, info.data_ptr(), None)
    assert rc == nat.FP_OK, lib.fp_last_error()
    torch.cuda.synchronize()
    assert _guards_intact(rbuf), "store outside rhs / out"
    if not in_place:
        assert _guards_intact(obuf), "store outside out"
        assert torch.equal(rhs.cpu(), torch.from_numpy(rhs_np.ravel()).to(dt)), "rhs modified"
    assert _guards_intact(wbuf), "store outside the workspace"
    return out.cpu().numpy().reshape(case.shape)


@pytest.mark.parametrize("name", sorted(CASES))
def test_guard_bands_poisoned_workspace_and_determinism(name, rng):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    lib = nat.load()
    case = CASES[name]
    rhs = rng.standard_normal(case.shape)
    if case.precision == "single":
        rhs = rhs.astype(np.float32)
    want, _ = orc.solve(case, rhs)
    h = _plan(lib, case)
    other = _plan(lib, CASES["dct3d" if name != "dct3d" else "per3d"])
    try:
        got = _solve(lib, h, torch, case, rhs)
        tol = 1e-5 if case.precision == "single" else 1e-12
        assert np.isfinite(got).all(), "NaN from the poisoned workspace / out reached the result"
        assert orc.relative_l2(got, want) <= tol
        # repeated, interleaved with another plan on the same stream, and in place: bit-identical
        for k in range(3):
            oc = CASES["dct3d" if name != "dct3d" else "per3d"]
            _solve(lib, other, torch, oc, np.random.default_rng(k).standard_normal(oc.shape).astype(
                np.float32 if oc.precision == "single" else np.float64))
            again = _solve(lib, h, torch, case, rhs, in_place=(k == 2))
            assert np.array_equal(again, got), f"run {k}: results differ between identical solves"
    finally:
        lib.fp_plan_destroy(h)
        lib.fp_plan_destroy(other)
