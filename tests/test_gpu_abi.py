"""GPU tier: the C ABI called directly (no Python host mirror), as a C/FFI host would.

Covers fp_solve_host (host buffers, strided host views, dtype cast on load,
FP_ERR_NONFINITE before `out` is touched), fp_solve with explicit strides and
a caller-managed workspace, fp_plan_info_get, and the status codes.
"""

import ctypes

import numpy as np
import pytest

from paper_1409_8116_b200 import _native as nat
from oracle import fastpoisson_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return nat.load()


def make_cfg(case):
    cfg = nat.FpConfig()
    cfg.ndim = len(case.axes)
    bc = {orc.PERIODIC: nat.FP_BC_PERIODIC, orc.DIRICHLET: nat.FP_BC_DIRICHLET, orc.NEUMANN: nat.FP_BC_NEUMANN}
    kind = {orc.REGULAR: nat.FP_GRID_REGULAR, orc.STAGGERED: nat.FP_GRID_STAGGERED}
    for a, ax in enumerate(case.axes):
        cfg.n[a] = ax.n
        cfg.length[a] = ax.length
        cfg.bc[a] = bc[ax.bc]
        cfg.kind[a] = kind[ax.kind]
    cfg.approx = nat.FP_APPROX_SPECTRAL if case.approx == orc.SPECTRAL else nat.FP_APPROX_FD2
    cfg.precision = nat.FP_F32 if case.precision == "single" else nat.FP_F64
    return cfg


def create(lib, case):
    cfg = make_cfg(case)
    h = ctypes.c_void_p()
    assert lib.fp_plan_create(ctypes.byref(cfg), 0, ctypes.byref(h)) == nat.FP_OK, lib.fp_last_error()
    return h


CASES = {
    "neu3d": orc.Case([(32, 1.0, orc.NEUMANN, orc.STAGGERED), (64, 1.5, orc.NEUMANN, orc.STAGGERED), (32, 2.0, orc.NEUMANN, orc.STAGGERED)], orc.FD2),
    "c4like": orc.Case([(64, orc.TWO_PI, orc.PERIODIC), (32, orc.TWO_PI, orc.PERIODIC), (32, 2.0, orc.NEUMANN, orc.STAGGERED)], orc.FD2),
    "dirreg2d": orc.Case([(9, 1.0, orc.DIRICHLET, orc.REGULAR), (33, 2.0, orc.DIRICHLET, orc.REGULAR)], orc.SPECTRAL),
    "neureg": orc.Case([(17, 1.0, orc.NEUMANN, orc.REGULAR), (32, 1.0, orc.NEUMANN, orc.REGULAR)], orc.FD2),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_solve_host_dense(lib, name, rng):
    case = CASES[name]
    h = create(lib, case)
    rhs = rng.standard_normal(case.shape)
    out = np.zeros(case.shape)
    res = nat.FpSolveResult()
    st = lib.fp_solve_host(h, rhs.ctypes.data, nat.FP_F64, None, out.ctypes.data, None, ctypes.byref(res))
    assert st == nat.FP_OK, lib.fp_last_error()
    want, rm = orc.solve(case, rhs)
    assert orc.relative_l2(out, want) <= 1e-12
    assert res.removed_mean == pytest.approx(rm, abs=1e-12)
    assert res.total_seconds > 0 and all(x >= 0 for x in res.timing)
    lib.fp_plan_destroy(h)


def test_solve_host_strided_views_and_cast(lib, rng):
    case = CASES["neu3d"]
    h = create(lib, case)
    parent = np.full((40, 70, 36), 5.0, dtype=np.float32)
    view = parent[3:35, 2:66, 1:33]
    view[...] = rng.standard_normal(case.shape).astype(np.float32)
    out_parent = np.full((34, 66, 34), -1.0)
    out_view = out_parent[1:33, 1:65, 1:33]
    st_in = (ctypes.c_int64 * 3)(*[s // 4 for s in view.strides])
    st_out = (ctypes.c_int64 * 3)(*[s // 8 for s in out_view.strides])
    res = nat.FpSolveResult()
    base_in = view.ctypes.data
    base_out = out_view.ctypes.data
    st = lib.fp_solve_host(h, base_in, nat.FP_F32, st_in, base_out, st_out, ctypes.byref(res))
    assert st == nat.FP_OK, lib.fp_last_error()
    want, rm = orc.solve(case, view.astype(np.float64))
    assert orc.relative_l2(out_view, want) <= 1e-12
    mask = np.ones(out_parent.shape, bool)
    mask[1:33, 1:65, 1:33] = False
    assert np.all(out_parent[mask] == -1.0)
    lib.fp_plan_destroy(h)


def test_solve_host_nonfinite_leaves_out_untouched(lib, rng):
    case = CASES["c4like"]
    h = create(lib, case)
    rhs = rng.standard_normal(case.shape)
    rhs[3, 4, 5] = np.inf
    out = np.full(case.shape, 7.0)
    res = nat.FpSolveResult()
    st = lib.fp_solve_host(h, rhs.ctypes.data, nat.FP_F64, None, out.ctypes.data, None, ctypes.byref(res))
    assert st == nat.FP_ERR_NONFINITE
    assert b"non-finite" in lib.fp_last_error()
    assert np.all(out == 7.0)
    lib.fp_plan_destroy(h)


def test_device_solve_with_strides_and_workspace(lib, rng):
    import torch

    case = CASES["c4like"]
    h = create(lib, case)
    info = nat.FpPlanInfo()
    assert lib.fp_plan_info_get(h, ctypes.byref(info)) == nat.FP_OK
    assert info.num_passes == 5 and info.middle_axis == 0 and info.singular == 1 and info.periodic_mask == 0b011
    rhs = torch.from_numpy(rng.standard_normal(case.shape)).cuda()
    out_parent = torch.zeros((66, 34, 36), dtype=torch.float64, device="cuda")
    out = out_parent[1:65, 1:33, 2:34]
    ws = ctypes.c_size_t()
    lib.fp_plan_workspace_bytes(h, 0, ctypes.byref(ws))
    small = torch.empty(16, dtype=torch.uint8, device="cuda")
    dinfo = torch.zeros(16, dtype=torch.uint8, device="cuda")
    st_out = (ctypes.c_int64 * 3)(*out.stride())
    st = lib.fp_solve(h, rhs.data_ptr(), nat.FP_F64, None, out.data_ptr(), st_out, small.data_ptr(), 16,
                      torch.cuda.current_stream().cuda_stream, dinfo.data_ptr(), None)
    assert st == nat.FP_ERR_VALUE and b"workspace" in lib.fp_last_error()
    work = torch.empty(ws.value, dtype=torch.uint8, device="cuda")
    st = lib.fp_solve(h, rhs.data_ptr(), nat.FP_F64, None, out.data_ptr(), st_out, work.data_ptr(), ws.value,
                      torch.cuda.current_stream().cuda_stream, dinfo.data_ptr(), None)
    assert st == nat.FP_OK, lib.fp_last_error()
    torch.cuda.synchronize()
    want, rm = orc.solve(case, rhs.cpu().numpy())
    assert orc.relative_l2(out.cpu().numpy(), want) <= 1e-12
    hinfo = nat.FpSolveInfo.from_buffer_copy(dinfo.cpu().numpy().tobytes())
    got_rm = ctypes.c_double()
    lib.fp_removed_mean(h, ctypes.byref(hinfo), ctypes.byref(got_rm))
    assert got_rm.value == pytest.approx(rm, abs=1e-12)
    lib.fp_plan_destroy(h)


def test_status_codes(lib):
    cfg = make_cfg(CASES["neu3d"])
    h = ctypes.c_void_p()
    assert lib.fp_plan_create(ctypes.byref(cfg), 99, ctypes.byref(h)) == nat.FP_ERR_VALUE
    cfg.n[0] = 5000 * 3 + 1  # odd, above the dense limit, not on the FFT engine: Bluestein (used to be unsupported)
    cfg.bc[0] = nat.FP_BC_DIRICHLET
    cfg.kind[0] = nat.FP_GRID_REGULAR
    cfg.bc[1] = cfg.bc[2] = nat.FP_BC_DIRICHLET
    cfg.kind[1] = cfg.kind[2] = nat.FP_GRID_REGULAR
    assert lib.fp_plan_create(ctypes.byref(cfg), 0, ctypes.byref(h)) == nat.FP_OK, lib.fp_last_error()
    lib.fp_plan_destroy(h)
    # a slab decomposition needs axis 0 on the FFT engine: 15001 points -> FP_ERR_UNSUPPORTED
    assert lib.fp_plan_create_dist(ctypes.byref(cfg), 0, 2, 0, ctypes.byref(h)) == nat.FP_ERR_UNSUPPORTED
    assert b"FFT engine" in lib.fp_last_error()
