"""GPU tier: the PyTorch-extension binding (torch.ops.fastpoisson_b200.solve) against the
plain ctypes call of the same C ABI entry point: bit-identical results on dense, strided,
in-place and override (`_inv_lam`) solves, on the current stream of the plan's device."""

import numpy as np
import pytest

import paper_1409_8116_b200 as fp
from paper_1409_8116_b200 import _native as nat
from oracle import fastpoisson_oracle as orc

pytestmark = pytest.mark.gpu

P, D, N = "periodic", "dirichlet", "neumann"
R, S = "regular", "staggered"
TWO_PI = 2 * np.pi

CASES = {
    "neumann3d_fd2": ([(32, 1.0, N, S), (16, 1.0, N, S), (24, 1.0, N, S)], "fd2", "double"),
    "mixed_c4_like": ([(32, TWO_PI, P), (16, TWO_PI, P), (32, 2.0, N, S)], "fd2", "double"),
    "dirichlet2d": ([(64, 1.0, D, S), (128, 1.0, D, S)], "fd2", "double"),
    "neumann_regular2d": ([(33, 1.0, N, R), (17, 1.0, N, R)], "fd2", "double"),
    "fp32_periodic": ([(32, TWO_PI, P)] * 3, "spectral", "single"),
}


def _plan(name):
    axes, approx, prec = CASES[name]
    case = orc.Case(axes, approx, prec)
    grids = tuple(fp.GridSpec(a.n, a.length, fp.BoundaryCondition(a.bc), fp.GridKind(a.kind)) for a in case.axes)
    return case, fp.SolverPlan(fp.SolverConfig(grids, fp.Approximation(case.approx), case.precision))


@pytest.fixture
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.parametrize("name", sorted(CASES))
def test_extension_matches_ctypes_and_oracle(torch_cuda, name, monkeypatch):
    t = torch_cuda
    case, plan = _plan(name)
    rng = np.random.default_rng(11)
    rhs = rng.standard_normal(case.shape).astype(case.dtype)
    rhs -= rhs.mean()
    x = t.from_numpy(rhs).cuda()
    assert nat.use_torch_ext()
    got_ext, rep_ext = plan.solve(x)
    monkeypatch.setenv("FP_BINDING", "ctypes")
    assert not nat.use_torch_ext()
    got_ct, rep_ct = plan.solve(x)
    monkeypatch.delenv("FP_BINDING")
    assert t.equal(got_ext, got_ct)
    assert rep_ext.removed_mean == rep_ct.removed_mean
    want, rm = orc.solve(case, rhs)
    tol = 1e-12 if case.precision == "double" else 1e-5   # north_star: <=1e-12 fp64, <=1e-5 fp32
    assert orc.relative_l2(got_ext.cpu().numpy(), want) <= tol
    assert abs(rep_ext.removed_mean - rm) <= (1e-12 if case.precision == "double" else 1e-5)


def test_extension_strided_inplace_and_stream(torch_cuda):
    t = torch_cuda
    case, plan = _plan("neumann3d_fd2")
    rng = np.random.default_rng(5)
    parent = t.from_numpy(rng.standard_normal((36, 20, 28))).cuda()
    view = parent[2:34, 2:18, 2:26]
    ref, _ = plan.solve(view.contiguous())
    side = t.cuda.Stream()
    with t.cuda.stream(side):      # the extension reads the CURRENT stream natively
        out, _ = plan.solve(view, out=view)
    side.synchronize()
    assert out.data_ptr() == view.data_ptr()
    assert t.equal(view, ref)
    # ghost cells untouched
    assert t.equal(parent[:2], t.from_numpy(np.random.default_rng(5).standard_normal((36, 20, 28))).cuda()[:2])


def test_extension_override_table(torch_cuda, monkeypatch):
    t = torch_cuda
    case, plan = _plan("mixed_c4_like")
    rng = np.random.default_rng(3)
    x = t.from_numpy(rng.standard_normal(case.shape)).cuda()
    plan._inv_lam[1, 2, 3] *= 1.5      # the reference's fault injection (verifysuite.py:83-88)
    got_ext, _ = plan.solve(x)
    monkeypatch.setenv("FP_BINDING", "ctypes")
    got_ct, _ = plan.solve(x)
    assert t.equal(got_ext, got_ct)


def test_extension_rejects_cpu_tensors(torch_cuda):
    z = torch_cuda.zeros(4)
    with pytest.raises(RuntimeError, match="CUDA tensors only"):
        nat.torch_ext().solve(0, z, z, z, z, 0, None)
