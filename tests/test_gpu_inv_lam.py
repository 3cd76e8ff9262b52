"""GPU tier: the writable ``SolverPlan._inv_lam`` contract (reference solver.py:151-159,221;
verifysuite.py:83-88 mutates it for fault injection).  A mutated table must change
the solve exactly as it changes the reference's; an untouched one must not."""

import numpy as np
import pytest

import paper_1409_8116_b200 as fp
from oracle import fastpoisson_oracle as orc

pytestmark = pytest.mark.gpu

P, D, N = "periodic", "dirichlet", "neumann"
R, S = "regular", "staggered"
TWO_PI = 2 * np.pi

CASES = {
    "neumann3d_fd2": ([(32, 1.0, N, S), (16, 1.0, N, S), (24, 1.0, N, S)], "fd2"),
    "periodic3d_spectral": ([(16, TWO_PI, P)] * 3, "spectral"),
    "periodic2d_fd2": ([(32, 1.0, P), (64, 2.0, P)], "fd2"),
    "mixed_c4_like": ([(32, TWO_PI, P), (16, TWO_PI, P), (32, 2.0, N, S)], "fd2"),
    "periodic_then_wall_2d": ([(64, 1.0, P), (32, 1.0, D, S)], "fd2"),
    "dirichlet1d": ([(64, 1.0, D, S)], "fd2"),
    "periodic1d": ([(128, 1.0, P)], "spectral"),
    "neumann_regular2d": ([(33, 1.0, N, R), (17, 1.0, N, R)], "fd2"),
    "odd_lengths": ([(30, 1.0, D, R), (21, 1.0, D, R)], "fd2"),
    "mixed_radix": ([(48, 1.0, N, S), (40, 1.0, N, S), (36, 1.0, N, S)], "fd2"),
    "fp32_periodic": ([(32, TWO_PI, P)] * 3, "spectral", "single"),
}


def _case(name):
    spec = CASES[name]
    return orc.Case(spec[0], spec[1], spec[2] if len(spec) > 2 else "double")


def _plan(case):
    grids = tuple(fp.GridSpec(a.n, a.length, fp.BoundaryCondition(a.bc), fp.GridKind(a.kind)) for a in case.axes)
    return fp.SolverPlan(fp.SolverConfig(grids, fp.Approximation(case.approx), case.precision))


def _rhs(case, rng):
    x = rng.standard_normal(case.shape).astype(case.dtype)
    if case.singular:
        x -= x.mean(dtype=np.float64).astype(case.dtype)
    return x


def _tol(case):
    return 1e-5 if case.precision == "single" else 1e-12


@pytest.mark.parametrize("name", sorted(CASES))
def test_fault_injection_matches_reference(name, rng):
    """verifysuite.py:87: plan._inv_lam.flat[-1] /= 1 + fault."""
    case = _case(name)
    plan = _plan(case)
    x = _rhs(case, rng)
    base, _ = plan.solve(x)
    plan._inv_lam.flat[-1] /= 1.0 + 1e-3
    got, rep = plan.solve(x)
    ref = orc.OraclePlan(case)
    ref.inv.flat[-1] /= 1.0 + 1e-3
    want, rm = ref.solve(x)
    assert orc.relative_l2(got, want) <= _tol(case)
    assert abs(rep.removed_mean - rm) <= (1e-5 if case.precision == "single" else 1e-12)
    if case.precision == "double":
        assert orc.relative_l2(got, base) > 1e-10     # the fault is visible


@pytest.mark.parametrize("name", sorted(CASES))
def test_dense_random_override_matches_reference(name, rng):
    """Any table, including ones without the Hermitian symmetry of lambda."""
    case = _case(name)
    plan = _plan(case)
    x = _rhs(case, rng)
    pert = 1.0 + 1e-2 * rng.standard_normal(case.shape)
    plan._inv_lam[...] = plan._inv_lam * pert.astype(case.dtype)
    got, _ = plan.solve(x)
    ref = orc.OraclePlan(case)
    ref.inv[...] = (ref.inv.astype(case.dtype) * pert.astype(case.dtype)).astype(ref.inv.dtype)
    want, _ = ref.solve(x)
    assert orc.relative_l2(got, want) <= _tol(case) * 10


def test_read_only_access_keeps_fused_path(rng):
    """Reading _inv_lam (reference tests/test_solver.py:235-240) changes nothing."""
    case = _case("neumann3d_fd2")
    plan = _plan(case)
    snap = plan._inv_lam.copy()
    x = _rhs(case, rng)
    for _ in range(3):
        got, _ = plan.solve(x)
    np.testing.assert_array_equal(plan._inv_lam, snap)
    assert plan._override_table() is None
    want, _ = orc.solve(case, x)
    assert orc.relative_l2(got, want) <= 1e-12


def test_restoring_the_table_restores_the_solve(rng):
    case = _case("periodic3d_spectral")
    plan = _plan(case)
    x = _rhs(case, rng)
    base, _ = plan.solve(x)
    saved = plan._inv_lam.copy()
    plan._inv_lam.flat[5] *= 2.0
    assert plan._override_table() is not None
    plan._inv_lam[...] = saved
    assert plan._override_table() is None
    again, _ = plan.solve(x)
    np.testing.assert_array_equal(again, base)


def test_device_tensor_solve_honours_override(torch_cuda, rng):
    t = torch_cuda
    case = _case("mixed_c4_like")
    plan = _plan(case)
    x = _rhs(case, rng)
    plan._inv_lam.flat[-1] *= 1.5
    got, _ = plan.solve(t.from_numpy(x).cuda())
    ref = orc.OraclePlan(case)
    ref.inv.flat[-1] *= 1.5
    want, _ = ref.solve(x)
    assert orc.relative_l2(got.cpu().numpy(), want) <= 1e-12


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch
