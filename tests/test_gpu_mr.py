"""GPU tier: the mixed-radix engine (fp_mr.cu) -- every transform kind at lengths
whose FFT length factors into primes <= 61 (radix 2/4/8/16, 3, 5, 7 and the
generic odd-prime butterfly), including lengths above the dense engine's 8192
limit.  Transforms are compared with scipy (oracle.forward_1d, the reference's
own call, transforms.py:157-172), solves with the oracle (solver.py:191-249).
"""

import numpy as np
import pytest

import paper_1409_8116_b200 as fp
from paper_1409_8116_b200.grid import Approximation as AP, BoundaryCondition as BC, GridKind as GK
from oracle import fastpoisson_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _check_transform(kind, n, axis, shape, torch_cuda, rng, precision="double"):
    shape = list(shape)
    shape[axis] = n
    x = rng.standard_normal(shape)
    if kind.is_complex:
        x = x + 1j * rng.standard_normal(shape)
    want = orc.forward_1d(kind.value, x, axis=axis)
    if precision == "single":
        x = x.astype(np.complex64 if kind.is_complex else np.float32)
    got = fp.TransformPlan(kind, n, axis=axis).execute(  # precision follows the operand dtype
        torch_cuda.from_numpy(x).cuda())
    got = got.cpu().numpy()
    tol = (2e-6 if precision == "single" else 1e-14) * np.log2(n) * np.abs(want).max()
    assert np.abs(got - want).max() <= tol, (kind, n, axis)


# lengths: 48 = 16*3, 60 = 4*3*5, 77 = 7*11 (generic radix), 99, 125 = 5^3,
# 243 = 3^5, 1000 = 8*5^3, 1001 = 7*11*13, 2046 = 2*3*11*31, 4913 = 17^3
@pytest.mark.parametrize("kind", list(fp.TransformKind))
@pytest.mark.parametrize("n", [48, 60, 77, 99, 125, 243, 1000, 1001, 2046, 4913])
@pytest.mark.parametrize("axis", [0, 1, 2])
def test_transform_mixed_radix(kind, n, axis, torch_cuda, rng):
    _check_transform(kind, n, axis, [3, 5, 4], torch_cuda, rng)


@pytest.mark.parametrize("kind", list(fp.TransformKind))
@pytest.mark.parametrize("n", [120, 1000])
def test_transform_mixed_radix_single(kind, n, torch_cuda, rng):
    _check_transform(kind, n, 1, [4, n, 6], torch_cuda, rng, precision="single")


@pytest.mark.parametrize("kind,n,precision", [
    (fp.TransformKind.DFT, 10000, "double"), (fp.TransformKind.IDFT, 9000, "double"),
    (fp.TransformKind.DCT2, 9000, "double"), (fp.TransformKind.DCT3, 9000, "double"),
    (fp.TransformKind.DST2, 10125, "double"), (fp.TransformKind.DST3, 12000, "double"),
    # type I runs on the 2(n -+ 1)-point extension: above 8192 points only the
    # fp32 line fits one CTA's shared memory
    (fp.TransformKind.DCT1, 9001, "single"), (fp.TransformKind.DST1, 9999, "single"),
    (fp.TransformKind.DCT2, 20000, "single")])
def test_transform_beyond_dense_limit(kind, n, precision, torch_cuda, rng):
    # lengths above 8192 used to be unsupported (dense engine limit)
    _check_transform(kind, n, 0, [n, 3], torch_cuda, rng, precision=precision)


@pytest.mark.parametrize("kind,n", [(fp.TransformKind.DCT1, 9001), (fp.TransformKind.DST1, 9999)])
def test_fp64_type1_beyond_dense_limit(kind, n, torch_cuda, rng):
    # type I on the half-length recipe: the 2(n -+ 1)-point extension packed into n -+ 1 complex points
    _check_transform(kind, n, 0, [n, 3], torch_cuda, rng)


def test_large_prime_length_beyond_dense_limit(torch_cuda, rng):
    # 8209 is prime: no mixed-radix plan, beyond the dense engine -- the Bluestein engine
    # (fp_blue.cu) takes it (it used to raise NotImplementedError)
    _check_transform(fp.TransformKind.DCT2, 8209, 0, [8209, 2], torch_cuda, rng)


def _solve_case(axes, approx, precision, torch_cuda, rng, device=False):
    case = orc.Case(axes, approx, precision)
    grids = tuple(fp.GridSpec(a.n, a.length, BC(a.bc), GK(a.kind)) for a in case.axes)
    plan = fp.SolverPlan(fp.SolverConfig(grids, AP(case.approx), case.precision))
    rhs = rng.standard_normal(case.shape)
    if device:
        got, rep = plan.solve(torch_cuda.from_numpy(rhs).cuda())
        got = got.cpu().numpy()
    else:
        got, rep = plan.solve(rhs)
    want, rm = orc.solve(case, rhs)
    tol = 1e-5 if precision == "single" else 1e-12
    assert orc.relative_l2(got, want) <= tol
    assert rep.removed_mean == pytest.approx(rm, abs=1e-6 if precision == "single" else 1e-12)
    return plan


@pytest.mark.parametrize("axes,approx,precision", [
    # staggered Neumann / Dirichlet (DCT-II/III, DST-II/III) at odd and even non-power-of-two lengths
    ([(100, 1.0, orc.NEUMANN, orc.STAGGERED), (75, 1.5, orc.NEUMANN, orc.STAGGERED), (120, 2.0, orc.NEUMANN, orc.STAGGERED)], orc.FD2, "double"),
    ([(243, 1.0, orc.DIRICHLET, orc.STAGGERED), (96, 1.0, orc.DIRICHLET, orc.STAGGERED), (35, 1.0, orc.DIRICHLET, orc.STAGGERED)], orc.FD2, "double"),
    # periodic (real FFT on the last axis, complex DFT elsewhere) with a wall axis
    ([(90, orc.TWO_PI, orc.PERIODIC), (70, orc.TWO_PI, orc.PERIODIC), (66, 2.0, orc.NEUMANN, orc.STAGGERED)], orc.SPECTRAL, "double"),
    ([(60, orc.TWO_PI, orc.PERIODIC), (45, orc.TWO_PI, orc.PERIODIC), (125, orc.TWO_PI, orc.PERIODIC)], orc.SPECTRAL, "double"),
    # regular grids (DCT-I / DST-I via the 2(n-1) / 2(n+1) extensions)
    ([(101, 1.0, orc.NEUMANN, orc.REGULAR), (121, 1.0, orc.NEUMANN, orc.REGULAR)], orc.FD2, "double"),
    ([(120, 1.0, orc.DIRICHLET, orc.REGULAR), (44, 1.0, orc.DIRICHLET, orc.REGULAR), (80, 1.0, orc.DIRICHLET, orc.REGULAR)], orc.FD2, "double"),
    # single precision
    ([(100, 1.0, orc.NEUMANN, orc.STAGGERED), (75, 1.5, orc.NEUMANN, orc.STAGGERED), (120, 2.0, orc.NEUMANN, orc.STAGGERED)], orc.FD2, "single"),
    ([(60, orc.TWO_PI, orc.PERIODIC), (45, orc.TWO_PI, orc.PERIODIC), (125, orc.TWO_PI, orc.PERIODIC)], orc.SPECTRAL, "single"),
    # beyond the dense engine's 8192 limit
    ([(9000, 1.0, orc.NEUMANN, orc.STAGGERED), (12, 1.0, orc.NEUMANN, orc.STAGGERED)], orc.FD2, "double"),
    ([(10000, orc.TWO_PI, orc.PERIODIC), (16, orc.TWO_PI, orc.PERIODIC)], orc.SPECTRAL, "double"),
    ([(6, 1.0, orc.DIRICHLET, orc.STAGGERED), (12000, 1.0, orc.DIRICHLET, orc.STAGGERED)], orc.FD2, "double"),
])
def test_solves_on_mixed_radix_axes(axes, approx, precision, torch_cuda, rng):
    _solve_case(axes, approx, precision, torch_cuda, rng)


def test_mixed_radix_device_solve_and_residual(torch_cuda, rng):
    # 3D 200 x 150 x 180 Neumann-staggered FD2 through device tensors, plus the
    # FD2 residual of the solution
    axes = [(200, 1.0, orc.NEUMANN, orc.STAGGERED), (150, 1.0, orc.NEUMANN, orc.STAGGERED),
            (180, 1.0, orc.NEUMANN, orc.STAGGERED)]
    case = orc.Case(axes, orc.FD2)
    grids = tuple(fp.GridSpec(a.n, a.length, BC(a.bc), GK(a.kind)) for a in case.axes)
    plan = fp.SolverPlan(fp.SolverConfig(grids, AP.FINITE_DIFFERENCE_2, "double"))
    rhs = rng.standard_normal(case.shape)
    rhs -= rhs.mean()
    got, rep = plan.solve(torch_cuda.from_numpy(rhs).cuda())
    got = got.cpu().numpy()
    want, rm = orc.solve(case, rhs)
    assert orc.relative_l2(got, want) <= 1e-12
    res = orc.laplacian(case, got) - (rhs - rep.removed_mean)
    assert np.abs(res).max() <= 1e-8 * np.abs(rhs).max()


def test_mixed_radix_nonfinite_rhs(torch_cuda, rng):
    grids = (fp.GridSpec(100, 1.0, BC.NEUMANN, GK.STAGGERED), fp.GridSpec(60, 1.0, BC.NEUMANN, GK.STAGGERED))
    plan = fp.SolverPlan(fp.SolverConfig(grids, AP.FINITE_DIFFERENCE_2, "double"))
    rhs = rng.standard_normal((100, 60))
    rhs[37, 11] = np.nan
    with pytest.raises(ValueError):
        plan.solve(rhs)
