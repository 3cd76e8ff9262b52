"""GPU tier: the dense engine (every length the FFT engine does not take).

The register-tiled product runs for lines of 64+ points (shorter lines use the
simple kernel); lines up to 8192 points.  Transforms are compared with scipy
(oracle.forward_1d), solves with the oracle.
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


@pytest.mark.parametrize("kind", list(fp.TransformKind))
@pytest.mark.parametrize("n", [63, 100, 383, 1000, 3001])
@pytest.mark.parametrize("axis", [0, 2])
def test_transform_dense_lengths(kind, n, axis, torch_cuda, rng):
    shape = [3, 5, 4]
    shape[axis] = n
    x = rng.standard_normal(shape)
    if kind.is_complex:
        x = x + 1j * rng.standard_normal(shape)
    want = orc.forward_1d(kind.value, x, axis=axis)
    got = fp.TransformPlan(kind, n, axis=axis).execute(torch_cuda.from_numpy(x).cuda()).cpu().numpy()
    assert np.abs(got - want).max() <= 1e-13 * n * np.abs(x).max() * 4


@pytest.mark.parametrize("kind", [fp.TransformKind.DFT, fp.TransformKind.DCT2, fp.TransformKind.DST1])
def test_transform_dense_longest(kind, torch_cuda, rng):
    n = 8191 if kind is not fp.TransformKind.DFT else 6000
    x = rng.standard_normal((n, 3))
    if kind.is_complex:
        x = x + 1j * rng.standard_normal((n, 3))
    want = orc.forward_1d(kind.value, x, axis=0)
    got = fp.TransformPlan(kind, n, axis=0).execute(torch_cuda.from_numpy(x).cuda()).cpu().numpy()
    assert np.abs(got - want).max() <= 1e-13 * n * np.abs(x).max() * 4


@pytest.mark.parametrize("axes,approx,precision", [
    ([(100, 1.0, orc.NEUMANN, orc.STAGGERED), (96, 1.5, orc.NEUMANN, orc.STAGGERED), (120, 2.0, orc.NEUMANN, orc.STAGGERED)], orc.FD2, "double"),
    ([(1000, 1.0, orc.DIRICHLET, orc.STAGGERED), (384, 1.0, orc.DIRICHLET, orc.STAGGERED)], orc.FD2, "double"),
    ([(90, orc.TWO_PI, orc.PERIODIC), (70, orc.TWO_PI, orc.PERIODIC), (66, 2.0, orc.NEUMANN, orc.STAGGERED)], orc.SPECTRAL, "double"),
    ([(300, 1.0, orc.NEUMANN, orc.REGULAR), (200, 1.0, orc.NEUMANN, orc.REGULAR)], orc.FD2, "double"),
    ([(300, orc.TWO_PI, orc.PERIODIC), (256, orc.TWO_PI, orc.PERIODIC)], orc.SPECTRAL, "double"),
    ([(100, 1.0, orc.NEUMANN, orc.STAGGERED), (96, 1.5, orc.NEUMANN, orc.STAGGERED), (120, 2.0, orc.NEUMANN, orc.STAGGERED)], orc.FD2, "single"),
    ([(5000, 1.0, orc.NEUMANN, orc.STAGGERED), (6, 1.0, orc.NEUMANN, orc.STAGGERED)], orc.FD2, "double"),
])
def test_solves_on_dense_axes(axes, approx, precision, torch_cuda, rng):
    case = orc.Case(axes, approx, precision)
    grids = tuple(fp.GridSpec(a.n, a.length, BC(a.bc), GK(a.kind)) for a in case.axes)
    plan = fp.SolverPlan(fp.SolverConfig(grids, AP(case.approx), case.precision))
    rhs = rng.standard_normal(case.shape)
    got, rep = plan.solve(rhs)
    want, rm = orc.solve(case, rhs)
    tol = 1e-5 if precision == "single" else 1e-12
    assert orc.relative_l2(got, want) <= tol
    assert rep.removed_mean == pytest.approx(rm, abs=1e-6 if precision == "single" else 1e-12)
