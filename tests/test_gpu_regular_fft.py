"""GPU tier: regular-grid Neumann / Dirichlet axes (DCT-I / DST-I) on the FFT engine.

For n = 2^k + 1 (Neumann, regular grid) and n = 2^k - 1 (Dirichlet, regular grid)
the transforms run as the half-length real FFT of the 2(n -+ 1)-point even / odd
extension instead of the dense O(n^2) engine.  Every case checks that the axis
really is on the FFT engine (plan info) and compares with the oracle.
"""

import numpy as np
import pytest

import paper_1409_8116_b200 as fp
from paper_1409_8116_b200.grid import Approximation as AP, BoundaryCondition as BC, GridKind as GK
from oracle import fastpoisson_oracle as orc

pytestmark = pytest.mark.gpu

N, D, P = orc.NEUMANN, orc.DIRICHLET, orc.PERIODIC
R = orc.REGULAR


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _solve_and_check(case, rng, expect_fft_axes):
    grids = tuple(fp.GridSpec(a.n, a.length, BC(a.bc), GK(a.kind)) for a in case.axes)
    plan = fp.SolverPlan(fp.SolverConfig(grids, AP(case.approx), case.precision))
    mask = int(plan._info.fft_axes_mask)
    for a in expect_fft_axes:
        assert mask >> a & 1, f"axis {a} of {case.axes} not on the FFT engine (mask {mask:b})"
    rhs = rng.standard_normal(case.shape)
    got, rep = plan.solve(rhs)
    want, rm = orc.solve(case, rhs)
    tol = 1e-5 if case.precision == "single" else 1e-12
    err = orc.relative_l2(got, want)
    assert err <= tol, (case.axes, err)
    assert rep.removed_mean == pytest.approx(rm, abs=1e-6 if case.precision == "single" else 1e-12)
    return err


NEU_N = [17, 33, 65, 129, 257, 513, 1025, 2049, 4097]
DIR_N = [15, 31, 63, 127, 255, 511, 1023, 2047, 4095]


@pytest.mark.parametrize("n", NEU_N + DIR_N)
@pytest.mark.parametrize("approx", [orc.FD2, orc.SPECTRAL])
def test_1d_every_length(n, approx, torch_cuda, rng):
    bc = N if n in NEU_N else D
    _solve_and_check(orc.Case([(n, 1.5, bc, R)], approx), rng, [0])


@pytest.mark.parametrize("n", NEU_N[:7] + DIR_N[:7])
def test_2d_contig_and_strided(n, torch_cuda, rng):
    # both families: axis 1 contiguous (first forward pass), axis 0 strided (the MID)
    bc = N if n in NEU_N else D
    m = 33 if bc == N else 31
    _solve_and_check(orc.Case([(n, 1.0, bc, R), (m, 2.0, bc, R)], orc.FD2), rng, [0, 1])
    _solve_and_check(orc.Case([(m, 1.0, bc, R), (n, 2.0, bc, R)], orc.FD2), rng, [0, 1])


@pytest.mark.parametrize("axes,fft_axes", [
    ([(33, 1.0, N, R), (65, 1.5, N, R), (17, 2.0, N, R)], [0, 1, 2]),
    ([(31, 1.0, D, R), (63, 1.5, D, R), (15, 2.0, D, R)], [0, 1, 2]),
    ([(129, 1.0, N, R)] * 3, [0, 1, 2]),
    ([(127, 1.0, D, R)] * 3, [0, 1, 2]),
    ([(64, orc.TWO_PI, P), (32, orc.TWO_PI, P), (33, 2.0, N, R)], [0, 1, 2]),   # periodic + DCT-I
    ([(64, orc.TWO_PI, P), (31, 2.0, D, R), (64, orc.TWO_PI, P)], [0, 1, 2]),   # DST-I between
    ([(513, 1.0, N, R), (17, 1.0, N, R)], [0, 1]),
])
@pytest.mark.parametrize("approx", [orc.FD2, orc.SPECTRAL])
def test_3d_and_mixed(axes, fft_axes, approx, torch_cuda, rng):
    _solve_and_check(orc.Case(axes, approx), rng, fft_axes)


@pytest.mark.parametrize("axes", [[(129, 1.0, N, R)] * 3, [(127, 1.0, D, R)] * 3, [(1025, 1.0, N, R), (65, 1.0, N, R)]])
def test_single_precision(axes, torch_cuda, rng):
    _solve_and_check(orc.Case(axes, orc.FD2, "single"), rng, list(range(len(axes))))


def test_neumann_regular_constant_and_mean(torch_cuda, rng):
    # the DCT-I null mode: removed_mean is the trapezoid-weighted mean and the
    # solution has exactly zero arithmetic mean (solver.py:218-225)
    case = orc.Case([(65, 1.0, N, R), (33, 2.0, N, R)], orc.FD2)
    grids = tuple(fp.GridSpec(a.n, a.length, BC(a.bc), GK(a.kind)) for a in case.axes)
    plan = fp.SolverPlan(fp.SolverConfig(grids, AP(case.approx)))
    rhs = rng.standard_normal(case.shape) + 3.0
    got, rep = plan.solve(rhs)
    want, rm = orc.solve(case, rhs)
    assert orc.relative_l2(got, want) <= 1e-12
    assert rep.removed_mean == pytest.approx(rm, abs=1e-12)
    assert abs(float(np.mean(got))) <= 1e-13 * float(np.abs(got).max())


@pytest.mark.parametrize("kind", [fp.TransformKind.DCT1, fp.TransformKind.DST1])
@pytest.mark.parametrize("M", [16, 64, 512, 4096])
@pytest.mark.parametrize("axis", [0, 1, 2])
def test_transform_plan_dct1_dst1(kind, M, axis, torch_cuda, rng):
    n = M + 1 if kind == fp.TransformKind.DCT1 else M - 1
    shape = [3, 5, 4]
    shape[axis] = n
    x = rng.standard_normal(shape)
    want = orc.forward_1d(kind.value, x, axis=axis)
    got = fp.TransformPlan(kind, n, axis=axis).execute(torch_cuda.from_numpy(x).cuda()).cpu().numpy()
    assert np.abs(got - want).max() <= 1e-13 * n * np.abs(x).max() * 4


# -- the longest FFT lines: M = 8192 complex (periodic n = 8192, real lines n = 16384) --
@pytest.mark.parametrize("axes,fft_axes", [
    ([(8192, orc.TWO_PI, P), (64, orc.TWO_PI, P)], [0, 1]),                      # CFFT 8192 as the MID
    ([(32, 1.0, N, orc.STAGGERED), (16384, 1.0, N, orc.STAGGERED)], [0, 1]),      # DCT-II n = 16384, contiguous
    ([(16384, 1.0, D, orc.STAGGERED), (32, 1.0, D, orc.STAGGERED)], [0, 1]),      # DST-II 16384, strided MID
    ([(32, orc.TWO_PI, P), (16384, orc.TWO_PI, P)], [0, 1]),                     # real FFT n = 16384
    ([(8193, 1.0, N, R), (17, 1.0, N, R)], [0, 1]),                              # DCT-I, M = 8192
])
@pytest.mark.parametrize("precision", ["double", "single"])
def test_longest_fft_lines(axes, fft_axes, precision, torch_cuda, rng):
    _solve_and_check(orc.Case(axes, orc.FD2 if axes[0][2] != P else orc.SPECTRAL, precision), rng, fft_axes)


@pytest.mark.parametrize("kind,n", [(fp.TransformKind.DFT, 8192), (fp.TransformKind.IDFT, 8192),
                                    (fp.TransformKind.DCT2, 16384), (fp.TransformKind.DST3, 16384)])
@pytest.mark.parametrize("axis", [0, 1])
def test_transform_plan_longest(kind, n, axis, torch_cuda, rng):
    shape = [3, 4]
    shape[axis] = n
    x = rng.standard_normal(shape)
    if kind.is_complex:
        x = x + 1j * rng.standard_normal(shape)
    want = orc.forward_1d(kind.value, x, axis=axis)
    got = fp.TransformPlan(kind, n, axis=axis).execute(torch_cuda.from_numpy(x).cuda()).cpu().numpy()
    assert np.abs(got - want).max() <= 1e-13 * n * np.abs(x).max() * 4
