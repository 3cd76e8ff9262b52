"""GPU tier: the Bluestein engine (fp_blue.cu) -- every transform kind at ANY length:
lengths with a prime factor above 61 (no mixed-radix plan) and lines longer than one
CTA's shared memory (four-step FFT_L).  The reference handles every n through
scipy.fft (transforms.py:70-77,128-177): transforms are compared with
scipy (oracle.forward_1d), solves with the oracle (solver.py:191-249).
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
    got = fp.TransformPlan(kind, n, axis=axis).execute(torch_cuda.from_numpy(x).cuda()).cpu().numpy()
    tol = (4e-6 if precision == "single" else 1e-14) * np.log2(n) * np.abs(want).max()
    err = np.abs(got - want).max()
    assert err <= tol, (kind, n, axis, err / np.abs(want).max())


# 131, 257, 1009 prime; 134 = 2 * 67; 8209 prime (L = 32768: four-step 16 x 2048)
@pytest.mark.parametrize("kind", list(fp.TransformKind))
@pytest.mark.parametrize("n", [131, 134, 257, 1009])
@pytest.mark.parametrize("axis", [0, 1, 2])
def test_transform_bluestein(kind, n, axis, torch_cuda, rng):
    _check_transform(kind, n, axis, [3, 5, 4], torch_cuda, rng)


@pytest.mark.parametrize("kind", list(fp.TransformKind))
@pytest.mark.parametrize("n", [257, 8209])
def test_transform_bluestein_single(kind, n, torch_cuda, rng):
    _check_transform(kind, n, 0, [n, 3], torch_cuda, rng, precision="single")


@pytest.mark.parametrize("kind", list(fp.TransformKind))
def test_transform_bluestein_four_step(kind, torch_cuda, rng):
    # 8209 (prime) and 20011 (prime; L = 65536 = 16 x 4096) fp64 lines
    _check_transform(kind, 8209, 0, [8209, 3], torch_cuda, rng)
    _check_transform(kind, 20011, 1, [2, 20011], torch_cuda, rng)


def _solve_case(axes, approx="fd2", precision="double"):
    case = orc.Case([tuple(a) for a in axes], approx, precision)
    grids = tuple(fp.GridSpec(a.n, a.length, BC(a.bc), GK(a.kind)) for a in case.axes)
    return case, fp.SolverConfig(grids, AP(case.approx), case.precision)


SOLVES = [
    # (axes, approx): every boundary row with a Bluestein axis (n >= 128, prime factor > 61)
    ([(131, 1.0, "neumann", "staggered"), (100, 1.5, "neumann", "staggered")], "fd2"),
    ([(137, 1.0, "dirichlet", "staggered"), (64, 2.0, "dirichlet", "staggered")], "fd2"),
    ([(131, 2 * np.pi, "periodic", "regular"), (96, 2 * np.pi, "periodic", "regular")], "spectral"),
    ([(135, 1.0, "neumann", "regular"), (40, 1.0, "neumann", "regular")], "fd2"),        # DCT-I, N = 268 = 4 * 67
    ([(133, 1.0, "dirichlet", "regular"), (48, 1.0, "dirichlet", "regular")], "fd2"),     # DST-I, N = 268
    ([(40, 1.0, "periodic", "regular"), (139, 1.0, "periodic", "regular"), (36, 1.0, "neumann", "staggered")], "fd2"),
    ([(149, 1.0, "neumann", "staggered"), (20, 1.0, "periodic", "regular"), (151, 1.0, "neumann", "staggered")], "spectral"),
    ([(8209, 1.0, "neumann", "staggered"), (8, 1.0, "periodic", "regular")], "fd2"),      # four-step, middle axis
    ([(6, 1.0, "neumann", "staggered"), (8209, 1.0, "periodic", "regular")], "fd2"),      # four-step, real FFT axis
]


@pytest.mark.parametrize("idx", range(len(SOLVES)))
def test_solve_bluestein_axes(idx, torch_cuda, rng):
    axes, approx = SOLVES[idx]
    case, cfg = _solve_case(axes, approx)
    rhs = rng.standard_normal(case.shape)
    want, rm_ref = orc.solve(case, rhs)
    got, rep = fp.SolverPlan(cfg).solve(rhs)
    err = orc.relative_l2(got, want)
    assert err <= 1e-12, (axes, err)
    assert rep.removed_mean == pytest.approx(rm_ref, abs=1e-12)


def test_solve_bluestein_single(torch_cuda, rng):
    case, cfg = _solve_case([(131, 1.0, "neumann", "staggered"), (257, 2.0, "periodic", "regular")], "fd2", "single")
    rhs = rng.standard_normal(case.shape).astype(np.float32)
    want, _ = orc.solve(case, rhs)
    got, _ = fp.SolverPlan(cfg).solve(rhs)
    assert orc.relative_l2(got, want) <= 1e-5


def test_solve_bluestein_device_strided(torch_cuda, rng):
    # a ghost-cell sub-block on the device through a Bluestein axis (strided I/O)
    t = torch_cuda
    case, cfg = _solve_case([(131, 1.0, "dirichlet", "staggered"), (70, 1.0, "dirichlet", "staggered")])
    big = t.from_numpy(rng.standard_normal((133, 72))).cuda()
    rhs = big[1:-1, 1:-1]
    want, _ = orc.solve(case, rhs.cpu().numpy())
    out = t.zeros_like(big)
    fp.SolverPlan(cfg).solve(rhs, out=out[1:-1, 1:-1])
    assert orc.relative_l2(out[1:-1, 1:-1].cpu().numpy(), want) <= 1e-12
    assert float(out[0].abs().max()) == 0.0
