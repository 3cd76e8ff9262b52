"""GPU tier: seeded random sweep over the configuration space (1-3 axes, every
(bc, grid) row, both approximations, both precisions, lengths that land on the
FFT, mixed-radix and dense engines, strided device views) -- every solve
against the oracle (solver.py:191-249) at the parity bar."""

import numpy as np
import pytest

import paper_1409_8116_b200 as fp
from oracle import fastpoisson_oracle as orc

pytestmark = pytest.mark.gpu

ROWS = [(orc.PERIODIC, orc.REGULAR), (orc.DIRICHLET, orc.REGULAR), (orc.DIRICHLET, orc.STAGGERED),
        (orc.NEUMANN, orc.REGULAR), (orc.NEUMANN, orc.STAGGERED)]
# FFT-engine lengths (powers of two, 2^k +- 1 for type I), mixed-radix, dense (primes > 61, short)
LENGTHS = [1, 2, 3, 5, 8, 12, 16, 17, 31, 32, 33, 45, 48, 60, 63, 64, 65, 67, 96, 100, 127, 128, 129, 150, 255, 256]


def random_case(r):
    d = int(r.integers(1, 4))
    cap = {1: 4096, 2: 256, 3: 64}[d]
    axes = []
    # SolverConfig (solver.py:84-91): the non-periodic axes share one (bc, grid) row
    wall = ROWS[1 + int(r.integers(len(ROWS) - 1))]
    for _ in range(d):
        bc, kind = ROWS[0] if r.random() < 0.4 else wall
        n = int(r.choice([x for x in LENGTHS if x <= cap] + ([cap] if cap > 256 else [])))
        if bc == orc.NEUMANN and kind == orc.REGULAR and n < 2:
            n = 2
        axes.append((n, float(r.choice([1.0, 2.0, orc.TWO_PI])), bc, kind))
    approx = orc.SPECTRAL if r.random() < 0.4 else orc.FD2
    precision = "single" if r.random() < 0.25 else "double"
    return orc.Case(axes, approx, precision)


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.parametrize("seed", range(400))
def test_random_configuration(seed, torch_cuda):
    t = torch_cuda
    r = np.random.default_rng(1409 + seed)
    case = random_case(r)
    grids = tuple(fp.GridSpec(a.n, a.length, fp.BoundaryCondition(a.bc), fp.GridKind(a.kind)) for a in case.axes)
    plan = fp.SolverPlan(fp.SolverConfig(grids, fp.Approximation(case.approx), case.precision))
    rhs = r.standard_normal(case.shape)
    want, rm = orc.solve(case, rhs)
    tol = 1e-5 if case.precision == "single" else 1e-12
    mode = int(r.integers(3))
    if mode == 0:          # host arrays through the C ABI's host path
        got, rep = plan.solve(rhs)
    elif mode == 1:        # device tensor, fresh output
        got, rep = plan.solve(t.from_numpy(rhs).cuda())
        got = got.cpu().numpy()
    else:                  # strided device sub-block in and out (ghost cells)
        big = t.zeros(tuple(n + 2 for n in case.shape), dtype=t.float64, device="cuda")
        inner = tuple(slice(1, 1 + n) for n in case.shape)
        big[inner] = t.from_numpy(rhs).cuda()
        out = t.zeros(tuple(n + 3 for n in case.shape), dtype=t.float64 if case.precision == "double" else t.float32,
                      device="cuda")
        oin = tuple(slice(2, 2 + n) for n in case.shape)
        _, rep = plan.solve(big[inner], out=out[oin])
        got = out[oin].cpu().numpy()
    scale = max(np.abs(want).max(), 1e-300)
    assert orc.relative_l2(got, want) <= tol or np.abs(got - want).max() <= tol * scale, (case.axes, case.approx)
    assert rep.removed_mean == pytest.approx(rm, abs=(1e-5 if case.precision == "single" else 1e-12) * max(1.0, abs(rm)))
