"""GPU tier: SolverPlan.capture -- one solve recorded as a CUDA graph (the
launch-bound 64^3 case of bench.py), replayed on refilled inputs."""

import numpy as np
import pytest

import paper_1409_8116_b200 as fp
from oracle import fastpoisson_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_captured_solve_matches_oracle_on_refilled_inputs(name, torch_cuda, rng):
    t = torch_cuda
    case = orc.config_case(name, scale=1 if name == "c1" else 16)
    grids = tuple(fp.GridSpec(a.n, a.length, fp.BoundaryCondition(a.bc), fp.GridKind(a.kind)) for a in case.axes)
    plan = fp.SolverPlan(fp.SolverConfig(grids, fp.Approximation(case.approx), case.precision))
    rhs = t.zeros(case.shape, dtype=t.float64, device="cuda")
    cap = plan.capture(rhs)
    for _ in range(3):
        x = rng.standard_normal(case.shape)
        if case.singular:
            x -= x.mean()
        rhs.copy_(t.from_numpy(x))           # refill in place, replay the same graph
        got = cap.replay().cpu().numpy()
        want, _ = orc.solve(case, x)
        assert orc.relative_l2(got, want) <= 1e-12
