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


def _plan(name, scale):
    case = orc.config_case(name, scale=scale)
    grids = tuple(fp.GridSpec(a.n, a.length, fp.BoundaryCondition(a.bc), fp.GridKind(a.kind)) for a in case.axes)
    return case, fp.SolverPlan(fp.SolverConfig(grids, fp.Approximation(case.approx), case.precision))


def test_captured_solve_outlives_its_plan(torch_cuda, rng):
    """The graph reads the plan's device tables: dropping the plan must not free them."""
    import gc

    t = torch_cuda
    case, plan = _plan("c3", 16)
    rhs = t.zeros(case.shape, dtype=t.float64, device="cuda")
    cap = plan.capture(rhs)
    del plan
    gc.collect()
    junk = [t.full((1 << 20,), 7.0, dtype=t.float64, device="cuda") for _ in range(8)]  # reuse freed blocks
    x = rng.standard_normal(case.shape)
    x -= x.mean()
    rhs.copy_(t.from_numpy(x))
    got = cap.replay().cpu().numpy()
    want, _ = orc.solve(case, x)
    assert orc.relative_l2(got, want) <= 1e-12
    del junk


def test_solve_batch_memory_bounded(torch_cuda, rng):
    """solve_batch keeps two workspaces, not one per step (periodic plans need a
    half-spectrum workspace)."""
    t = torch_cuda
    case, plan = _plan("c4", 8)
    xs = []
    for _ in range(12):
        x = rng.standard_normal(case.shape)
        xs.append(x - x.mean())
    t.cuda.synchronize()
    t.cuda.reset_peak_memory_stats()
    base = t.cuda.memory_allocated()
    res = plan.solve_batch(xs)
    peak = t.cuda.max_memory_allocated() - base
    field = int(np.prod(case.shape)) * 8
    ws = plan.workspace_bytes(True)
    assert peak <= 4 * field + 2 * ws + (64 << 20), (peak, field, ws)
    for x, (got, rep) in zip(xs[:3], res[:3]):
        want, rm = orc.solve(case, x)
        assert orc.relative_l2(got, want) <= 1e-12
        assert abs(rep.removed_mean - rm) <= 1e-12


def test_solve_on_non_current_device(torch_cuda, rng):
    """Events are created on the plan's device, not the current one."""
    t = torch_cuda
    if t.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    case = orc.config_case("c1", scale=4)
    grids = tuple(fp.GridSpec(a.n, a.length, fp.BoundaryCondition(a.bc), fp.GridKind(a.kind)) for a in case.axes)
    plan = fp.SolverPlan(fp.SolverConfig(grids, fp.Approximation(case.approx), case.precision), device="cuda:1")
    x = rng.standard_normal(case.shape)
    x -= x.mean()
    with t.cuda.device(0):
        got, _ = plan.solve(x)
        got_d, _ = plan.solve(t.from_numpy(x).to("cuda:1"))
    want, _ = orc.solve(case, x)
    assert orc.relative_l2(got, want) <= 1e-12
    assert orc.relative_l2(got_d.cpu().numpy(), want) <= 1e-12


def test_events_created_on_requested_device(torch_cuda, native_lib):
    import ctypes

    h = ctypes.c_void_p()
    assert native_lib.fp_event_create_on(0, ctypes.byref(h)) == 0
    assert native_lib.fp_event_destroy(h) == 0
