"""GPU tier: the distributed kernels (exchange layout, blocked MID) on one B200.

The P ranks of a slab decomposition are emulated sequentially on one GPU --
phase 0 for every rank, the all-to-all as device copies between the ranks'
buffers, phase 1 for every rank, the copies back, phase 2 -- so no kernel ever
waits on another rank.  The assembled solution must match the single-GPU solve.
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


def _config(case):
    grids = tuple(fp.GridSpec(a.n, a.length, BC(a.bc), GK(a.kind)) for a in case.axes)
    return fp.SolverConfig(grids, AP(case.approx), case.precision)


def emulate(config, P, rhs):
    """Run the three native phases for P ranks on this GPU; returns (solution, raw dc sum)."""
    import torch
    from paper_1409_8116_b200.distributed import NativeBackend

    bes = [NativeBackend(config, P, r) for r in range(P)]
    outs = []
    for r, be in enumerate(bes):
        out = be.new_output()
        off, a0 = int(be.info.offset0), int(be.info.local_n0)
        be.forward(rhs[off:off + a0].contiguous(), out)
        outs.append(out)
    blk = bes[0].send.numel() // P
    for r in range(P):
        for s in range(P):
            bes[r].recv[s * blk:(s + 1) * blk].copy_(bes[s].send[r * blk:(r + 1) * blk])
    for be in bes:
        be.middle()
    for r in range(P):
        for s in range(P):
            bes[s].send[r * blk:(r + 1) * blk].copy_(bes[r].recv[s * blk:(s + 1) * blk])
    for r, be in enumerate(bes):
        be.backward(outs[r])
    if bes[0].exact_mean:   # DCT-I: the global arithmetic mean (an all-reduce between ranks)
        total = sum(be.local_sum(outs[r]) for r, be in enumerate(bes))
        for r, be in enumerate(bes):
            be.subtract_mean(outs[r], total)
    torch.cuda.synchronize()
    dc = sum(float(be.read_status()[0]) for be in bes)
    nonfinite = sum(float(be.read_status()[1]) for be in bes)
    return torch.cat(outs, dim=0), dc, nonfinite


def emulate_chunked(config, P, rhs, C):
    """The pipelined exchange (DistributedSolverPlan._pipelined_exchange) emulated: per chunk of
    axis-1 rows, the chunk's pieces of every peer block copied, the MID on those rows
    (fp_solve_mid_rows), the pieces copied back."""
    import torch
    from paper_1409_8116_b200.distributed import NativeBackend

    bes = [NativeBackend(config, P, r) for r in range(P)]
    outs = []
    for r, be in enumerate(bes):
        out = be.new_output()
        off, a0 = int(be.info.offset0), int(be.info.local_n0)
        be.forward(rhs[off:off + a0].contiguous(), out)
        outs.append(out)
    B = int(bes[0].info.block_n1)
    C = max(1, min(C, B))   # (as DistributedSolverPlan does: no empty chunks)
    blk = bes[0].send.numel() // P
    row = blk // B
    for c in range(C):
        a, b = c * B // C, (c + 1) * B // C
        for r in range(P):
            for s in range(P):
                bes[r].recv[s * blk + a * row:s * blk + b * row].copy_(bes[s].send[r * blk + a * row:r * blk + b * row])
        for be in bes:
            be.middle_rows(a, b - a)
        for r in range(P):
            for s in range(P):
                bes[s].send[r * blk + a * row:r * blk + b * row].copy_(bes[r].recv[s * blk + a * row:s * blk + b * row])
    for r, be in enumerate(bes):
        be.backward(outs[r])
    if bes[0].exact_mean:
        total = sum(be.local_sum(outs[r]) for r, be in enumerate(bes))
        for r, be in enumerate(bes):
            be.subtract_mean(outs[r], total)
    torch.cuda.synchronize()
    dc = sum(float(be.read_status()[0]) for be in bes)
    return torch.cat(outs, dim=0), dc


SMALL = {
    "c3": orc.Case([(64, 1.0, orc.NEUMANN, orc.STAGGERED), (32, 1.0, orc.NEUMANN, orc.STAGGERED), (32, 1.0, orc.NEUMANN, orc.STAGGERED)], orc.FD2),
    "c4": orc.Case([(64, orc.TWO_PI, orc.PERIODIC), (64, orc.TWO_PI, orc.PERIODIC), (32, 2.0, orc.NEUMANN, orc.STAGGERED)], orc.FD2),
    "c5": orc.Case([(64, orc.TWO_PI, orc.PERIODIC)] * 3, orc.SPECTRAL, "single"),
    "c5d": orc.Case([(64, orc.TWO_PI, orc.PERIODIC)] * 3, orc.SPECTRAL),
    "dst2d": orc.Case([(64, 1.0, orc.DIRICHLET, orc.STAGGERED), (48, 1.5, orc.DIRICHLET, orc.STAGGERED)], orc.FD2),
    "perx": orc.Case([(64, 2.0, orc.PERIODIC), (12, 1.0, orc.DIRICHLET, orc.REGULAR), (10, 1.0, orc.DIRICHLET, orc.REGULAR)], orc.FD2),
    # local axes on the mixed-radix engine (non-power-of-two lengths)
    "mrwall": orc.Case([(64, 1.0, orc.NEUMANN, orc.STAGGERED), (60, 1.0, orc.NEUMANN, orc.STAGGERED), (45, 2.0, orc.NEUMANN, orc.STAGGERED)], orc.FD2),
    "mrper": orc.Case([(64, orc.TWO_PI, orc.PERIODIC), (48, orc.TWO_PI, orc.PERIODIC), (30, orc.TWO_PI, orc.PERIODIC)], orc.SPECTRAL),
    # a wall axis 0 after periodic local axes: complex exchanged state, real-view MID
    "wall0per3d": orc.Case([(64, 1.0, orc.NEUMANN, orc.STAGGERED), (48, orc.TWO_PI, orc.PERIODIC), (30, orc.TWO_PI, orc.PERIODIC)], orc.FD2),
    "wall0per2d": orc.Case([(64, 1.0, orc.DIRICHLET, orc.STAGGERED), (40, 2.0, orc.PERIODIC)], orc.SPECTRAL),
    # DCT-I / DST-I (regular walls): axis 0 (n0 = 2^k +- 1) on the FFT engine's type-I MID over the
    # receive layout, local axes on the mixed-radix / dense engines, exact global mean removal
    "dct1": orc.Case([(65, 1.0, orc.NEUMANN, orc.REGULAR), (33, 1.0, orc.NEUMANN, orc.REGULAR), (17, 2.0, orc.NEUMANN, orc.REGULAR)], orc.FD2),
    "dst1": orc.Case([(63, 1.0, orc.DIRICHLET, orc.REGULAR), (31, 1.0, orc.DIRICHLET, orc.REGULAR)], orc.FD2),
    "per_dct1": orc.Case([(64, orc.TWO_PI, orc.PERIODIC), (33, 1.0, orc.NEUMANN, orc.REGULAR), (17, 1.0, orc.NEUMANN, orc.REGULAR)], orc.FD2),
    "dct1_wall0per": orc.Case([(65, 1.0, orc.NEUMANN, orc.REGULAR), (24, orc.TWO_PI, orc.PERIODIC), (20, orc.TWO_PI, orc.PERIODIC)], orc.FD2),
    "wall0per3d_f32": orc.Case([(64, 1.0, orc.NEUMANN, orc.STAGGERED), (32, orc.TWO_PI, orc.PERIODIC), (16, orc.TWO_PI, orc.PERIODIC)], orc.FD2, "single"),
}


# P = 3, 5, 6, 7: uneven slabs (64 planes split 22/21/21, ...) through the MID's row table
@pytest.mark.parametrize("P", [2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("name", sorted(SMALL))
def test_dist_emulated_matches_single_gpu(name, P, torch_cuda, rng):
    t = torch_cuda
    case = SMALL[name]
    config = _config(case)
    rhs = rng.standard_normal(case.shape)
    if case.singular:
        rhs -= rhs.mean()
    dt = t.float32 if case.precision == "single" else t.float64
    rhs_t = t.from_numpy(rhs).to("cuda", dt)
    want, rep = fp.SolverPlan(config).solve(rhs_t)
    got, dc, nonfinite = emulate(config, P, rhs_t)
    tol = 1e-5 if case.precision == "single" else 1e-12
    err = (t.linalg.vector_norm((got - want).double()) / t.linalg.vector_norm(want.double())).item()
    assert err <= tol, err
    assert nonfinite == 0
    if case.singular:
        plan = fp.SolverPlan(config)
        np_prod = np.prod([a.n for a in case.axes if a.bc == orc.PERIODIC]) if case.periodic_axes else 1.0
        rm = (dc / np_prod) / plan._null_scale
        assert rm == pytest.approx(rep.removed_mean, abs=1e-6 if case.precision == "single" else 1e-12)


@pytest.mark.parametrize("P,C", [(2, 3), (3, 2), (4, 4)])
@pytest.mark.parametrize("name", sorted(SMALL))
def test_dist_pipelined_exchange_matches_single_gpu(name, P, C, torch_cuda, rng):
    # the exchange in C chunks of axis-1 rows with the MID per chunk (fp_solve_mid_rows)
    t = torch_cuda
    case = SMALL[name]
    config = _config(case)
    rhs = rng.standard_normal(case.shape)
    if case.singular:
        rhs -= rhs.mean()
    dt = t.float32 if case.precision == "single" else t.float64
    rhs_t = t.from_numpy(rhs).to("cuda", dt)
    want, rep = fp.SolverPlan(config).solve(rhs_t)
    got, dc = emulate_chunked(config, P, rhs_t, C)
    tol = 1e-5 if case.precision == "single" else 1e-12
    err = (t.linalg.vector_norm((got - want).double()) / t.linalg.vector_norm(want.double())).item()
    assert err <= tol, err
    if case.singular:
        plan = fp.SolverPlan(config)
        np_prod = np.prod([a.n for a in case.axes if a.bc == orc.PERIODIC]) if case.periodic_axes else 1.0
        assert (dc / np_prod) / plan._null_scale == pytest.approx(rep.removed_mean, abs=1e-6 if case.precision == "single" else 1e-12)


@pytest.mark.slow
@pytest.mark.parametrize("name,P", [("c3", 8), ("c4", 8), ("c4", 2)])
def test_dist_emulated_full_size(name, P, torch_cuda):
    t = torch_cuda
    case = orc.config_case(name)
    config = _config(case)
    gen = t.Generator(device="cuda")
    gen.manual_seed(3)
    rhs = t.randn(case.shape, dtype=t.float64, device="cuda", generator=gen)
    rhs -= rhs.mean()
    want, _ = fp.SolverPlan(config).solve(rhs)
    got, _, _ = emulate(config, P, rhs)
    err = (t.linalg.vector_norm(got - want) / t.linalg.vector_norm(want)).item()
    print(f"{name} P={P}: relative L2 vs single-GPU solve {err:.3e}")
    assert err <= 1e-12


@pytest.mark.parametrize("P", [2, 3, 4])
@pytest.mark.parametrize("name", ["c3", "c4", "c5d", "mrper", "wall0per3d"])
def test_multi_device_wrapper_matches_single_gpu(name, P, torch_cuda, rng):
    # the single-process multi-device wrapper; ranks share cuda:0 here
    from paper_1409_8116_b200.distributed import MultiDeviceSolverPlan

    case = SMALL[name]
    config = _config(case)
    rhs = rng.standard_normal(case.shape)
    if case.singular:
        rhs -= rhs.mean()
    want, rep = fp.SolverPlan(config).solve(rhs)
    plan = MultiDeviceSolverPlan(config, ["cuda:0"] * P)
    got, rep2 = plan.solve(rhs)
    assert isinstance(got, np.ndarray)
    assert orc.relative_l2(got, want) <= 1e-12
    assert rep2.removed_mean == pytest.approx(rep.removed_mean, abs=1e-12)
    got_t, _ = plan.solve(torch_cuda.from_numpy(rhs).cuda())
    assert orc.relative_l2(got_t.cpu().numpy(), want) <= 1e-12


def test_distributed_plan_world_one_nccl(torch_cuda, rng):
    # DistributedSolverPlan on a one-rank NCCL group: the whole grid is the slab
    import os
    import socket

    import torch.distributed as dist
    from paper_1409_8116_b200.distributed import DistributedSolverPlan

    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", world_size=1, rank=0,
                            device_id=torch_cuda.device("cuda", 0))
    try:
        case = SMALL["c4"]
        config = _config(case)
        rhs = rng.standard_normal(case.shape)
        want, rep = fp.SolverPlan(config).solve(rhs)
        plan = DistributedSolverPlan(config)
        assert plan.local_shape == tuple(case.shape)
        got, rep2 = plan.solve(torch_cuda.from_numpy(rhs).cuda())
        assert orc.relative_l2(got.cpu().numpy(), want) <= 1e-12
        assert rep2.removed_mean == pytest.approx(rep.removed_mean, abs=1e-12)
        out = plan.solve_async(torch_cuda.from_numpy(rhs).cuda())
        torch_cuda.cuda.synchronize()
        assert orc.relative_l2(out.cpu().numpy(), want) <= 1e-12
    finally:
        dist.destroy_process_group()
