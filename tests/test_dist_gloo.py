"""CPU tier: the multi-rank path (slab decomposition + all-to-all) with gloo, world size 2 and 4.

Each rank runs paper_1409_8116_b200.distributed.DistributedSolverPlan with the
native library's own layout rules (fp_dist_layout, device-free) and the numpy
backend of tests/dist_numpy_backend.py for the local phases; the exchanges are
real torch.distributed all_to_all_single calls over gloo.  The assembled
solution must equal the oracle's single-process solve.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import fastpoisson_oracle as orc

CASES = {
    "c3_small": orc.Case([(32, 1.0, orc.NEUMANN, orc.STAGGERED), (16, 1.0, orc.NEUMANN, orc.STAGGERED), (16, 1.0, orc.NEUMANN, orc.STAGGERED)], orc.FD2),
    "c4_small": orc.Case([(16, orc.TWO_PI, orc.PERIODIC), (16, orc.TWO_PI, orc.PERIODIC), (8, 2.0, orc.NEUMANN, orc.STAGGERED)], orc.FD2),
    "c5_small": orc.Case([(16, orc.TWO_PI, orc.PERIODIC)] * 3, orc.SPECTRAL),
    "dst_2d": orc.Case([(32, 1.0, orc.DIRICHLET, orc.STAGGERED), (12, 1.5, orc.DIRICHLET, orc.STAGGERED)], orc.FD2),
    "per_x_only": orc.Case([(32, 2.0, orc.PERIODIC), (8, 1.0, orc.DIRICHLET, orc.REGULAR), (6, 1.0, orc.DIRICHLET, orc.REGULAR)], orc.FD2),
    # a wall axis 0 after periodic local axes (complex exchanged state, real-view MID)
    "wall0_per_3d": orc.Case([(32, 1.0, orc.NEUMANN, orc.STAGGERED), (12, orc.TWO_PI, orc.PERIODIC), (10, orc.TWO_PI, orc.PERIODIC)], orc.FD2),
    "dct1_3d": orc.Case([(33, 1.0, orc.NEUMANN, orc.REGULAR), (9, 1.0, orc.NEUMANN, orc.REGULAR), (7, 1.0, orc.NEUMANN, orc.REGULAR)], orc.FD2),
    "per_dct1": orc.Case([(32, orc.TWO_PI, orc.PERIODIC), (9, 1.0, orc.NEUMANN, orc.REGULAR)], orc.FD2),
    "wall0_per_2d": orc.Case([(32, 1.0, orc.DIRICHLET, orc.STAGGERED), (10, 2.0, orc.PERIODIC)], orc.SPECTRAL),
}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1409_8116_b200 as fp
        from paper_1409_8116_b200.distributed import DistributedSolverPlan, dist_layout
        from dist_numpy_backend import NumpyBackend

        case = CASES[name]
        grids = tuple(fp.GridSpec(a.n, a.length, fp.BoundaryCondition(a.bc), fp.GridKind(a.kind)) for a in case.axes)
        config = fp.SolverConfig(grids, fp.Approximation(case.approx))
        info = dist_layout(config, world, rank)
        plan = DistributedSolverPlan(config, backend=NumpyBackend(case, info, world, rank))
        rng = np.random.default_rng(7)
        rhs = rng.standard_normal(case.shape)
        local = torch.from_numpy(np.ascontiguousarray(rhs[plan.local_slice]))
        out, rep = plan.solve(local)
        q.put((rank, plan.local_slice.start, out.numpy().copy(), rep.removed_mean))
    except Exception as exc:  # pragma: no cover - surfaced by the parent
        q.put((rank, -1, repr(exc), 0.0))
    finally:
        dist.destroy_process_group()


def _run(name, world):
    case = CASES[name]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, start, arr, _ in results:
        assert start >= 0, f"rank {rank} failed: {arr}"
    results.sort(key=lambda r: r[1])
    got = np.concatenate([r[2] for r in results], axis=0)
    rng = np.random.default_rng(7)
    rhs = rng.standard_normal(case.shape)
    want, rm = orc.solve(case, rhs, extended=False)
    assert orc.relative_l2(got, want) <= 1e-12
    for r in results:
        assert r[3] == pytest.approx(rm, abs=1e-12)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("name", sorted(CASES))
def test_distributed_orchestration_matches_oracle(name, world, native_lib):
    _run(name, world)


# uneven slabs: 32 planes over 3 ranks (11, 11, 10) -- any rank count, balanced split
@pytest.mark.parametrize("name", ["c3_small", "c4_small", "wall0_per_3d", "dst_2d", "dct1_3d"])
def test_distributed_uneven_slabs_world3(name, native_lib):
    _run(name, 3)
