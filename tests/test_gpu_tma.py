"""GPU tier: the TMA-staged strided passes (csrc/fp_tma.cuh) -- fp64 DCT / DST lines of
256 and 512 points over 16-column tiles: the forward pass, the MID and the inverse pass
on the cp.async.bulk.tensor path, including ragged column counts (the last tile's
columns out of bounds: zero-filled loads, clipped stores), a missing line axis (2D),
the first pass's non-finite check, and strided operands that are not eligible (they
fall back to the regular kernel).  Results against the oracle (solver.py:191-249).
"""

import numpy as np
import pytest

import paper_1409_8116_b200 as fp
from paper_1409_8116_b200.grid import Approximation as AP, BoundaryCondition as BC, GridKind as GK
from oracle import fastpoisson_oracle as orc

pytestmark = pytest.mark.gpu
N_, D_, P_, S_ = orc.NEUMANN, orc.DIRICHLET, orc.PERIODIC, orc.STAGGERED

CASES = {
    "mid512_2d": orc.Case([(512, 1.0, N_, S_), (40, 1.5, N_, S_)], orc.FD2),
    "mid256_dst_2d": orc.Case([(256, 1.0, D_, S_), (100, 2.0, D_, S_)], orc.FD2),
    "fwd_inv512_3d": orc.Case([(24, 1.0, N_, S_), (512, 1.0, N_, S_), (33, 2.0, N_, S_)], orc.FD2),
    "mid_fwd256_3d": orc.Case([(256, 1.0, D_, S_), (256, 1.0, D_, S_), (20, 1.0, D_, S_)], orc.FD2),
    "wall_first_pass": orc.Case([(512, 1.0, N_, S_), (48, orc.TWO_PI, P_), (32, orc.TWO_PI, P_)], orc.SPECTRAL),
    "c3_quarter": orc.Case([(128, 1.0, N_, S_), (256, 1.0, N_, S_), (512, 1.0, N_, S_)], orc.FD2),
    "dst_c3_like": orc.Case([(256, 1.0, D_, S_), (512, 1.0, D_, S_), (64, 1.0, D_, S_)], orc.SPECTRAL),
    # 512-point DST MID and inverse on the interleaved-lines mapping (two lines per warp), > 148 tiles
    # along the strided passes so the L2 prefetch of a later tile fires
    "dst_mid512_3d": orc.Case([(512, 1.0, D_, S_), (56, 1.0, D_, S_), (48, 1.5, D_, S_)], orc.FD2),
    "neu_y512_many_tiles": orc.Case([(64, 1.0, N_, S_), (512, 1.0, N_, S_), (48, 1.0, N_, S_)], orc.FD2),
    # c4's pattern: the real-FFT axis (1024 points) strided between the wall axis and the MID:
    # the real-FFT forward / inverse on the TMA kernel (8-column tiles, ragged: 36 columns)
    "rfft_c4_like": orc.Case([(16, orc.TWO_PI, P_), (1024, orc.TWO_PI, P_), (36, 2.0, N_, S_)], orc.FD2),
    "rfft_dir": orc.Case([(8, 1.0, P_), (1024, 2.0, P_), (64, 1.0, D_, S_)], orc.SPECTRAL),
    # the MID over a complex state (c4's x axis): 1024-point complex lines, 4-column tiles (ragged: 22)
    # contiguous 512-point DCT / DST lines (c3's z passes) on the 4D-map kernel; odd line count: fallback
    "z512_dst": orc.Case([(6, 1.0, D_, S_), (10, 1.0, D_, S_), (512, 1.0, D_, S_)], orc.FD2),
    "z512_neu_2d": orc.Case([(30, 1.0, N_, S_), (512, 2.0, N_, S_)], orc.SPECTRAL),
    "z512_odd_nb": orc.Case([(4, 1.0, N_, S_), (7, 1.0, N_, S_), (512, 1.0, N_, S_)], orc.FD2),
    "cmid_c4_like": orc.Case([(1024, orc.TWO_PI, P_), (16, orc.TWO_PI, P_), (22, 2.0, N_, S_)], orc.FD2),
    "cmid_spectral": orc.Case([(1024, orc.TWO_PI, P_), (10, orc.TWO_PI, P_), (32, 1.0, D_, S_)], orc.SPECTRAL),
}


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _config(case):
    grids = tuple(fp.GridSpec(a.n, a.length, BC(a.bc), GK(a.kind)) for a in case.axes)
    return fp.SolverConfig(grids, AP(case.approx), case.precision)


@pytest.mark.parametrize("name", sorted(CASES))
def test_tma_passes_match_oracle(name, torch_cuda, rng):
    case = CASES[name]
    rhs = rng.standard_normal(case.shape)
    want, rm = orc.solve(case, rhs)
    plan = fp.SolverPlan(_config(case))
    got, rep = plan.solve(rhs)
    assert orc.relative_l2(got, want) <= 1e-12
    assert rep.removed_mean == pytest.approx(rm, abs=1e-12)
    # device tensors, in place
    x = torch_cuda.from_numpy(rhs).cuda()
    plan.solve(x, out=x)
    assert orc.relative_l2(x.cpu().numpy(), want) <= 1e-12


def test_tma_first_pass_nonfinite(torch_cuda, rng):
    case = CASES["wall_first_pass"]
    rhs = rng.standard_normal(case.shape)
    rhs[300, 7, 5] = np.nan
    with pytest.raises(ValueError):
        fp.SolverPlan(_config(case)).solve(rhs)


@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
@pytest.mark.parametrize("name", ["z512_dst", "z512_neu_2d"])
def test_tma_contiguous_first_pass_nonfinite(torch_cuda, rng, name, bad):
    # the contiguous 512-point first pass checks its inputs through 0 * x accumulated over the
    # registers that hold the line (NaN and both infinities must trip it, finite data must not)
    case = CASES[name]
    plan = fp.SolverPlan(_config(case))
    rhs = rng.standard_normal(case.shape)
    plan.solve(rhs)                      # finite: no error
    idx = tuple(int(v) for v in rng.integers(0, np.array(case.shape)))
    rhs[idx] = bad
    with pytest.raises(ValueError):
        plan.solve(rhs)
    big = rng.standard_normal(case.shape) * 1e300   # huge but finite values stay legal
    plan.solve(big)


def test_tma_ineligible_strides_fall_back(torch_cuda, rng):
    # a ghost-cell sub-block: rows 8-B aligned only -> the regular strided kernel
    t = torch_cuda
    case = CASES["mid512_2d"]
    big = t.from_numpy(rng.standard_normal((514, 42))).cuda()
    want, _ = orc.solve(case, big[1:-1, 1:-1].cpu().numpy())
    out = t.zeros_like(big)
    fp.SolverPlan(_config(case)).solve(big[1:-1, 1:-1], out=out[1:-1, 1:-1])
    assert orc.relative_l2(out[1:-1, 1:-1].cpu().numpy(), want) <= 1e-12
    assert float(out[0].abs().max()) == 0.0 and float(out[:, 0].abs().max()) == 0.0
