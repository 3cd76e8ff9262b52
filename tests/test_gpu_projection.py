"""GPU tier: the fused projection step against the reference flow.

ProjectionStep.project = divergence formed inside the solve's first pass (or by
a stand-alone kernel when z is on the dense engine) + the corrector kernel.
Compared with fixtures produced by the reference flow module and with the oracle.
"""

from pathlib import Path

import numpy as np
import pytest

import paper_1409_8116_b200 as fp
from oracle import fastpoisson_oracle as orc

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden" / "projection_v1.npz"


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


@pytest.mark.parametrize("name", ["periodic", "walls", "walls_dense"])
def test_projection_matches_reference_fixture(name, torch_cuda):
    z = np.load(GOLD)
    nx, nz, lx, lz, walls, scale = z[f"{name}/meta"]
    step = fp.ProjectionStep((int(nx), int(nz)), (lx, lz), z_walls=bool(walls))
    u, w, phi, rep = step.project(z[f"{name}/ustar"], z[f"{name}/wstar"], scale)
    u, w, phi = u.cpu().numpy(), w.cpu().numpy(), phi.cpu().numpy()
    assert _rel(phi, z[f"{name}/phi"]) <= 1e-12
    assert _rel(u, z[f"{name}/u"]) <= 1e-12
    assert _rel(w, z[f"{name}/w"]) <= 1e-12
    assert np.abs(orc.staggered_divergence(u, w, (lx, lz), bool(walls))).max() <= 1e-9
    assert rep.removed_mean == pytest.approx(float(np.mean(orc.staggered_divergence(
        z[f"{name}/ustar"], z[f"{name}/wstar"], (lx, lz), bool(walls)) / scale)), abs=1e-10)


@pytest.mark.parametrize("cells,walls", [((1024, 512), True), ((512, 1024), False), ((96, 256), True), ((256, 100), False)])
def test_projection_larger_vs_oracle(cells, walls, torch_cuda, rng):
    L = (2.0, 1.0)
    nx, nz = cells
    ustar = rng.standard_normal((nx, nz))
    wstar = rng.standard_normal((nx, nz + 1) if walls else (nx, nz))
    if walls:
        wstar[:, [0, -1]] = 0.0
    scale = 0.013
    step = fp.ProjectionStep(cells, L, z_walls=walls)
    u, w, phi, _ = step.project(torch_cuda.from_numpy(ustar).cuda(), torch_cuda.from_numpy(wstar).cuda(), scale)
    want_u, want_w, want_phi = orc.project_step(ustar, wstar, scale, L, walls)
    assert _rel(phi.cpu().numpy(), want_phi) <= 1e-12
    assert _rel(u.cpu().numpy(), want_u) <= 1e-12
    assert _rel(w.cpu().numpy(), want_w) <= 1e-12


def test_projection_in_place_pressure_and_fp32(torch_cuda, rng):
    t = torch_cuda
    cells, L = (256, 128), (2 * np.pi, 1.0)
    ustar = rng.standard_normal(cells)
    wstar = rng.standard_normal((256, 129))
    wstar[:, [0, -1]] = 0.0
    want_u, want_w, want_phi = orc.project_step(ustar, wstar, 0.02, L, True)
    step = fp.ProjectionStep(cells, L, z_walls=True)
    u_d, w_d = t.from_numpy(ustar).cuda(), t.from_numpy(wstar).cuda()
    p = t.ones(cells, dtype=t.float64, device="cuda")
    u, w, phi, _ = step.project(u_d, w_d, 0.02, p=p, u_out=u_d, w_out=w_d)   # in place
    assert u.data_ptr() == u_d.data_ptr() and w.data_ptr() == w_d.data_ptr()
    assert _rel(u_d.cpu().numpy(), want_u) <= 1e-12 and _rel(w_d.cpu().numpy(), want_w) <= 1e-12
    assert _rel(p.cpu().numpy() - 1.0, want_phi) <= 1e-12
    s32 = fp.ProjectionStep(cells, L, z_walls=True, precision="single")
    u32, w32, phi32, _ = s32.project(ustar.astype(np.float32), wstar.astype(np.float32), 0.02)
    assert _rel(u32.cpu().numpy(), want_u) <= 1e-5 and _rel(phi32.cpu().numpy(), want_phi) <= 1e-5


def test_projection_nonfinite_and_wrong_plan(torch_cuda, rng):
    step = fp.ProjectionStep((64, 32), (1.0, 1.0), z_walls=False)
    ustar = rng.standard_normal((64, 32))
    ustar[3, 4] = np.nan
    with pytest.raises(ValueError):
        step.project(ustar, rng.standard_normal((64, 32)), 0.1)
    with pytest.raises(ValueError):
        step.project(rng.standard_normal((64, 31)), rng.standard_normal((64, 32)), 0.1)
