"""GPU tier: parity of the sm_100a solve path with the reference / oracle.

Every solve here goes through the drop-in API -> ctypes -> C ABI -> kernels.
Bars (BASELINE.json north_star): relative L2 <= 1e-12 in fp64, <= 1e-5 in fp32,
plus the discrete residual of the chosen operator.
"""

import threading

import numpy as np
import pytest

import paper_1409_8116_b200 as fp
from paper_1409_8116_b200.grid import Approximation as AP, BoundaryCondition as BC, GridKind as GK
from oracle import fastpoisson_oracle as orc

pytestmark = pytest.mark.gpu

F64_TOL = 1e-12
F32_TOL = 1e-5


def fp_config(case):
    grids = tuple(fp.GridSpec(a.n, a.length, BC(a.bc), GK(a.kind)) for a in case.axes)
    return fp.SolverConfig(grids, AP(case.approx), case.precision)


def entry_case(e):
    return orc.Case([tuple(a) for a in e["axes"]], e["approx"], e["precision"])


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


# -- golden vectors produced by the reference itself ----------------------------
def test_golden_solves(golden, torch_cuda):
    meta, arrays = golden
    worst = 0.0
    for e in meta["solves"]:
        if e["sampled"]:
            continue
        case = entry_case(e)
        plan = fp.SolverPlan(fp_config(case))
        rhs = arrays[f"{e['id']}/rhs"]
        want = arrays[f"{e['id']}/sol"]
        got, rep = plan.solve(rhs)
        assert got.dtype == case.dtype
        tol = F32_TOL if case.precision == "single" else F64_TOL
        err = orc.relative_l2(got, want)
        worst = max(worst, err if case.precision == "double" else 0.0)
        assert err <= tol, (e["id"], e["axes"], e["approx"], err)
        atol = 1e-6 if case.precision == "single" else 1e-12
        assert rep.removed_mean == pytest.approx(e["removed_mean"], abs=atol), e["id"]
        assert rep.mode == e["mode"] and list(rep.periodic_axes) == e["periodic_axes"]
        assert set(rep.timing) == {"forward", "diagonal", "backward"}
    print(f"worst fp64 relative L2 vs reference: {worst:.3e}")


def test_golden_scaled_configs(golden, torch_cuda):
    meta, arrays = golden
    stride = meta["sample_stride"]
    for e in meta["solves"]:
        if not e["sampled"]:
            continue
        case = orc.config_case(e["generator"], e["scale"])
        rhs = orc.config_rhs(e["generator"], case, seed=e["seed"])
        plan = fp.SolverPlan(fp_config(case))
        got, rep = plan.solve(rhs)
        tol = F32_TOL if case.precision == "single" else F64_TOL
        assert orc.relative_l2(got.ravel()[::stride], arrays[f"{e['id']}/sol_sample"]) <= tol, e["id"]
        assert rep.removed_mean == pytest.approx(e["removed_mean"], abs=1e-12 if case.precision == "double" else 1e-6)


def test_golden_transforms(golden, torch_cuda):
    meta, arrays = golden
    for e in meta["transforms"]:
        kind = fp.TransformKind(e["kind"])
        x = arrays[f"{e['id']}/x"]
        y = arrays[f"{e['id']}/y"]
        got = fp.TransformPlan(kind, e["n"]).execute(x)
        assert np.abs(got - y).max() <= 1e-12 * e["n"] * max(np.abs(x).max(), 1.0), e["id"]


@pytest.mark.parametrize("kind", list(fp.TransformKind))
@pytest.mark.parametrize("n", [32, 64, 1024, 8192])
@pytest.mark.parametrize("axis", [0, 1, 2])
def test_transform_plan_batched(kind, n, axis, torch_cuda, rng):
    # FFT engine (pow2) and dense engine, contiguous and strided axes, device tensors
    # (n = 8192: FFT engine for the half-length kinds, the dense engine's longest line for the others)
    shape = [3, 5, 4]
    shape[axis] = n
    x = rng.standard_normal(shape)
    if kind.is_complex:
        x = x + 1j * rng.standard_normal(shape)
    want = orc.forward_1d(kind.value, x, axis=axis)
    xt = torch_cuda.from_numpy(x).cuda()
    got = fp.TransformPlan(kind, n, axis=axis).execute(xt).cpu().numpy()
    assert np.abs(got - want).max() <= 1e-13 * n * np.abs(x).max() * 4


# -- BASELINE configs: oracle parity at full size + residual --------------------
def _residual_rel(case, sol, rhs, rm):
    res = orc.laplacian(case, sol) - (rhs - rm)
    return np.linalg.norm(res.ravel()) / np.linalg.norm(rhs.ravel())


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_config_full_size_parity(name, torch_cuda):
    case = orc.config_case(name)
    rhs = orc.config_rhs(name, case, seed=0)
    want, rm_ref = orc.solve(case, rhs, workers=-1)
    plan = fp.SolverPlan(fp_config(case))
    got, rep = plan.solve(rhs)
    err = orc.relative_l2(got, want)
    print(f"{name}: relative L2 vs oracle {err:.3e}, removed_mean {rep.removed_mean:.3e} vs {rm_ref:.3e}")
    assert err <= F64_TOL
    assert rep.removed_mean == pytest.approx(rm_ref, abs=1e-12)
    if case.approx == orc.FD2:
        r_gpu = _residual_rel(case, got, rhs, rep.removed_mean)
        r_ref = _residual_rel(case, want, rhs, rm_ref)
        print(f"{name}: FD2 residual gpu {r_gpu:.3e} ref {r_ref:.3e}")
        assert r_gpu <= 10 * r_ref + 1e-15
    else:
        # spectral: transform the solution forward and multiply by lambda
        lam = sum(np.meshgrid(*[orc.eigenvalues(a, case.approx) for a in case.axes], indexing="ij"))
        spec = np.fft.fftn(got) * lam
        target = np.fft.fftn(rhs - rm_ref)
        target.flat[0] = 0.0
        assert np.linalg.norm((spec - target).ravel()) <= 1e-11 * np.linalg.norm(target.ravel())


@pytest.mark.slow
def test_config_c4_full_size_parity(torch_cuda):
    import psutil

    if psutil.virtual_memory().total < 96e9:
        pytest.skip("host RAM too small for the c4 oracle")
    case = orc.config_case("c4")
    rhs = orc.config_rhs("c4", case, seed=0)
    want, rm_ref = orc.solve(case, rhs, workers=-1)
    got, rep = fp.SolverPlan(fp_config(case)).solve(rhs)
    assert orc.relative_l2(got, want) <= F64_TOL
    assert rep.removed_mean == pytest.approx(rm_ref, abs=1e-12)


@pytest.mark.parametrize("name,scale", [("c4", 2), ("c5", 4), ("c5", 2)])
def test_config_reduced_parity(name, scale, torch_cuda):
    case = orc.config_case(name, scale)
    rhs = orc.config_rhs(name, case, seed=1)
    want, rm_ref = orc.solve(case, rhs, workers=-1)
    got, rep = fp.SolverPlan(fp_config(case)).solve(rhs)
    tol = F32_TOL if case.precision == "single" else F64_TOL
    err = orc.relative_l2(got, want)
    print(f"{name}/{scale}: relative L2 {err:.3e}")
    assert err <= tol
    assert rep.removed_mean == pytest.approx(rm_ref, abs=1e-6 if case.precision == "single" else 1e-12)


@pytest.mark.slow
def test_c5_full_size_planted_modes(torch_cuda):
    """2048^3 fp32 spectral: planted eigenmodes come back exactly (size-independent property)."""
    t = torch_cuda
    case = orc.config_case("c5")
    n = case.axes[0].n
    dev = t.device("cuda")
    x = t.arange(n, device=dev, dtype=t.float64) * (2 * np.pi / n)
    modes = [(3, 5, 7, 1.0), (100, 1, 1000, 0.5), (1024, 0, 2, -0.25)]
    sol_want = t.zeros((n, n, n), dtype=t.float32, device=dev)
    rhs = t.zeros((n, n, n), dtype=t.float32, device=dev)
    for kx, ky, kz, amp in modes:
        m = (t.cos(kx * x)[:, None, None] * t.cos(ky * x)[None, :, None]).to(t.float32) * t.cos(kz * x).to(t.float32)[None, None, :]
        lam = -float(min(kx, n - kx) ** 2 + min(ky, n - ky) ** 2 + min(kz, n - kz) ** 2)
        sol_want.add_(m, alpha=amp)
        rhs.add_(m, alpha=amp * lam)
        del m
    plan = fp.SolverPlan(fp_config(case))
    out, rep = plan.solve(rhs)
    num = den = 0.0
    for i in range(0, n, 64):   # fp64 accumulation without a 64 GiB temporary
        dlt = (out[i:i + 64] - sol_want[i:i + 64]).double()
        num += float((dlt * dlt).sum())
        den += float((sol_want[i:i + 64].double() ** 2).sum())
    err = (num / den) ** 0.5
    print(f"c5 planted-mode relative L2 {err:.3e}")
    assert err <= F32_TOL
    assert abs(rep.removed_mean) <= 1e-6


def _c5_spectral_norms(t, S, lam0, lam12, chunk):
    """Axis-0 FFT of the (axes-1,2 transformed) fp64 half spectrum S in column
    chunks; returns (sum |E|^2, sum lam^2 |E|^2) with lam = lam0[k0] + lam12[k1, k2]."""
    e2 = r2 = 0.0
    for c in range(0, S.shape[1], chunk):
        blk = t.fft.fft(S[:, c:c + chunk], dim=0)
        a2 = blk.real.square_() + blk.imag.square_()
        lam = lam0[:, None, None] + lam12[None, c:c + chunk]
        # rfft half spectrum: interior k2 columns stand for two modes of the full spectrum
        w = t.full((S.shape[2],), 2.0, dtype=t.float64, device=S.device)
        w[0] = 1.0
        if S.shape[2] % 2 == 1:
            w[-1] = 1.0
        e2 += float((a2 * w).sum())
        r2 += float((a2 * lam.square() * w).sum())
        del blk, a2, lam
    return e2, r2


@pytest.mark.slow
def test_c5_full_size_seeded_vs_fp64(torch_cuda):
    """c5 at FULL size (2048^3 fp32 periodic spectral) on a seeded N(0,1) RHS with its
    mean removed (BASELINE.json configs[4]).

    The reference needs ~270 GB of host RAM here (dense _inv_lam + full complex
    spectra, solver.py:147-159,239-245) and the GPU box has 196 GB
    (profiles/r02/gpu_box_host.txt), so the checker is an on-device fp64 spectral solve
    with torch.fft (test-only; cuFFT is never on the product path), chunked so that
    rhs-derived data, the GPU solution and one fp64 half spectrum fit in HBM:
      * relative L2 of the GPU solution vs the exact fp64 solve of the same fp32 RHS
        <= 1e-5 (the north_star's fp32 bar; the reference's own fp32 solve is itself
        ~1e-7 away from that exact solution);
      * spectral residual ||lam F(u) - F(f - mean)|| / ||F(f - mean)||, obtained as
        ||lam F(u - u_exact)|| (u_exact solves the system exactly), must be <= 10x the
        residual of u_exact rounded to fp32 -- the best any fp32 output can do.
    """
    t = torch_cuda
    case = orc.config_case("c5")
    n = case.axes[0].n
    dev = t.device("cuda")
    gen = t.Generator(device=dev)
    gen.manual_seed(5)
    f = t.randn((n, n, n), generator=gen, dtype=t.float32, device=dev)
    f -= float(f.mean(dtype=t.float64))
    plan = fp.SolverPlan(fp_config(case))
    out, rep = plan.solve(f)
    del plan
    t.cuda.synchronize()
    t.cuda.empty_cache()
    fm = rep.removed_mean
    lam = [t.as_tensor(orc.eigenvalues(a, case.approx), device=dev) for a in case.axes]
    lam12 = lam[1][:, None] + lam[2][None, : n // 2 + 1]
    B = 32       # planes per rfft2 batch (~2 GB of fp64)
    C = 32       # axis-1 rows per axis-0 chunk (~2 GB of complex128)
    f_norm2 = 0.0
    S = t.empty((n, n, n // 2 + 1), dtype=t.complex128, device=dev)   # 68.7 GB
    for i in range(0, n, B):
        x = f[i:i + B].double() - fm
        f_norm2 += float(x.square().sum())
        S[i:i + B] = t.fft.rfft2(x)
        del x
    del f
    t.cuda.empty_cache()
    for c in range(0, n, C):   # exact solve in fp64: U = F(f - mean) / lam, zero mode 0
        blk = t.fft.fft(S[:, c:c + C], dim=0)
        lamc = lam[0][:, None, None] + lam12[None, c:c + C]
        if c == 0:
            lamc[0, 0, 0] = 1.0
        blk /= lamc
        if c == 0:
            blk[0, 0, 0] = 0.0
        S[:, c:c + C] = t.fft.ifft(blk, dim=0)
        del blk, lamc
    err2 = ex2 = 0.0
    d = t.empty((n, n, n), dtype=t.float32, device=dev)   # u_exact rounded to fp32, minus u_exact
    for i in range(0, n, B):
        ue = t.fft.irfft2(S[i:i + B], s=(n, n))
        ex2 += float(ue.square().sum())
        e = out[i:i + B].double() - ue
        err2 += float(e.square().sum())
        d[i:i + B] = (ue.float().double() - ue).float()
        S[i:i + B] = t.fft.rfft2(e)
        del ue, e
    err = (err2 / ex2) ** 0.5
    _, r_gpu = _c5_spectral_norms(t, S, lam[0], lam12, C)
    for i in range(0, n, B):
        S[i:i + B] = t.fft.rfft2(d[i:i + B].double())
    _, r_round = _c5_spectral_norms(t, S, lam[0], lam12, C)
    del S, d
    t.cuda.empty_cache()
    target = (n ** 3 * f_norm2) ** 0.5   # ||F(f - mean)|| by Parseval
    res_gpu, res_round = r_gpu ** 0.5 / target, r_round ** 0.5 / target
    print(f"c5 full size: rel L2 vs fp64 exact {err:.3e}; spectral residual gpu {res_gpu:.3e}, "
          f"exact-rounded-to-fp32 {res_round:.3e}; removed_mean {fm:.3e}")
    assert err <= F32_TOL
    assert res_gpu <= 10 * res_round
    assert abs(fm) <= 1e-6


# -- semantics of the drop-in --------------------------------------------------------
def _plan(bc, kind, shape, approx=AP.FINITE_DIFFERENCE_2, precision="double"):
    lengths = [1.0 + 0.5 * i for i in range(len(shape))]
    return fp.SolverPlan(fp.SolverConfig(tuple(fp.GridSpec(n, L, bc, kind) for n, L in zip(shape, lengths)), approx, precision))


def test_zero_rhs_and_constant_neumann(torch_cuda):
    plan = _plan(BC.DIRICHLET, GK.REGULAR, (8, 8))
    sol, rep = plan.solve(np.zeros((8, 8)))
    assert np.all(sol == 0.0) and rep.removed_mean == 0.0
    plan = _plan(BC.NEUMANN, GK.STAGGERED, (64, 32))
    sol, rep = plan.solve(np.full((64, 32), -2.75))
    assert np.abs(sol).max() <= 1e-13
    assert rep.removed_mean == pytest.approx(-2.75, rel=1e-12)


def test_validation_errors(torch_cuda):
    plan = _plan(BC.PERIODIC, GK.REGULAR, (32, 32))
    with pytest.raises(ValueError):
        plan.solve(np.zeros((32, 31)))
    bad = np.zeros((32, 32))
    bad[1, 2] = np.nan
    out = np.full((32, 32), 7.0)
    with pytest.raises(ValueError, match="non-finite"):
        plan.solve(bad, out=out)
    assert np.all(out == 7.0)  # nothing written before the error
    bad[1, 2] = np.inf
    with pytest.raises(ValueError):
        plan.solve(torch_cuda.from_numpy(bad).cuda())
    with pytest.raises(ValueError):
        plan.solve(np.zeros((32, 32)), out=np.zeros((33, 32)))
    with pytest.raises(fp.ConfigurationError):
        fp.solve_mixed(plan, np.zeros((32, 32)))


@pytest.mark.parametrize("shape", [(6, 7), (64, 32), (32, 64, 32)])
def test_subblock_transparency_host_and_device(shape, torch_cuda, rng):
    plan = _plan(BC.NEUMANN, GK.STAGGERED, shape)
    rhs_tight = rng.standard_normal(shape)
    pshape = tuple(n + 4 for n in shape)
    off = (2,) * len(shape)
    rhs_parent = np.full(pshape, 123.0)
    rhs_field = fp.Field.subblock(rhs_parent, off, shape)
    rhs_field.data[...] = rhs_tight
    sol_parent = np.full(pshape, -9.0)
    sol_field = fp.Field.subblock(sol_parent, (1,) * len(shape), shape)
    tight, _ = plan.solve(rhs_tight)
    plan.solve(rhs_field, out=sol_field)
    assert np.abs(sol_field.data - tight).max() <= 1e-14 * max(1.0, np.abs(tight).max())
    mask = np.ones(pshape, bool)
    mask[tuple(slice(1, 1 + n) for n in shape)] = False
    assert np.all(sol_parent[mask] == -9.0)
    np.testing.assert_array_equal(rhs_field.data, rhs_tight)
    # device: ghost-cell sub-blocks solved in place through their strides
    t = torch_cuda
    rp = t.from_numpy(rhs_parent).cuda()
    sp = t.full(pshape, -9.0, dtype=t.float64, device="cuda")
    rf = fp.Field.subblock(rp, off, shape)
    sf = fp.Field.subblock(sp, (1,) * len(shape), shape)
    plan.solve(rf, out=sf)
    assert np.abs(sf.data.cpu().numpy() - tight).max() <= 1e-14 * max(1.0, np.abs(tight).max())
    spn = sp.cpu().numpy()
    assert np.all(spn[mask] == -9.0)
    np.testing.assert_array_equal(rp.cpu().numpy(), rhs_parent)


@pytest.mark.parametrize("shape", [(8, 5), (64, 64), (32, 32, 32)])
def test_in_place_aliasing(shape, torch_cuda, rng):
    plan = _plan(BC.DIRICHLET, GK.STAGGERED, shape)
    rhs = rng.standard_normal(shape)
    expected, _ = plan.solve(rhs)
    buf = rhs.copy()
    plan.solve(buf, out=buf)
    np.testing.assert_array_equal(buf, expected)
    d = torch_cuda.from_numpy(rhs).cuda()
    plan.solve(d, out=d)
    np.testing.assert_array_equal(d.cpu().numpy(), expected)


def test_linearity_and_translation(torch_cuda, rng):
    plan = _plan(BC.DIRICHLET, GK.STAGGERED, (64, 32))
    f, g = rng.standard_normal((64, 32)), rng.standard_normal((64, 32))
    c, _ = plan.solve(0.6 * f - 2.2 * g)
    a, _ = plan.solve(f)
    b, _ = plan.solve(g)
    np.testing.assert_allclose(c, 0.6 * a - 2.2 * b, atol=1e-12 * np.abs(c).max())
    plan = _plan(BC.PERIODIC, GK.REGULAR, (32, 64))
    r = rng.standard_normal((32, 64))
    r -= r.mean()
    base, _ = plan.solve(r)
    sh, _ = plan.solve(np.roll(r, (3, 5), axis=(0, 1)))
    np.testing.assert_allclose(sh, np.roll(base, (3, 5), axis=(0, 1)), atol=1e-12 * np.abs(base).max())


def test_concurrent_solves_on_shared_plan(torch_cuda, rng):
    plan = _plan(BC.DIRICHLET, GK.STAGGERED, (64, 64))
    inputs = [rng.standard_normal((64, 64)) for _ in range(8)]
    expected = [plan.solve(r)[0] for r in inputs]
    results = [None] * 8

    def work(i):
        results[i] = plan.solve(inputs[i])[0]

    threads = [threading.Thread(target=work, args=(i,)) for i in range(8)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    for got, want in zip(results, expected):
        np.testing.assert_array_equal(got, want)


def test_single_precision_and_input_casts(torch_cuda, rng):
    plan = _plan(BC.NEUMANN, GK.STAGGERED, (64, 32), precision="single")
    rhs = rng.standard_normal((64, 32))
    rhs -= rhs.mean()
    got, _ = plan.solve(rhs.astype(np.float32))
    assert got.dtype == np.float32
    case = orc.Case([(64, 1.0, "neumann", "staggered"), (32, 1.5, "neumann", "staggered")], "fd2")
    want, _ = orc.solve(case, rhs)
    assert orc.relative_l2(got, want) <= F32_TOL
    # float32 rhs into a double plan, integer rhs
    plan64 = _plan(BC.NEUMANN, GK.STAGGERED, (64, 32))
    got64, _ = plan64.solve(rhs.astype(np.float32))
    want64, _ = orc.solve(case, rhs.astype(np.float32).astype(np.float64))
    assert orc.relative_l2(got64, want64) <= F64_TOL
    ints = np.arange(64 * 32).reshape(64, 32) % 7
    goti, _ = plan64.solve(ints)
    wanti, _ = orc.solve(case, ints.astype(np.float64))
    assert orc.relative_l2(goti, wanti) <= F64_TOL


def test_device_tensor_path_returns_tensor(torch_cuda, rng):
    t = torch_cuda
    plan = _plan(BC.PERIODIC, GK.REGULAR, (64, 64, 64), AP.PSEUDO_SPECTRAL)
    rhs = rng.standard_normal((64, 64, 64))
    d = t.from_numpy(rhs).cuda()
    out, rep = plan.solve(d)
    assert isinstance(out, t.Tensor) and out.is_cuda
    host, rep2 = plan.solve(rhs)
    np.testing.assert_array_equal(out.cpu().numpy(), host)
    assert rep.removed_mean == rep2.removed_mean


def test_laplacian_aid_device_matches_host(torch_cuda, rng):
    cfg = fp.SolverConfig(tuple(fp.GridSpec(n, 1.0, BC.NEUMANN, GK.REGULAR) for n in (9, 7)), AP.FINITE_DIFFERENCE_2)
    x = rng.standard_normal((9, 7))
    h = fp.apply_discrete_laplacian(cfg, x)
    d = fp.apply_discrete_laplacian(cfg, torch_cuda.from_numpy(x).cuda()).cpu().numpy()
    np.testing.assert_allclose(d, h, atol=1e-12 * np.abs(h).max())
    case = orc.Case([(9, 1.0, "neumann", "regular"), (7, 1.0, "neumann", "regular")], "fd2")
    np.testing.assert_allclose(h, orc.laplacian(case, x), atol=1e-12 * np.abs(h).max())


def test_solve_batch_matches_individual_solves(torch_cuda, rng):
    plan = _plan(BC.NEUMANN, GK.STAGGERED, (64, 32, 32))
    rhs = [rng.standard_normal((64, 32, 32)) for _ in range(5)]
    single = [plan.solve(r) for r in rhs]
    outs = [np.empty((64, 32, 32)) for _ in range(5)]
    batch = plan.solve_batch(rhs, outs)
    for (a, ra), (b, rb), o in zip(single, batch, outs):
        np.testing.assert_array_equal(a, b)
        assert b is o
        assert ra.removed_mean == rb.removed_mean
    bad = [r.copy() for r in rhs[:3]]
    bad[1][0, 0, 0] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        plan.solve_batch(bad)


def test_reorder_seam_keys_match_reference(torch_cuda, rng):
    # tests/test_solver.py:291-320 assert these keys of plan._reorder; the GPU
    # path transforms those axes in place through strides
    BC, GK, AP = fp.BoundaryCondition, fp.GridKind, fp.Approximation
    cfg = fp.SolverConfig((fp.GridSpec(6, 1.0, BC.PERIODIC), fp.GridSpec(5, 1.5, BC.NEUMANN, GK.STAGGERED),
                           fp.GridSpec(4, 2.0, BC.NEUMANN, GK.STAGGERED)), AP.FINITE_DIFFERENCE_2)
    plan = fp.SolverPlan(cfg)
    assert 1 in plan._reorder and 2 not in plan._reorder
    cfg2 = fp.SolverConfig((fp.GridSpec(5, 1.0, BC.DIRICHLET, GK.STAGGERED), fp.GridSpec(6, 2.0, BC.PERIODIC)),
                           AP.FINITE_DIFFERENCE_2)
    plan2 = fp.SolverPlan(cfg2)
    assert plan2._reorder.keys() == {0}
    rhs = rng.standard_normal((5, 6))
    sol, rep = plan2.solve(rhs)
    assert rep.periodic_axes == (1,)
    want, _ = orc.solve(orc.Case([(5, 1.0, orc.DIRICHLET, orc.STAGGERED), (6, 2.0, orc.PERIODIC)], orc.FD2), rhs)
    assert orc.relative_l2(sol, want) <= 1e-12
    uniform = fp.SolverPlan(fp.SolverConfig((fp.GridSpec(8, 1.0, BC.NEUMANN, GK.STAGGERED),) * 2, AP.FINITE_DIFFERENCE_2))
    assert uniform._reorder == {}


@pytest.mark.parametrize("kind", [fp.TransformKind.DFT, fp.TransformKind.IDFT])
@pytest.mark.parametrize("n", [2048, 4096])
def test_wide_strided_tiles_fp32_complex(kind, n, torch_cuda, rng):
    # long complex fp32 lines on a strided axis run on the wide-tile kernel
    # (I/O tile twice the 512-thread compute width); also through a solve (c5-like)
    x = (rng.standard_normal((n, 3, 24)) + 1j * rng.standard_normal((n, 3, 24))).astype(np.complex64)
    want = orc.forward_1d(kind.value, x.astype(np.complex128), axis=0)
    got = fp.TransformPlan(kind, n, axis=0).execute(torch_cuda.from_numpy(x).cuda()).cpu().numpy()
    assert np.abs(got - want).max() <= 2e-6 * np.log2(n) * np.abs(want).max()


def test_wide_tiles_in_a_periodic_fp32_solve(torch_cuda, rng):
    case = orc.Case([(2048, orc.TWO_PI, orc.PERIODIC), (2048, orc.TWO_PI, orc.PERIODIC), (16, orc.TWO_PI, orc.PERIODIC)],
                    orc.SPECTRAL, "single")
    grids = tuple(fp.GridSpec(a.n, a.length, fp.BoundaryCondition(a.bc), fp.GridKind(a.kind)) for a in case.axes)
    plan = fp.SolverPlan(fp.SolverConfig(grids, fp.Approximation(case.approx), case.precision))
    rhs = rng.standard_normal(case.shape).astype(np.float32)
    rhs -= rhs.mean(dtype=np.float64)
    got, rep = plan.solve(torch_cuda.from_numpy(rhs).cuda())
    want, rm = orc.solve(case, rhs.astype(np.float64))
    assert orc.relative_l2(got.cpu().numpy(), want) <= 1e-5
