"""CPU tier: pin the oracle against the reference's own outputs and known answers.

The golden vectors (tests/golden/make_golden.py) were produced by running the
reference package itself; the known answers below are the ones the reference
tests hold (test_transforms.py:55-94, test_verify.py:28-33, test_solver.py:108-146).
"""

import math

import numpy as np
import pytest

from oracle import fastpoisson_oracle as orc


def case_of(entry):
    return orc.Case([tuple(a) for a in entry["axes"]], entry["approx"], entry["precision"])


def test_golden_solves_match_oracle(golden):
    meta, arrays = golden
    checked = 0
    for e in meta["solves"]:
        if e["sampled"]:
            continue
        case = case_of(e)
        rhs = arrays[f"{e['id']}/rhs"]
        want = arrays[f"{e['id']}/sol"]
        got, rm = orc.solve(case, rhs)
        tol = 1e-6 if case.precision == "single" else 1e-13
        scale = max(np.abs(want).max(), 1e-30)
        assert np.abs(got - want).max() <= tol * scale, e["id"]
        assert rm == pytest.approx(e["removed_mean"], abs=1e-13 if case.precision == "double" else 1e-6)
        checked += 1
    assert checked > 100


def test_golden_sampled_configs_match_oracle(golden):
    meta, arrays = golden
    stride = meta["sample_stride"]
    for e in meta["solves"]:
        if not e["sampled"]:
            continue
        case = orc.config_case(e["generator"], e["scale"])
        rhs = orc.config_rhs(e["generator"], case, seed=e["seed"])
        # the generator still produces the same field as when the goldens were made
        assert float(np.sum(rhs, dtype=np.float64)) == pytest.approx(e["rhs_sum"], abs=1e-9)
        assert float(np.sum(np.square(rhs, dtype=np.float64))) == pytest.approx(e["rhs_sumsq"], rel=1e-12)
        got, rm = orc.solve(case, rhs)
        want = arrays[f"{e['id']}/sol_sample"]
        tol = 1e-6 if case.precision == "single" else 1e-12
        assert orc.relative_l2(got.ravel()[::stride], want) <= tol, e["id"]
        assert rm == pytest.approx(e["removed_mean"], abs=1e-12 if case.precision == "double" else 1e-6)


def test_golden_transforms_match_oracle(golden):
    meta, arrays = golden
    for e in meta["transforms"]:
        x = arrays[f"{e['id']}/x"]
        y = arrays[f"{e['id']}/y"]
        got = orc.forward_1d(e["kind"], x)
        assert np.abs(got - y).max() <= 1e-12 * e["n"] * max(np.abs(x).max(), 1.0), e["id"]
        if f"{e['id']}/naive" in arrays:
            nv = orc.naive_transform(e["kind"], x)
            assert np.abs(nv - arrays[f"{e['id']}/naive"]).max() <= 1e-12 * e["n"]
            assert np.abs(nv - y).max() <= 1e-11 * e["n"] * max(np.abs(x).max(), 1.0)


@pytest.mark.parametrize("n", [8, 16, 64, 512, 4096, 60, 250, 1000, 2046])
def test_makhoul_recipes_match_scipy(n, rng):
    # the half-length FFT recipes the GPU kernels implement (FFT engine at 2^k, and the
    # mixed-radix engine's half-length path at any even n)
    x = rng.standard_normal((3, n))
    np.testing.assert_allclose(orc.makhoul_dct2(x), orc.forward_1d("dct2", x), atol=1e-12 * n)
    np.testing.assert_allclose(orc.makhoul_dct3(x), orc.forward_1d("dct3", x), atol=1e-12 * n)
    s = (-1.0) ** np.arange(n)
    np.testing.assert_allclose(orc.makhoul_dct2(s * x)[..., ::-1], orc.forward_1d("dst2", x), atol=1e-12 * n)
    np.testing.assert_allclose(s * orc.makhoul_dct3(x[..., ::-1]), orc.forward_1d("dst3", x), atol=1e-12 * n)


@pytest.mark.parametrize("M", [16, 32, 256])
def test_regular_grid_recipes_match_scipy(M, rng):
    # DCT-I / DST-I via the real FFT of the extension (the FFT-engine recipe for
    # regular grids) against scipy's type-1 transforms, forward and inverse legs
    for kind, n in (("dct1", M + 1), ("dst1", M - 1)):
        x = rng.standard_normal((3, n))
        want = orc.forward_1d(kind, x)
        np.testing.assert_allclose(orc.r1_via_rfft(x, kind), want, atol=1e-12 * n)
        np.testing.assert_allclose(orc.r1_inverse_via_irfft(x, kind), want, atol=1e-12 * n)


@pytest.mark.parametrize("n", [16, 45, 48, 77, 99, 125, 243, 1000, 1001, 2046])
def test_mixed_radix_recipes_match_scipy(n, rng):
    # the mixed-radix engine's algorithm (digit-reversed scatter + in-place DIT
    # stages; Makhoul / extension recipes at any parity) against scipy.fft, and
    # against the reference's own golden transforms where the length matches
    x = rng.standard_normal((3, n))
    c = x + 1j * rng.standard_normal((3, n))
    for kind in ("dct1", "dct2", "dct3", "dst1", "dst2", "dst3", "dft", "idft"):
        N = {"dct1": 2 * (n - 1), "dst1": 2 * (n + 1)}.get(kind, n)
        xx = c if kind in ("dft", "idft") else x
        if not orc.mr_factors(N):
            with pytest.raises(ValueError):
                orc.mr_transform(kind, xx)
            continue
        want = orc.forward_1d(kind, xx)
        np.testing.assert_allclose(orc.mr_transform(kind, xx), want, atol=1e-13 * n * np.abs(want).max())


@pytest.mark.parametrize("n", [2, 3, 16, 67, 97, 131, 250, 1009])
def test_bluestein_recipes_match_scipy(n, rng):
    # the Bluestein engine's algorithm (fp_blue.cu: chirp, zero-padded cyclic convolution of
    # power-of-two length, the same recipes as the mixed-radix engine) against scipy.fft at
    # lengths with large prime factors, plus the real FFT and its inverse (plan kinds 100/101)
    x = rng.standard_normal((3, n))
    c = x + 1j * rng.standard_normal((3, n))
    for kind in ("dct1", "dct2", "dct3", "dst1", "dst2", "dst3", "dft", "idft"):
        if kind == "dct1" and n < 2:
            continue
        xx = c if kind in ("dft", "idft") else x
        want = orc.forward_1d(kind, xx)
        np.testing.assert_allclose(orc.blue_transform(kind, xx), want, atol=1e-13 * n * np.abs(want).max())
    want = np.fft.rfft(x)
    np.testing.assert_allclose(orc.blue_transform("rfft", x), want, atol=1e-13 * n * np.abs(want).max())
    X = np.fft.rfft(x)
    np.testing.assert_allclose(orc.blue_irfft(X, n), n * np.fft.irfft(X, n), atol=1e-12 * n * np.abs(x).max())


def test_bluestein_matches_golden_transforms(golden):
    meta, arrays = golden
    seen = 0
    for e in meta["transforms"]:
        n = e["n"]
        if n < 2:
            continue
        x = arrays[f"{e['id']}/x"]
        y = arrays[f"{e['id']}/y"]
        assert np.abs(orc.blue_transform(e["kind"], x) - y).max() <= 1e-12 * n * max(np.abs(x).max(), 1.0), e["id"]
        seen += 1
    assert seen > 50


def test_mixed_radix_matches_golden_transforms(golden):
    meta, arrays = golden
    seen = 0
    for e in meta["transforms"]:
        n = e["n"]
        N = {"dct1": 2 * (n - 1), "dst1": 2 * (n + 1)}.get(e["kind"], n)
        if n < 2 or not orc.mr_factors(N):
            continue
        x = arrays[f"{e['id']}/x"]
        y = arrays[f"{e['id']}/y"]
        assert np.abs(orc.mr_transform(e["kind"], x) - y).max() <= 1e-12 * n * max(np.abs(x).max(), 1.0), e["id"]
        seen += 1
    assert seen > 20


def test_known_answers_transforms():
    # reference tests/test_transforms.py:55-94
    np.testing.assert_allclose(orc.forward_1d("dst1", np.array([1.0, 0.0])), [math.sqrt(3), math.sqrt(3)], atol=1e-14)
    for n in (2, 3, 8, 17):
        out = orc.forward_1d("dct2", np.ones(n))
        assert out[0] == pytest.approx(2.0 * n)
        assert np.abs(out[1:]).max() <= 1e-12
    np.testing.assert_allclose(orc.forward_1d("dst3", np.array([1.0, 0.0])), [2 * math.sin(math.pi / 4), 2 * math.sin(3 * math.pi / 4)], atol=1e-14)
    np.testing.assert_allclose(orc.forward_1d("dct1", np.array([1.0, 2.0])), [3.0, -1.0], atol=1e-14)
    x = np.array([1.0, 2.0, 3.0, 4.0])
    np.testing.assert_allclose(orc.forward_1d("dft", x), np.fft.fft(x) / 4, atol=1e-14)


def test_known_answer_tridiagonal():
    # reference tests/test_verify.py:28-33: Dirichlet regular n=3, dx=1, f=1 -> [-1.5,-2,-1.5]
    case = orc.Case([(3, 4.0, orc.DIRICHLET, orc.REGULAR)], orc.FD2)
    sol, rm = orc.solve(case, np.ones(3))
    np.testing.assert_allclose(orc.laplacian(case, sol), np.ones(3), atol=1e-13)
    np.testing.assert_allclose(sol, [-1.5, -2.0, -1.5], atol=1e-13)
    assert rm == 0.0


def test_constant_neumann_removed_mean():
    # reference tests/test_solver.py:140-146
    case = orc.Case([(6, 1.0, orc.NEUMANN, orc.STAGGERED), (5, 1.5, orc.NEUMANN, orc.STAGGERED)], orc.FD2)
    sol, rm = orc.solve(case, np.full((6, 5), -2.75))
    assert np.abs(sol).max() <= 1e-13
    assert rm == pytest.approx(-2.75, rel=1e-12)


@pytest.mark.parametrize("row", [(orc.PERIODIC, orc.REGULAR), (orc.DIRICHLET, orc.REGULAR),
                                 (orc.DIRICHLET, orc.STAGGERED), (orc.NEUMANN, orc.REGULAR),
                                 (orc.NEUMANN, orc.STAGGERED)])
def test_oracle_matches_dense_fd2(row, rng):
    # verify.py:81-104 dense factorization vs the transform pipeline
    bc, kind = row
    case = orc.Case([(5, 1.0, bc, kind), (4, 1.5, bc, kind)], orc.FD2)
    mat = orc.dense_matrix(case)
    rhs = (mat @ rng.standard_normal(20)).reshape(5, 4)
    sol, _ = orc.solve(case, rhs)
    ref = orc.dense_solve(case, rhs)
    assert np.abs(sol - ref).max() <= 1e-9 * np.abs(ref).max()


def test_config_rhs_compatibility():
    # c4's divergence RHS sums to zero (compatible with the Neumann/periodic null space)
    case = orc.config_case("c4", 16)
    rhs = orc.config_rhs("c4", case)
    assert abs(rhs.sum()) <= 1e-9 * np.abs(rhs).sum()


@pytest.mark.parametrize("name", ["periodic", "walls", "walls_dense"])
def test_projection_oracle_matches_reference_flow(name):
    # fixtures made by the reference flow module (tests/golden/make_projection_golden.py)
    from pathlib import Path

    z = np.load(Path(__file__).resolve().parent / "golden" / "projection_v1.npz")
    nx, nz, lx, lz, walls, scale = z[f"{name}/meta"]
    L = (lx, lz)
    u, w, phi = orc.project_step(z[f"{name}/ustar"], z[f"{name}/wstar"], scale, L, bool(walls))
    for got, key in ((u, "u"), (w, "w"), (phi, "phi")):
        np.testing.assert_allclose(got, z[f"{name}/{key}"], rtol=0, atol=1e-13 * np.abs(z[f"{name}/{key}"]).max())
    assert np.abs(orc.staggered_divergence(u, w, L, bool(walls))).max() <= 1e-10
