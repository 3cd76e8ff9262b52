"""Small solves / transforms over every kernel family, for compute-sanitizer
(memcheck, racecheck, synccheck, initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py

Covers: FFT-engine contiguous / strided passes and the MID (register path M <= 512,
shared-memory path beyond), in-place solves and strided sub-blocks (aliasing), the
type-I (DCT-I / DST-I) placements, the mixed-radix, dense and Bluestein engines, fp32
(incl. the wide and pipelined strided kernels), the distributed phases emulated on
one device (uneven slabs, real-view MID, exact mean), TransformPlan and the fused
projection step.  Every result is checked against the oracle so a silent corruption
fails too.
"""

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))

import torch  # noqa: E402

import paper_1409_8116_b200 as fp  # noqa: E402
from paper_1409_8116_b200.grid import Approximation as AP, BoundaryCondition as BC, GridKind as GK  # noqa: E402
from oracle import fastpoisson_oracle as orc  # noqa: E402

PI2 = 2 * np.pi
CASES = [
    ("dct3d", [(32, 1.0, "neumann", "staggered"), (32, 1.0, "neumann", "staggered"), (32, 1.0, "neumann", "staggered")], "fd2", "double"),
    ("per3d", [(32, PI2, "periodic", "regular")] * 3, "spectral", "double"),
    ("dst2d_long", [(2048, 1.0, "dirichlet", "staggered"), (64, 1.0, "dirichlet", "staggered")], "fd2", "double"),
    ("mixed3d", [(64, PI2, "periodic", "regular"), (32, PI2, "periodic", "regular"), (32, 2.0, "neumann", "staggered")], "fd2", "double"),
    ("dct1", [(33, 1.0, "neumann", "regular"), (65, 1.0, "neumann", "regular")], "fd2", "double"),
    ("dst1", [(63, 1.0, "dirichlet", "regular"), (31, 1.0, "dirichlet", "regular")], "fd2", "double"),
    ("mr", [(60, 1.0, "neumann", "staggered"), (45, 1.0, "neumann", "staggered"), (100, 1.0, "neumann", "staggered")], "fd2", "double"),
    ("dense", [(67, 1.0, "dirichlet", "staggered"), (40, 1.0, "dirichlet", "staggered")], "fd2", "double"),
    ("blue", [(131, 1.0, "neumann", "staggered"), (64, PI2, "periodic", "regular")], "fd2", "double"),
    ("f32_per", [(64, PI2, "periodic", "regular")] * 3, "spectral", "single"),
    ("f32_long", [(2048, PI2, "periodic", "regular"), (4, PI2, "periodic", "regular"), (2048, PI2, "periodic", "regular")], "spectral", "single"),
]


def config(axes, approx, prec):
    grids = tuple(fp.GridSpec(n, L, BC(bc), GK(kind)) for n, L, bc, kind in axes)
    return fp.SolverConfig(grids, AP(approx), prec)


def check(name, got, want, tol):
    err = orc.relative_l2(np.asarray(got), want)
    status = "ok" if err <= tol else "FAIL"
    print(f"{name:24s} rel L2 {err:.2e} {status}", flush=True)
    return err <= tol


def main():
    rng = np.random.default_rng(11)
    ok = True
    for name, axes, approx, prec in CASES:
        case = orc.Case([tuple(a) for a in axes], approx, prec)
        cfg = config(axes, approx, prec)
        rhs = rng.standard_normal(case.shape)
        if prec == "single":
            rhs = rhs.astype(np.float32)
        want, _ = orc.solve(case, rhs)
        tol = 1e-5 if prec == "single" else 1e-12
        plan = fp.SolverPlan(cfg)
        got, _ = plan.solve(rhs)
        ok &= check(name, got, want, tol)
        # device, in place (out is rhs), and a strided ghost-cell sub-block
        dt = torch.float32 if prec == "single" else torch.float64
        x = torch.from_numpy(np.ascontiguousarray(rhs)).cuda()
        plan.solve(x, out=x)
        ok &= check(name + " in-place", x.cpu().numpy(), want, tol)
        big = torch.zeros(tuple(n + 2 for n in case.shape), dtype=dt, device="cuda")
        inner = tuple(slice(1, -1) for _ in case.shape)
        big[inner] = torch.from_numpy(np.ascontiguousarray(rhs)).cuda()
        out = torch.zeros_like(big)
        plan.solve(big[inner], out=out[inner])
        ok &= check(name + " sub-block", out[inner].cpu().numpy(), want, tol)
    # distributed phases emulated on this device: uneven slabs, real-view MID, exact mean
    from test_gpu_dist import emulate

    for name, axes, approx, P in [
        ("dist c4 P=3", [(64, PI2, "periodic", "regular"), (32, PI2, "periodic", "regular"), (16, 2.0, "neumann", "staggered")], "fd2", 3),
        ("dist wall0 P=2", [(64, 1.0, "neumann", "staggered"), (24, PI2, "periodic", "regular"), (20, PI2, "periodic", "regular")], "fd2", 2),
        ("dist dct1 P=3", [(65, 1.0, "neumann", "regular"), (17, 1.0, "neumann", "regular")], "fd2", 3),
    ]:
        case = orc.Case([tuple(a) for a in axes], approx)
        cfg = config(axes, approx, "double")
        rhs = rng.standard_normal(case.shape)
        rhs -= rhs.mean()
        want, _ = fp.SolverPlan(cfg).solve(rhs)
        got, _, _ = emulate(cfg, P, torch.from_numpy(rhs).cuda())
        ok &= check(name, got.cpu().numpy(), want, 1e-12)
    # TransformPlan on every kind through the three non-power-of-two engines
    for n in (24, 100, 131):
        for kind in fp.TransformKind:
            x = rng.standard_normal((3, n, 5))
            if kind.is_complex:
                x = x + 1j * rng.standard_normal(x.shape)
            want = orc.forward_1d(kind.value, x, axis=1)
            got = fp.TransformPlan(kind, n, axis=1).execute(torch.from_numpy(x).cuda()).cpu().numpy()
            err = np.abs(got - want).max() / np.abs(want).max()
            good = err <= 1e-12
            ok &= good
            print(f"transform {kind.value:5s} n={n:4d} max rel {err:.1e} {'ok' if good else 'FAIL'}", flush=True)
    torch.cuda.synchronize()
    print("ALL OK" if ok else "FAILURES", flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
