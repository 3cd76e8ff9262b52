"""Run a few device-resident solves of one BASELINE config (profiling driver for ncu).

    python tools/one_solve.py --config c5 --repeat 2
"""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_1409_8116_b200 as fp  # noqa: E402
from paper_1409_8116_b200.grid import Approximation as AP, BoundaryCondition as BC, GridKind as GK  # noqa: E402

SHAPES = {
    "c1": ([(64, 6.283185307179586, "periodic", "regular")] * 3, "spectral", "double"),
    "c2": ([(4096, 1.0, "dirichlet", "staggered")] * 2, "fd2", "double"),
    "c3": ([(512, 1.0, "neumann", "staggered")] * 3, "fd2", "double"),
    "c4": ([(1024, 6.283185307179586, "periodic", "regular")] * 2 + [(512, 2.0, "neumann", "staggered")], "fd2", "double"),
    "c5": ([(2048, 6.283185307179586, "periodic", "regular")] * 3, "spectral", "single"),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3", choices=sorted(SHAPES))
    ap.add_argument("--repeat", type=int, default=2)
    a = ap.parse_args()
    axes, approx, prec = SHAPES[a.config]
    grids = tuple(fp.GridSpec(n, L, BC(bc), GK(kind)) for n, L, bc, kind in axes)
    cfg = fp.SolverConfig(grids, AP(approx), prec)
    plan = fp.SolverPlan(cfg)
    dt = torch.float32 if prec == "single" else torch.float64
    rhs = torch.randn(cfg.shape, dtype=dt, device="cuda")
    out = torch.empty_like(rhs)
    for _ in range(a.repeat):
        plan.solve(rhs, out=out)
    torch.cuda.synchronize()
    print("ok", a.config, plan.num_passes)


if __name__ == "__main__":
    main()
