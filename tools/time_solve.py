"""Device-resident solve time for an arbitrary configuration (A/B helper).

    python tools/time_solve.py --axes 513:1:neumann:regular,513:1:neumann:regular,513:1:neumann:regular
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_1409_8116_b200 as fp  # noqa: E402
from paper_1409_8116_b200.grid import Approximation as AP, BoundaryCondition as BC, GridKind as GK  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--axes", required=True)
ap.add_argument("--approx", default="fd2")
ap.add_argument("--precision", default="double")
ap.add_argument("--steps", type=int, default=10)
a = ap.parse_args()
grids = []
for spec in a.axes.split(","):
    n, L, bc, kind = spec.split(":")
    grids.append(fp.GridSpec(int(n), float(L), BC(bc), GK(kind)))
cfg = fp.SolverConfig(tuple(grids), AP(a.approx), a.precision)
plan = fp.SolverPlan(cfg)
dt = torch.float32 if a.precision == "single" else torch.float64
rhs = torch.randn(cfg.shape, dtype=dt, device="cuda")
out = torch.empty_like(rhs)
for _ in range(3):
    plan.solve(rhs, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
keep = []
e0.record()
for _ in range(a.steps):
    keep.append(plan.solve_async(rhs, out))   # (out, info, workspace): alive until the sync
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.steps
print(json.dumps({"axes": a.axes, "ms": round(ms, 4), "passes": plan.num_passes,
                  "fft_axes_mask": int(plan._info.fft_axes_mask)}))
