"""Fused projection step vs the unfused sequence (torch divergence -> SolverPlan solve ->
torch gradient / updates), device-resident, CUDA events.

    python tools/time_projection.py --cells 4096,4096 [--walls]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_1409_8116_b200 as fp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cells", default="4096,4096")
ap.add_argument("--walls", action="store_true")
ap.add_argument("--steps", type=int, default=10)
a = ap.parse_args()
nx, nz = (int(x) for x in a.cells.split(","))
L = (2.0, 1.0)
dx, dz = L[0] / nx, L[1] / nz
step = fp.ProjectionStep((nx, nz), L, z_walls=a.walls)
plan = step.plan
u = torch.randn(nx, nz, dtype=torch.float64, device="cuda")
w = torch.randn(nx, nz + 1 if a.walls else nz, dtype=torch.float64, device="cuda")
if a.walls:
    w[:, 0] = 0
    w[:, -1] = 0
p = torch.zeros(nx, nz, dtype=torch.float64, device="cuda")
scale = 0.01
uo, wo, phi = torch.empty_like(u), torch.empty_like(w), torch.empty_like(p)


def fused():
    step.project(u, w, scale, p=p, u_out=uo, w_out=wo, phi_out=phi)


def unfused():
    div = (torch.roll(u, -1, 0) - u) / dx
    div += ((w[:, 1:] - w[:, :-1]) if a.walls else (torch.roll(w, -1, 1) - w)) / dz
    ph, _ = plan.solve(div / scale)
    gx = (ph - torch.roll(ph, 1, 0)) / dx
    if a.walls:
        gz = torch.zeros_like(w)
        gz[:, 1:-1] = (ph[:, 1:] - ph[:, :-1]) / dz
    else:
        gz = (ph - torch.roll(ph, 1, 1)) / dz
    uo.copy_(u - scale * gx)
    wo.copy_(w - scale * gz)
    p.add_(ph)


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.steps


tf, tu = timed(fused), timed(unfused)
print(json.dumps({"cells": [nx, nz], "walls": a.walls, "fused_ms": round(tf, 4), "unfused_ms": round(tu, 4),
                  "speedup": round(tu / tf, 2)}))
