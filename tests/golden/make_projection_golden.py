"""Golden vectors of the projection step, produced by the REFERENCE flow module.

Run in the build container (where /root/reference exists):

    python tests/golden/make_projection_golden.py

For seeded predictor velocities it runs exactly the reference stage
(flow.py:290-295): ``rhs = divergence(star) / scale``, ``phi, _ =
flow.poisson.solve(rhs)``, ``gradient(vel, phi)`` and the velocity update, for
a periodic (Taylor-Green geometry) and a walled (channel geometry) case, and
writes ``projection_v1.npz``.  Nothing at test time reads /root/reference.
"""

import sys
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent

CASES = {
    "periodic": dict(cells=(64, 32), lengths=(2 * np.pi, 2 * np.pi), z_walls=False, scale=0.35 * 0.01),
    "walls": dict(cells=(48, 32), lengths=(3.0, 1.0), z_walls=True, scale=0.5 * 0.02),
    "walls_dense": dict(cells=(32, 24), lengths=(2.0, 1.5), z_walls=True, scale=0.04),
}


def main():
    sys.path.insert(0, REF_SRC)
    from fastpoisson import flow

    rng = np.random.default_rng(20261020)
    out = {}
    for name, c in CASES.items():
        nx, nz = c["cells"]
        wshape = (nx, nz + 1) if c["z_walls"] else (nx, nz)
        ustar = rng.standard_normal((nx, nz))
        wstar = rng.standard_normal(wshape)
        if c["z_walls"]:
            wstar[:, 0] = 0.0
            wstar[:, -1] = 0.0
        vel = flow.StaggeredVelocity(ustar.copy(), wstar.copy(), c["lengths"], 0.0, c["z_walls"])
        fl = flow.ProjectionFlow(vel)
        star = flow.StaggeredVelocity(ustar, wstar, vel.lengths, vel.nu, vel.z_walls)
        rhs = flow.divergence(star) / c["scale"]
        phi, _ = fl.poisson.solve(rhs)
        gfx, gfz = flow.gradient(vel, phi)
        u = ustar - c["scale"] * gfx
        w = wstar - c["scale"] * gfz
        for k, v in dict(ustar=ustar, wstar=wstar, rhs=rhs, phi=phi, u=u, w=w).items():
            out[f"{name}/{k}"] = v
        out[f"{name}/meta"] = np.array([nx, nz, c["lengths"][0], c["lengths"][1], float(c["z_walls"]), c["scale"]])
    np.savez_compressed(HERE / "projection_v1.npz", **out)
    print("wrote", HERE / "projection_v1.npz", len(out), "arrays")


if __name__ == "__main__":
    main()
