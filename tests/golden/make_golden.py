"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``fastpoisson`` from /root/reference/pkg/src, runs
``SolverPlan(config).solve(rhs)`` and ``TransformPlan.execute_*`` on seeded
inputs, and writes ``golden_v1.npz`` + ``golden_v1.json`` next to this file.
Small cases store full arrays; cases at BASELINE-config shapes store the seed,
input fingerprints and a strided sample of the solution.  Nothing at test
time reads /root/reference -- only these committed fixtures.
"""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent
SAMPLE_STRIDE = 97


def axes_json(grids):
    return [[g.n, g.length, g.bc.value, g.kind.value] for g in grids]


def main():
    sys.path.insert(0, REF_SRC)
    import fastpoisson as ref
    from fastpoisson.grid import BoundaryCondition as BC, GridKind as GK, Approximation as AP

    rows = [(BC.PERIODIC, GK.REGULAR), (BC.DIRICHLET, GK.REGULAR), (BC.DIRICHLET, GK.STAGGERED),
            (BC.NEUMANN, GK.REGULAR), (BC.NEUMANN, GK.STAGGERED)]
    arrays = {}
    meta = {"reference": "fastpoisson " + ref.__version__, "numpy": np.__version__,
            "sample_stride": SAMPLE_STRIDE, "solves": [], "transforms": []}
    import scipy

    meta["scipy"] = scipy.__version__

    def add_solve(cid, grids, approx, precision, rhs, sampled=False, seed=None, gen=None):
        cfg = ref.SolverConfig(tuple(grids), approx, precision)
        plan = ref.SolverPlan(cfg)
        sol, rep = plan.solve(rhs)
        entry = {"id": cid, "axes": axes_json(grids), "approx": approx.value, "precision": precision,
                 "removed_mean": rep.removed_mean, "mode": rep.mode, "periodic_axes": list(rep.periodic_axes),
                 "sampled": sampled, "shape": list(rhs.shape),
                 "rhs_sum": float(np.sum(rhs, dtype=np.float64)),
                 "rhs_sumsq": float(np.sum(np.square(rhs, dtype=np.float64))),
                 "sol_norm": float(np.linalg.norm(sol.astype(np.float64).ravel())),
                 "sol_sum": float(np.sum(sol, dtype=np.float64))}
        if sampled:
            entry["seed"] = seed
            entry["generator"] = gen
            arrays[f"{cid}/sol_sample"] = sol.ravel()[::SAMPLE_STRIDE].copy()
        else:
            arrays[f"{cid}/rhs"] = rhs
            arrays[f"{cid}/sol"] = sol
        meta["solves"].append(entry)

    rng = np.random.default_rng(20240901)
    k = 0
    # small cases on every row, both approximations (dense engine + odd sizes)
    for bc, kind in rows:
        for shape in [(1,), (2,), (7,), (8,), (5, 4), (8, 8), (4, 7), (6, 5, 4), (3, 1, 2)]:
            if bc is BC.NEUMANN and kind is GK.REGULAR and min(shape) < 2:
                continue
            for approx in (AP.FINITE_DIFFERENCE_2, AP.PSEUDO_SPECTRAL):
                lengths = [1.0 + 0.5 * i for i in range(len(shape))]
                grids = [ref.GridSpec(n, L, bc, kind) for n, L in zip(shape, lengths)]
                rhs = rng.standard_normal(shape)
                add_solve(f"s{k:03d}", grids, approx, "double", rhs)
                k += 1
    # power-of-two cases that run on the GPU FFT engine (rows with FFT kernels)
    fft_rows = [(BC.PERIODIC, GK.REGULAR), (BC.DIRICHLET, GK.STAGGERED), (BC.NEUMANN, GK.STAGGERED)]
    for bc, kind in fft_rows:
        for shape in [(64,), (32, 64), (64, 32), (32, 32, 32), (16, 32, 32)]:
            approxes = (AP.FINITE_DIFFERENCE_2, AP.PSEUDO_SPECTRAL) if len(shape) < 3 else (AP.FINITE_DIFFERENCE_2,)
            for approx in approxes:
                lengths = [1.0 + 0.5 * i for i in range(len(shape))]
                grids = [ref.GridSpec(n, L, bc, kind) for n, L in zip(shape, lengths)]
                rhs = rng.standard_normal(shape)
                add_solve(f"p{k:03d}", grids, approx, "double", rhs)
                k += 1
    # mixed periodic + wall configurations, including permuted axis roles
    P = ref.GridSpec
    mixed = [
        [P(32, 2.0, BC.PERIODIC), P(32, 2.0, BC.PERIODIC), P(16, 1.0, BC.NEUMANN, GK.STAGGERED)],
        [P(32, 2.0, BC.PERIODIC), P(32, 1.0, BC.DIRICHLET, GK.STAGGERED)],
        [P(32, 1.0, BC.DIRICHLET, GK.STAGGERED), P(64, 2.0, BC.PERIODIC)],
        [P(6, 1.0, BC.PERIODIC), P(5, 1.5, BC.NEUMANN, GK.STAGGERED), P(4, 2.0, BC.NEUMANN, GK.STAGGERED)],
        [P(8, 2.0, BC.PERIODIC), P(6, 1.0, BC.DIRICHLET, GK.REGULAR)],
        [P(32, 1.0, BC.NEUMANN, GK.STAGGERED), P(32, 2.0, BC.PERIODIC), P(16, 2.0, BC.PERIODIC)],
        [P(10, 2.0, BC.PERIODIC), P(7, 1.0, BC.DIRICHLET, GK.STAGGERED)],
    ]
    for grids in mixed:
        for approx in (AP.FINITE_DIFFERENCE_2, AP.PSEUDO_SPECTRAL):
            shape = tuple(g.n for g in grids)
            rhs = rng.standard_normal(shape)
            add_solve(f"m{k:03d}", grids, approx, "double", rhs)
            k += 1
    # single precision
    for bc, kind in rows:
        grids = [P(32, 1.0, bc, kind), P(16, 1.5, bc, kind)]
        rhs = rng.standard_normal((32, 16)).astype(np.float32)
        add_solve(f"f{k:03d}", grids, AP.FINITE_DIFFERENCE_2, "single", rhs)
        k += 1

    # BASELINE configs: c1 at full size, the others scaled down (sampled outputs)
    sys.path.insert(0, str(HERE.parents[1]))
    from oracle import fastpoisson_oracle as orc

    def ref_grids(case):
        return [P(a.n, a.length, BC(a.bc), GK(a.kind)) for a in case.axes]

    for name, scale in [("c1", 1), ("c2", 16), ("c3", 8), ("c4", 16), ("c5", 32)]:
        case = orc.config_case(name, scale)
        rhs = orc.config_rhs(name, case, seed=0)
        approx = AP(case.approx)
        add_solve(f"{name}_div{scale}", ref_grids(case), approx, case.precision, rhs,
                  sampled=True, seed=0, gen=name)
        meta["solves"][-1]["scale"] = scale

    # transforms: every kind, lengths covering dense and FFT engines
    tk = ref.TransformKind
    for kind in tk:
        for n in [1, 2, 3, 4, 5, 7, 8, 16, 17, 31, 32, 64, 127, 128, 257, 512]:
            if kind is tk.DCT1 and n < 2:
                continue
            x = rng.standard_normal(n)
            if kind.is_complex:
                x = x + 1j * rng.standard_normal(n)
            plan = ref.TransformPlan(kind, n)
            y = plan.execute(x)
            tid = f"t_{kind.value}_{n}"
            arrays[f"{tid}/x"] = x
            arrays[f"{tid}/y"] = y
            entry = {"id": tid, "kind": kind.value, "n": n}
            if n <= 64:
                arrays[f"{tid}/naive"] = ref.naive_transform(kind, x)
            meta["transforms"].append(entry)

    np.savez_compressed(HERE / "golden_v1.npz", **arrays)
    (HERE / "golden_v1.json").write_text(json.dumps(meta, indent=1))
    size = (HERE / "golden_v1.npz").stat().st_size
    print(f"wrote {len(meta['solves'])} solve cases, {len(meta['transforms'])} transform cases, {size/1e6:.2f} MB")


if __name__ == "__main__":
    main()
