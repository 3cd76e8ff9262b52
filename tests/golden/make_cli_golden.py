"""Field files and CLI outputs produced by the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_cli_golden.py

Writes, under ``tests/golden/cli_v1/``:
  * ``rhs.json/.bin`` (fp64, 2D, with grids) and ``rhs32.json/.bin`` (fp32, 1D,
    no grids) via the reference's ``fieldio.write_field`` (fieldio.py:49-75);
  * ``ref_run/`` = the reference's ``fastpoisson solve --in rhs.json --out ref_run``
    (cli.py:175-225): ``solution.json/.bin`` and ``report.json`` (the manifest
    carries a timestamp and absolute paths, so only its key set is pinned in the
    tests).
Nothing at test time reads /root/reference -- only these committed files.
"""

import sys
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent / "cli_v1"


def main():
    sys.path.insert(0, REF_SRC)
    from fastpoisson.cli import main as ref_main
    from fastpoisson.fieldio import write_field
    from fastpoisson.grid import BoundaryCondition as BC, GridKind as GK, GridSpec

    rng = np.random.default_rng(1409)
    grids = (GridSpec(12, 1.0, BC.NEUMANN, GK.STAGGERED), GridSpec(10, 2.0, BC.NEUMANN, GK.STAGGERED))
    HERE.mkdir(parents=True, exist_ok=True)
    np.save(HERE / "rhs_values.npy", rng.standard_normal((12, 10)))
    rhs = np.load(HERE / "rhs_values.npy")
    write_field(HERE / "rhs", rhs, grids)
    write_field(HERE / "rhs32", rng.standard_normal(16).astype(np.float32))
    code = ref_main(["solve", "--in", str(HERE / "rhs.json"), "--out", str(HERE / "ref_run")])
    assert code == 0, code
    (HERE / "ref_run" / "manifest.json").unlink()   # timestamp + absolute paths
    print("wrote", sorted(p.name for p in HERE.rglob("*")))


if __name__ == "__main__":
    main()
