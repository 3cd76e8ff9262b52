"""Run the REFERENCE's own test suite against this package.

    python tools/run_reference_suite.py [pytest args...]

The reference tests (`/root/reference/pkg/tests`, staged unmodified into the
git-ignored `baseline/_reftests/` so they travel to the GPU box) import
`fastpoisson.<module>`.  A shim package named `fastpoisson` maps every module this
package re-implements (grid, solver, transforms, eigenvalues, field, fieldio, cli)
onto `paper_1409_8116_b200.*`, so those tests drive the GPU solve path.  Modules
outside the hot path -- the reference's test utilities and consumers (verify,
flow, reorder) -- are loaded from the unmodified reference package in
`baseline/_ref/fastpoisson`, as submodules of the shim: their relative imports
(`from .solver import SolverPlan`) resolve to this package too.
"""

import os
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF_PKG = ROOT / "baseline" / "_ref" / "fastpoisson"
REF_TESTS = ROOT / "baseline" / "_reftests"
MAPPED = ("grid", "solver", "transforms", "eigenvalues", "field", "fieldio", "cli")

SHIM = '''
import importlib as _il
import sys as _sys

import paper_1409_8116_b200 as _pkg
from paper_1409_8116_b200 import *  # noqa: F401,F403

for _m in {mapped!r}:
    _sys.modules[__name__ + "." + _m] = _il.import_module("paper_1409_8116_b200." + _m)
    globals()[_m] = _sys.modules[__name__ + "." + _m]
# verify / flow / reorder: the reference's own files, found through __path__
__path__.append({ref!r})
__version__ = getattr(_pkg, "__version__", "0.1.0")
'''


def main(argv):
    if not REF_TESTS.exists() or not REF_PKG.exists():
        print("reference tests or package not staged (baseline/_reftests, baseline/_ref)", file=sys.stderr)
        return 2
    shim_root = Path(tempfile.mkdtemp(prefix="fp_shim_"))
    (shim_root / "fastpoisson").mkdir()
    (shim_root / "fastpoisson" / "__init__.py").write_text(SHIM.format(mapped=MAPPED, ref=str(REF_PKG)))
    sys.path[:0] = [str(shim_root), str(ROOT), str(REF_TESTS)]
    os.environ["PYTHONPATH"] = os.pathsep.join([str(shim_root), str(ROOT), str(REF_TESTS), os.environ.get("PYTHONPATH", "")])
    import pytest

    import fastpoisson

    assert fastpoisson.solver.__name__ == "paper_1409_8116_b200.solver", fastpoisson.solver
    return pytest.main([str(REF_TESTS), "-p", "no:cacheprovider", "--rootdir", str(REF_TESTS), *argv])


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
