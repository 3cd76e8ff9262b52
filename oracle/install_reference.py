"""Install the UNMODIFIED reference package for the CPU baseline arm and stage its tests.

    python oracle/install_reference.py

Test / bench infrastructure only (bench.py --impl reference, cpu_baseline,
tools/run_reference_suite.py) -- nothing on the product path imports it.

* `baseline/_ref/`      <- `pip install --no-index --no-build-isolation --no-deps --target`
                           of a scratch copy of /root/reference/pkg (the source tree is
                           read-only; --no-deps because the offline wheelhouse has no numpy
                           wheel -- the image's numpy / scipy serve it)
* `baseline/_reftests/` <- /root/reference/pkg/tests, unmodified

Both directories are git-ignored (no reference sources in history) but travel to the
GPU box with the snapshot.  A no-op when /root/reference is absent (the GPU box).
"""

from __future__ import annotations

import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REFERENCE = Path("/root/reference/pkg")
TARGET = ROOT / "baseline" / "_ref"
TESTS = ROOT / "baseline" / "_reftests"


def install(force: bool = False) -> bool:
    if not REFERENCE.exists():
        return False
    if force or not (TARGET / "fastpoisson" / "solver.py").exists():
        with tempfile.TemporaryDirectory(prefix="fp_ref_") as tmp:
            src = Path(tmp) / "pkg"
            shutil.copytree(REFERENCE, src)
            if TARGET.exists():
                shutil.rmtree(TARGET)
            TARGET.mkdir(parents=True)
            cmd = [sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation", "--no-deps",
                   "--find-links", "/opt/wheelhouse", "--target", str(TARGET), str(src)]
            proc = subprocess.run(cmd, capture_output=True, text=True)
            if proc.returncode != 0:
                raise RuntimeError(f"reference install failed:\n{proc.stdout}\n{proc.stderr}")
    if force or not TESTS.exists():
        if TESTS.exists():
            shutil.rmtree(TESTS)
        shutil.copytree(REFERENCE / "tests", TESTS)
    return True


if __name__ == "__main__":
    print("installed" if install(force="--force" in sys.argv) else "no /root/reference here: nothing to do")
