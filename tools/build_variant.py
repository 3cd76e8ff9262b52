"""Build a variant of the native library with extra nvcc flags (A/B benchmarks).

    python tools/build_variant.py variants/tw2f64 -DFP_TW2_F64=1
    FP_NATIVE_LIB=variants/tw2f64/libfastpoisson_b200.so python bench.py ...
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1409_8116_b200 import _build  # noqa: E402

out = Path(sys.argv[1]) / "libfastpoisson_b200.so"
print(_build.build(force=True, extra_flags=tuple(sys.argv[2:]), lib_path=out))
