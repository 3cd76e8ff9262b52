"""Build the in-tree shared library ``lib/libfastpoisson_b200.so`` with nvcc.

The library is plain C ABI (include/fastpoisson_b200.h) over sm_100a kernels;
it links the CUDA runtime statically so it loads without a GPU (symbol checks
in the CPU test tier) and travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB_DIR = PKG / "lib"
LIB_PATH = LIB_DIR / "libfastpoisson_b200.so"

SOURCES = [f"fp_fft_{t}_l{g}.cu" for t in ("d", "f") for g in (4, 6, 8, 9, 11, 12)] + [
    "fp_kernels.cu", "fp_mr.cu", "fp_blue.cu", "fp_tma.cu", "fp_plan.cu", "fp_tables.cpp"]
HEADERS = ["fp_types.h", "fp_tables.h", "fp_common.cuh", "fp_fft.cuh", "fp_tma.cuh", "fp_attr.h"]
OBJ_DIR = PKG / "build"

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMPILE_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden"]
LINK_FLAGS = ["-shared", "-cudart", "static"]


def nvcc_path() -> str:
    cand = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(cand):
        raise RuntimeError("nvcc not found: cannot build the sm_100a extension")
    return cand


def _inputs():
    files = [CSRC / s for s in SOURCES] + [CSRC / h for h in HEADERS]
    files.append(ROOT / "include" / "fastpoisson_b200.h")
    return files


def is_stale() -> bool:
    if not LIB_PATH.exists():
        return True
    t = LIB_PATH.stat().st_mtime
    return any(f.stat().st_mtime > t for f in _inputs())


def build(force: bool = False, verbose: bool = False, extra_flags=(), lib_path=None) -> Path:
    """Compile the library if missing or older than its sources (one nvcc per
    translation unit, in parallel, then one link).  ``extra_flags`` / ``lib_path``
    build a variant library elsewhere (A/B benchmarks, tools/build_variant.py)."""
    if lib_path is None and not extra_flags and not force and not is_stale():
        return LIB_PATH
    lib_out = Path(lib_path) if lib_path is not None else LIB_PATH
    obj_dir = OBJ_DIR if lib_path is None else lib_out.parent / (lib_out.stem + "_obj")
    from concurrent.futures import ThreadPoolExecutor

    lib_out.parent.mkdir(parents=True, exist_ok=True)
    obj_dir.mkdir(parents=True, exist_ok=True)
    nvcc = nvcc_path()

    def compile_one(src):
        obj = obj_dir / (src + ".o")
        cmd = [nvcc, *ARCH_FLAGS, *COMPILE_FLAGS, *extra_flags, "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        proc = subprocess.run(cmd, capture_output=True, text=True)
        if proc.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src} ({proc.returncode}):\n{proc.stdout}\n{proc.stderr}")
        return obj

    workers = max(1, min(len(SOURCES), os.cpu_count() or 1))
    with ThreadPoolExecutor(max_workers=workers) as pool:
        objs = list(pool.map(compile_one, SOURCES))
    tmp = lib_out.with_suffix(".so.tmp")
    cmd = [nvcc, *ARCH_FLAGS, *LINK_FLAGS, "-o", str(tmp), *map(str, objs)]
    if verbose:
        print(" ".join(cmd), flush=True)
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"nvcc link failed ({proc.returncode}):\n{proc.stdout}\n{proc.stderr}")
    os.replace(tmp, lib_out)
    return lib_out


TORCH_EXT_SRC = CSRC / "fp_torch_ext.cpp"
TORCH_EXT_PATH = LIB_DIR / "fastpoisson_b200_torch.so"


def torch_ext_is_stale() -> bool:
    return (not TORCH_EXT_PATH.exists()) or TORCH_EXT_SRC.stat().st_mtime > TORCH_EXT_PATH.stat().st_mtime


def build_torch_ext(force: bool = False, verbose: bool = False) -> Path:
    """Compile the PyTorch extension in front of the C ABI (csrc/fp_torch_ext.cpp) into
    ``lib/fastpoisson_b200_torch.so`` (in-tree: it travels with the kernel library).  It is
    host C++ only -- it takes tensors, reads the current stream and calls fp_solve through
    the address Python binds -- so it links libtorch but not the kernel library."""
    if not force and not torch_ext_is_stale():
        return TORCH_EXT_PATH
    import sys

    bdir = OBJ_DIR / "torch_ext"
    bdir.mkdir(parents=True, exist_ok=True)
    LIB_DIR.mkdir(parents=True, exist_ok=True)
    name = "fastpoisson_b200_torch"
    # in a child process: cpp_extension.load also LOADS what it built, and a second copy of the
    # same TORCH_LIBRARY (lib/..., loaded by _native.torch_ext) in one process aborts
    code = (
        "from torch.utils import cpp_extension\n"
        f"cpp_extension.load(name={name!r}, sources=[{str(TORCH_EXT_SRC)!r}], build_directory={str(bdir)!r}, "
        f"extra_cflags=['-O2'], with_cuda=True, is_python_module=False, verbose={bool(verbose)!r})\n"
    )
    proc = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    if verbose:
        print(proc.stdout, proc.stderr, flush=True)
    if proc.returncode != 0:
        raise RuntimeError(f"torch extension build failed ({proc.returncode}):\n{proc.stdout}\n{proc.stderr}")
    built = bdir / f"{name}.so"
    if not built.exists():
        raise RuntimeError(f"torch extension build produced no {built}")
    tmp = TORCH_EXT_PATH.with_suffix(".so.tmp")
    shutil.copyfile(built, tmp)
    os.replace(tmp, TORCH_EXT_PATH)
    return TORCH_EXT_PATH


if __name__ == "__main__":  # pragma: no cover
    print(build(force=True, verbose=True))
    print(build_torch_ext(force=True, verbose=True))
