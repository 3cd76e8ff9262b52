"""CPU tier: host-side logic of the drop-in API and the C-ABI library surface.

Mirrors the reference's unit tests for configuration handling
(tests/test_grid.py, test_solver.py:55-105, test_transforms.py:22-49,
test_eigenvalues.py) -- everything that does not launch a kernel.
"""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1409_8116_b200 as fp
from paper_1409_8116_b200 import _native
from paper_1409_8116_b200.grid import Approximation as AP, BoundaryCondition as BC, GridKind as GK
from oracle import fastpoisson_oracle as orc

ROOT = Path(__file__).resolve().parents[1]

ROWS = [(BC.PERIODIC, GK.REGULAR), (BC.DIRICHLET, GK.REGULAR), (BC.DIRICHLET, GK.STAGGERED),
        (BC.NEUMANN, GK.REGULAR), (BC.NEUMANN, GK.STAGGERED)]


def test_public_names_match_reference_surface():
    expected = {"Approximation", "BoundaryCondition", "CombinedEigenvalues", "ConfigurationError",
                "EigenvalueTable", "Field", "GridKind", "GridSpec", "SolveReport", "SolverConfig",
                "SolverPlan", "TransformKind", "TransformPair", "TransformPlan", "apply_discrete_laplacian",
                "as_array", "combine_eigenvalues", "eigenvalue_table", "execute_complex", "execute_real",
                "fd2_eigenvalues", "grid_dx", "grid_points", "naive_transform", "plan_create", "solve",
                "solve_mixed", "spectral_eigenvalues", "transform_pair_for", "__version__"}
    assert set(fp.__all__) == expected
    assert fp.__version__ == "0.1.0"
    assert issubclass(fp.ConfigurationError, ValueError)


@pytest.mark.parametrize("bad", [dict(n=0), dict(length=0.0), dict(length=-1.0)])
def test_gridspec_validation(bad):
    kw = dict(n=4, length=1.0, bc=BC.PERIODIC)
    kw.update(bad)
    with pytest.raises(fp.ConfigurationError):
        fp.GridSpec(**kw)


def test_gridspec_rules():
    with pytest.raises(fp.ConfigurationError):
        fp.GridSpec(4, 1.0, BC.PERIODIC, GK.STAGGERED)
    with pytest.raises(fp.ConfigurationError):
        fp.GridSpec(1, 1.0, BC.NEUMANN, GK.REGULAR)
    fp.GridSpec(1, 1.0, BC.DIRICHLET, GK.REGULAR)
    # dx / points against the oracle's restatement of grid.py:80-100
    for bc, kind in ROWS:
        for n in (2, 5, 8):
            g = fp.GridSpec(n, 3.0, bc, kind)
            a = orc.Axis(n, 3.0, bc.value, kind.value)
            assert g.dx == orc.axis_dx(a)
            np.testing.assert_array_equal(g.points(), orc.axis_points(a))
            assert fp.grid_dx(g) == g.dx


@pytest.mark.parametrize("approx", [AP.PSEUDO_SPECTRAL, AP.FINITE_DIFFERENCE_2])
@pytest.mark.parametrize("row", ROWS, ids=["per-reg", "dir-reg", "dir-stag", "neu-reg", "neu-stag"])
def test_eigenvalue_tables_bitwise_match_oracle(row, approx):
    bc, kind = row
    for n in (2, 7, 64, 512):
        g = fp.GridSpec(n, 1.7, bc, kind)
        tab = fp.eigenvalue_table(g, approx)
        np.testing.assert_array_equal(tab.values, orc.eigenvalues(orc.Axis(n, 1.7, bc.value, kind.value), approx.value))
        assert tab.null_indices == (frozenset() if bc is BC.DIRICHLET else frozenset({0}))


def test_transform_pairs_and_scales():
    TK = fp.TransformKind
    assert fp.transform_pair_for(BC.NEUMANN, GK.STAGGERED).backward_scale(6) == 1.0 / 12.0
    assert fp.transform_pair_for(BC.DIRICHLET, GK.REGULAR).backward_scale(5) == 1.0 / 12.0
    assert fp.transform_pair_for(BC.NEUMANN, GK.REGULAR).backward_scale(7) == 1.0 / 12.0
    assert fp.transform_pair_for(BC.PERIODIC, GK.REGULAR).backward_scale(9) == 1.0
    assert (fp.transform_pair_for(BC.DIRICHLET, GK.STAGGERED).forward, fp.transform_pair_for(BC.DIRICHLET, GK.STAGGERED).backward) == (TK.DST2, TK.DST3)
    with pytest.raises(fp.ConfigurationError):
        fp.transform_pair_for(BC.PERIODIC, GK.STAGGERED)
    with pytest.raises(fp.ConfigurationError):
        fp.TransformPlan(TK.DCT1, 1)


def test_naive_transform_matches_oracle(rng):
    for kind in fp.TransformKind:
        for n in (2, 5, 16):
            x = rng.standard_normal(n)
            np.testing.assert_allclose(fp.naive_transform(kind, x), orc.naive_transform(kind.value, x), atol=1e-13)


def test_solver_config_validation():
    g = fp.GridSpec(4, 1.0, BC.PERIODIC)
    with pytest.raises(fp.ConfigurationError):
        fp.SolverConfig((g,) * 4, AP.FINITE_DIFFERENCE_2)
    with pytest.raises(fp.ConfigurationError):
        fp.SolverConfig((), AP.FINITE_DIFFERENCE_2)
    with pytest.raises(fp.ConfigurationError):
        fp.SolverConfig((g,), AP.FINITE_DIFFERENCE_2, precision="half")
    with pytest.raises(fp.ConfigurationError):
        fp.SolverConfig((fp.GridSpec(4, 1.0, BC.DIRICHLET, GK.REGULAR), fp.GridSpec(4, 1.0, BC.NEUMANN, GK.STAGGERED)), AP.FINITE_DIFFERENCE_2)
    with pytest.raises(fp.ConfigurationError):
        fp.SolverConfig((fp.GridSpec(4, 1.0, BC.DIRICHLET, GK.REGULAR), fp.GridSpec(4, 1.0, BC.DIRICHLET, GK.STAGGERED)), AP.FINITE_DIFFERENCE_2)
    per, neu = g, fp.GridSpec(4, 1.0, BC.NEUMANN, GK.STAGGERED)
    c = fp.SolverConfig((fp.GridSpec(4, 1.0, BC.DIRICHLET, GK.STAGGERED), fp.GridSpec(6, 1.0, BC.PERIODIC)), AP.FINITE_DIFFERENCE_2)
    assert c.mode == "mixed" and c.periodic_axes == (1,)
    assert fp.SolverConfig((per, per, neu), AP.FINITE_DIFFERENCE_2).mode == "mixed"
    assert fp.SolverConfig((per, per, per), AP.FINITE_DIFFERENCE_2).mode == "uniform"
    assert fp.SolverConfig((g,), AP.FINITE_DIFFERENCE_2, precision="single").dtype == np.float32
    assert fp.SolverConfig((per, neu), AP.FINITE_DIFFERENCE_2).singular
    assert not c.singular


def test_field_subblock_views():
    parent = np.full((10, 11), 123.0)
    f = fp.Field.subblock(parent, (2, 2), (6, 7))
    assert f.extents == (6, 7) and f.offsets == (2, 2) and f.strides == (11, 1)
    f.data[...] = 1.0
    assert parent[2:8, 2:9].sum() == 42.0 and parent.sum() == 42.0 + 123.0 * (110 - 42)
    with pytest.raises(ValueError):
        fp.Field.subblock(parent, (5, 5), (6, 7))
    with pytest.raises(TypeError):
        fp.Field((3, 3), dtype=np.int32)
    with pytest.raises(ValueError):
        fp.Field((1, 1, 1, 1))


# -- C ABI -----------------------------------------------------------------------
def _header_symbols():
    text = (ROOT / "include" / "fastpoisson_b200.h").read_text()
    return set(re.findall(r"FP_API\s+[\w\s\*]+?\b(fp_\w+)\s*\(", text))


def test_abi_exports_every_declared_symbol(native_lib):
    declared = _header_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(native_lib, name), name
    # the ctypes signature table covers exactly the declared surface
    assert declared == set(_native.SIGNATURES)
    assert native_lib.fp_abi_version() == 1


def test_abi_config_struct_layout():
    # fp_config: int ndim; int64 n[3]; double length[3]; int bc[3], kind[3]; int approx, precision; ptr eig[3]
    assert ctypes.sizeof(_native.FpConfig) == 4 + 4 + 24 + 24 + 12 + 12 + 4 + 4 + 24
    assert ctypes.sizeof(_native.FpSolveInfo) == 16


def test_abi_rejects_bad_config_without_gpu(native_lib):
    cfg = _native.FpConfig()
    cfg.ndim = 4
    h = ctypes.c_void_p()
    assert native_lib.fp_plan_create(ctypes.byref(cfg), 0, ctypes.byref(h)) == _native.FP_ERR_CONFIG
    assert b"dimensions" in native_lib.fp_last_error()
    cfg.ndim = 1
    cfg.n[0] = 8
    cfg.length[0] = 1.0
    cfg.bc[0] = _native.FP_BC_PERIODIC
    cfg.kind[0] = _native.FP_GRID_STAGGERED
    assert native_lib.fp_plan_create(ctypes.byref(cfg), 0, ctypes.byref(h)) == _native.FP_ERR_CONFIG
    assert b"periodic" in native_lib.fp_last_error()


def test_no_cpu_fallback_on_cpu_host():
    # the product path must refuse to run without a GPU instead of computing on the host
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    g = fp.GridSpec(8, 1.0, BC.PERIODIC)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        fp.SolverPlan(fp.SolverConfig((g,), AP.PSEUDO_SPECTRAL))


def test_product_never_imports_oracle():
    for p in (ROOT / "paper_1409_8116_b200").rglob("*.py"):
        text = p.read_text()
        assert "import oracle" not in text and "from oracle" not in text, p


def test_torch_extension_loads_and_registers_ops(native_lib):
    # the PyTorch extension in front of the C ABI (csrc/fp_torch_ext.cpp): in-tree, loadable
    # without a GPU, bound to the loaded kernel library; it has no CPU path
    import torch

    from paper_1409_8116_b200 import _build

    assert _build.TORCH_EXT_PATH.exists(), "build it: python -c 'import __graft_entry__ as g; g.build()'"
    ops = _native.torch_ext()
    assert hasattr(ops, "solve") and hasattr(ops, "bind")
    z = torch.zeros(4)
    with pytest.raises(RuntimeError, match="CUDA tensors only"):
        ops.solve(0, z, z, z, z, 0, None)
