"""GPU tier: ``solve`` / ``bench`` of the CLI (cli.py:175-306) and the field
files streamed through HBM (fieldio.py), against the reference's own outputs
(tests/golden/cli_v1, made by tests/golden/make_cli_golden.py) and the
reference tests (tests/test_cli.py:21-51,103-119)."""

import csv
import json
from pathlib import Path

import numpy as np
import pytest

from paper_1409_8116_b200 import BoundaryCondition as BC, GridKind as GK, GridSpec
from paper_1409_8116_b200.cli import main
from paper_1409_8116_b200.fieldio import read_field, write_field
from oracle import fastpoisson_oracle as orc

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden" / "cli_v1"


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def test_solve_matches_reference_run(tmp_path, torch_cuda):
    out = tmp_path / "run"
    assert main(["solve", "--in", str(GOLD / "rhs.json"), "--out", str(out)]) == 0
    # same header bytes as the reference's solution file, values within the fp64 parity bar
    assert (out / "solution.json").read_bytes() == (GOLD / "ref_run" / "solution.json").read_bytes()
    got, _ = read_field(out / "solution.json")
    want, _ = read_field(GOLD / "ref_run" / "solution.json")
    assert orc.relative_l2(got, want) <= 1e-12
    rep = json.loads((out / "report.json").read_text())
    ref = json.loads((GOLD / "ref_run" / "report.json").read_text())
    assert set(rep) == set(ref) == {"removed_mean", "mode", "periodic_axes", "timing_seconds"}
    assert set(rep["timing_seconds"]) == set(ref["timing_seconds"])
    assert rep["mode"] == ref["mode"] and rep["periodic_axes"] == ref["periodic_axes"]
    assert rep["removed_mean"] == pytest.approx(ref["removed_mean"], abs=1e-12)
    manifest = json.loads((out / "manifest.json").read_text())
    assert manifest["subcommand"] == "solve" and manifest["library_version"] and manifest["seed"] == 0
    assert any("solution" in o for o in manifest["outputs"])


def test_solve_reruns_byte_identical(tmp_path, torch_cuda):
    a, b = tmp_path / "a", tmp_path / "b"
    assert main(["solve", "--in", str(GOLD / "rhs.json"), "--out", str(a)]) == 0
    assert main(["solve", "--in", str(GOLD / "rhs.json"), "--out", str(b)]) == 0
    assert (a / "solution.bin").read_bytes() == (b / "solution.bin").read_bytes()
    assert (a / "solution.json").read_text() == (b / "solution.json").read_text()


def test_solve_singular_reports_removed_mean(tmp_path, rng, torch_cuda):
    rhs = rng.standard_normal(64) + 2.0
    header = write_field(tmp_path / "r", rhs, (GridSpec(64, 1.0, BC.PERIODIC),))
    out = tmp_path / "out"
    assert main(["solve", "--in", str(header), "--out", str(out)]) == 0
    assert json.loads((out / "report.json").read_text())["removed_mean"] == pytest.approx(rhs.mean(), rel=1e-12)


def test_solve_flags_override_header_and_single_precision(tmp_path, rng, torch_cuda):
    rhs = rng.standard_normal((40, 48)).astype(np.float32)
    header = write_field(tmp_path / "r", rhs)
    out = tmp_path / "o"
    assert main(["solve", "--in", str(header), "--bc", "dirichlet", "--grid", "staggered", "--length", "1,2",
                 "--out", str(out)]) == 0
    got, grids = read_field(out / "solution.json")
    assert got.dtype == np.float32 and grids[1].length == 2.0
    case = orc.Case([(40, 1.0, orc.DIRICHLET, orc.STAGGERED), (48, 2.0, orc.DIRICHLET, orc.STAGGERED)], orc.FD2, "single")
    want, _ = orc.solve(case, rhs)
    assert orc.relative_l2(got, want) <= 1e-5


def test_field_streaming_large_through_hbm(tmp_path, rng, torch_cuda, monkeypatch):
    # chunked pinned streaming (3 chunks + remainder) both ways, device tensors in/out
    from paper_1409_8116_b200 import fieldio

    monkeypatch.setattr(fieldio, "_CHUNK_BYTES", 1 << 16)
    x = rng.standard_normal((50, 41, 17))
    write_field(tmp_path / "big", x)
    t, _ = read_field(tmp_path / "big.json", device="cuda")
    assert t.is_cuda and t.dtype == torch_cuda.float64
    np.testing.assert_array_equal(t.cpu().numpy(), x)
    write_field(tmp_path / "back", t * 2.0)
    back, _ = read_field(tmp_path / "back.json")
    np.testing.assert_array_equal(back, 2.0 * x)


def test_bench_csv_output(tmp_path, torch_cuda):
    out = tmp_path / "bench.csv"
    assert main(["bench", "--sizes", "16,32", "--dims", "2", "--bc", "periodic", "--approx", "spectral",
                 "--reps", "3", "--out", str(out)]) == 0
    with open(out, newline="") as fh:
        rows = list(csv.DictReader(fh))
    assert {r["phase"] for r in rows} == {"forward", "diagonal", "backward", "total"}
    assert {int(r["size"]) for r in rows} == {16, 32}
    for r in rows:
        assert float(r["min_seconds"]) <= float(r["median_seconds"])
        assert r["threads"] == "1"
    for n in (16, 32):
        by_phase = {r["phase"]: float(r["median_seconds"]) for r in rows if int(r["size"]) == n}
        assert by_phase["forward"] + by_phase["diagonal"] + by_phase["backward"] <= by_phase["total"] * 1.05
    assert json.loads((tmp_path / "manifest.json").read_text())["subcommand"] == "bench"
