"""CPU tier: field files (fieldio.py:1-116) and the CLI's pre-device paths
(cli.py:47-66,175-200,261-268), checked against files the reference wrote
(tests/golden/make_cli_golden.py) and against the reference tests
(tests/test_fieldio.py, tests/test_cli.py)."""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_1409_8116_b200 import BoundaryCondition as BC, GridKind as GK, GridSpec
from paper_1409_8116_b200.cli import main
from paper_1409_8116_b200.fieldio import FieldFormatError, read_field, write_field

GOLD = Path(__file__).resolve().parent / "golden" / "cli_v1"


def grids_for(shape):
    return tuple(GridSpec(n, 1.0, BC.DIRICHLET, GK.STAGGERED) for n in shape)


def test_writer_is_byte_identical_to_the_reference(tmp_path):
    rhs = np.load(GOLD / "rhs_values.npy")
    grids = (GridSpec(12, 1.0, BC.NEUMANN, GK.STAGGERED), GridSpec(10, 2.0, BC.NEUMANN, GK.STAGGERED))
    write_field(tmp_path / "rhs", rhs, grids)
    assert (tmp_path / "rhs.json").read_bytes() == (GOLD / "rhs.json").read_bytes()
    assert (tmp_path / "rhs.bin").read_bytes() == (GOLD / "rhs.bin").read_bytes()
    x32, grids32 = read_field(GOLD / "rhs32.json")
    assert grids32 is None and x32.dtype == np.float32
    write_field(tmp_path / "rhs32", x32)
    assert (tmp_path / "rhs32.json").read_bytes() == (GOLD / "rhs32.json").read_bytes()
    assert (tmp_path / "rhs32.bin").read_bytes() == (GOLD / "rhs32.bin").read_bytes()


def test_reader_matches_reference_files():
    x, grids = read_field(GOLD / "rhs.json")
    np.testing.assert_array_equal(x, np.load(GOLD / "rhs_values.npy"))
    assert grids[0].bc is BC.NEUMANN and grids[1].length == 2.0
    sol, g2 = read_field(GOLD / "ref_run" / "solution.json")
    assert sol.shape == (12, 10) and g2 == grids


def test_round_trip(tmp_path, rng):
    data = rng.standard_normal((5, 7, 3))
    back, grids = read_field(write_field(tmp_path / "f", data, grids_for(data.shape)))
    np.testing.assert_array_equal(back, data)
    assert grids[0].bc is BC.DIRICHLET and grids[0].kind is GK.STAGGERED


def test_payload_is_raw_little_endian(tmp_path):
    data = np.array([1.0, 2.0, -3.5])
    write_field(tmp_path / "raw", data)
    np.testing.assert_array_equal(np.frombuffer((tmp_path / "raw.bin").read_bytes(), "<f8"), data)


@pytest.mark.parametrize("mutate,expect", [
    (lambda h: h.update(format_version=99), "format version"),
    (lambda h: h.pop("precision"), "missing header key"),
    (lambda h: h.update(byte_order="big"), "byte order"),
    (lambda h: h.update(order="F"), "storage order"),
    (lambda h: h.update(precision="half"), "precision"),
    (lambda h: h.update(dims=3), "dims"),
    (lambda h: h.update(grids=[{"n": 3, "length": 1.0, "bc": "neumann", "kind": "staggered"}] * 2), "grid point counts"),
    (lambda h: h.update(grids=[{"n": 4, "bc": "neumann"}] * 2), "bad grid entry"),
])
def test_bad_headers_rejected(tmp_path, mutate, expect):
    hp = write_field(tmp_path / "h", np.zeros((4, 4)), grids_for((4, 4)))
    header = json.loads(hp.read_text())
    mutate(header)
    hp.write_text(json.dumps(header))
    with pytest.raises(FieldFormatError, match=expect):
        read_field(hp)


def test_truncated_payload_and_invalid_json_rejected(tmp_path):
    write_field(tmp_path / "t", np.zeros(8))
    (tmp_path / "t.bin").write_bytes((tmp_path / "t.bin").read_bytes()[:-8])
    with pytest.raises(FieldFormatError, match="expected 64"):
        read_field(tmp_path / "t.json")
    (tmp_path / "j.json").write_text("{not json")
    with pytest.raises(FieldFormatError, match="invalid JSON"):
        read_field(tmp_path / "j.json")


def test_unsupported_dtype_rejected(tmp_path):
    with pytest.raises(FieldFormatError):
        write_field(tmp_path / "i", np.zeros(4, dtype=np.int32))


# -- CLI paths that exit before any device work (tests/test_cli.py:54-70,122-125)
def test_cli_flag_header_mismatch_exits_2(tmp_path, capsys):
    code = main(["solve", "--in", str(GOLD / "rhs.json"), "--size", "8,8", "--out", str(tmp_path / "x")])
    assert code == 2
    err = capsys.readouterr().err
    assert "(8, 8)" in err and "(12, 10)" in err


def test_cli_missing_input_exits_3(tmp_path):
    assert main(["solve", "--in", str(tmp_path / "nope.json"), "--out", str(tmp_path / "x")]) == 3


def test_cli_bad_payload_exits_3(tmp_path):
    write_field(tmp_path / "t", np.zeros(8))
    (tmp_path / "t.bin").write_bytes(b"\0" * 8)
    assert main(["solve", "--in", str(tmp_path / "t.json"), "--out", str(tmp_path / "x")]) == 3


def test_cli_bad_config_exits_2(tmp_path, rng):
    header = write_field(tmp_path / "r", rng.standard_normal((6, 6)))
    code = main(["solve", "--in", str(header), "--bc", "periodic,dirichlet", "--grid", "staggered,regular",
                 "--out", str(tmp_path / "x")])
    assert code == 2  # periodic is regular-only


def test_cli_cpu_device_rejected(tmp_path):
    code = main(["solve", "--in", str(GOLD / "rhs.json"), "--bc", "neumann", "--grid", "staggered",
                 "--device", "cpu", "--out", str(tmp_path / "x")])
    assert code == 2


def test_cli_bench_rejects_bad_sizes():
    assert main(["bench", "--sizes", "0", "--dims", "1"]) == 2
    assert main(["bench", "--sizes", "8", "--dims", "1", "--reps", "0"]) == 2
