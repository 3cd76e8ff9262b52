"""CPU tier: bench.py's workload table and reference arm (no GPU needed)."""

import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_1409_8116_b200 as fp  # noqa: E402
from oracle import fastpoisson_oracle as orc  # noqa: E402


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_bench_configs_match_baseline_table(name):
    cfg = bench.build_config(fp, name)
    case = orc.config_case(name)
    assert cfg.shape == case.shape
    assert cfg.precision == case.precision
    for g, a in zip(cfg.grids, case.axes):
        assert (g.n, g.bc.value, g.kind.value) == (a.n, a.bc, a.kind)
        assert g.length == pytest.approx(a.length)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_host_rhs_distribution(name):
    cfg = bench.build_config(fp, name, scale=8 if name != "c1" else 2)
    r = bench.host_rhs(name, cfg)
    assert r.shape == cfg.shape and np.isfinite(r).all()
    if name in ("c1", "c3", "c4"):
        assert abs(r.mean()) < 1e-9 * max(1.0, np.abs(r).max())   # compatible (solvable) rhs


def test_reference_arm_json_line():
    proc = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", "c1",
                           "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, proc.stderr
    line = json.loads(proc.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert line["cpu_baseline"]["t1"]["cores"] == 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_oracle_plan_matches_one_shot_solve():
    case = orc.config_case("c3", scale=32)
    rhs = orc.config_rhs("c3", case, seed=3)
    a, ma = orc.solve(case, rhs)
    b, mb = orc.OraclePlan(case).solve(rhs)
    assert np.array_equal(a, b) and ma == mb
