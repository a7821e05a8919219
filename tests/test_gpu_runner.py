"""GPU: the config runner end to end (point formula, last passage, field eval,
biewos_dtn) with deterministic CSV output (tests/test_cli.cpp of the reference:
byte-identical CSV bodies across runs and worker counts)."""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from paper_1210_1491_b200 import runner

pytestmark = pytest.mark.gpu
CFG = Path(__file__).resolve().parents[1] / "configs"


def _rows(rec):
    return np.array(rec.rows, dtype=float)


def test_point_config_analytic(gpu):
    c = runner.parse_config_file(str(CFG / "halfspace_point_b200.cfg"))
    rec = runner.run(c)
    assert rec.schema == "biewos_point/v1" and len(rec.rows) == 5
    r = _rows(rec)
    total, se, ref = r[:, 8], r[:, 9], r[:, 10]
    assert (np.abs(total - ref) < 4 * se + 3e-3).all()
    again = runner.run(runner.parse_config_file(str(CFG / "halfspace_point_b200.cfg")), workers=7)
    assert again.csv_text == rec.csv_text  # workers never change results


def test_lp_config(gpu):
    c = runner.parse_config_file(str(CFG / "disk_lastpassage_b200.cfg"))
    runner.apply_override(c, "method.n_path=20000")
    rec = runner.run(c)
    r = _rows(rec)
    assert (np.abs(r[:, 3] - r[:, 6]) < 4 * r[:, 4] + 0.03 * r[:, 6]).all()


def test_field_eval_config(gpu):
    c = runner.parse_config_text("""
[scene]
kind = sphere
R = 3
potential = 0.25
[method]
name = field_eval
targets = 4 0 0 ; 0 0 5
n_panels = 2000 8000
""", "fe.cfg")
    r = _rows(runner.run(c))
    assert (np.abs(r[:, 6]) < 1.0).all()  # err_pct below 1 %


def test_dtn_config_small(gpu):
    c = runner.parse_config_file(str(CFG / "baseline_cfg1.cfg"))
    runner.apply_override(c, "method.n_bp=20")
    runner.apply_override(c, "method.n_path=2000")
    rec = runner.run(c)
    r = _rows(rec)
    assert rec.schema == "biewos_dtn/v1" and len(r) == 20
    assert (r[:, 9] == 0).all()
    assert (np.abs(r[:, 5] - r[:, 7]) < 5 * r[:, 6] + 5e-3 * np.abs(r[:, 7]).max()).all()


SMALL_POINT_RUN = """
# half-space point formula, two radii, small budget
[scene]
kind = half_space
charge_height = 1.0
charge_scale = 1.0
[method]
name = biewos_point
x = 0.5 0
a = 0.2 0.5
n_g1 = 8
n_g2 = 20
n_path = 200
reference = analytic
[wos]
seed = 7
eps_shell = 1e-5
trunc_radius = 1e5
"""


def test_point_run_bookkeeping_and_determinism(gpu):  # test_cli.cpp:52-75
    c = runner.parse_config_text(SMALL_POINT_RUN, "small")
    r1 = runner.run(c)
    assert len(r1.rows) == 2 and len(r1.columns) == 13
    assert r1.rows[0][12] == 8.0 * 8.0 * 200.0
    assert r1.paths_total == 2 * 8.0 * 8.0 * 200.0
    for row in r1.rows:
        assert abs(row[8] / 0.71554 - 1.0) < 0.05
    assert runner.run(c).csv_text == r1.csv_text
    assert runner.run(c, workers=4).csv_text == r1.csv_text
    assert runner.run(c, seed=8, workers=1).csv_text != r1.csv_text
