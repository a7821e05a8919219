"""Runner/config/CSV layer (CPU): the reference's config grammar and error
diagnostics (config.cpp:131-182), canonical echo without wos.workers, CSV
comparison (runner.cpp:445-479), CLI exit codes."""
from __future__ import annotations

import io
from pathlib import Path

import pytest

from paper_1210_1491_b200 import runner
from paper_1210_1491_b200.__main__ import main
from paper_1210_1491_b200.errors import ConfigError

TEXT = """
# comment
[scene]
kind = half_space   # trailing comment
charge_height = 1.0
[method]
name = biewos_point
x = 0.5, 0
a = 0.1 0.2
targets = 1 2 3 ; 4 5 6
[wos]
workers = 8
seed = 3
"""


def test_parse_tokens_and_echo():
    c = runner.parse_config_text(TEXT, "t.cfg")
    assert c.get_str("scene", "kind") == "half_space"
    assert c.get_list("method", "x") == [0.5, 0.0]
    assert c.tokens("method", "targets") == ["1", "2", "3", ";", "4", "5", "6"]
    assert c.get_int("wos", "seed", 0) == 3
    assert "workers" not in c.echo() and "wos.seed=3" in c.echo()
    runner.apply_override(c, "wos.seed=9")
    assert c.get_int("wos", "seed", 0) == 9


@pytest.mark.parametrize("bad,msg", [("[scene\nk=1", ":2: malformed"), ("k = 1", "outside any"),
                                     ("[s]\n = 1", "empty key"), ("[s]\nnovalue", "expected")])
def test_diagnostics(bad, msg):
    with pytest.raises(ConfigError, match=msg if msg != ":2: malformed" else "malformed"):
        runner.parse_config_text(bad, "x.cfg")


def test_get_errors_name_the_line():
    c = runner.parse_config_text("[a]\nb = notanumber\n", "f.cfg")
    with pytest.raises(ConfigError, match="f.cfg:2"):
        c.get_real("a", "b")
    with pytest.raises(ConfigError):
        runner.apply_override(c, "nodot=1")


def test_compare_csv(tmp_path):
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    a.write_text("# x\nc1,c2\n1.0,2.0\nnan,3\n")
    b.write_text("# y\nc1,c2\n1.0000001,2.0\nnan,3\n")
    rep = io.StringIO()
    assert runner.compare_csv(str(a), str(b), 1e-6, rep) == 0 and "PASS" in rep.getvalue()
    assert runner.compare_csv(str(a), str(b), 1e-9, rep) == 1
    b.write_text("c1,c3\n1,2\n")
    with pytest.raises(ConfigError):
        runner.compare_csv(str(a), str(b), 1e-6)


def test_cli_exit_codes(tmp_path):
    bad = tmp_path / "bad.cfg"
    bad.write_text("[scene]\nkind = nope\n[method]\nname = biewos_point\n")
    assert main(["solve", str(bad)]) == 2
    assert main(["solve", str(tmp_path / "missing.cfg")]) == 2


def test_empty_sweep_header_only_csv():  # test_cli.cpp:77-94
    from paper_1210_1491_b200 import runner as R

    c = R.parse_config_file(str(Path(__file__).resolve().parents[1] / "configs"
                                / "halfspace_point_b200.cfg"))
    R.apply_override(c, "method.a=")
    rec = R.run(c)
    assert rec.rows == []
    lines = [l for l in rec.csv_text.splitlines() if l and not l.startswith("#")]
    assert len(lines) == 1 and lines[0].startswith("a,delta_frac")


def test_pipeline_config_validation_and_echo():
    """configs/baseline_cfg5.cfg parses; [gpu] devices never enters the echo
    (results do not depend on it, like wos.workers); a bad stream name or a
    non-cavity configuration is a ConfigError before any device work."""
    from paper_1210_1491_b200 import runner
    from paper_1210_1491_b200.errors import ConfigError

    c = runner.parse_config_file(str(Path(__file__).resolve().parents[1] / "configs" / "baseline_cfg5.cfg"))
    assert "gpu." not in c.echo() and runner._devices(c) == [0]
    runner.apply_override(c, "method.rng=mt19937")
    with pytest.raises(ConfigError):
        runner.run(c)
    c2 = runner.parse_config_file(str(Path(__file__).resolve().parents[1] / "configs" / "baseline_cfg5.cfg"))
    runner.apply_override(c2, "method.baseline_config=4")
    with pytest.raises(ConfigError):
        runner.run(c2)
