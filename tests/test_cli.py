"""CLI harness parity (unimul.cli, cli.py:30-470) against the reference's own
command-line output (tests/golden/cli, made by tests/golden/make_cli_golden.py).

dump-ops / dump-ir plan on a placement-only fabric, so they run on CPU; `run`
and `sweep` execute on the GPU and compare the CSV with the reference's."""

import contextlib
import io
import os

import pytest

from paper_2510_08874_b200 import cli
from paper_2510_08874_b200.errors import ConfigError

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")
NAMES = sorted(f[:-4] for f in os.listdir(GOLD) if f.endswith(".cfg"))


def capture(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.main(argv)
    return rc, buf.getvalue()


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("cmd,ext", [("dump-ops", "ops"), ("dump-ir", "ir")])
def test_dump_matches_reference(name, cmd, ext):
    rc, out = capture([cmd, os.path.join(GOLD, name + ".cfg")])
    assert rc == 0
    with open(os.path.join(GOLD, f"{name}.{ext}")) as f:
        assert out == f.read()


def test_grammar_errors(tmp_path):
    bad = tmp_path / "bad.cfg"
    bad.write_text("m = 8\nbogus = 1\n")
    with pytest.raises(ConfigError, match="unknown key"):
        cli.load_config(str(bad))
    bad.write_text("m 8\n")
    with pytest.raises(ConfigError, match="expected 'key = value'"):
        cli.load_config(str(bad))
    bad.write_text("m = 8, 16\n")
    with pytest.raises(ConfigError, match="single-valued"):
        cli.load_config(str(bad))
    bad.write_text("m =\n")
    with pytest.raises(ConfigError, match="no value"):
        cli.load_config(str(bad))
    with pytest.raises(ConfigError, match="replication must divide"):
        cli.RunConfig(8, 8, 8, 4, c_c=3).validate()


def test_sweep_order_matches_reference():
    """Cross product in file key order (cli.py:340-347): same config ids, same order."""
    ids = [c.config_id() for c in cli.iter_sweep_configs(os.path.join(GOLD, "sweep.sweep"))]
    with open(os.path.join(GOLD, "sweep.csv")) as f:
        ref = [line.split(",")[0] for line in f.read().splitlines()[1:]]
    assert ids == ref


@pytest.mark.gpu
def test_sweep_csv_matches_reference(cuda):
    """Same pass verdicts, bytes, flops, modeled cost and op counts as the reference's sweep."""
    rc, out = capture(["sweep", os.path.join(GOLD, "sweep.sweep")])
    with open(os.path.join(GOLD, "sweep.csv")) as f:
        assert out == f.read()
    assert rc == 0


@pytest.mark.gpu
def test_run_writes_counters(cuda, tmp_path):
    rc, out = capture(["run", os.path.join(GOLD, "rep_cost.cfg"), "--counters", str(tmp_path / "ctr")])
    assert rc == 0
    assert out.splitlines()[0] == cli.CSV_HEADER
    assert ",pass," in out.splitlines()[1]
    assert (tmp_path / "ctr_links.csv").read_text().startswith("src,dst")
