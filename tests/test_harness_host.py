"""Host-side contracts of the experiment harness and CLI (no GPU needed): the
reference's tests/test_harness.py cases that do not solve anything — configuration
validation, the worker cap, CSV schema/appending, plot-data format, the rate fit
and the CLI's usage exit code (cli.py:1-5)."""

import csv
import json
import math
from pathlib import Path

import pytest

import paper_2006_12883_b200 as pd
from paper_2006_12883_b200.cli import main as cli_main
from paper_2006_12883_b200.harness import (CSV_FIELDS, METHODS, ExperimentConfig, append_rows,
                                            worker_limit, write_series)
from paper_2006_12883_b200.harness_util import fit_slope

GOLD = json.loads((Path(__file__).parent / "golden" / "harness.json").read_text())


def test_schema_matches_reference_rows():
    assert METHODS == ("smg", "stmg", "smmg", "pfasst", "direct")
    for item in GOLD["single"]:
        assert tuple(item["row"]) == CSV_FIELDS


def test_validation_and_worker_cap(monkeypatch):
    with pytest.raises(pd.ConfigurationError):
        ExperimentConfig(method="jacobi").validate()
    with pytest.raises(pd.ConfigurationError):
        ExperimentConfig(P=0).validate()
    with pytest.raises(pd.ConfigurationError, match="divide"):
        ExperimentConfig(method="pfasst", Nt=6, P=4).validate()
    with pytest.raises(pd.ConfigurationError):
        ExperimentConfig(mode="explicit").validate()
    monkeypatch.setenv("PARADIFF_MAX_THREADS", "2")
    assert worker_limit() == 2
    with pytest.raises(pd.ConfigurationError, match="cap"):
        pd.run_experiment(ExperimentConfig(method="pfasst", P=4, Nt=16, Nx=32, L=2, nu=1))
    monkeypatch.setenv("PARADIFF_MAX_THREADS", "many")
    assert worker_limit() == 16
    assert ExperimentConfig().resolved_mode(0.0) == "implicit"
    assert ExperimentConfig().resolved_mode(5.0) == "imex"
    assert ExperimentConfig(mode="implicit").resolved_mode(5.0) == "implicit"


def test_csv_appends_with_one_header(tmp_path):
    out = tmp_path / "sub" / "runs.csv"
    row = GOLD["single"][0]["row"]
    append_rows(str(out), [row])
    append_rows(str(out), [row, {"method": "direct"}])
    with out.open() as fh:
        rows = list(csv.reader(fh))
    assert rows[0] == list(CSV_FIELDS) and len(rows) == 4
    assert rows[3][0] == "direct" and rows[3][1] == ""


def test_series_format(tmp_path):
    path = tmp_path / "a" / "s.dat"
    write_series(str(path), [(4.0, 1e-3), (8.0, 1.25e-4)])
    lines = path.read_text().strip().splitlines()
    assert [len(line.split()) for line in lines] == [2, 2]
    assert float(lines[1].split()[1]) == 1.25e-4


def test_fit_slope_contract():
    # order 3, then a round-off floor (reference test_fit_slope_skips_floor_points)
    assert 2.5 < fit_slope([2, 4, 8, 16], [1e-2, 1.25e-3, 1e-13, 9e-14], floor=5e-13) < 3.5
    assert math.isnan(fit_slope([2, 4], [1e-15, 1e-16]))
    # a pre-asymptotic transient is left out of the fit
    s = fit_slope([2, 4, 8, 16, 32], [1.0, 1e-3, 1.25e-4, 1.5625e-5, 1.953125e-6])
    assert abs(s - 3.0) < 0.05
    # the reference's fitted slopes from its own error tables
    by_m = {}
    for row in GOLD["order"]["rows"]:
        by_m.setdefault(row["M"], []).append((row["Nt"], row["error_vs_semidiscrete"]))
    for M, pts in by_m.items():
        got = fit_slope([p[0] for p in pts], [p[1] for p in pts], floor=1e-14)
        assert got == pytest.approx(GOLD["order"]["slopes"][str(M)], rel=1e-12)


def test_cli_usage_errors_exit_two(capsys):
    with pytest.raises(SystemExit) as exc:
        cli_main(["solve", "--method", "sor"])
    assert exc.value.code == 2
    assert cli_main(["solve", "--method", "pfasst", "--nt", "6", "-P", "4", "--nx", "32",
                     "-L", "2"]) == 2
    assert "error:" in capsys.readouterr().err
