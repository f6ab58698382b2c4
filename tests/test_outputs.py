"""§8(f) rank 1: output files byte-identical to the reference's.

tests/golden/outputs/ holds files written by the REAL reference
(oracle/gen_golden_outputs.py): ``write_outputs`` (requests.csv,
summary.json, monitor.csv, decisions.jsonl; report.py:217-238) for three
golden scenarios, and the ``pdsim compare`` summary CSV (cli.py:26,
96-117).  The package's public API must reproduce them byte for byte: on
the B200 (gpu marker) and, for the host-side assembly and writers, with the
CPU oracle standing in for the device (OracleEvaluator, test-only)."""

from __future__ import annotations

import filecmp
import sys
from pathlib import Path

import pytest

import harness as H
import paper_2505_11916_b200 as arrow
from paper_2505_11916_b200 import cli

OUT = H.GOLDEN / "outputs"
NAMES = ("c1_rate4", "conservation_slo", "overload_flips")
FILES = ("requests.csv", "summary.json", "monitor.csv", "decisions.jsonl")


def _scenario(name):
    sys.path.insert(0, str(H.ROOT / "oracle"))
    import scenarios as S

    sc = next(s for s in S.catalogue(arrow.TraceRequest) if s["name"] == name)
    config = arrow.config_from_values(sc["values"])
    trace = arrow.scale_trace(sc["trace"], sc["scale"]) if sc["scale"] != 1.0 else sc["trace"]
    return trace, config


def _check_run_outputs(tmp_path, name):
    trace, config = _scenario(name)
    result = arrow.run(trace, config)
    arrow.write_outputs(result, config.slo, tmp_path / name, decisions=True)
    for f in FILES:
        assert filecmp.cmp(tmp_path / name / f, OUT / name / f, shallow=False), f"{name}/{f} differs"


def _check_compare(tmp_path):
    out = tmp_path / "compare.csv"
    rc = cli.main(["compare", str(OUT / "compare_trace.csv"), "--config", str(OUT / "compare_config.txt"),
                   "--rates", "4", "8", "12", "--strategies", "slo-aware", "minimal-load", "round-robin",
                   "--out", str(out)])
    assert rc == 0
    assert out.read_bytes() == (OUT / "compare.csv").read_bytes()


@pytest.mark.parametrize("name", NAMES)
def test_write_outputs_byte_identical_host_path(tmp_path, monkeypatch, name):
    H.use_oracle_backend(monkeypatch)
    _check_run_outputs(tmp_path, name)


def test_compare_csv_byte_identical_host_path(tmp_path, monkeypatch):
    H.use_oracle_backend(monkeypatch)
    _check_compare(tmp_path)


def test_cli_usage_and_runtime_exit_codes(tmp_path, monkeypatch, capsys):
    """cli.py:29-33, 224-230: usage errors exit 1, runtime errors 2."""
    H.use_oracle_backend(monkeypatch)
    with pytest.raises(SystemExit) as e:
        cli.main(["compare", str(OUT / "compare_trace.csv"), "--out", str(tmp_path / "x.csv")])
    assert e.value.code == 1
    assert cli.main(["run", str(tmp_path / "missing.csv"), "--out-dir", str(tmp_path / "o")]) == 2
    assert "pdsim: error:" in capsys.readouterr().err


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_write_outputs_byte_identical_gpu(tmp_path, name):
    _check_run_outputs(tmp_path, name)


@pytest.mark.gpu
def test_compare_csv_byte_identical_gpu(tmp_path):
    _check_compare(tmp_path)
