"""CLI (paper_1807_01751_b200/cli.py) — the reference's pkg/tests/test_cli.py cases.

Argument handling and the data/usage error paths run on CPU (they fail before any device
work); the monitor / critical-value runs that reach the kernel are marked gpu.
"""
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_1807_01751_b200 import SeriesStack, regular_axis, write_stack
from paper_1807_01751_b200.cli import dispatch

REPO = Path(__file__).resolve().parents[1]


def make_stack_file(tmp_path, name="stack.bts", m=60, n_obs=200, seed=0):
    path = tmp_path / name
    code = dispatch(["generate", "--m", str(m), "--N", str(n_obs), "--freq", "23", "--noise-std", "0.02",
                     "--break-mag", "0.5", "--seed", str(seed), "--out", str(path)])
    assert code == 0
    return path


def test_generate_reports(tmp_path, capsys):
    make_stack_file(tmp_path, m=10, n_obs=30)
    out = capsys.readouterr().out
    assert "30 observations x 10 pixels, 5 break series" in out


def test_bandwidth_above_history_is_usage_error(tmp_path, capsys):
    p = make_stack_file(tmp_path, m=5)
    assert dispatch(["monitor", "--input", str(p), "--h", "150", "--n", "100", "--out", str(tmp_path / "x")]) == 1
    assert "h <= n" in capsys.readouterr().err


def test_missing_input_is_data_error(tmp_path, capsys):
    code = dispatch(["monitor", "--input", str(tmp_path / "missing.bts"), "--lambda", "4.9",
                     "--out", str(tmp_path / "x.csv")])
    assert code == 2
    assert capsys.readouterr().err


def test_malformed_input_is_data_error(tmp_path, capsys):
    bad = tmp_path / "bad.bts"
    bad.write_bytes(b"XXXX" + bytes(40))
    assert dispatch(["monitor", "--input", str(bad), "--lambda", "4.9", "--out", str(tmp_path / "x.csv")]) == 2
    assert "magic" in capsys.readouterr().err


def test_unknown_backend_is_usage_error(tmp_path, capsys):
    p = make_stack_file(tmp_path, m=5)
    assert dispatch(["monitor", "--input", str(p), "--backend", "bogus", "--out", str(tmp_path / "x")]) == 1


def test_unknown_flag_rejected(tmp_path, capsys):
    assert dispatch(["generate", "--m", "5", "--N", "20", "--frobnicate", "--out", str(tmp_path / "x.bts")]) == 1
    assert "--frobnicate" in capsys.readouterr().err


def test_missing_subcommand():
    assert dispatch([]) == 1


def test_bad_m_list(tmp_path, capsys):
    assert dispatch(["bench", "--m-list", "10,oops", "--out", str(tmp_path / "b.csv")]) == 1
    assert "m-list" in capsys.readouterr().err


def test_invalid_critical_value_request_is_usage_error():
    assert dispatch(["critical-value", "--alpha", "2.0", "--reps", "1000"]) == 1


def test_help_exits_zero():
    assert dispatch(["--help"]) == 0


def test_module_entry_point_runs():
    r = subprocess.run([sys.executable, "-m", "paper_1807_01751_b200", "--help"], capture_output=True, text=True,
                       cwd=REPO)
    assert r.returncode == 0
    assert "generate" in r.stdout


# ---- through the kernel ------------------------------------------------------------------
@pytest.mark.gpu
def test_monitor_happy_path(tmp_path, capsys):
    p = make_stack_file(tmp_path)
    out = tmp_path / "breaks.csv"
    code = dispatch(["monitor", "--input", str(p), "--n", "100", "--h", "50", "--k", "3", "--freq", "23",
                     "--lambda", "4.9", "--out", str(out)])
    assert code == 0
    o = capsys.readouterr().out
    assert "lambda: 4.9" in o and "breaks:" in o
    lines = out.read_text().splitlines()
    assert lines[0] == "pixel,valid,detected,first_break,max_abs_mo"
    assert len(lines) == 61


@pytest.mark.gpu
def test_monitor_profile_lines(tmp_path, capsys):
    p = make_stack_file(tmp_path, m=20)
    assert dispatch(["monitor", "--input", str(p), "--lambda", "4.9", "--profile", "--out", str(tmp_path / "p")]) == 0
    o = capsys.readouterr().out
    for name in ("ingest", "model", "predictions", "residuals", "mosum", "breaks", "total"):
        assert f"{name}:" in o


@pytest.mark.gpu
def test_identical_invocations_identical_csvs(tmp_path):
    p = make_stack_file(tmp_path, m=30, n_obs=40)
    args = ["monitor", "--input", str(p), "--n", "20", "--h", "10", "--k", "1", "--freq", "10"]
    assert dispatch(args + ["--out", str(tmp_path / "a.csv")]) == 0
    assert dispatch(args + ["--out", str(tmp_path / "b.csv")]) == 0
    assert (tmp_path / "a.csv").read_bytes() == (tmp_path / "b.csv").read_bytes()


@pytest.mark.gpu
def test_zero_residual_is_numeric_error(tmp_path, capsys):
    flat = tmp_path / "flat.bts"
    write_stack(SeriesStack(np.zeros((200, 3), dtype=np.float32), regular_axis(200)), flat)
    assert dispatch(["monitor", "--input", str(flat), "--lambda", "4.9", "--out", str(tmp_path / "x")]) == 3
    assert "sigma" in capsys.readouterr().err


@pytest.mark.gpu
def test_critical_value_prints_lambda(capsys):
    assert dispatch(["critical-value", "--alpha", "0.05", "--h-frac", "0.5", "--horizon", "2", "--n-sim", "30",
                     "--reps", "1000", "--seed", "9"]) == 0
    o = capsys.readouterr().out
    assert o.startswith("lambda: ") and float(o.split()[1]) > 0


@pytest.mark.gpu
def test_bench_writes_csv(tmp_path, capsys):
    out = tmp_path / "bench.csv"
    assert dispatch(["bench", "--m-list", "200,600", "--n", "20", "--h", "10", "--k", "1", "--freq", "10",
                     "--seed", "4", "--out", str(out)]) == 0
    lines = out.read_text().splitlines()
    assert lines[0] == "m,ingest,model,predictions,residuals,mosum,breaks,total"
    assert len(lines) == 3
    assert capsys.readouterr().out.count("m=") == 2
