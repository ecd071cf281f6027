"""Host-side pieces of bench.py that the JSON line depends on (CPU, no GPU)."""
import subprocess
import sys
from pathlib import Path

import bench

ROOT = Path(__file__).resolve().parents[1]


def _row(sm, smax, power_cap="Not Active", thermal="Not Active"):
    return f"0, {sm}, {smax}, 700.0, 0x0, Not Active, Not Active, {thermal}, {power_cap}\n"


def test_clock_summary_median_under_load_and_reasons():
    c = bench.ClockSampler(0)
    c.lines = [_row(345, 1965), _row(1965, 1965), _row(1950, 1965, power_cap="Active"), _row(1965, 1965)]
    s = c.summary()
    assert s["sm_mhz"] == 1965.0 and s["sm_max_mhz"] == 1965.0     # the idle 345 MHz sample is dropped
    assert s["reasons"] == ["sw_power_cap"] and s["samples"] == 4


def test_clock_summary_thermal_reason():
    c = bench.ClockSampler(0)
    c.lines = [_row(1500, 1965, thermal="Active")]
    assert c.summary()["reasons"] == ["sw_thermal_slowdown"]


def test_clock_summary_without_samples():
    c = bench.ClockSampler(0)
    s = c.summary()
    assert s["samples"] == 0 and s["sm_mhz"] is None and s["reasons"]


def test_rejects_zero_steps():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "0"], capture_output=True, text=True,
                       cwd=ROOT, timeout=120)
    assert r.returncode == 2 and "--steps" in r.stderr
