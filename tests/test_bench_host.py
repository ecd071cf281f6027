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


def test_default_workload_follows_gpu_count():
    # BASELINE.json: config 2 on 1 GPU, the config-3 scene (north-star gate) on 2/4/8
    assert bench.parse(["--gpus", "1"]).workload == "C2"
    for n in (2, 4, 8):
        assert bench.parse(["--gpus", str(n)]).workload == "C3"
    assert bench.parse(["--gpus", "8", "--workload", "C5"]).workload == "C5"


def test_world_size_must_match_gpus():
    assert bench.check_world(4, {"WORLD_SIZE": "4"}) == 4
    assert bench.check_world(1, {}) == 1
    import pytest

    with pytest.raises(SystemExit, match="WORLD_SIZE=2 but --gpus 8"):
        bench.check_world(8, {"WORLD_SIZE": "2"})


def test_launcher_command():
    cmd = bench.launcher_command(["--gpus", "8", "--steps", "3"], 8, 29511)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "127.0.0.1" in cmd and "29511" in cmd
    assert cmd[-3:] == ["--gpus", "8", "--steps", "3"][-3:]


def test_spawns_ranks_and_bands_the_c3_scene():
    """`python bench.py --gpus 2` (no torchrun environment) spawns two ranks itself; rank 0
    reports world size 2 and the C3 scene cut into two 256-aligned bands."""
    import json
    import os

    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run"], capture_output=True,
                       text=True, cwd=ROOT, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["n_gpus"] == 2 and d["workload"] == "C3" and d["scaling"] == "strong"
    assert d["pixels_total"] == 16384 * 16384
    (a0, b0), (a1, b1) = d["bands"]
    assert a0 == 0 and b0 == a1 and b1 == 16384 * 16384 and a1 % 256 == 0


def test_mismatched_world_exits_nonzero():
    import os

    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4", "--dry-run"], capture_output=True,
                       text=True, cwd=ROOT, timeout=120, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=2 but --gpus 4" in r.stderr
