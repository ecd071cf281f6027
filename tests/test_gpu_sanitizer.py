"""compute-sanitizer over the hand-rolled mbarrier / TMA / TMEM pipelines: memcheck
(out-of-bounds and misaligned accesses) and synccheck (barrier misuse) on C1-sized calls of every
fill/masked kernel variant, through the public API (tests/tools/sanitize_c1.py)."""
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _sanitizer():
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not Path(exe).exists():
        pytest.skip("compute-sanitizer not installed")
    return exe


@pytest.mark.parametrize("tool", ["memcheck", "synccheck"])
def test_sanitizer_clean(tool):
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "17", "--target-processes", "all",
           sys.executable, str(ROOT / "tests" / "tools" / "sanitize_c1.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=1800)
    tail = (r.stdout + r.stderr)[-4000:]
    if r.returncode != 0 and "closed on this pool" in tail:
        # the GPU pool's compute-sanitizer wrapper refuses to run (pool policy, not a finding)
        pytest.skip("compute-sanitizer is disabled on this GPU pool")
    assert r.returncode == 0, tail
    assert "sanitize workload ok" in r.stdout, tail
    assert "ERROR SUMMARY: 0 errors" in r.stdout + r.stderr, tail
