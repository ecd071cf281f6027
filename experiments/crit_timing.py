"""Time lambda calibration (critical_value) on the GPU vs the pinned reference values.
First call per geometry includes plan creation (host QR, tables, kernel setup); the second
is the steady state (device draws + one monitor launch + quantile)."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1807_01751_b200 as pkg  # noqa: E402

pinned = json.load(open(ROOT / "tests" / "golden" / "pinned.json"))
for key in ("crit_20k", "crit_c1", "crit_100k"):
    r = pinned[key]["request"]
    req = pkg.CriticalValueRequest(**r)
    for run in ("cold", "warm"):
        t0 = time.perf_counter()
        lam = pkg.critical_value(req)
        dt = time.perf_counter() - t0
        print(key, r["reps"], "reps", run, f"{dt * 1e3:.1f} ms", lam, pinned[key]["value"],
              f"rel {abs(lam / pinned[key]['value'] - 1):.2e}", flush=True)
