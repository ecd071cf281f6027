"""Time lambda calibration (critical_value) on the GPU vs the pinned reference values."""
import json, time, sys
sys.path.insert(0, "/root/repo")
import paper_1807_01751_b200 as pkg
pinned = json.load(open("/root/repo/tests/golden/pinned.json"))
for key in ("crit_20k", "crit_c1", "crit_100k"):
    r = pinned[key]["request"]
    req = pkg.CriticalValueRequest(**r)
    t0 = time.perf_counter()
    lam = pkg.critical_value(req, threads=16)
    dt = time.perf_counter() - t0
    print(key, r["reps"], "reps", f"{dt:.2f} s", lam, pinned[key]["value"], flush=True)
