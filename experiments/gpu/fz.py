"""Debug: the masked fuzz geometry 8 against the oracle, per-pixel error report (beta, MO)."""
import math
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import paper_1807_01751_b200 as pkg
from oracle import bfast_oracle as bo
from paper_1807_01751_b200.synth import host_stack
i, N, n, h, k, P, nan = 8, 141, 133, 68, 5, 600, 0.6
rng = np.random.default_rng(300 + i)
t = np.cumsum(rng.uniform(1, 9, N)) + 1.0
y = host_stack(P, t, 365.25, n, nan, seed=400 + i)
ref = bo.monitor_masked(y, t, n, h, k, 365.25, 3.0, keep_mosum=True)
cfg = pkg.MonitorConfig(history=n, bandwidth=h, harmonics=k, freq=365.25, crit_value=3.0, nan_mode="mask")
bm = pkg.monitor_batch(pkg.SeriesStack(y, pkg.TimeAxis(t)), cfg, return_beta=True, keep_mosum=True)
v = ref.valid
err = np.abs(bm.max_abs_mo - ref.max_abs_mo) / np.maximum(ref.max_abs_mo, 1e-30)
bad = np.flatnonzero(v & (err > 1e-4))
print("valid eq", np.array_equal(bm.valid, ref.valid), "max err", err[v].max(), "bad", bad[:20], err[bad][:10])
for px in bad[:3]:
    bk, br = bm.beta[:, px], ref.beta[:, px]
    print("px", px, "beta rel err", np.max(np.abs(bk - br) / (np.abs(br) + 1e-12)), "beta", br[:4], bk[:4])
    mk, mr = bm.mosum[:, px], ref.mosum[:, px]
    ok = np.isfinite(mr)
    print("   mosum ratio", (mk[ok] / mr[ok])[:8], "diff", (mk[ok] - mr[ok])[:8])
