import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_1807_01751_b200 as pkg
from paper_1807_01751_b200.synth import host_stack
from oracle import bfast_oracle as bo
for (i, N, n, h, k, P, nan, irr) in [(16, 313, 20, 5, 2, 2704, 0.2, True)]:
    rng = np.random.default_rng(100 + i)
    t = np.cumsum(rng.uniform(1, 9, N)) + 1.0 if irr else np.arange(1.0, N + 1.0)
    freq = 365.25 if irr else 23.0
    y = host_stack(P, t, freq, n, nan, seed=200 + i)
    cfg = pkg.MonitorConfig(history=n, bandwidth=h, harmonics=k, freq=freq, crit_value=3.0)
    ref = bo.monitor(y, t, n, h, k, freq, 3.0, keep_mosum=True, want_beta=True)
    bm = pkg.monitor_batch(pkg.SeriesStack(y, pkg.TimeAxis(t)), cfg, keep_mosum=True, return_beta=True)
    ok = ref.valid
    rel = np.abs(bm.max_abs_mo - ref.max_abs_mo) / np.maximum(ref.max_abs_mo, 1e-30)
    worst = np.argsort(-np.where(ok, rel, 0))[:3]
    print("case", i, "max rel err max_abs", rel[ok].max(), "worst px", worst, rel[worst])
    # sigma ratio: MO = acc/(sigma sqrt n): compare mosum columns
    for px in worst[:2]:
        r = bm.mosum[:, px] / ref.mosum[:, px]
        print("  px", px, "mosum ratio min/max", np.nanmin(r), np.nanmax(r), "sigma_ref", ref.sigma[px] if ref.sigma is not None else None)
        d = np.abs(bm.mosum[:, px] - ref.mosum[:, px])
        j = np.argmax(d); print("  max abs diff at j", j, bm.mosum[j, px], ref.mosum[j, px])
        print("  beta rel", np.abs(bm.beta[:, px] - ref.beta[:, px]) / (np.abs(ref.beta[:, px]) + 1e-12))
