"""C1-sized libbwm calls for compute-sanitizer (tests/test_gpu_sanitizer.py): the fill kernels
(TMA tiles + LDG tail + float64 fixup + finalize), the lagging-cursor TMA kernels (16-warp CTAs
with smem tables; tables through L1 for long series), the masked kernel, the host pipeline and
the device null draws of critical_value."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1807_01751_b200 as pkg  # noqa: E402
from paper_1807_01751_b200.synth import host_stack  # noqa: E402

N, n, h, k, f, crit = 228, 114, 28, 3, 23.0, 2.96519227
t = np.arange(1.0, N + 1)
y = host_stack(128 * 128 + 100, t, f, n, 0.2, seed=5)
axis = pkg.TimeAxis(t)
for mode in ("fill", "mask"):
    cfg = pkg.MonitorConfig(history=n, bandwidth=h, harmonics=k, freq=f, crit_value=crit, nan_mode=mode)
    bm = pkg.monitor_batch(pkg.SeriesStack(torch.as_tensor(y, device="cuda"), axis), cfg, keep_mosum=True,
                           return_beta=True, return_mean=True)
    bl = pkg.monitor_batch(pkg.SeriesStack(torch.as_tensor(y, device="cuda"), axis), cfg)   # LEAN variant
    bh = pkg.monitor_batch(pkg.SeriesStack(y, axis), cfg)                                   # host pipeline
    assert np.array_equal(bh.first_break, bl.first_break)
# lagging cursor (h > 120): 16-warp CTAs with the window-sum table in smem, and (long series)
# the table read through L1; P = 2 tiles of 1,024 px + an LDG tail
tl = np.cumsum(np.random.default_rng(3).uniform(1, 9, 1000)) + 1.0
yl = host_stack(2 * 1024 + 77, tl, 365.25, 500, 0.5, seed=6)
cfg = pkg.MonitorConfig(history=500, bandwidth=250, harmonics=6, freq=365.25, crit_value=3.0)
for kw in (dict(), dict(keep_mosum=True, return_mean=True)):
    pkg.monitor_batch(pkg.SeriesStack(torch.as_tensor(yl, device="cuda"), pkg.TimeAxis(tl)), cfg, **kw)
t2 = np.cumsum(np.random.default_rng(4).uniform(1, 9, 2600)) + 1.0
y2 = host_stack(300, t2, 365.25, 1300, 0.3, seed=7)
cfg = pkg.MonitorConfig(history=1300, bandwidth=400, harmonics=6, freq=365.25, crit_value=3.0)
pkg.monitor_batch(pkg.SeriesStack(torch.as_tensor(y2, device="cuda"), pkg.TimeAxis(t2)), cfg)
# lambda: device null draws + the sup_stat launch
pkg.critical_value(pkg.CriticalValueRequest(alpha=0.05, h_frac=0.5, horizon=2.0, n_sim=100, reps=2000, seed=1))
torch.cuda.synchronize()
print("sanitize workload ok")
