"""C1-sized libbwm calls for compute-sanitizer (tests/test_gpu_sanitizer.py): the fill kernels
(TMA tiles + LDG tail + float64 fixup + finalize), the masked kernel and the host pipeline."""
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
torch.cuda.synchronize()
print("sanitize workload ok")
