"""Where an end-to-end monitor_batch step spends its time (C2, pinned host stack)."""
import time

import numpy as np
import torch

from paper_1807_01751_b200 import MonitorConfig, SeriesStack, TimeAxis, monitor_batch, profile_run
from paper_1807_01751_b200.synth import WORKLOADS, device_stack, time_axis

w = WORKLOADS["C2"]
t = time_axis(w)
y = device_stack(w.n_pixels, t, w.freq, w.n_hist, w.nan_frac, seed=1)
host = torch.empty(y.shape, dtype=torch.float32, pin_memory=True)
host.copy_(y)
del y
torch.cuda.empty_cache()
stack = SeriesStack(host.numpy(), TimeAxis(t))
cfg = MonitorConfig(history=w.n_hist, bandwidth=w.bandwidth, harmonics=w.harmonics, freq=w.freq, crit_value=w.crit)
monitor_batch(stack, cfg)
for _ in range(3):
    t0 = time.perf_counter()
    bm, tm = profile_run(stack, cfg)
    wall = time.perf_counter() - t0
    print(f"wall {wall*1e3:7.1f} ms | ingest(H2D+D2H) {tm.ingest*1e3:7.1f} model {tm.model*1e3:6.1f} "
          f"kernel {tm.mosum*1e3:6.1f} breaks {tm.breaks*1e3:6.1f} total {tm.total*1e3:7.1f}")
from paper_1807_01751_b200.device import DevicePlan
plan = DevicePlan.get(stack.time_axis, cfg.freq, cfg.harmonics, cfg.history, cfg.bandwidth, cfg.crit_value)
for _ in range(2):
    t0 = time.perf_counter()
    r = plan.run_host(stack.data, ref_dtypes=True)
    print(f"run_host wall {(time.perf_counter()-t0)*1e3:7.1f} ms, lib total {r.total_ms:7.1f} kernel {r.kernel_ms:6.2f}"
          f" h2d {r.h2d_bytes/1e9:.2f} GB d2h {r.d2h_bytes/1e6:.0f} MB")
