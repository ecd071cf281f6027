"""Where the C2 end-to-end step goes: profile_run phases over a pinned C2 stack (1 GPU).

    python experiments/e2e_phases.py [steps]
"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1807_01751_b200 import MonitorConfig, SeriesStack, TimeAxis, monitor_batch, profile_run  # noqa: E402
from paper_1807_01751_b200.synth import WORKLOADS, device_stack, time_axis  # noqa: E402

w = WORKLOADS["C2"]
t = time_axis(w)
y = device_stack(w.n_pixels, t, w.freq, w.n_hist, w.nan_frac, seed=1, device=torch.device("cuda", 0))
host = torch.empty(tuple(y.shape), dtype=torch.float32, pin_memory=True)
host.copy_(y)
del y
torch.cuda.empty_cache()
stack = SeriesStack(host.numpy(), TimeAxis(t))
cfg = MonitorConfig(history=w.n_hist, bandwidth=w.bandwidth, harmonics=w.harmonics, freq=w.freq, crit_value=w.crit)
monitor_batch(stack, cfg)
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
for _ in range(steps):
    t0 = time.perf_counter()
    _, ph = profile_run(stack, cfg)
    wall = time.perf_counter() - t0
    print(f"wall {wall*1e3:7.1f} ms | " + " ".join(f"{k} {getattr(ph, k)*1e3:.1f}" for k in
                                              ("ingest", "model", "mosum", "breaks", "total")))
walls = []
for _ in range(steps):
    t0 = time.perf_counter()
    bm = monitor_batch(stack, cfg)
    walls.append((time.perf_counter() - t0) * 1e3)
print("monitor_batch wall ms:", " ".join(f"{x:.1f}" for x in walls))
