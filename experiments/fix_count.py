"""How many pixels the float64 fixup re-evaluates on the bench workloads (fix_ratio default)."""
import sys, ctypes as C, torch
sys.path.insert(0, "/root/repo")
from paper_1807_01751_b200 import TimeAxis
from paper_1807_01751_b200.device import DevicePlan
from paper_1807_01751_b200.synth import WORKLOADS, device_stack, time_axis
for name in ("C2", "C5", "C4"):
    w = WORKLOADS[name]; t = time_axis(w)
    plan = DevicePlan(TimeAxis(t), w.freq, w.harmonics, w.n_hist, w.bandwidth, w.crit, "cuda")
    y = device_stack(w.n_pixels, t, w.freq, w.n_hist, w.nan_frac, seed=20261017, device="cuda")
    plan.run_device(y); torch.cuda.synchronize()
    # read the plan's device-side count through a tiny ctypes peek is not exposed: time with and without instead
    import time, os
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(); [plan.run_device(y, check_zero=False) for _ in range(10)]; ev[1].record(); torch.cuda.synchronize()
    print(name, "ms/step", ev[0].elapsed_time(ev[1]) / 10, flush=True)
    del y, plan; torch.cuda.empty_cache()
