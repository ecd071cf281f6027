import time, numpy as np, torch, sys
sys.path.insert(0, "/root/repo")
from paper_1807_01751_b200 import MonitorConfig, SeriesStack, TimeAxis, monitor_batch
from paper_1807_01751_b200.synth import WORKLOADS, device_stack, time_axis
w = WORKLOADS["C2"]; t = time_axis(w)
y = device_stack(w.n_pixels, t, w.freq, w.n_hist, w.nan_frac, seed=1, device="cuda")
pin = torch.empty(y.shape, dtype=torch.float32, pin_memory=True); pin.copy_(y)
pag = np.empty(y.shape, dtype=np.float32); pag[...] = pin.numpy()
del y; torch.cuda.empty_cache()
cfg = MonitorConfig(history=w.n_hist, bandwidth=w.bandwidth, harmonics=w.harmonics, freq=w.freq, crit_value=w.crit)
for name, arr in (("pinned", pin.numpy()), ("pageable", pag)):
    st = SeriesStack(arr, TimeAxis(t))
    monitor_batch(st, cfg)
    t0 = time.perf_counter()
    for _ in range(2): bm = monitor_batch(st, cfg)
    dt = (time.perf_counter() - t0) / 2
    print(name, f"{dt*1e3:.1f} ms  {arr.nbytes/dt/1e9:.1f} GB/s  {w.n_pixels/dt/1e6:.1f} Mpix/s", flush=True)
