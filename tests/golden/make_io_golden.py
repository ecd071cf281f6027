"""Golden vectors for the I/O surfaces, made by running the REFERENCE in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_io_golden.py

  io_generate.bts   reference `generate` (synth.py:65-105) + write_stack (dataio.py:44-71) for
                    SynthSpec(m=300, N=60, freq=23, noise_std=0.02, break_mag=0.5, seed=5)
  io_axis.bts       a small stack with an irregular (explicit) axis and NaN/Inf samples
  io_breaks.npz/csv a break map with edge-case magnitudes and the reference's
                    write_break_map output (dataio.py:168-182) for it
The GPU box has no /root/reference; the tests compare against these files.
"""
from pathlib import Path

import numpy as np
from breakwatch import BreakMap, MonitorConfig, SeriesStack, TimeAxis, write_break_map, write_stack
from breakwatch.synth import SynthSpec, generate

HERE = Path(__file__).resolve().parent

stack, _ = generate(SynthSpec(n_pixels=300, n_obs=60, freq=23.0, noise_std=0.02, break_mag=0.5, seed=5))
write_stack(stack, HERE / "io_generate.bts")

rng = np.random.default_rng(3)
y = rng.normal(size=(12, 7)).astype(np.float32)
y[2, 1] = np.nan
y[5, 3] = np.inf
y[7, 0] = -np.inf
axis = TimeAxis(np.cumsum(rng.uniform(1, 9, size=12)))
write_stack(SeriesStack(y, axis), HERE / "io_axis.bts")

P = 64
mx = np.concatenate([
    [0.0, 1e-5, 1.5e-7, 123456789.0, 1.23456789e16, 2.5, 3.0, 0.1, 1 / 3, 2 / 3, 1e300, 5e-324, 65504.0,
     4.892936439219294, 0.5, 1e-10],
    np.abs(rng.standard_cauchy(P - 16)),
])
fb = np.where(rng.random(P) < 0.5, rng.integers(101, 200, P), 0).astype(np.int64)
valid = rng.random(P) < 0.9
fb[~valid] = 0
mx[~valid] = 0.0
bm = BreakMap(detected=fb > 0, first_break=fb, max_abs_mo=mx, valid=valid,
              config=MonitorConfig(history=100, bandwidth=50, harmonics=3, freq=23.0), crit_value=4.9)
np.savez(HERE / "io_breaks.npz", detected=fb > 0, first_break=fb, max_abs_mo=mx, valid=valid)
write_break_map(bm, HERE / "io_breaks.csv")
print("wrote io_generate.bts io_axis.bts io_breaks.npz io_breaks.csv")
