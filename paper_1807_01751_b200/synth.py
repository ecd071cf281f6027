"""Synthetic NDVI-like stacks for tests and benchmarks.

  y = 0.5 + 0.2 sin(2 pi t / f + phi_px) + 1e-5 t + eps,   eps ~ N(0, 0.03^2)
  half the pixels get a level drop c ~ U(-0.3, -0.1) from a random monitoring date on,
  missing samples: i.i.d. Bernoulli(nan_frac), or clustered "cloud" discs per date,
  plus a small fraction of dead (all-NaN) pixels.

Two generators with the same recipe: ``host_stack`` (numpy, seeded PCG64; used by the
tests so a fixture can be regenerated bit-for-bit) and ``device_stack`` (torch on the GPU,
seeded Philox; used by bench.py for multi-GB stacks).  They are statistically equal, not
bitwise equal.  Irregular axes follow §8(d): days since the first acquisition, i.i.d.
U(lo, hi) gaps.  The reference's own generator (synth.py:65-105) is not NDVI-like (mean 0).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json configuration."""

    name: str
    rows: int            # image rows
    cols: int            # image cols  -> n_pixels = rows * cols
    n_obs: int
    n_hist: int
    harmonics: int
    bandwidth: int
    freq: float
    nan_frac: float
    axis: str = "regular"      # "regular" | "irregular"
    gap: tuple = (1.0, 9.0)    # irregular spacing U(lo, hi) days
    clustered: bool = False
    crit: Optional[float] = None

    @property
    def n_pixels(self) -> int:
        return self.rows * self.cols


# BASELINE.json "configs" (SURVEY.md §8 shorthand C1..C5).  lambda for C1-C3 is the
# reference's resolve_crit_value at (n=114, h=28, k=3, f=23) measured in SURVEY §8(d).
WORKLOADS = {
    "C1": Workload("C1", 128, 128, 228, 114, 3, 28, 23.0, 0.20, crit=2.96519227),
    "C2": Workload("C2", 4096, 4096, 228, 114, 3, 28, 23.0, 0.20, crit=2.96519227),
    "C3": Workload("C3", 16384, 16384, 228, 114, 3, 28, 23.0, 0.20, crit=2.96519227),
    "C4": Workload("C4", 2048, 2048, 1000, 500, 6, 250, 365.25, 0.50, axis="irregular", gap=(1.0, 9.0), crit=3.0),
    "C5": Workload("C5", 7000, 7000, 400, 200, 3, 50, 365.25, 0.19, axis="irregular", gap=(8.0, 24.0),
                   clustered=True, crit=3.0),
}


def time_axis(w: Workload, seed: int = 20261017) -> np.ndarray:
    if w.axis == "regular":
        return np.arange(1.0, w.n_obs + 1.0)
    rng = np.random.default_rng(seed)
    gaps = rng.uniform(w.gap[0], w.gap[1], w.n_obs - 1)
    return np.concatenate([[1.0], 1.0 + np.cumsum(gaps)])


def host_stack(n_pixels: int, t: np.ndarray, freq: float, n_hist: int, nan_frac: float, seed: int,
               clustered: bool = False, dead_frac: float = 1e-4, cols: Optional[int] = None) -> np.ndarray:
    """float32 (N, P) NDVI-like stack on the host (numpy)."""
    rng = np.random.default_rng(seed)
    N = t.size
    phi = rng.uniform(0.0, 2.0 * np.pi, n_pixels)
    y = 0.5 + 0.2 * np.sin(2.0 * np.pi * t[:, None] / freq + phi[None, :]) + 1e-5 * t[:, None]
    y += rng.normal(0.0, 0.03, (N, n_pixels))
    brk = rng.random(n_pixels) < 0.5
    start = rng.integers(n_hist, N, n_pixels)
    drop = rng.uniform(-0.3, -0.1, n_pixels)
    y += ((np.arange(N)[:, None] >= start[None, :]) & brk[None, :]) * drop[None, :]
    y = y.astype(np.float32)
    if clustered:
        y[_cloud_mask(rng, N, n_pixels, cols or int(np.sqrt(n_pixels)))] = np.nan
    else:
        y[rng.random((N, n_pixels)) < nan_frac] = np.nan
    dead = rng.random(n_pixels) < dead_frac
    y[:, dead] = np.nan
    return y


def _cloud_mask(rng, N: int, P: int, cols: int) -> np.ndarray:
    """Per-date random discs (radius U(20,150) px, 0-5 per 512^2 area), §8(d) C5."""
    rows = (P + cols - 1) // cols
    mask = np.zeros((N, P), dtype=bool)
    rr, cc = np.divmod(np.arange(P), cols)
    per = max(1.0, rows * cols / 512.0**2)
    for d in range(N):
        for _ in range(rng.integers(0, int(round(5 * per)) + 1)):
            r0, c0 = rng.uniform(0, rows), rng.uniform(0, cols)
            rad = rng.uniform(20, 150)
            mask[d] |= (rr - r0) ** 2 + (cc - c0) ** 2 <= rad * rad
    return mask


def cloud_discs(n_obs: int, rows: int, cols: int, seed: int) -> list:
    """Per-date cloud discs of a rows x cols scene, §8(d) C5: 0-5 discs per 512^2 area per
    date (scaled to the scene), centres uniform over the scene, radius U(20, 150) px.  Drawn
    from the SCENE seed on the host, so every rank's pixel band sees the same clouds.
    Returns one float64 array [k, 3] (row, col, radius) per date."""
    rng = np.random.default_rng(seed)
    per = max(1.0, rows * cols / 512.0**2)
    out = []
    for _ in range(n_obs):
        k = int(rng.integers(0, int(round(5 * per)) + 1))
        out.append(np.stack([rng.uniform(0, rows, k), rng.uniform(0, cols, k), rng.uniform(20, 150, k)], axis=1))
    return out


def _apply_clouds(y, discs, cols: int, first_pixel: int):
    """NaN every pixel of the band [first_pixel, first_pixel + P) of a row-major scene that lies
    inside a disc of its date: each disc's 301x301 bounding box is tested on the device."""
    import torch

    dev = y.device
    P = int(y.shape[1])
    g0, g1 = first_pixel, first_pixel + P
    r_lo, r_hi = g0 // cols, (g1 - 1) // cols
    off = torch.arange(-150, 151, device=dev, dtype=torch.float64)
    dr, dc = torch.meshgrid(off, off, indexing="ij")
    dr, dc = dr.reshape(-1), dc.reshape(-1)
    for d, disc in enumerate(discs):
        keep = (disc[:, 0] + disc[:, 2] >= r_lo) & (disc[:, 0] - disc[:, 2] <= r_hi + 1)
        disc = disc[keep]
        for c0 in range(0, len(disc), 256):                     # bound the candidate tensor
            q = torch.as_tensor(disc[c0:c0 + 256], device=dev)
            rr = torch.floor(q[:, 0:1]) + dr[None, :]           # candidate pixel rows / cols
            cc = torch.floor(q[:, 1:2]) + dc[None, :]
            inside = ((rr - q[:, 0:1]) ** 2 + (cc - q[:, 1:2]) ** 2 <= q[:, 2:3] ** 2) & (cc >= 0) & (cc < cols)
            gidx = (rr * cols + cc)[inside].long() - first_pixel
            gidx = gidx[(gidx >= 0) & (gidx < P)]
            y[d].index_fill_(0, gidx, float("nan"))
    return y


def device_stack(n_pixels: int, t: np.ndarray, freq: float, n_hist: int, nan_frac: float, seed: int,
                 device="cuda", out=None, chunk: int = 1 << 22, clustered: bool = False,
                 cols: Optional[int] = None, first_pixel: int = 0, scene_rows: Optional[int] = None,
                 scene_seed: int = 20261022):
    """float32 (N, P) NDVI-like stack generated directly in HBM (torch Philox).

    clustered: missing values are the cloud discs of a scene_rows x cols scene (this stack is
    the band [first_pixel, first_pixel + P) of it; the discs come from `scene_seed`, identical
    on every rank) instead of i.i.d. Bernoulli(nan_frac) samples."""
    import torch

    N = t.size
    dev = torch.device(device)
    if out is None:
        out = torch.empty((N, n_pixels), dtype=torch.float32, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    tt = torch.as_tensor(t, dtype=torch.float32, device=dev)[:, None]
    rows = torch.arange(N, device=dev)[:, None]
    for p0 in range(0, n_pixels, chunk):
        w = min(chunk, n_pixels - p0)
        phi = torch.rand(w, generator=g, device=dev) * (2 * np.pi)
        blk = 0.5 + 0.2 * torch.sin(2 * np.pi * tt / freq + phi[None, :]) + 1e-5 * tt
        blk += 0.03 * torch.randn((N, w), generator=g, device=dev)
        brk = torch.rand(w, generator=g, device=dev) < 0.5
        start = torch.randint(n_hist, N, (w,), generator=g, device=dev)
        drop = -0.1 - 0.2 * torch.rand(w, generator=g, device=dev)
        blk += ((rows >= start[None, :]) & brk[None, :]) * drop[None, :]
        if not clustered:
            blk[torch.rand((N, w), generator=g, device=dev) < nan_frac] = float("nan")
        dead = torch.rand(w, generator=g, device=dev) < 1e-4
        blk[:, dead] = float("nan")
        out[:, p0:p0 + w] = blk
    if clustered:
        cols = cols or int(np.sqrt(first_pixel + n_pixels))
        scene_rows = scene_rows or (first_pixel + n_pixels + cols - 1) // cols
        _apply_clouds(out, cloud_discs(N, scene_rows, cols, scene_seed), cols, first_pixel)
    return out


# ---- the reference's benchmark recipe (CLI `generate` / `bench`) -------------------------
# Restated from its documented contract (reference synth.py:29-105): a sine of amplitude
# 0.05 with period `freq` plus N(0, noise_std^2) noise; the first floor(break_ratio * m)
# pixels get +break_mag over the last floor(break_frac * N) dates.  Pixels are generated
# in 4096-column blocks, block i drawing from Philox(key=seed, counter=i << 128), so files
# written by `generate` are bit-identical to the reference's for the same flags.
SYNTH_AMPLITUDE = 0.05
SYNTH_BLOCK = 4096


@dataclass(frozen=True)
class SynthSpec:
    n_pixels: int
    n_obs: int
    freq: float
    noise_std: float = 0.01
    break_mag: float = 0.1
    break_frac: float = 0.4
    break_ratio: float = 0.5
    seed: int = 0

    def __post_init__(self):
        checks = [
            (self.n_pixels >= 1, "n_pixels must be >= 1"),
            (self.n_obs >= 2, "n_obs must be >= 2"),
            (self.freq > 0, "freq must be positive"),
            (self.noise_std >= 0, "noise_std must be >= 0"),
            (0.0 <= self.break_frac <= 1.0, "break_frac must lie in [0, 1]"),
            (0.0 <= self.break_ratio <= 1.0, "break_ratio must lie in [0, 1]"),
            (0 <= self.seed < 2**64, "seed must be an unsigned 64-bit integer"),
        ]
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)


def generate(spec: SynthSpec, threads: Optional[int] = None):
    """(SeriesStack, truth) for a SynthSpec; deterministic per seed, any thread count."""
    import math
    from concurrent.futures import ThreadPoolExecutor

    from .engine import SeriesStack, resolve_threads
    from .model import regular_axis

    N, m = spec.n_obs, spec.n_pixels
    t = np.arange(1.0, N + 1.0)
    season = SYNTH_AMPLITUDE * np.sin(2.0 * np.pi * t / spec.freq)
    n_break = int(math.floor(spec.break_ratio * m + 1e-9))
    n_shift = int(math.floor(spec.break_frac * N + 1e-9))
    out = np.empty((N, m), dtype=np.float32)

    def block(i):
        a, b = i * SYNTH_BLOCK, min(m, (i + 1) * SYNTH_BLOCK)
        rng = np.random.Generator(np.random.Philox(key=spec.seed, counter=i << 128))
        v = season[:, None] + spec.noise_std * rng.standard_normal((N, b - a))
        k = min(b, n_break) - a
        if k > 0 and n_shift > 0 and spec.break_mag != 0.0:
            v[N - n_shift:, :k] += spec.break_mag
        out[:, a:b] = v

    n_blocks = (m + SYNTH_BLOCK - 1) // SYNTH_BLOCK
    threads = resolve_threads(threads)
    if threads > 1 and n_blocks > 1:
        with ThreadPoolExecutor(max_workers=threads) as pool:
            list(pool.map(block, range(n_blocks)))
    else:
        for i in range(n_blocks):
            block(i)
    return SeriesStack(out, regular_axis(N)), np.arange(m) < n_break


# ---- the reference's scaling benchmark (synth.py:108-149) -----------------------------------
BENCH_CSV_HEADER = "m,ingest,model,predictions,residuals,mosum,breaks,total"


def bench_scaling(m_values, config, template: SynthSpec, threads: Optional[int] = None, sink=None):
    """profile_run of one freshly generated stack per pixel count (reference synth.py:108-135).

    Same contract: lambda is resolved once up front (it depends on the monitoring geometry,
    not on the pixel count), each m gets `generate(replace(template, n_pixels=m))`, and
    (m, PhaseTimings) rows are returned — and written as CSV when a sink is given.  The
    timings are the GPU path's (PhaseTimings: ingest = H2D, mosum = the fused kernel).
    """
    from dataclasses import replace

    from .engine import profile_run, resolve_crit_value, resolve_threads

    m_values = [int(m) for m in m_values]
    if not m_values:
        raise ValueError("need at least one pixel count")
    if any(m < 1 for m in m_values):
        raise ValueError("pixel counts must be >= 1")
    if config.crit_value is None:
        config = replace(config, crit_value=resolve_crit_value(config, template.n_obs, resolve_threads(threads)))
    rows = []
    for m in m_values:
        stack, _ = generate(replace(template, n_pixels=m), threads=threads)
        _, timings = profile_run(stack, config, threads=threads)
        rows.append((m, timings))
    if sink is not None:
        write_bench_csv(rows, sink)
    return rows


def write_bench_csv(rows, sink) -> int:
    """bench_scaling rows as CSV, six decimals per phase (reference synth.py:138-149)."""
    from .dataio import _open

    with _open(sink, "w") as out:
        out.write(BENCH_CSV_HEADER + "\n")
        for m, tm in rows:
            fields = [tm.ingest, tm.model, tm.predictions, tm.residuals, tm.mosum, tm.breaks, tm.total]
            out.write(f"{m}," + ",".join(f"{v:.6f}" for v in fields) + "\n")
    return len(rows)
