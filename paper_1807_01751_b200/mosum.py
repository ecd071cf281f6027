"""MOSUM boundary and critical value — host setup (reference pkg/src/breakwatch/mosum.py).

``log_plus`` and ``boundary_values`` are the per-geometry constants the kernel compares
against (mosum.py:27-32, 68-79).  ``critical_value`` is the Monte Carlo calibration of
lambda (mosum.py:166-227): the null draws come from the same per-replication Philox
substreams as the reference, and the replications run through the same fused GPU kernel
as the data (libbwm), so there is no CPU MOSUM in this package.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .errors import DegreesOfFreedomError

REPLICATION_BLOCK = 2048


def log_plus(x) -> np.ndarray:
    """1 for x <= e, natural log above (mosum.py:27-32)."""
    x = np.asarray(x, dtype=np.float64)
    return np.where(x > np.e, np.log(np.maximum(x, np.e)), 1.0)


def boundary_values(n_history: int, n_obs: int, crit_value: float) -> np.ndarray:
    """crit * sqrt(log_plus(t/n)) for observation counts t = n+1..N (mosum.py:68-79)."""
    if n_obs <= n_history:
        raise ValueError("need at least one monitored observation (n < N)")
    if crit_value <= 0:
        raise ValueError("critical value must be positive")
    t = np.arange(n_history + 1, n_obs + 1, dtype=np.float64)
    return crit_value * np.sqrt(log_plus(t / n_history))


@dataclass(frozen=True)
class BreakResult:
    """Monitoring outcome of one series (mosum.py:101-111)."""

    detected: bool
    first_break: Optional[int]
    max_abs_mo: float


@dataclass(frozen=True)
class CriticalValueRequest:
    """Monte Carlo calibration request (mosum.py:125-163), same validation."""

    alpha: float
    h_frac: float
    horizon: float
    n_sim: int
    reps: int
    seed: int
    harmonics: int = 3
    freq: float = 23.0

    def __post_init__(self):
        if not 0.0 < self.alpha < 1.0:
            raise ValueError("alpha must lie in (0, 1)")
        if not 0.0 < self.h_frac <= 1.0:
            raise ValueError("h_frac must lie in (0, 1]")
        if not self.horizon > 1.0:
            raise ValueError("monitoring horizon must exceed 1")
        if self.reps < 1000:
            raise ValueError("need at least 1000 replications")
        if not 0 <= self.seed < 2**64:
            raise ValueError("seed must be an unsigned 64-bit integer")
        if self.harmonics < 1:
            raise ValueError("harmonics must be >= 1")
        if self.freq <= 0:
            raise ValueError("freq must be positive")
        if self.n_sim <= 2 + 2 * self.harmonics:
            raise DegreesOfFreedomError(
                f"n_sim must exceed the coefficient count ({2 + 2 * self.harmonics})"
            )


def null_draws(request: CriticalValueRequest, start: int, stop: int, n_obs: int) -> np.ndarray:
    """Standard-normal draws of replications [start, stop), time-major (n_obs, width).

    Replication r uses Philox(key=seed, counter=r << 128), exactly the reference's
    substreams (mosum.py:195-198), so results do not depend on batching.
    """
    out = np.empty((n_obs, stop - start))
    for j in range(stop - start):
        rng = np.random.Generator(np.random.Philox(key=request.seed, counter=(start + j) << 128))
        out[:, j] = rng.standard_normal(n_obs)
    return out


def critical_value(request: CriticalValueRequest, threads: int = 1, device=None) -> float:
    """(1 - alpha) quantile of sup_t |MO_t| / sqrt(log_plus(t/n)) under the null.

    Same geometry rules as the reference (mosum.py:166-227): regular axis 1..N with
    N = round(horizon * n_sim), h = round(h_frac * n_sim), the full season-trend fit per
    replication.  The replications are monitored on the GPU by libbwm (keep_mosum), so
    the statistic sees float32 residual arithmetic: agreement with the float64 reference
    is ~1e-6 relative, not bit-exact.
    """
    from concurrent.futures import ThreadPoolExecutor

    from .device import DevicePlan

    import torch

    n_hist = request.n_sim
    n_obs = int(round(request.horizon * n_hist))
    bandwidth = int(round(request.h_frac * n_hist))
    if n_obs <= n_hist:
        raise ValueError("horizon too small: no monitor period to simulate")
    if bandwidth < 1:
        raise ValueError("h_frac too small: bandwidth rounds to zero")
    from .model import regular_axis

    axis = regular_axis(n_obs)
    # unit boundary: the kernel's own crossing test is irrelevant here; only MO is kept
    plan = DevicePlan.get(axis, request.freq, request.harmonics, n_hist, bandwidth, 1.0, device)
    t = np.arange(n_hist + 1, n_obs + 1, dtype=np.float64)
    inv_shape = torch.as_tensor(1.0 / np.sqrt(log_plus(t / n_hist)), dtype=torch.float32,
                                device=plan.torch_device)[:, None]
    blocks = [(s, min(s + REPLICATION_BLOCK, request.reps)) for s in range(0, request.reps, REPLICATION_BLOCK)]
    sup = np.empty(request.reps)

    def draws(block):
        return null_draws(request, block[0], block[1], n_obs).astype(np.float32)

    with ThreadPoolExecutor(max_workers=max(1, threads)) as pool:
        for (start, stop), y in zip(blocks, pool.map(draws, blocks)):
            res = plan.run_device(torch.as_tensor(y, device=plan.torch_device), keep_mosum=True)
            if res.zero_sigma is not None:
                from .errors import ZeroResidualError

                raise ZeroResidualError("a simulated null series produced a zero residual scale")
            stat = (res.mosum.abs() * inv_shape).amax(dim=0)
            sup[start:stop] = stat.double().cpu().numpy()
    return float(np.quantile(sup, 1.0 - request.alpha))
