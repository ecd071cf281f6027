"""MOSUM boundary and critical value — host setup (reference pkg/src/breakwatch/mosum.py).

``log_plus`` and ``boundary_values`` are the per-geometry constants the kernel compares
against (mosum.py:27-32, 68-79).  ``critical_value`` is the Monte Carlo calibration of
lambda (mosum.py:166-227), entirely on the device: libbwm draws every replication's null
series from the reference's own per-replication Philox substreams (bwm_null_draws: numpy's
Philox4x64-10 + ziggurat restated bit for bit, one thread per replication, straight into a
time-major stack), and ALL replications run as one stack through the same fused kernel as the
data, which emits the per-replication statistic sup_j |MO_j| / sqrt(log_plus) directly
(bwm_outputs.sup_stat) — no host draws, no MOSUM matrix, no CPU MOSUM in this package.
``null_draws`` is the host restatement of the same streams (numpy), kept for the checks.
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


def null_draws(request: CriticalValueRequest, start: int, stop: int, n_obs: int,
               dtype=np.float64, out: Optional[np.ndarray] = None) -> np.ndarray:
    """Standard-normal draws of replications [start, stop), time-major (n_obs, width).

    Replication r uses Philox(key=seed, counter=r << 128), exactly the reference's
    substreams (mosum.py:195-198), so results do not depend on batching.  One bit generator
    is re-keyed per replication by resetting its counter state (the same stream as a fresh
    ``Philox(key, counter)``: the 4-word buffer is emptied), half the cost of constructing
    a generator per replication.  ``out`` (n_obs, stop - start) receives the draws cast to
    its dtype (float32 for the kernel).
    """
    width = stop - start
    if out is None:
        out = np.empty((n_obs, width), dtype=dtype)
    bg = np.random.Philox(key=request.seed)
    gen = np.random.Generator(bg)
    state = bg.state
    mask = (1 << 64) - 1
    for j in range(width):
        c = (start + j) << 128
        state["state"]["counter"][:] = [(c >> (64 * i)) & mask for i in range(4)]
        state["buffer_pos"] = 4
        state["has_uint32"] = 0
        bg.state = state
        out[:, j] = gen.standard_normal(n_obs)
    return out


def critical_value(request: CriticalValueRequest, threads: int = 1, device=None) -> float:
    """(1 - alpha) quantile of sup_t |MO_t| / sqrt(log_plus(t/n)) under the null.

    Same geometry rules as the reference (mosum.py:166-227): regular axis 1..N with
    N = round(horizon * n_sim), h = round(h_frac * n_sim), the full season-trend fit per
    replication.  The draws are the reference's (bit-identical Philox substreams), generated
    on the device in float32 — the dtype the monitor kernel reads; one libbwm launch over all
    replications emits each one's statistic (sup_stat), so the statistic sees float32 residual
    arithmetic: agreement with the float64 reference is ~1e-6 relative, not bit-exact.
    `threads` is accepted for the reference signature and unused (no host work).
    """
    import ctypes as C

    import torch

    from . import _lib
    from .device import DevicePlan

    del threads
    n_hist = request.n_sim
    n_obs = int(round(request.horizon * n_hist))
    bandwidth = int(round(request.h_frac * n_hist))
    if n_obs <= n_hist:
        raise ValueError("horizon too small: no monitor period to simulate")
    if bandwidth < 1:
        raise ValueError("h_frac too small: bandwidth rounds to zero")
    from .model import regular_axis

    axis = regular_axis(n_obs)
    # unit lambda: bound_j = sqrt(log_plus((n+1+j)/n)), so sup_stat is the reference statistic
    plan = DevicePlan.get(axis, request.freq, request.harmonics, n_hist, bandwidth, 1.0, device)
    dev = plan.torch_device
    y = torch.empty((n_obs, request.reps), dtype=torch.float32, device=dev)
    seed = int(request.seed)
    with torch.cuda.device(dev):
        stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        _lib.check(plan._lib.bwm_null_draws(seed & ((1 << 64) - 1), seed >> 64, 0, request.reps, n_obs,
                                            y.data_ptr(), request.reps, stream), "bwm_null_draws")
    res = plan.run_device(y, sup=True)
    if res.zero_sigma is not None:
        from .errors import ZeroResidualError

        raise ZeroResidualError("a simulated null series produced a zero residual scale")
    sup = res.sup.double().cpu().numpy()
    return float(np.quantile(sup, 1.0 - request.alpha))
