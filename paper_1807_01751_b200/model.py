"""Season-trend design and the shared history mapping — host setup in float64.

These run once per batch geometry on the host, exactly as in the reference
(pkg/src/breakwatch/model.py): they are the constants of the hot path, not part of it.
The per-pixel contraction they feed runs in libbwm (csrc/bwm_kernel_tma.cuh).

Reference anchors:
  TimeAxis            model.py:23-45   strictly increasing, finite, >= 2 stamps
  regular_axis        model.py:48-50   1..N
  build_design_matrix model.py:90-110  rows 1, t, sin(2 pi j t/f), cos(2 pi j t/f)
  fit_mapping         model.py:118-152 Gram + cond <= 1e12 + Cholesky, pinv(1e-10)
                                       fallback, identity gap <= 1e-9
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.linalg import LinAlgError, cho_factor, cho_solve

from .errors import DegreesOfFreedomError, RankDeficiencyError

GRAM_CONDITION_LIMIT = 1e12
PINV_RELATIVE_CUTOFF = 1e-10
MAPPING_IDENTITY_TOL = 1e-9


@dataclass(frozen=True)
class TimeAxis:
    """Strictly increasing observation time stamps (model.py:23-45)."""

    values: np.ndarray

    def __post_init__(self):
        v = np.asarray(self.values, dtype=np.float64)
        if v.ndim != 1 or v.size < 2:
            raise ValueError("time axis needs at least two observations")
        if not np.isfinite(v).all():
            raise ValueError("time axis values must be finite")
        if not (np.diff(v) > 0).all():
            raise ValueError("time axis must be strictly increasing")
        object.__setattr__(self, "values", v)

    def __len__(self) -> int:
        return int(self.values.size)


def regular_axis(n_obs: int) -> TimeAxis:
    """Evenly sampled axis 1, 2, ..., n_obs (model.py:48-50)."""
    return TimeAxis(np.arange(1.0, n_obs + 1.0))


@dataclass(frozen=True)
class DesignMatrix:
    """Season-trend regressors, one column per observation: (2 + 2k, N)."""

    matrix: np.ndarray
    freq: float
    harmonics: int

    @property
    def n_params(self) -> int:
        return 2 + 2 * self.harmonics

    @property
    def n_obs(self) -> int:
        return int(self.matrix.shape[1])


@dataclass(frozen=True)
class MappingMatrix:
    """coefficients = matrix @ y_history, shared by every series on one axis."""

    matrix: np.ndarray
    n_history: int


def _trend_rows(t: np.ndarray, freq: float, harmonics: int, trend: np.ndarray) -> np.ndarray:
    out = np.empty((2 + 2 * harmonics, t.size))
    out[0] = 1.0
    out[1] = trend
    for j in range(1, harmonics + 1):
        w = (2.0 * np.pi * j / freq) * t
        out[2 * j] = np.sin(w)
        out[2 * j + 1] = np.cos(w)
    return out


def build_design_matrix(axis, freq: float, harmonics: int) -> DesignMatrix:
    """Intercept, raw-axis trend and `harmonics` sin/cos pairs (model.py:90-110)."""
    if harmonics < 1:
        raise ValueError("harmonics must be >= 1")
    if freq <= 0:
        raise ValueError("freq must be positive")
    if not isinstance(axis, TimeAxis):
        axis = TimeAxis(axis)
    t = axis.values
    return DesignMatrix(_trend_rows(t, freq, harmonics, t), float(freq), int(harmonics))


def _identity_gap(mapping: np.ndarray, hist: np.ndarray) -> float:
    return float(np.abs(mapping @ hist.T - np.eye(mapping.shape[0])).max())


def _solve_mapping(hist: np.ndarray) -> tuple[np.ndarray, float]:
    """(X_h X_h^T)^-1 X_h by Cholesky when well conditioned, else SVD pseudo-inverse."""
    gram = hist @ hist.T
    mapping = None
    if np.linalg.cond(gram) <= GRAM_CONDITION_LIMIT:
        try:
            mapping = cho_solve(cho_factor(gram), hist)
        except LinAlgError:
            mapping = None
    if mapping is None or _identity_gap(mapping, hist) > MAPPING_IDENTITY_TOL:
        mapping = np.linalg.pinv(hist.T, rcond=PINV_RELATIVE_CUTOFF)
    return np.ascontiguousarray(mapping), _identity_gap(mapping, hist)


def fit_mapping(design: DesignMatrix, n_history: int) -> MappingMatrix:
    """Solve the history normal equations once (model.py:118-152), same error contract."""
    p = design.n_params
    if n_history <= p:
        raise DegreesOfFreedomError(
            f"history of {n_history} cannot identify {p} coefficients; need n > {p}"
        )
    if n_history > design.n_obs:
        raise ValueError("history length exceeds the design matrix")
    mapping, gap = _solve_mapping(design.matrix[:, :n_history])
    if gap > MAPPING_IDENTITY_TOL:
        raise RankDeficiencyError(f"history design is rank deficient (identity gap {gap:.3e})")
    return MappingMatrix(mapping, int(n_history))


@dataclass(frozen=True)
class KernelBasis:
    """Constants handed to libbwm (include/bwm.h, struct bwm_tables).

    The kernel fits the same model in the basis where the trend regressor is
    (t - trend_center) / trend_scale — an invertible reparametrisation, so fitted values,
    residuals, sigma and MOSUM are unchanged in exact arithmetic, while the float32
    contraction over the history stays well conditioned.
    """

    mapping: np.ndarray      # (p, n)  float64, C-contiguous
    design: np.ndarray       # (p, N)  float64, C-contiguous
    trend_center: float
    trend_scale: float


def kernel_basis(axis: TimeAxis, freq: float, harmonics: int, n_history: int) -> KernelBasis:
    """Centred-trend design/mapping for the device.  Call after fit_mapping succeeded on the
    raw design (the reference's error contract is decided there)."""
    t = axis.values
    th = t[:n_history]
    center = 0.5 * (th[0] + th[-1])
    scale = 0.5 * (th[-1] - th[0])
    if not scale > 0:
        scale = 1.0
    rows = _trend_rows(t, freq, harmonics, (t - center) / scale)
    mapping, _ = _solve_mapping(rows[:, :n_history])
    return KernelBasis(np.ascontiguousarray(mapping), np.ascontiguousarray(rows), float(center), float(scale))
