"""Batch monitoring over pixel stacks — the drop-in for breakwatch's engine.

Same entry points, arguments and outputs as the reference (pkg/src/breakwatch/engine.py):

  monitor_batch(stack, config, threads=None, block_size=4096, keep_mosum=False) -> BreakMap
  profile_run(stack, config, threads=None, block_size=4096) -> (BreakMap, PhaseTimings)

but the whole fused backend (_fused_phases, engine.py:322-411: ingest/fill, model,
predictions, residuals, mosum, breaks) is one sm_100a kernel launch per pixel chunk in
libbwm.  The host does what the reference's host does once per batch, in float64:
validation, lambda, the design/mapping matrices and the boundary.

Differences a caller can observe (documented in DESIGN.md):
  * every backend — "fused" (default), "naive" and "cuda" — runs the same GPU kernel.  The
    reference's "naive" backend is its per-pixel CPU restatement, contractually identical to
    "fused" (test_acceptance.py:67-95: indices equal, MO within 1e-9); here both names
    select the one fused kernel, so the contract holds exactly and a reference caller that
    passes backend="naive" keeps working.  There is no CPU path.
  * `threads` and `block_size` are validated like the reference and otherwise ignored:
    the CUDA grid replaces the thread pool and the 4096-pixel blocks.
  * the kernel computes in float32 (compensated where it matters); max_abs_mo agrees
    with the float64 reference to rtol 1e-4 and break indices are identical except on
    pixels whose MOSUM touches the boundary within that tolerance.
  * stack.data may also be a float32 CUDA torch tensor (N, P): then nothing crosses PCIe
    but the result maps.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass
from typing import ClassVar, Optional

import numpy as np

from .device import DevicePlan, DeviceResult
from .errors import ZeroResidualError
from .model import TimeAxis, build_design_matrix, fit_mapping

DEFAULT_BLOCK_SIZE = 4096
THREADS_ENV_VAR = "BREAKWATCH_THREADS"
CALIBRATION_REPS = 50_000
CALIBRATION_SEED = 7
PHASE_NAMES = ("ingest", "model", "predictions", "residuals", "mosum", "breaks")
BACKENDS = ("fused", "naive", "cuda")
NAN_MODES = ("fill", "mask")


def resolve_threads(threads: Optional[int] = None) -> int:
    """Explicit argument, else BREAKWATCH_THREADS, else machine parallelism (engine.py:53-68)."""
    if threads is None:
        env = os.environ.get(THREADS_ENV_VAR)
        if env is not None:
            try:
                threads = int(env)
            except ValueError:
                raise ValueError(f"{THREADS_ENV_VAR} must be an integer, got {env!r}") from None
        else:
            threads = os.cpu_count() or 1
    if threads < 1:
        raise ValueError("thread count must be >= 1")
    return threads


def _is_cuda_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor) and x.is_cuda


@dataclass(frozen=True)
class SeriesStack:
    """Time-major stack (n_obs, n_pixels) of float32 series; NaN/Inf = missing (engine.py:71-99).

    data: numpy array (cast to C-contiguous float32, as the reference does) or a float32
    CUDA tensor already resident in HBM (kept as is).
    """

    data: object
    time_axis: TimeAxis

    def __post_init__(self):
        if not isinstance(self.time_axis, TimeAxis):
            object.__setattr__(self, "time_axis", TimeAxis(self.time_axis))
        data = self.data
        if _is_cuda_tensor(data):
            import torch

            if data.dtype != torch.float32:
                data = data.float()
            if data.dim() != 2:
                raise ValueError("stack data must be 2-D (n_obs, n_pixels)")
            if data.stride(1) != 1:
                data = data.contiguous()
        else:
            data = np.ascontiguousarray(data, dtype=np.float32)
            if data.ndim != 2:
                raise ValueError("stack data must be 2-D (n_obs, n_pixels)")
        if data.shape[1] < 1:
            raise ValueError("stack needs at least one pixel")
        if data.shape[0] != len(self.time_axis):
            raise ValueError("time axis length must match the number of rows")
        object.__setattr__(self, "data", data)

    @property
    def n_obs(self) -> int:
        return int(self.data.shape[0])

    @property
    def n_pixels(self) -> int:
        return int(self.data.shape[1])


@dataclass(frozen=True)
class MonitorConfig:
    """Monitoring parameters shared by every pixel of a batch (engine.py:102-134)."""

    history: int
    bandwidth: int
    harmonics: int
    freq: float
    alpha: float = 0.05
    crit_value: Optional[float] = None
    backend: str = "fused"
    # "fill": the reference's forward/back gap fill (engine.py:305-319).  "mask": each pixel
    # is fitted on its valid history dates and monitored over its compacted valid series
    # (include/bwm.h BWM_NAN_MASK) — an extension, not in the reference.
    nan_mode: str = "fill"

    def __post_init__(self):
        if self.harmonics < 1:
            raise ValueError("harmonics must be >= 1")
        if self.freq <= 0:
            raise ValueError("freq must be positive")
        if self.history <= self.n_params:
            raise ValueError(f"history must exceed the coefficient count (n > {self.n_params})")
        if not 1 <= self.bandwidth <= self.history:
            raise ValueError("bandwidth must satisfy 1 <= h <= n")
        if not 0.0 < self.alpha < 1.0:
            raise ValueError("alpha must lie in (0, 1)")
        if self.crit_value is not None and not self.crit_value > 0:
            raise ValueError("explicit critical value must be positive")
        if self.nan_mode not in NAN_MODES:
            raise ValueError(f"nan_mode must be 'fill' or 'mask', got {self.nan_mode!r}")
        if self.backend not in BACKENDS:
            raise ValueError("backend must be 'fused', 'naive' or 'cuda'")

    @property
    def n_params(self) -> int:
        return 2 + 2 * self.harmonics


@dataclass(frozen=True)
class BreakMap:
    """Per-pixel break decisions (engine.py:137-168), plus optional GPU extras.

    first_break: 1-based observation number of the first strict crossing, 0 if none.
    beta / mosum_mean are filled only when requested (return_beta / return_mean).
    """

    detected: np.ndarray
    first_break: np.ndarray
    max_abs_mo: np.ndarray
    valid: np.ndarray
    config: MonitorConfig
    crit_value: float
    mosum: Optional[np.ndarray] = None
    beta: Optional[np.ndarray] = None
    mosum_mean: Optional[np.ndarray] = None

    def __len__(self) -> int:
        return int(self.detected.size)

    @property
    def break_count(self) -> int:
        return int(self.detected.sum())

    def result(self, pixel: int):
        from .mosum import BreakResult

        first = int(self.first_break[pixel])
        return BreakResult(bool(self.detected[pixel]), first if first else None, float(self.max_abs_mo[pixel]))


@dataclass(frozen=True)
class PhaseTimings:
    """Seconds per phase (engine.py:171-192).

    On the GPU the five compute phases are one fused kernel: `mosum` holds the kernel time,
    `ingest` the host->device transfer (the paper's "transfer" phase), `model` the host
    setup (design, mapping, boundary, plan), `breaks` the device->host result copy and map
    assembly; `predictions` and `residuals` are 0.
    """

    ingest: float
    model: float
    predictions: float
    residuals: float
    mosum: float
    breaks: float
    total: float

    names: ClassVar[tuple] = PHASE_NAMES

    @property
    def phase_sum(self) -> float:
        return sum(getattr(self, name) for name in PHASE_NAMES)


def fill_gaps(series) -> np.ndarray:
    """Forward fill from the first finite value; back-fill the leading gap (engine.py:195-211).

    The per-series statement of the gap fill the kernel applies to every pixel (a host numpy
    helper of the reference's public API, not a compute path): a series without gaps is
    returned unchanged, one with no finite value raises AllNanSeriesError.
    """
    from .errors import AllNanSeriesError

    values = np.asarray(series)
    finite = np.isfinite(values)
    if finite.all():
        return values
    if not finite.any():
        raise AllNanSeriesError("series has no finite values")
    # index of the latest finite sample at or before each position; leading gap -> first finite
    last = np.maximum.accumulate(np.where(finite, np.arange(values.size), -1))
    return values[np.where(last < 0, int(np.argmax(finite)), last)]


def resolve_crit_value(config: MonitorConfig, n_obs: int, threads: int = 1) -> float:
    """config.crit_value, else one simulation at the batch geometry (engine.py:214-228)."""
    if config.crit_value is not None:
        return float(config.crit_value)
    from .mosum import CriticalValueRequest, critical_value

    request = CriticalValueRequest(
        alpha=config.alpha,
        h_frac=config.bandwidth / config.history,
        horizon=n_obs / config.history,
        n_sim=config.history,
        reps=CALIBRATION_REPS,
        seed=CALIBRATION_SEED,
        harmonics=config.harmonics,
        freq=config.freq,
    )
    return critical_value(request, threads=threads)


def monitor_batch(stack: SeriesStack, config: MonitorConfig, threads: Optional[int] = None,
                  block_size: int = DEFAULT_BLOCK_SIZE, keep_mosum: bool = False, *,
                  return_beta: bool = False, return_mean: bool = False, device=None) -> BreakMap:
    """Monitor every pixel of a stack on the GPU (engine.py:231-244)."""
    break_map, _ = _run(stack, config, threads, block_size, keep_mosum, return_beta, return_mean, device)
    return break_map


def profile_run(stack: SeriesStack, config: MonitorConfig, threads: Optional[int] = None,
                block_size: int = DEFAULT_BLOCK_SIZE, *, device=None) -> tuple[BreakMap, PhaseTimings]:
    """monitor_batch plus seconds per phase (engine.py:247-254)."""
    return _run(stack, config, threads, block_size, False, False, False, device)


def _run(stack, config, threads, block_size, keep_mosum, return_beta, return_mean, device, source=None):
    """One batch through the GPU.  `source` = (path, payload_offset) monitors a BTS1 file's
    payload directly (dataio.monitor_file); `stack` then only needs n_obs, n_pixels and the
    time axis."""
    clock = time.perf_counter
    started = clock()
    if config.history >= stack.n_obs:
        raise ValueError("history must end before the series does (n < N)")
    threads = resolve_threads(threads)
    if block_size < 1:
        raise ValueError("block size must be >= 1")
    crit = resolve_crit_value(config, stack.n_obs, threads)

    mark = clock()
    design = build_design_matrix(stack.time_axis, config.freq, config.harmonics)
    fit_mapping(design, config.history)        # the reference's error contract (model.py:118-152)
    on_device = source is None and _is_cuda_tensor(stack.data)
    if on_device and device is None:
        device = stack.data.device
    plan = DevicePlan.get(stack.time_axis, config.freq, config.harmonics, config.history,
                          config.bandwidth, crit, device, nan_mode=config.nan_mode)
    t_model = clock() - mark

    if on_device:
        import torch

        mark = clock()
        res = plan.run_device(stack.data, keep_mosum=keep_mosum, beta=return_beta, mean=return_mean,
                              ref_dtypes=True)
        torch.cuda.synchronize(plan.torch_device)
        t_kernel = clock() - mark
        mark = clock()
        host = lambda t: None if t is None else t.cpu().numpy()  # noqa: E731
        res = DeviceResult(valid=host(res.valid), first_idx=None, max_abs=None, beta=host(res.beta),
                           mo_mean=host(res.mo_mean), mosum=host(res.mosum), zero_sigma=res.zero_sigma,
                           first_break=host(res.first_break), max_abs_f64=host(res.max_abs_f64),
                           detected=host(res.detected))
        t_ingest, t_d2h = 0.0, clock() - mark
    else:
        if source is None:
            res = plan.run_host(stack.data, keep_mosum=keep_mosum, beta=return_beta, mean=return_mean,
                                ref_dtypes=True)
        else:
            first, total = (source[2], source[3]) if len(source) > 2 else (0, stack.n_pixels)
            res = plan.run_file(source[0], source[1], stack.n_pixels, keep_mosum=keep_mosum, beta=return_beta,
                                mean=return_mean, ref_dtypes=True, first_pixel=first, file_pixels=total)
        t_kernel = res.kernel_ms * 1e-3
        t_ingest = max(0.0, (res.total_ms - res.kernel_ms) * 1e-3)
        t_d2h = 0.0
    if res.zero_sigma is not None:
        raise ZeroResidualError(f"pixel {res.zero_sigma} fits its history exactly (sigma = 0)")

    # the maps arrive in the reference dtypes (engine.py:147-150, 297-299): no conversion pass
    mark = clock()
    break_map = BreakMap(
        detected=res.detected.view(bool),
        first_break=res.first_break,
        max_abs_mo=res.max_abs_f64,
        valid=res.valid.view(bool),
        config=config,
        crit_value=crit,
        mosum=None if res.mosum is None else res.mosum.astype(np.float64),
        beta=None if res.beta is None else res.beta.astype(np.float64),
        mosum_mean=None if res.mo_mean is None else res.mo_mean.astype(np.float64),
    )
    t_breaks = t_d2h + (clock() - mark)
    timings = PhaseTimings(ingest=t_ingest, model=t_model, predictions=0.0, residuals=0.0,
                           mosum=t_kernel, breaks=t_breaks, total=clock() - started)
    return break_map, timings
