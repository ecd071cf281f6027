"""backend="cuda" for the UNMODIFIED reference package — the INTEGRATION.md stub, importable.

The reference selects its batch backend in ``_run`` (pkg/src/breakwatch/engine.py:287):
``_fused_phases`` for ``config.backend == "fused"``, ``_naive_phases`` otherwise, after
``MonitorConfig.__post_init__`` (engine.py:129-130) admitted only those two names.  A
backend has the signature (engine.py:322, 411)

    (stack, config, crit, blocks, pool, keep_mosum, clock)
        -> ((first_idx int64[P], max_abs float64[P], valid bool[P], mosum float64[N-n, P] | None),
            {phase: seconds})

with first_idx 0 (no break) or the 1-based offset into the monitoring period; ``_run`` then
assembles the BreakMap (engine.py:297-301).  ``install(breakwatch)`` adds a third name,
"cuda", whose backend is one libbwm call through the C ABI (bwm_monitor_host, include/bwm.h):
the reference's own host setup runs first — ``build_design_matrix`` and ``fit_mapping``
(model.py:90-152), so its RankDeficiencyError / DegreesOfFreedomError contract is the
reference's — then the stack crosses PCIe once and the maps come back.  A zero-sigma pixel
raises the reference's own ZeroResidualError with its message (engine.py:373-378).  Nothing
else in the reference changes; "fused" and "naive" keep running on the CPU, so the reference's
own tests can compare them with "cuda" on the same stacks (tests/test_integration.py).
"""

from __future__ import annotations


import numpy as np

_INSTALLED = "_bwm_cuda_installed"


def cuda_phases(ref, stack, config, crit, blocks, pool, keep_mosum, clock):
    """The reference backend contract on the GPU (see the module docstring)."""
    from .device import DevicePlan
    from .model import TimeAxis

    n = config.history
    design = ref.build_design_matrix(stack.time_axis, config.freq, config.harmonics)
    ref.fit_mapping(design, n)                 # the reference's own error contract (model.py:118-152)
    t0 = clock()
    plan = DevicePlan.get(TimeAxis(np.asarray(stack.time_axis.values, dtype=np.float64)), config.freq,
                          config.harmonics, n, config.bandwidth, crit)
    t1 = clock()
    res = plan.run_host(stack.data, keep_mosum=keep_mosum)
    t2 = clock()
    if res.zero_sigma is not None:
        raise ref.ZeroResidualError(f"pixel {res.zero_sigma} fits its history exactly (sigma = 0)")
    mosum = None if res.mosum is None else res.mosum.astype(np.float64)
    outputs = (res.first_idx.astype(np.int64), res.max_abs.astype(np.float64), res.valid.astype(bool), mosum)
    h2d_s = max(0.0, (res.total_ms - res.kernel_ms) * 1e-3)
    times = {"ingest": h2d_s, "model": t1 - t0, "predictions": 0.0, "residuals": 0.0,
             "mosum": res.kernel_ms * 1e-3, "breaks": max(0.0, (t2 - t1) - res.total_ms * 1e-3)}
    return outputs, times


def install(ref) -> None:
    """Teach the reference package `ref` (breakwatch) the "cuda" backend, in place."""
    engine = ref.engine
    if getattr(engine, _INSTALLED, False):
        return
    original_post_init = engine.MonitorConfig.__post_init__
    original_naive = engine._naive_phases

    def post_init(self):
        if self.backend != "cuda":
            return original_post_init(self)
        object.__setattr__(self, "backend", "fused")       # validate everything else as the reference does
        try:
            original_post_init(self)
        finally:
            object.__setattr__(self, "backend", "cuda")

    def dispatch(stack, config, crit, blocks, pool, keep_mosum, clock):
        # _run sends every non-"fused" backend here (engine.py:287)
        if config.backend == "cuda":
            return cuda_phases(ref, stack, config, crit, blocks, pool, keep_mosum, clock)
        return original_naive(stack, config, crit, blocks, pool, keep_mosum, clock)

    engine.MonitorConfig.__post_init__ = post_init
    engine._naive_phases = dispatch
    setattr(engine, _INSTALLED, True)


def load_reference(path=None):
    """Import the unmodified reference from baseline/_ref (the pip-installed copy that travels
    to the GPU box) or the read-only source tree; None when neither exists."""
    import sys
    from pathlib import Path

    repo = Path(__file__).resolve().parents[1]
    for d in ([Path(path)] if path else []) + [repo / "baseline" / "_ref", Path("/root/reference/pkg/src")]:
        if (d / "breakwatch" / "__init__.py").exists():
            if str(d) not in sys.path:
                sys.path.insert(0, str(d))
            import breakwatch

            return breakwatch
    return None


__all__ = ["cuda_phases", "install", "load_reference"]
