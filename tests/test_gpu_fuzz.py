"""Seeded random geometries through the whole GPU path against the float64 oracle.

Covers the rarely hit corners in one sweep: every kernel mode (TMEM ring with and without
wrapping lag windows, both lagging-cursor modes, the LDG kernels for h < 8 and the tail tile),
harmonic orders 1-8, regular and irregular axes, pixel counts that are not multiples of a
tile, NaN fractions from none to most, monitoring horizons up to 4x the history.
Tolerances as in test_gpu_parity.py.
"""
import numpy as np
import pytest

from oracle import bfast_oracle as bo

pytestmark = pytest.mark.gpu

RTOL = 1e-4


def _geometries(count=20, seed=20261017):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(count):
        k = int(rng.integers(1, 9))
        p = 2 + 2 * k
        N = int(rng.integers(max(40, 3 * p), 420))
        # monitoring horizons up to 4x the history (the float32 trend extrapolation
        # error grows with N/n; the BASELINE geometries use N/n = 2)
        n = int(rng.integers(max(p + 4, (N + 3) // 4), N - 4))
        h = int(rng.choice([int(rng.integers(1, 8)), int(rng.integers(8, 40)), int(rng.integers(1, n + 1))]))
        h = max(1, min(h, n))
        P = int(rng.integers(1, 3000))
        nan = float(rng.choice([0.0, 0.2, 0.6]))
        irregular = bool(rng.integers(0, 2))
        out.append((i, N, n, h, k, P, nan, irregular))
    return out


@pytest.mark.parametrize("i,N,n,h,k,P,nan,irregular", _geometries())
def test_random_geometry(i, N, n, h, k, P, nan, irregular):
    import paper_1807_01751_b200 as pkg
    from paper_1807_01751_b200.synth import host_stack

    rng = np.random.default_rng(100 + i)
    t = np.cumsum(rng.uniform(1, 9, N)) + 1.0 if irregular else np.arange(1.0, N + 1.0)
    freq = 365.25 if irregular else 23.0
    y = host_stack(P, t, freq, n, nan, seed=200 + i)
    crit = 3.0
    cfg = pkg.MonitorConfig(history=n, bandwidth=h, harmonics=k, freq=freq, crit_value=crit)
    try:
        ref = bo.monitor(y, t, n, h, k, freq, crit, keep_mosum=True)
    except Exception as exc:                      # geometry the reference rejects: so must we
        want = (pkg.ZeroResidualError if isinstance(exc, bo.OracleZeroResidual)
                else pkg.RankDeficiencyError if "rank deficient" in str(exc) else type(exc))
        with pytest.raises(want):
            pkg.monitor_batch(pkg.SeriesStack(y, pkg.TimeAxis(t)), cfg)
        return
    bm = pkg.monitor_batch(pkg.SeriesStack(y, pkg.TimeAxis(t)), cfg)
    assert np.array_equal(bm.valid, ref.valid)
    first_gpu = np.where(bm.first_break > 0, bm.first_break - n, 0)
    pairs = bo.near_pairs(ref.mosum, bo.boundary(n, N, crit))
    border = bo.borderline_from_pairs(pairs, N - n, P, ref.first_idx, first_gpu)
    filled, _ = bo.fill_block(y)
    degen = (filled[:n] == filled[0]).all(axis=0)
    bad = np.flatnonzero((first_gpu != ref.first_idx) & ~border & ~degen & ref.valid)
    assert bad.size == 0, f"{bad.size} mismatches, e.g. {bad[:5]}"
    ok = ref.valid & ~degen
    np.testing.assert_allclose(bm.max_abs_mo[ok], ref.max_abs_mo[ok], rtol=RTOL, atol=0)


@pytest.mark.parametrize("i,N,n,h,k,P,nan,irregular", _geometries(count=10, seed=7))
def test_random_geometry_masked(i, N, n, h, k, P, nan, irregular):
    """The same sweep in nan_mode="mask" against the per-pixel masked oracle (600 px each)."""
    import paper_1807_01751_b200 as pkg
    from paper_1807_01751_b200.synth import host_stack

    P = min(P, 600)
    rng = np.random.default_rng(300 + i)
    t = np.cumsum(rng.uniform(1, 9, N)) + 1.0 if irregular else np.arange(1.0, N + 1.0)
    freq = 365.25 if irregular else 23.0
    y = host_stack(P, t, freq, n, nan, seed=400 + i)
    crit = 3.0
    cfg = pkg.MonitorConfig(history=n, bandwidth=h, harmonics=k, freq=freq, crit_value=crit, nan_mode="mask")
    try:
        ref = bo.monitor_masked(y, t, n, h, k, freq, crit)
    except bo.OracleZeroResidual:
        with pytest.raises(pkg.ZeroResidualError):
            pkg.monitor_batch(pkg.SeriesStack(y, pkg.TimeAxis(t)), cfg)
        return
    try:
        bm = pkg.monitor_batch(pkg.SeriesStack(y, pkg.TimeAxis(t)), cfg)
    except pkg.RankDeficiencyError:
        pytest.skip("full-history design rank deficient (checked before any pixel is fitted)")
    assert np.array_equal(bm.valid, ref.valid)
    bad = np.flatnonzero((bm.first_break != ref.first_break) & ~ref.near & ref.valid)
    assert bad.size == 0, f"{bad.size} mismatches, e.g. {bad[:5]}"
    v = ref.valid
    np.testing.assert_allclose(bm.max_abs_mo[v], ref.max_abs_mo[v], rtol=RTOL, atol=0)


@pytest.mark.parametrize("i,N,n,h,k,P,irregular", [(16, 313, 20, 5, 2, 2704, True), (30, 600, 40, 12, 3, 2000, False),
                                                   (31, 900, 60, 30, 4, 1500, True)])
def test_long_horizon_precise(i, N, n, h, k, P, irregular):
    """Monitoring horizons far beyond 4x the history (N/n = 10-16): the plan switches to float64
    fitted values (plan_info precise) and stays within tolerance where float32 did not (case 16
    reached 2e-4 on max |MO| before)."""
    import paper_1807_01751_b200 as pkg
    from paper_1807_01751_b200.device import DevicePlan
    from paper_1807_01751_b200.synth import host_stack

    rng = np.random.default_rng(100 + i)
    t = np.cumsum(rng.uniform(1, 9, N)) + 1.0 if irregular else np.arange(1.0, N + 1.0)
    freq = 365.25 if irregular else 23.0
    y = host_stack(P, t, freq, n, 0.2, seed=200 + i)
    cfg = pkg.MonitorConfig(history=n, bandwidth=h, harmonics=k, freq=freq, crit_value=3.0)
    assert DevicePlan.get(pkg.TimeAxis(t), freq, k, n, h, 3.0).info()["precise"] == 1
    ref = bo.monitor(y, t, n, h, k, freq, 3.0, keep_mosum=True)
    bm = pkg.monitor_batch(pkg.SeriesStack(y, pkg.TimeAxis(t)), cfg)
    assert np.array_equal(bm.valid, ref.valid)
    first_gpu = np.where(bm.first_break > 0, bm.first_break - n, 0)
    pairs = bo.near_pairs(ref.mosum, bo.boundary(n, N, 3.0))
    border = bo.borderline_from_pairs(pairs, N - n, P, ref.first_idx, first_gpu)
    assert not np.any((first_gpu != ref.first_idx) & ~border & ref.valid)
    np.testing.assert_allclose(bm.max_abs_mo[ref.valid], ref.max_abs_mo[ref.valid], rtol=RTOL, atol=0)


def test_precise_mode_on_baseline_geometry(monkeypatch):
    """BWM_PRECISE=1 forces the float64 fitted values on a C1 geometry: same decisions, within
    tolerance of the float32 default."""
    import paper_1807_01751_b200 as pkg
    from paper_1807_01751_b200.device import DevicePlan
    from tests.golden_cases import load
    from tests.test_gpu_parity import check_parity, config_for

    case = load("c1")
    monkeypatch.setenv("BWM_PRECISE", "1")
    DevicePlan._cache.clear()
    bm = pkg.monitor_batch(pkg.SeriesStack(case.y, pkg.TimeAxis(case.t)), config_for(case))
    assert DevicePlan.get(pkg.TimeAxis(case.t), case.freq, case.k, case.n, case.h, case.crit).info()["precise"] == 1
    DevicePlan._cache.clear()
    check_parity(case, bm.first_break, bm.max_abs_mo, bm.valid)


@pytest.mark.parametrize("i,sigma", [(0, 0.005), (1, 0.002), (2, 0.001), (3, 0.003)])
def test_low_noise(i, sigma):
    """Low-noise stacks (||y - c||^2 / RSS up to ~1e4, the cancellation the one-pass RSS must
    survive) with leading gaps and long NaN runs; C1-C3 and C4/C5-like geometries."""
    import paper_1807_01751_b200 as pkg

    rng = np.random.default_rng(500 + i)
    N, n, h, k, freq = [(228, 114, 28, 3, 23.0), (400, 200, 50, 3, 365.25), (1000, 500, 250, 6, 365.25),
                        (160, 80, 8, 8, 23.0)][i]
    t = np.arange(1.0, N + 1.0) if freq == 23.0 else np.cumsum(rng.uniform(1, 9, N)) + 1.0
    P = 1500
    phi = rng.uniform(0, 2 * np.pi, P)
    y = 0.5 + 0.2 * np.sin(2 * np.pi * t[:, None] / freq + phi[None, :]) + rng.normal(0, sigma, (N, P))
    brk = rng.random(P) < 0.5
    start = rng.integers(n, N, P)
    y += ((np.arange(N)[:, None] >= start[None, :]) & brk[None, :]) * rng.uniform(-0.05, -0.01, P)[None, :]
    y = y.astype(np.float32)
    y[rng.random((N, P)) < 0.2] = np.nan
    y[: rng.integers(1, 30), : P // 10] = np.nan            # leading gaps
    for c in rng.integers(0, P, 50):                          # long NaN runs
        a = int(rng.integers(0, N - 20))
        y[a:a + int(rng.integers(5, 20)), c] = np.nan
    cfg = pkg.MonitorConfig(history=n, bandwidth=h, harmonics=k, freq=freq, crit_value=3.0)
    ref = bo.monitor(y, t, n, h, k, freq, 3.0, keep_mosum=True)
    bm = pkg.monitor_batch(pkg.SeriesStack(y, pkg.TimeAxis(t)), cfg)
    assert np.array_equal(bm.valid, ref.valid)
    first_gpu = np.where(bm.first_break > 0, bm.first_break - n, 0)
    pairs = bo.near_pairs(ref.mosum, bo.boundary(n, N, 3.0))
    border = bo.borderline_from_pairs(pairs, N - n, P, ref.first_idx, first_gpu)
    filled, _ = bo.fill_block(y)
    degen = (filled[:n] == filled[0]).all(axis=0)
    assert not np.any((first_gpu != ref.first_idx) & ~border & ~degen & ref.valid)
    ok = ref.valid & ~degen
    np.testing.assert_allclose(bm.max_abs_mo[ok], ref.max_abs_mo[ok], rtol=RTOL, atol=0)


@pytest.mark.parametrize("i,sigma", [(0, 0.003), (1, 0.001)])
def test_low_noise_masked(i, sigma):
    """Masked mode on near-noiseless series with per-pixel gaps (per-pixel float32 Cholesky
    plus one refinement step, against the per-pixel float64 oracle)."""
    import paper_1807_01751_b200 as pkg

    rng = np.random.default_rng(700 + i)
    N, n, h, k, freq = [(228, 114, 28, 3, 23.0), (400, 200, 50, 3, 365.25)][i]
    t = np.arange(1.0, N + 1.0) if freq == 23.0 else np.cumsum(rng.uniform(8, 24, N)) + 1.0
    P = 600
    phi = rng.uniform(0, 2 * np.pi, P)
    y = 0.5 + 0.2 * np.sin(2 * np.pi * t[:, None] / freq + phi[None, :]) + rng.normal(0, sigma, (N, P))
    brk = rng.random(P) < 0.5
    start = rng.integers(n, N, P)
    y += ((np.arange(N)[:, None] >= start[None, :]) & brk[None, :]) * rng.uniform(-0.05, -0.01, P)[None, :]
    y = y.astype(np.float32)
    y[rng.random((N, P)) < 0.25] = np.nan
    cfg = pkg.MonitorConfig(history=n, bandwidth=h, harmonics=k, freq=freq, crit_value=3.0, nan_mode="mask")
    ref = bo.monitor_masked(y, t, n, h, k, freq, 3.0)
    bm = pkg.monitor_batch(pkg.SeriesStack(y, pkg.TimeAxis(t)), cfg)
    assert np.array_equal(bm.valid, ref.valid)
    assert not np.any((bm.first_break != ref.first_break) & ~ref.near & ref.valid)
    np.testing.assert_allclose(bm.max_abs_mo[ref.valid], ref.max_abs_mo[ref.valid], rtol=RTOL, atol=0)


@pytest.mark.parametrize("i,N,n,h,k", [(0, 600, 150, 30, 3), (1, 320, 80, 12, 2), (2, 400, 100, 25, 4),
                                       (3, 600, 60, 15, 3), (4, 313, 30, 6, 2)])
def test_long_horizon_masked(i, N, n, h, k):
    """Masked mode with monitoring horizons of 4x the history (float32 kernel) and of 10x
    (the plan switches to the per-pixel float64 masked kernel)."""
    import paper_1807_01751_b200 as pkg
    from paper_1807_01751_b200.synth import host_stack

    rng = np.random.default_rng(800 + i)
    t = np.cumsum(rng.uniform(1, 9, N)) + 1.0
    y = host_stack(600, t, 365.25, n, 0.2, seed=900 + i)
    cfg = pkg.MonitorConfig(history=n, bandwidth=h, harmonics=k, freq=365.25, crit_value=3.0, nan_mode="mask")
    from paper_1807_01751_b200.device import DevicePlan

    precise = DevicePlan.get(pkg.TimeAxis(t), 365.25, k, n, h, 3.0, nan_mode="mask").info()["precise"]
    assert precise == (1 if N >= 5 * n else 0)
    ref = bo.monitor_masked(y, t, n, h, k, 365.25, 3.0)
    bm = pkg.monitor_batch(pkg.SeriesStack(y, pkg.TimeAxis(t)), cfg)
    assert np.array_equal(bm.valid, ref.valid)
    assert not np.any((bm.first_break != ref.first_break) & ~ref.near & ref.valid)
    np.testing.assert_allclose(bm.max_abs_mo[ref.valid], ref.max_abs_mo[ref.valid], rtol=RTOL, atol=0)
