"""The reference package itself, unmodified, with backend="cuda" installed
(paper_1807_01751_b200.integration, the INTEGRATION.md stub): its own public API and its own
test scenarios — backend equivalence (test_engine.py:150-158, test_acceptance.py:67-95),
duplicated pixels (160-167), worker-count determinism and pixel permutation (170-193), dead
pixels (196-204), the zero-sigma failure (206-215) — run "cuda" against its CPU "fused"
backend.  The comparison is the north star's parity contract (float32 kernel vs float64
reference): valid identical, first_break identical except on borderline pixels, MOSUM and
max |MO| within rtol 1e-4.  The reference comes from baseline/_ref (pip-installed; travels to
the GPU box) or the read-only source tree here.
"""
import numpy as np
import pytest

from paper_1807_01751_b200.integration import install, load_reference

RTOL = 1e-4


@pytest.fixture(scope="module")
def bw():
    ref = load_reference()
    if ref is None:
        pytest.skip("reference package not available (baseline/_ref or /root/reference)")
    install(ref)
    return ref


def _configs(bw, **kw):
    base = dict(history=100, bandwidth=50, harmonics=3, freq=23.0, crit_value=4.9)
    base.update(kw)
    return bw.MonitorConfig(**base), bw.MonitorConfig(**base, backend="cuda")


def _small_stack(bw, seed=0, m=300, noise=0.02, break_mag=0.4):
    spec = bw.SynthSpec(n_pixels=m, n_obs=200, freq=23.0, noise_std=noise, break_mag=break_mag, seed=seed)
    return bw.generate(spec)[0]


def _with_nans(bw, stack, seed=0, fraction=0.05, dead_pixels=()):
    data = stack.data.copy()
    rng = np.random.default_rng(seed)
    data[rng.random(data.shape) < fraction] = np.nan
    for p in dead_pixels:
        data[:, p] = np.nan
    return bw.SeriesStack(data, stack.time_axis)


def _assert_parity(fused, cuda, n):
    assert np.array_equal(fused.valid, cuda.valid)
    mo = fused.mosum                                # float64 [N-n, P]
    # borderline: some window up to the later of the two first crossings within 1e-4 b of b
    b = fused.crit_value * np.sqrt(np.where(
        np.arange(n + 1, n + 1 + mo.shape[0]) / n > np.e,
        np.log(np.maximum(np.arange(n + 1, n + 1 + mo.shape[0]) / n, np.e)), 1.0))
    j_f = np.where(fused.first_break > 0, fused.first_break - n, mo.shape[0])
    j_c = np.where(cuda.first_break > 0, cuda.first_break - n, mo.shape[0])
    reach = np.maximum(j_f, j_c)
    near = np.abs(np.abs(mo) - b[:, None]) <= 1e-4 * b[:, None]
    near &= np.arange(mo.shape[0])[:, None] < reach[None, :]
    border = near.any(axis=0)
    assert not np.any((fused.first_break != cuda.first_break) & ~border)
    assert np.array_equal(fused.detected | border, cuda.detected | border)
    v = fused.valid
    np.testing.assert_allclose(cuda.max_abs_mo[v], fused.max_abs_mo[v], rtol=RTOL, atol=0)
    if cuda.mosum is not None:
        scale = np.abs(mo).max(axis=0, keepdims=True)
        assert np.all(np.abs(cuda.mosum - mo)[:, v] <= RTOL * scale[:, v] + 1e-6)


def test_install_is_cpu_safe_and_validates(bw):
    # the reference validation still applies to "cuda"; unknown names still fail
    with pytest.raises(ValueError):
        bw.MonitorConfig(history=100, bandwidth=0, harmonics=3, freq=23.0, backend="cuda")
    with pytest.raises(ValueError):
        bw.MonitorConfig(history=100, bandwidth=50, harmonics=3, freq=23.0, backend="bogus")
    assert bw.MonitorConfig(history=100, bandwidth=50, harmonics=3, freq=23.0, backend="cuda").backend == "cuda"


@pytest.mark.gpu
def test_seeded_stack_with_gaps(bw):
    stack = _with_nans(bw, _small_stack(bw, seed=11), seed=11, dead_pixels=(7, 42))
    fused_cfg, cuda_cfg = _configs(bw)
    fused = bw.monitor_batch(stack, fused_cfg, keep_mosum=True)
    cuda = bw.monitor_batch(stack, cuda_cfg, keep_mosum=True)
    _assert_parity(fused, cuda, 100)
    assert not cuda.valid[7] and not cuda.valid[42]


@pytest.mark.gpu
def test_acceptance_backend_equivalence(bw):
    """Criterion 1 of the reference's acceptance suite with "cuda" in place of "naive"."""
    rng = np.random.default_rng(12345)
    for trial in range(10):
        spec = bw.SynthSpec(n_pixels=1000, n_obs=200, freq=23.0, noise_std=float(rng.uniform(0.005, 0.05)),
                            break_mag=float(rng.uniform(0.05, 0.5)), seed=int(rng.integers(0, 2**32)))
        stack, _ = bw.generate(spec)
        fused_cfg, cuda_cfg = _configs(bw)
        _assert_parity(bw.monitor_batch(stack, fused_cfg, keep_mosum=True),
                       bw.monitor_batch(stack, cuda_cfg, keep_mosum=True), 100)


@pytest.mark.gpu
def test_duplicated_pixels_identical(bw):
    one = _small_stack(bw, seed=3, m=1)
    stack = bw.SeriesStack(np.repeat(one.data, 600, axis=1), one.time_axis)    # > 2 tiles: TMA + tail
    bm = bw.monitor_batch(stack, _configs(bw)[1])
    assert np.all(bm.detected == bm.detected[0])
    assert np.all(bm.first_break == bm.first_break[0])
    assert np.all(bm.max_abs_mo == bm.max_abs_mo[0])


@pytest.mark.gpu
def test_worker_count_and_permutation(bw):
    stack = _with_nans(bw, _small_stack(bw, seed=21, m=1500), seed=21)
    cfg = _configs(bw)[1]
    maps = [bw.monitor_batch(stack, cfg, threads=t, block_size=256) for t in (1, 2, 4)]
    for other in maps[1:]:
        for f in ("detected", "first_break", "max_abs_mo", "valid"):
            assert np.array_equal(getattr(maps[0], f), getattr(other, f))
    perm = np.random.default_rng(8).permutation(stack.n_pixels)
    shuffled = bw.monitor_batch(bw.SeriesStack(np.ascontiguousarray(stack.data[:, perm]), stack.time_axis), cfg)
    for f in ("detected", "first_break", "max_abs_mo"):
        assert np.array_equal(getattr(maps[0], f)[perm], getattr(shuffled, f))


@pytest.mark.gpu
def test_dead_pixel_masked(bw):
    stack = _with_nans(bw, _small_stack(bw, seed=13, m=50), seed=13, dead_pixels=(3,))
    bm = bw.monitor_batch(stack, _configs(bw)[1])
    assert not bm.valid[3] and not bm.detected[3] and bm.first_break[3] == 0 and bm.max_abs_mo[3] == 0.0
    assert bm.result(3).first_break is None


@pytest.mark.gpu
def test_exactly_fit_pixel_fails_the_batch(bw):
    stack = _small_stack(bw, seed=14, m=20)
    data = stack.data.copy()
    data[:, 5] = 0.0
    with pytest.raises(bw.ZeroResidualError):
        bw.monitor_batch(bw.SeriesStack(data, stack.time_axis), _configs(bw)[1])


@pytest.mark.gpu
def test_profile_run_phases(bw):
    stack = _small_stack(bw, seed=17, m=400)
    bm, tm = bw.profile_run(stack, _configs(bw)[1])
    assert tm.mosum > 0 and tm.total >= tm.phase_sum * 0.5
    assert bm.first_break.shape == (400,) and bm.first_break.dtype == np.int64
