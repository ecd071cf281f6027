"""nan_mode="mask": per-pixel fits on the valid history dates and a MOSUM
over the compacted valid series (include/bwm.h BWM_NAN_MASK).  The reference has no such
mode, so the oracle's restatement (oracle/bfast_oracle.py:monitor_masked) is pinned by the
reference itself on the two input classes where masked mode reduces to a reference run:

  mask_nanfree          no missing values: masked == fill == the reference
  mask_common_*         gaps on the same dates in every pixel: masked == the reference run
                        on the compacted series (n_v, h_v = floor(h n_v / n)), breaks mapped
                        back to the original dates (tests/golden/make_golden.py:masked)

The CUDA kernel is then checked against those fixtures and against the oracle on inputs
with per-pixel gaps.  Tolerances as in test_gpu_parity.py: valid identical, first_break
identical off the boundary (rtol 1e-4 near-pixels excluded), max_abs_mo rtol 1e-4.
"""

import json

import numpy as np
import pytest

from oracle import bfast_oracle as bo
from tests.golden_cases import GOLDEN, edge_stack

RTOL = 1e-4
MASK_CASES = ["mask_nanfree", "mask_common_c1", "mask_common_irregular", "mask_common_k8_h60"]


class Fixture:
    def __init__(self, name):
        z = np.load(GOLDEN / f"{name}.npz")
        self.name = name
        self.info = json.loads(str(z["info"]))
        self.y, self.t = z["y"], z["t"]
        self.n, self.h, self.k = self.info["n"], self.info["h"], self.info["k"]
        self.freq, self.crit = self.info["freq"], self.info["crit"]
        self.first_break = z["first_break"].astype(np.int64)
        self.max_abs_mo, self.valid = z["max_abs_mo"], z["valid"]
        self.mosum_mean = z["mosum_mean"]
        self.beta = z["beta"] if "beta" in z else None
        self.mosum = z["mosum"].astype(np.float64) if "mosum" in z else None
        near = z["near"]
        self.near_px = np.zeros(self.y.shape[1], dtype=bool)
        if near.size:
            self.near_px[np.unique(near[:, 1])] = True


def oracle_masked(y, t, n, h, k, freq, crit, keep_mosum=False):
    return bo.monitor_masked(y, t, n, h, k, freq, crit, keep_mosum=keep_mosum)


def compare(name, want_first, want_max, want_valid, got_first, got_max, got_valid, near):
    assert np.array_equal(got_valid, want_valid), f"{name}: valid mask differs"
    bad = np.flatnonzero((got_first != want_first) & ~near & want_valid)
    assert bad.size == 0, f"{name}: {bad.size} non-borderline break mismatches, e.g. {bad[:5]}"
    v = want_valid
    np.testing.assert_allclose(got_max[v], want_max[v], rtol=RTOL, atol=0)


# ---------------------------------------------------------------- oracle pinned (CPU)
@pytest.mark.parametrize("name", MASK_CASES)
def test_oracle_masked_matches_reference_fixture(name):
    f = Fixture(name)
    r = oracle_masked(f.y, f.t, f.n, f.h, f.k, f.freq, f.crit, keep_mosum=True)
    assert np.array_equal(r.valid, f.valid)
    assert np.array_equal(r.first_break, f.first_break)
    np.testing.assert_allclose(r.max_abs_mo, f.max_abs_mo, rtol=1e-9)
    np.testing.assert_allclose(r.mosum_mean, f.mosum_mean, rtol=1e-7, atol=1e-9)
    assert np.array_equal(np.isnan(r.mosum), np.isnan(f.mosum))
    np.testing.assert_allclose(r.mosum[~np.isnan(r.mosum)], f.mosum[~np.isnan(f.mosum)], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(r.beta, f.beta, rtol=1e-8, atol=1e-8)


def test_oracle_masked_equals_fill_without_gaps():
    from paper_1807_01751_b200.synth import host_stack

    t = np.arange(1.0, 161.0)
    y = host_stack(200, t, 23.0, 80, 0.0, seed=41, dead_frac=0.0)
    a = bo.monitor(y, t, 80, 20, 2, 23.0, 3.0)
    b = oracle_masked(y, t, 80, 20, 2, 23.0, 3.0)
    assert np.array_equal(a.first_break, b.first_break)
    np.testing.assert_allclose(a.max_abs_mo, b.max_abs_mo, rtol=1e-10)


def test_oracle_masked_invalid_pixels():
    t = np.arange(1.0, 61.0)
    rng = np.random.default_rng(3)
    y = (1.0 + 0.1 * rng.standard_normal((60, 6))).astype(np.float32)
    y[:, 0] = np.nan                       # no data
    y[:25, 1] = np.nan                     # n_v = 5 <= p = 6
    y[30:, 2] = np.nan                     # no valid monitoring date
    y[:27, 3] = np.nan                     # n_v = 3: h_v = floor(10*3/30) = 1 but n_v <= p
    r = oracle_masked(y, t, 30, 10, 2, 12.0, 2.5)
    assert r.valid.tolist() == [False, False, False, False, True, True]


# ---------------------------------------------------------------- CUDA kernel (B200)
def _pkg():
    import paper_1807_01751_b200 as pkg

    return pkg


def _config(f_or_args, **kw):
    pkg = _pkg()
    n, h, k, freq, crit = f_or_args
    return pkg.MonitorConfig(history=n, bandwidth=h, harmonics=k, freq=freq, crit_value=crit, nan_mode="mask", **kw)


@pytest.mark.gpu
@pytest.mark.parametrize("name", MASK_CASES)
@pytest.mark.parametrize("path", ["host", "device"])
def test_gpu_masked_matches_reference_fixture(name, path):
    import torch

    pkg = _pkg()
    f = Fixture(name)
    data = f.y if path == "host" else torch.as_tensor(f.y, device="cuda")
    stack = pkg.SeriesStack(data, pkg.TimeAxis(f.t))
    bm = pkg.monitor_batch(stack, _config((f.n, f.h, f.k, f.freq, f.crit)), keep_mosum=True, return_beta=True,
                           return_mean=True)
    compare(name, f.first_break, f.max_abs_mo, f.valid, bm.first_break, bm.max_abs_mo, bm.valid, f.near_px)
    v = f.valid
    scale = np.maximum(np.abs(f.mosum_mean), f.max_abs_mo)
    assert np.all((np.abs(bm.mosum_mean - f.mosum_mean) <= RTOL * scale)[v])
    assert np.array_equal(np.isnan(bm.mosum[:, v]), np.isnan(f.mosum[:, v])), "missing-date rows must be NaN"
    d = np.nan_to_num(np.abs(bm.mosum - f.mosum))
    assert np.all((d <= RTOL * f.max_abs_mo[None, :])[:, v])
    yinf = np.nanmax(np.abs(f.y[:f.n]), axis=0)
    assert np.all((np.abs(bm.beta - f.beta) <= 1e-4 * np.abs(f.beta) + 1e-4 * yinf[None, :])[:, v])
    assert np.array_equal(bm.detected, bm.first_break > 0)


def _gap_stack(P, t, freq, n, frac, seed, clustered=False):
    from paper_1807_01751_b200.synth import host_stack

    cols = int(round(P ** 0.5)) if clustered else None
    return host_stack(P, t, freq, n, frac, seed=seed, clustered=clustered, cols=cols)


@pytest.mark.gpu
@pytest.mark.parametrize("case", [
    dict(name="c1_like", N=228, n=114, h=28, k=3, freq=23.0, crit=2.96519227, P=3000, frac=0.2),
    dict(name="c5_like", N=400, n=200, h=50, k=3, freq=365.25, crit=3.0, P=96 * 96, frac=0.19, clustered=True,
         irregular=(8.0, 24.0)),
    dict(name="c4_like", N=1000, n=500, h=250, k=6, freq=365.25, crit=3.0, P=600, frac=0.5, irregular=(1.0, 9.0)),
    dict(name="k1_h1", N=90, n=45, h=1, k=1, freq=12.0, crit=2.5, P=777, frac=0.3),
    dict(name="k8_hn", N=120, n=60, h=60, k=8, freq=40.0, crit=2.7, P=513, frac=0.15),
])
def test_gpu_masked_matches_oracle(case):
    pkg = _pkg()
    N, n = case["N"], case["n"]
    if "irregular" in case:
        lo, hi = case["irregular"]
        t = np.cumsum(np.random.default_rng(1).uniform(lo, hi, N)) + 1.0
    else:
        t = np.arange(1.0, N + 1)
    y = _gap_stack(case["P"], t, case["freq"], n, case["frac"], 100 + N, case.get("clustered", False))
    args = (n, case["h"], case["k"], case["freq"], case["crit"])
    r = oracle_masked(y, t, *args)
    bm = pkg.monitor_batch(pkg.SeriesStack(y, pkg.TimeAxis(t)), _config(args), return_beta=True)
    compare(case["name"], r.first_break, r.max_abs_mo, r.valid, bm.first_break, bm.max_abs_mo, bm.valid, r.near)


@pytest.mark.gpu
def test_gpu_masked_edge_pixels():
    pkg = _pkg()
    rng = np.random.default_rng(7)
    N, n = 60, 30
    y = edge_stack(rng, N, 300, n)
    y[:25, 20] = np.nan                  # n_v = 5 <= p
    y[30:, 21] = np.nan                  # nothing to monitor
    y[:, 22] = np.inf
    t = np.arange(1.0, N + 1)
    for h, k in [(10, 2), (1, 1), (30, 3)]:
        args = (n, h, k, 12.0, 2.5)
        r = oracle_masked(y, t, *args)
        bm = pkg.monitor_batch(pkg.SeriesStack(y, pkg.TimeAxis(t)), _config(args))
        compare(f"edges h={h}", r.first_break, r.max_abs_mo, r.valid, bm.first_break, bm.max_abs_mo, bm.valid,
                r.near)
        assert not bm.valid[[0, 20, 21, 22]].any()


@pytest.mark.gpu
def test_gpu_masked_equals_fill_without_gaps():
    import torch

    pkg = _pkg()
    f = Fixture("mask_nanfree")
    y = torch.as_tensor(f.y, device="cuda")
    stack = pkg.SeriesStack(y, pkg.TimeAxis(f.t))
    a = pkg.monitor_batch(stack, _pkg().MonitorConfig(history=f.n, bandwidth=f.h, harmonics=f.k, freq=f.freq,
                                                      crit_value=f.crit))
    b = pkg.monitor_batch(stack, _config((f.n, f.h, f.k, f.freq, f.crit)))
    assert np.array_equal(a.valid, b.valid)
    assert np.array_equal(a.first_break, b.first_break)
    np.testing.assert_allclose(a.max_abs_mo, b.max_abs_mo, rtol=RTOL)


@pytest.mark.gpu
def test_gpu_masked_layout_invariance():
    """Misaligned / strided input and pixel sharding give bit-identical maps."""
    import torch

    from paper_1807_01751_b200.device import DevicePlan
    from paper_1807_01751_b200.model import TimeAxis

    f = Fixture("mask_common_c1")
    y = f.y.copy()
    rng = np.random.default_rng(5)
    y[rng.random(y.shape) < 0.2] = np.nan
    plan = DevicePlan(TimeAxis(f.t), f.freq, f.k, f.n, f.h, f.crit, "cuda", nan_mode="mask")
    yd = torch.as_tensor(y, device="cuda")
    base = plan.run_device(yd, beta=True, mean=True)
    big = torch.full((y.shape[0], y.shape[1] + 3), float("nan"), device="cuda")
    big[:, 1:-2] = yd
    mis = plan.run_device(big[:, 1:-2], beta=True, mean=True)
    half = y.shape[1] // 2 + 1
    s0 = plan.run_device(yd[:, :half].contiguous(), beta=True, mean=True)
    s1 = plan.run_device(yd[:, half:].contiguous(), beta=True, mean=True, pixel_offset=half)
    for key in ("valid", "first_idx", "max_abs", "mo_mean", "beta"):
        a = getattr(base, key).cpu().numpy()
        assert np.array_equal(a, getattr(mis, key).cpu().numpy()), key
        joined = np.concatenate([getattr(s0, key).cpu().numpy(), getattr(s1, key).cpu().numpy()], axis=-1)
        assert np.array_equal(a, joined), key
    assert plan.info()["nan_mode"] == "mask"


@pytest.mark.gpu
def test_gpu_masked_zero_sigma_raises():
    pkg = _pkg()
    z = np.load(GOLDEN / "zero_sigma.npz")
    y = z["y"]
    t = np.arange(1.0, y.shape[0] + 1)
    with pytest.raises(pkg.ZeroResidualError, match=r"pixel 5 fits its history exactly"):
        pkg.monitor_batch(pkg.SeriesStack(y, pkg.TimeAxis(t)), _config((100, 50, 3, 23.0, 4.9)))


@pytest.mark.gpu
@pytest.mark.parametrize("chunk", ["1024", "2560"])
def test_gpu_masked_global_scratch_chunked_pipeline(monkeypatch, chunk):
    """Masked mode on a global-scratch geometry (p = 14, h = 250: the x x^T table and the
    residual rings live in plan-owned global memory) through the chunked host pipeline, two
    chunks in flight on two streams.  Every launch that uses the plan's scratch (rings, float64
    fixup list) is ordered after the previous one, so the chunked run equals the one-launch run
    bit for bit, and matches the oracle."""
    from paper_1807_01751_b200.device import DevicePlan

    pkg = _pkg()
    N, n, h, k, freq = 1000, 500, 250, 6, 365.25
    t = np.cumsum(np.random.default_rng(1).uniform(1.0, 9.0, N)) + 1.0
    y = _gap_stack(3000, t, freq, n, 0.5, 77)
    args = (n, h, k, freq, 3.0)
    assert DevicePlan.get(pkg.TimeAxis(t), freq, k, n, h, 3.0, nan_mode="mask").info()["masked_global"] == 1
    stack = pkg.SeriesStack(y, pkg.TimeAxis(t))
    whole = pkg.monitor_batch(stack, _config(args), return_beta=True, return_mean=True)
    monkeypatch.setenv("BWM_HOST_CHUNK", chunk)
    parts = pkg.monitor_batch(stack, _config(args), return_beta=True, return_mean=True)
    monkeypatch.delenv("BWM_HOST_CHUNK")
    for f in ("valid", "first_break", "max_abs_mo", "mosum_mean", "beta"):
        assert np.array_equal(getattr(whole, f), getattr(parts, f), equal_nan=True), f
    sl = slice(0, 400)
    r = oracle_masked(y[:, sl], t, *args)
    compare("global scratch, chunked", r.first_break, r.max_abs_mo, r.valid, parts.first_break[sl],
            parts.max_abs_mo[sl], parts.valid[sl], r.near)
