"""Parity at BASELINE.json's full single-GPU sizes (C2: 4096^2 px x 228 dates, C4: 2048^2 px
x 1000 dates, C5: 7000^2 px x 400 dates), where the float64 oracle cannot run on everything:

  * a seeded random sample of pixels, copied back to the host, against the oracle
    (same tolerances as test_gpu_parity.py: valid identical, first_break identical off the
    boundary, max_abs_mo rtol 1e-4);
  * size-independent properties on the WHOLE stack: placement invariance (the view starting
    s pixels in gives the shifted maps) and shard invariance (two parts == whole), bit for bit;
  * sanity of the break statistics of the synthetic NDVI stacks (half the pixels carry a
    level drop inside the monitoring period; dead pixels are invalid).
"""
import numpy as np
import pytest

from oracle import bfast_oracle as bo

pytestmark = pytest.mark.gpu

RTOL = 1e-4


def _setup(name):
    import torch

    from paper_1807_01751_b200.device import DevicePlan
    from paper_1807_01751_b200.model import TimeAxis
    from paper_1807_01751_b200.synth import WORKLOADS, device_stack, time_axis

    w = WORKLOADS[name]
    t = time_axis(w)
    plan = DevicePlan(TimeAxis(t), w.freq, w.harmonics, w.n_hist, w.bandwidth, w.crit, "cuda")
    y = device_stack(w.n_pixels, t, w.freq, w.n_hist, w.nan_frac, seed=20261017, device="cuda",
                     clustered=w.clustered, cols=w.cols, scene_rows=w.rows)    # C5: cloud-disc NaNs
    torch.cuda.synchronize()
    return w, t, plan, y


def _maps(res):
    return [a.cpu().numpy() for a in (res.valid, res.first_idx, res.max_abs)]


@pytest.mark.parametrize("name", ["C2", "C4", "C5"])
def test_fullsize_sample_against_oracle(name):
    import torch

    w, t, plan, y = _setup(name)
    valid, first, mx = _maps(plan.run_device(y))
    rng = np.random.default_rng(7)
    idx = np.sort(rng.choice(w.n_pixels, size=6000, replace=False))
    ys = y[:, torch.as_tensor(idx, device="cuda")].cpu().numpy()
    del y
    torch.cuda.empty_cache()
    ref = bo.monitor(ys, t, w.n_hist, w.bandwidth, w.harmonics, w.freq, w.crit, keep_mosum=True)
    assert np.array_equal(valid[idx].astype(bool), ref.valid)
    bound = bo.boundary(w.n_hist, w.n_obs, w.crit)
    pairs = bo.near_pairs(ref.mosum, bound)
    border = bo.borderline_from_pairs(pairs, w.n_obs - w.n_hist, idx.size, ref.first_idx, first[idx])
    bad = np.flatnonzero((first[idx] != ref.first_idx) & ~border & ref.valid)
    assert bad.size == 0, f"{bad.size} non-borderline mismatches, e.g. pixels {idx[bad[:5]]}"
    filled, _ = bo.fill_block(ys)
    degen = (filled[:w.n_hist] == filled[0]).all(axis=0)       # constant history: sigma = 0 here
    v = ref.valid & ~degen
    np.testing.assert_allclose(mx[idx][v], ref.max_abs_mo[v], rtol=RTOL, atol=0)
    # synthetic statistics: roughly half the valid pixels break, dead pixels are invalid
    frac = (first[valid.astype(bool)] > 0).mean()
    assert 0.3 < frac < 0.9, frac          # C4/C5 use an uncalibrated lambda = 3 (more alarms)
    assert valid.mean() > 0.99
    if w.clustered:            # the C5 stack carries clustered clouds, ~19% missing
        assert 0.1 < float(np.isnan(ys).mean()) < 0.3


@pytest.mark.parametrize("name", ["C2", "C5"])
def test_fullsize_shift_and_shards(name):
    """Pixel-placement invariance on the whole stack, without copies: monitoring the view that
    starts s pixels in (a different tile / warp slice / lane for every pixel; s = 4 mod 256
    keeps the TMA path) gives the maps of the whole stack shifted by s, and so do two shards."""
    w, t, plan, y = _setup(name)
    P = w.n_pixels
    base = _maps(plan.run_device(y))
    s = 256 * 1001 + 4
    got = _maps(plan.run_device(y[:, s:], pixel_offset=s))
    for a, b in zip(base, got):
        assert np.array_equal(a[s:], b)
    cut = (P // 3) // 2 * 2 + 2                      # 8-byte aligned: LDG path for the upper shard
    lo = _maps(plan.run_device(y[:, :cut]))
    hi = _maps(plan.run_device(y[:, cut:], pixel_offset=cut))
    for a, b, c in zip(base, lo, hi):
        assert np.array_equal(a, np.concatenate([b, c]))


def _masked_plan(w, t):
    from paper_1807_01751_b200.device import DevicePlan
    from paper_1807_01751_b200.model import TimeAxis

    return DevicePlan(TimeAxis(t), w.freq, w.harmonics, w.n_hist, w.bandwidth, w.crit, "cuda", nan_mode="mask")


@pytest.mark.parametrize("name", ["C2", "C4"])
def test_fullsize_masked_sample_against_oracle(name):
    """nan_mode="mask" on the whole stack — C2: shared-memory residual rings,
    C4: the global-scratch variant (p = 14, h = 250) — and a 3,000-pixel sample against the
    per-pixel masked oracle: valid identical, first break identical off the boundary, max |MO|
    within rtol 1e-4."""
    import torch

    w, t, _, y = _setup(name)
    plan = _masked_plan(w, t)
    assert plan.info()["masked_global"] == (1 if name == "C4" else 0)
    valid, first, mx = _maps(plan.run_device(y))
    rng = np.random.default_rng(11)
    idx = np.sort(rng.choice(w.n_pixels, size=3000, replace=False))
    ys = y[:, torch.as_tensor(idx, device="cuda")].cpu().numpy()
    del y
    torch.cuda.empty_cache()
    ref = bo.monitor_masked(ys, t, w.n_hist, w.bandwidth, w.harmonics, w.freq, w.crit)
    assert np.array_equal(valid[idx].astype(bool), ref.valid)
    bad = np.flatnonzero((first[idx] != ref.first_idx) & ~ref.near & ref.valid)
    assert bad.size == 0, f"{bad.size} non-borderline mismatches, e.g. pixels {idx[bad[:5]]}"
    np.testing.assert_allclose(mx[idx][ref.valid], ref.max_abs_mo[ref.valid], rtol=RTOL, atol=0)
    assert valid.mean() > 0.99


def test_fullsize_masked_shift_and_shards():
    """The placement invariance of test_fullsize_shift_and_shards for the masked kernel at C2:
    one pixel per thread, but warp-wide decisions (the backward window sweep, the exact-sweep
    lanes) and the per-tile Gram MMAs must not leak between pixels."""
    w, t, _, y = _setup("C2")
    plan = _masked_plan(w, t)
    P = w.n_pixels
    base = _maps(plan.run_device(y))
    s = 128 * 1001 + 37
    got = _maps(plan.run_device(y[:, s:], pixel_offset=s))
    for a, b in zip(base, got):
        assert np.array_equal(a[s:], b)
    cut = P // 3 + 5
    lo = _maps(plan.run_device(y[:, :cut]))
    hi = _maps(plan.run_device(y[:, cut:], pixel_offset=cut))
    for a, b, c in zip(base, lo, hi):
        assert np.array_equal(a, np.concatenate([b, c]))


@pytest.mark.parametrize("name", ["C2", "C4", "C5"])
def test_fullsize_dynamic_schedule(name, monkeypatch):
    """The TMA kernel's dynamic per-warp slice scheduler (default) hands 64-px slices to
    whichever warp asks first, so a pixel's slice lands on a different warp, CTA and SM from
    run to run: the maps must equal the static schedule's bit for bit, and repeated calls on
    one plan (the scheduler's counters reset themselves at the end of every launch) must too."""
    from paper_1807_01751_b200.device import DevicePlan
    from paper_1807_01751_b200.model import TimeAxis

    w, t, plan, y = _setup(name)
    assert plan.info()["dyn_sched"] == 1
    runs = [_maps(plan.run_device(y)) for _ in range(3)]
    monkeypatch.setenv("BWM_DYN", "0")
    static = DevicePlan(TimeAxis(t), w.freq, w.harmonics, w.n_hist, w.bandwidth, w.crit, "cuda")
    monkeypatch.delenv("BWM_DYN")
    assert static.info()["dyn_sched"] == 0
    ref = _maps(static.run_device(y))
    for got in runs:
        for a, b in zip(ref, got):
            assert np.array_equal(a, b)
    # C2 runs its LEAN launches on the 16-date-stage (TALL) variant, C5 on the TALL variant without
    # ring mirror rows: same bits as 8-date stages
    assert plan.info()["tall_stages"] == {"C2": 1, "C4": 0, "C5": 2}[name]
    monkeypatch.setenv("BWM_TALL", "0")
    short = DevicePlan(TimeAxis(t), w.freq, w.harmonics, w.n_hist, w.bandwidth, w.crit, "cuda")
    monkeypatch.delenv("BWM_TALL")
    for a, b in zip(ref, _maps(short.run_device(y))):
        assert np.array_equal(a, b)
