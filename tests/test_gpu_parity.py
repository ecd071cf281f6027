"""Parity of the CUDA path (libbwm through the C ABI) against the reference's golden
outputs and the CPU oracle.  Tolerances (BASELINE.json north_star):

  valid        identical
  first_break  identical on every pixel that is not borderline (a window j <= the later of
               the two first crossings with | |MO_ref,j| - b_j | <= 1e-4 b_j)
  max_abs_mo   rtol 1e-4
  mosum_mean   |d| <= 1e-4 * max(|mean_ref|, max_abs_ref)  (a mean of signed terms)
  beta         |d_i| <= 1e-4 |beta_ref,i| + 1e-4 ||M_i,:||_1 ||y_hist||_inf

Degenerate pixels — a constant filled history (e.g. a leading gap covering the history) —
have sigma at float64 round-off in the reference: its MO is round-off / round-off (noise) on
windows without a real value change, and ~1e15 on windows with one.  The kernel computes
sigma = 0 exactly there, so its first break is the first window holding a real change.
Magnitudes are not compared; where the reference blew up (max |MO| > 1e10) the kernel must
blow up too and break no earlier than the reference (whose noise may cross sooner); a
constant whole series (noise-only decisions in the reference) is excluded.
"""

import re

import numpy as np
import pytest

from oracle import bfast_oracle as bo
from tests.golden_cases import CASES, load

pytestmark = pytest.mark.gpu

RTOL = 1e-4


def _pkg():
    import paper_1807_01751_b200 as pkg

    return pkg


def degenerate_pixels(case):
    filled, valid = bo.fill_block(case.y)
    return valid & (filled[:case.n] == filled[0]).all(axis=0)


def check_parity(case, first_break, max_abs, valid, mean=None, beta=None, mosum=None):
    n_mon = case.y.shape[0] - case.n
    P = case.y.shape[1]
    assert np.array_equal(valid, case.valid), "valid mask differs"
    first_gpu = np.where(first_break > 0, first_break - case.n, 0)
    border = bo.borderline_from_pairs(case.near, n_mon, P, case.first_idx, first_gpu)
    degen = degenerate_pixels(case)
    blown = degen & (case.max_abs_mo > 1e10)
    bad = np.flatnonzero((first_gpu != case.first_idx) & ~border & ~degen)
    assert bad.size == 0, f"{case.name}: {bad.size} non-borderline break mismatches, e.g. {bad[:5]}"
    assert np.all(max_abs[blown] > 1e10), "round-off-sigma pixels must blow up where the reference does"
    assert np.all(first_gpu[blown] >= case.first_idx[blown]) and np.all(case.first_idx[blown] > 0)
    assert degen.sum() <= max(12, P // 100), "degenerate pixels must stay rare in the fixtures"
    ok = ~degen
    np.testing.assert_allclose(max_abs[ok], case.max_abs_mo[ok], rtol=RTOL, atol=0)
    if mean is not None:
        scale = np.maximum(np.abs(case.mosum_mean), case.max_abs_mo)
        assert np.all((np.abs(mean - case.mosum_mean) <= RTOL * scale + 1e-30)[ok])
    if beta is not None and case.beta is not None:
        X = bo.design_matrix(case.t, case.freq, case.k)
        M = bo.mapping_matrix(X, case.n)
        filled, _ = bo.fill_block(case.y)
        yinf = np.abs(filled[:case.n]).max(axis=0)
        tol = RTOL * np.abs(case.beta) + RTOL * np.abs(M).sum(axis=1)[:, None] * yinf[None, :]
        assert np.all(np.abs(beta - case.beta) <= tol), f"{case.name}: beta out of tolerance"
    if mosum is not None and case.mosum is not None:
        scale = np.maximum(case.max_abs_mo, 1e-30)[None, :]
        assert np.all((np.abs(mosum - case.mosum) <= RTOL * scale)[:, ok])
    return int(border.sum())


def config_for(case, backend="fused"):
    return _pkg().MonitorConfig(history=case.n, bandwidth=case.h, harmonics=case.k, freq=case.freq,
                                crit_value=case.crit, backend=backend)


@pytest.mark.parametrize("name", CASES)
def test_golden_parity_host_path(name):
    pkg = _pkg()
    case = load(name)
    stack = pkg.SeriesStack(case.y, pkg.TimeAxis(case.t))
    bm = pkg.monitor_batch(stack, config_for(case), keep_mosum=True, return_beta=True, return_mean=True)
    assert bm.first_break.dtype == np.int64 and bm.max_abs_mo.dtype == np.float64 and bm.valid.dtype == bool
    check_parity(case, bm.first_break, bm.max_abs_mo, bm.valid, bm.mosum_mean, bm.beta, bm.mosum)
    assert np.array_equal(bm.detected, bm.first_break > 0)
    assert bm.crit_value == case.crit


@pytest.mark.parametrize("name", CASES)
def test_golden_parity_device_path(name):
    import torch

    pkg = _pkg()
    case = load(name)
    y = torch.as_tensor(case.y, device="cuda")
    stack = pkg.SeriesStack(y, pkg.TimeAxis(case.t))
    bm = pkg.monitor_batch(stack, config_for(case, "cuda"), keep_mosum=True, return_beta=True, return_mean=True)
    check_parity(case, bm.first_break, bm.max_abs_mo, bm.valid, bm.mosum_mean, bm.beta, bm.mosum)


def _plan(case, env=None, monkeypatch=None):
    from paper_1807_01751_b200.device import DevicePlan
    from paper_1807_01751_b200.model import TimeAxis

    if env is not None:
        monkeypatch.setenv("BWM_KERNEL", env)
    plan = DevicePlan(TimeAxis(case.t), case.freq, case.k, case.n, case.h, case.crit, "cuda")
    if env is not None:
        monkeypatch.delenv("BWM_KERNEL")
    return plan


def _maps(res):
    return [None if a is None else a.cpu().numpy() for a in (res.valid, res.first_idx, res.max_abs, res.mo_mean, res.beta)]


@pytest.mark.parametrize("name", ["c1", "c4_tile", "odd_pixels_k8", "edges_h10_k2", "lag_h100"])
def test_kernel_variants_bit_identical(name, monkeypatch):
    """TMA-staged kernel, register-prefetch kernel and the scalar safe kernel (misaligned
    input) run the same arithmetic in the same order: results must match bit for bit."""
    import torch

    case = load(name)
    y = torch.as_tensor(case.y, device="cuda")
    tma = _maps(_plan(case).run_device(y, beta=True, mean=True))
    ldg = _maps(_plan(case, "ldg", monkeypatch).run_device(y, beta=True, mean=True))
    # misaligned view: pixel 0 at a 4-byte offset -> safe kernel for every tile
    big = torch.empty((y.shape[0], y.shape[1] + 1), device="cuda")
    big[:, 1:] = y
    safe = _maps(_plan(case).run_device(big[:, 1:], beta=True, mean=True))
    for a, b, c in zip(tma, ldg, safe):
        assert np.array_equal(a, b)
        assert np.array_equal(a, c)
    # the LEAN TMA variant (no mean/MOSUM outputs requested; constant boundary hoisted)
    lean = _maps(_plan(case).run_device(y))
    for a, b in zip(lean[:3], ldg[:3]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("name", ["c1", "c4_tile", "lag_h100", "edges_h10_k2", "c5_tile", "three_pixels"])
def test_dynamic_schedule_bit_identical(name, monkeypatch):
    """The TMA kernel's dynamic slice scheduler (default) against the static schedule
    (BWM_DYN=0), and back-to-back calls on one plan (the counters reset in-kernel): same bits."""
    import torch

    from paper_1807_01751_b200.device import DevicePlan
    from paper_1807_01751_b200.model import TimeAxis

    case = load(name)
    y = torch.as_tensor(case.y, device="cuda")
    dyn = _plan(case)
    runs = [_maps(dyn.run_device(y, beta=True, mean=True)) for _ in range(3)]
    runs.append(_maps(dyn.run_device(y))[:3] + [None, None])           # LEAN variant
    monkeypatch.setenv("BWM_DYN", "0")
    static = DevicePlan(TimeAxis(case.t), case.freq, case.k, case.n, case.h, case.crit, "cuda")
    monkeypatch.delenv("BWM_DYN")
    assert static.info()["dyn_sched"] == 0
    ref = _maps(static.run_device(y, beta=True, mean=True))
    for got in runs:
        for a, b in zip(ref, got):
            if b is not None:
                assert np.array_equal(a, b)
    # the LEAN launch's 16-date-stage (TALL) variant against the 8-date kernel
    monkeypatch.setenv("BWM_TALL", "0")
    short = DevicePlan(TimeAxis(case.t), case.freq, case.k, case.n, case.h, case.crit, "cuda")
    monkeypatch.delenv("BWM_TALL")
    assert short.info()["tall_stages"] == 0
    # 16-date stages: c1 with mirror rows (1), c5_tile without (2: 64 + 16 rows would double the
    # TMEM allocation), the lagging cursor never
    expect = {"c1": 1, "c4_tile": 0, "c5_tile": 2, "lag_h100": 1}
    if name in expect:
        assert dyn.info()["tall_stages"] == expect[name]
    for a, b in zip(_maps(short.run_device(y))[:3], runs[-1][:3]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("P", [3000, 1024 + 2, 77])
def test_lagging_cursor_ragged_tail(P):
    """c4_tile (h = 250: the 16-warp lagging-cursor TMA kernel, 1,024-px tiles) cut to P pixels:
    whole tiles run on the TMA kernel, the rest on the LDG lagging cursor — both must give the
    bits the all-TMA run gives for those pixels, and match the reference's golden maps."""
    import torch

    case = load("c4_tile")
    plan = _plan(case)
    assert plan.info()["ring_mode"] == "lag_smem_tables"
    y = torch.as_tensor(case.y, device="cuda")
    whole = _maps(plan.run_device(y, mean=True))
    part = _maps(plan.run_device(y[:, :P].contiguous(), mean=True))
    for a, b in zip(whole[:4], part[:4]):
        assert np.array_equal(a[:P], b)
    n = case.n
    fi = part[1].astype(np.int64)
    near = case.near[case.near[:, 1] < P] if case.near.ndim == 2 else case.near[:P]   # (j, pixel) pairs
    sub = type(case)(case.name, case.y[:, :P], case.t, case.n, case.h, case.k, case.freq, case.crit,
                     case.first_break[:P], case.max_abs_mo[:P], case.valid[:P], near, case.bound,
                     case.mosum_mean[:P], None, None, case.info)
    check_parity(sub, np.where(fi > 0, fi + n, 0), part[2].astype(np.float64), part[0].astype(bool), part[3])


@pytest.mark.parametrize("shards", [2, 3, 8])
def test_shard_invariance(shards):
    """Results are bit-identical whatever the pixel sharding (the GPU analogue of
    test_engine.py:170-181 'results do not depend on the worker count')."""
    import torch

    case = load("c1")
    plan = _plan(case)
    y = torch.as_tensor(case.y, device="cuda")
    whole = _maps(plan.run_device(y, mean=True))
    P = y.shape[1]
    edges = np.linspace(0, P, shards + 1).astype(int)
    edges[1:-1] = (edges[1:-1] // 2) * 2          # keep float2 alignment of each shard
    parts = [_maps(plan.run_device(y[:, a:b], mean=True, pixel_offset=int(a))) for a, b in zip(edges[:-1], edges[1:])]
    for i in range(4):
        assert np.array_equal(whole[i], np.concatenate([p[i] for p in parts]))


def test_host_and_device_paths_identical():
    import torch

    case = load("c5_tile")
    plan = _plan(case)
    host = plan.run_host(case.y, beta=True, mean=True, keep_mosum=True)
    dev = plan.run_device(torch.as_tensor(case.y, device="cuda"), beta=True, mean=True, keep_mosum=True)
    for a, b in [(host.valid, dev.valid), (host.first_idx, dev.first_idx), (host.max_abs, dev.max_abs),
                 (host.mo_mean, dev.mo_mean), (host.beta, dev.beta), (host.mosum, dev.mosum)]:
        assert np.array_equal(a, b.cpu().numpy())
    assert host.h2d_bytes == case.y.nbytes


def test_zero_sigma_raises_for_lowest_pixel():
    import json

    from tests.golden_cases import GOLDEN

    pkg = _pkg()
    z = np.load(GOLDEN / "zero_sigma.npz")
    info = json.loads(str(z["info"]))
    cfg = pkg.MonitorConfig(history=100, bandwidth=50, harmonics=3, freq=23.0, crit_value=4.9)
    with pytest.raises(pkg.ZeroResidualError, match=re.escape(info["message"])):
        pkg.monitor_batch(pkg.SeriesStack(z["y"], pkg.regular_axis(200)), cfg)


def test_determinism_and_permutation_equivariance():
    import torch

    case = load("c4_tile")
    plan = _plan(case)
    y = torch.as_tensor(case.y, device="cuda")
    a = _maps(plan.run_device(y, mean=True))
    b = _maps(plan.run_device(y, mean=True))
    for u, v in zip(a[:4], b[:4]):
        assert np.array_equal(u, v)
    perm = torch.randperm(y.shape[1], generator=torch.Generator().manual_seed(3)).cuda()
    c = _maps(plan.run_device(y[:, perm].contiguous(), mean=True))
    p = perm.cpu().numpy()
    for u, v in zip(a[:4], c[:4]):
        assert np.array_equal(u[p], v)


@pytest.mark.parametrize("wname", ["C2", "C4", "C5"])
def test_large_stack_sampled_tiles(wname):
    """Full-size kernels on device-generated stacks; sampled tiles checked against the oracle
    (the f64 oracle of a whole C2 stack would need ~124 GB of host RAM)."""
    import torch

    from paper_1807_01751_b200.device import DevicePlan
    from paper_1807_01751_b200.model import TimeAxis
    from paper_1807_01751_b200.synth import WORKLOADS, device_stack, time_axis

    w = WORKLOADS[wname]
    t = time_axis(w)
    P = {"C2": 1 << 21, "C4": 1 << 18, "C5": 1 << 20}[wname]      # bounded for test time
    y = device_stack(P, t, w.freq, w.n_hist, w.nan_frac, seed=20261017, device="cuda")
    plan = DevicePlan(TimeAxis(t), w.freq, w.harmonics, w.n_hist, w.bandwidth, w.crit, "cuda")
    res = plan.run_device(y, mean=True)
    valid, first, mx, mean, _ = _maps(res)
    rng = np.random.default_rng(1)
    tiles = sorted(set(rng.integers(0, P // 256, 3).tolist()) | {P // 256 - 1})
    for tile in tiles:
        sl = slice(tile * 256, tile * 256 + 256)
        ys = y[:, sl].cpu().numpy()
        r = bo.monitor(ys, t, w.n_hist, w.bandwidth, w.harmonics, w.freq, w.crit, keep_mosum=True)
        assert np.array_equal(valid[sl].astype(bool), r.valid)
        border = bo.borderline(r.mosum, r.bound, r.first_idx, first[sl].astype(np.int64))
        assert not np.any((first[sl] != r.first_idx) & ~border)
        np.testing.assert_allclose(mx[sl], r.max_abs_mo, rtol=RTOL)
    # size-independent properties of the whole stack
    assert np.all((first >= 0) & (first <= t.size - w.n_hist))
    assert np.all(mx[valid == 0] == 0) and np.all(first[valid == 0] == 0)
    assert np.all(np.abs(mean) <= mx + 1e-6)
    del y
    torch.cuda.empty_cache()


def test_critical_value_matches_pinned():
    """lambda through the GPU kernel vs the reference's pinned value (test_mosum.py:20)."""
    import json

    from tests.golden_cases import GOLDEN

    pkg = _pkg()
    pinned = json.loads((GOLDEN / "pinned.json").read_text())["crit_20k"]
    req = pkg.CriticalValueRequest(**pinned["request"])
    lam = pkg.critical_value(req, threads=8)
    assert lam == pytest.approx(pinned["value"], rel=2e-5)


@pytest.mark.parametrize("seed,rep0,reps,n_obs", [(1, 0, 2048, 200), (7, 49000, 1000, 228), (2**64 - 5, 3, 300, 1000)])
def test_null_draws_match_numpy(seed, rep0, reps, n_obs):
    """bwm_null_draws (device Philox4x64-10 + ziggurat) reproduces the reference's null series
    bit for bit: replication r = Generator(Philox(key=seed, counter=r << 128)).standard_normal
    (reference mosum.py:195-198), as float32.  The samples cover ziggurat wedge and tail draws
    (~0.7% of draws leave the fast path)."""
    import ctypes as C

    import torch

    from paper_1807_01751_b200 import _lib
    from paper_1807_01751_b200.mosum import CriticalValueRequest, null_draws

    lib = _lib.load()
    ld = reps + 5                                  # padded leading dimension
    out = torch.full((n_obs, ld), float("nan"), dtype=torch.float32, device="cuda")
    _lib.check(lib.bwm_null_draws(seed & ((1 << 64) - 1), seed >> 64, rep0, reps, n_obs, out.data_ptr(), ld,
                                  C.c_void_p(torch.cuda.current_stream().cuda_stream)), "bwm_null_draws")
    req = CriticalValueRequest(alpha=0.05, h_frac=0.5, horizon=2.0, n_sim=100, reps=1000, seed=seed)
    ref = null_draws(req, rep0, rep0 + reps, n_obs, dtype=np.float32)
    got = out.cpu().numpy()
    assert np.array_equal(got[:, :reps].view(np.uint32), ref.view(np.uint32))
    assert np.isnan(got[:, reps:]).all()          # nothing written past the replications


@pytest.mark.parametrize("N,n,h,k", [(3000, 1500, 20, 8), (2600, 1300, 400, 6)])
def test_long_series(N, n, h, k):
    """Series too long for shared-memory tables (N * p floats > 227 KB): the lagging-cursor
    kernels read their tables through L1 — any N is supported, as in the reference."""
    pkg = _pkg()
    from paper_1807_01751_b200.synth import host_stack

    t = np.cumsum(np.random.default_rng(3).uniform(1, 9, N)) + 1.0
    y = host_stack(1500, t, 365.25, n, 0.3, seed=11)
    crit = 3.0
    cfg = pkg.MonitorConfig(history=n, bandwidth=h, harmonics=k, freq=365.25, crit_value=crit)
    bm = pkg.monitor_batch(pkg.SeriesStack(y, pkg.TimeAxis(t)), cfg)
    ref = bo.monitor(y, t, n, h, k, 365.25, crit, keep_mosum=True)
    assert np.array_equal(bm.valid, ref.valid)
    first_gpu = np.where(bm.first_break > 0, bm.first_break - n, 0)
    pairs = bo.near_pairs(ref.mosum, bo.boundary(n, N, crit))
    border = bo.borderline_from_pairs(pairs, N - n, y.shape[1], ref.first_idx, first_gpu)
    assert not np.any((first_gpu != ref.first_idx) & ~border & ref.valid)
    np.testing.assert_allclose(bm.max_abs_mo[ref.valid], ref.max_abs_mo[ref.valid], rtol=RTOL, atol=0)


@pytest.mark.parametrize("name", ["c4_tile", "c5_tile"])
def test_tensor_core_fitted_values(name, monkeypatch):
    """The opt-in lagging-cursor kernel with its fitted values on the tensor cores
    (BWM_MMA=1, bwm_kernel_mma.cuh: 3xTF32 tcgen05.mma) meets the same parity bar as the FFMA
    kernels: a different arithmetic for z_t^T beta_Q, so the check is the oracle tolerance, not
    bit identity.  c5_tile (h = 50) is forced onto the lagging cursor with a 64-column TMEM cap."""
    import torch

    from paper_1807_01751_b200.device import DevicePlan
    from paper_1807_01751_b200.model import TimeAxis

    case = load(name)
    monkeypatch.setenv("BWM_MMA", "1")
    monkeypatch.setenv("BWM_TMEM_COLS_MAX", "64")
    plan = DevicePlan(TimeAxis(case.t), case.freq, case.k, case.n, case.h, case.crit, "cuda")
    monkeypatch.delenv("BWM_MMA")
    monkeypatch.delenv("BWM_TMEM_COLS_MAX")
    assert plan.info()["mma"] == 1
    n = case.n
    y = torch.as_tensor(case.y, device="cuda")
    for kw in (dict(), dict(mean=True, keep_mosum=True)):         # LEAN and general variants
        res = plan.run_device(y, **kw)
        fi = res.first_idx.cpu().numpy()
        check_parity(case, np.where(fi > 0, fi + n, 0), res.max_abs.cpu().numpy().astype(np.float64),
                     res.valid.cpu().numpy().astype(bool),
                     None if res.mo_mean is None else res.mo_mean.cpu().numpy(),
                     None, None if res.mosum is None else res.mosum.cpu().numpy())
