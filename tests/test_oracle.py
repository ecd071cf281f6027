"""Pin the CPU oracle before trusting it: golden vectors of the reference, the reference's
own known-answer tests, and (in the build container) the live reference."""

import numpy as np
import pytest

from oracle import bfast_oracle as bo
from tests.golden_cases import CASES, load


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference_golden(name):
    c = load(name)
    r = bo.monitor(c.y, c.t, c.n, c.h, c.k, c.freq, c.crit, keep_mosum=True, want_beta=True)
    assert np.array_equal(r.valid, c.valid)
    assert np.array_equal(r.first_break, c.first_break)       # float64 restatement: exact decisions
    np.testing.assert_allclose(r.max_abs_mo, c.max_abs_mo, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(r.bound, c.bound, rtol=0, atol=0)
    np.testing.assert_allclose(r.mosum.mean(axis=0), c.mosum_mean, rtol=1e-9, atol=1e-12)
    if c.beta is not None:
        np.testing.assert_allclose(r.beta, c.beta, rtol=1e-9, atol=1e-12)
    if c.mosum is not None:
        np.testing.assert_allclose(r.mosum, c.mosum, rtol=1e-9, atol=1e-12)


def test_zero_sigma_contract_golden():
    from tests.golden_cases import GOLDEN
    import json

    z = np.load(GOLDEN / "zero_sigma.npz")
    info = json.loads(str(z["info"]))
    with pytest.raises(bo.OracleZeroResidual, match=f"pixel {info['pixel']} "):
        bo.monitor(z["y"], np.arange(1.0, 201.0), 100, 50, 3, 23.0, 4.9)


# ---- known-answer tests of the reference's own suite -------------------------------------

def test_detect_kat():
    # pkg/tests/test_kernels.py:88-96
    mo = np.array([[0.5, -0.1], [0.2, 3.0], [2.5, 0.0]])
    first, mx = bo.detect_block(mo, np.array([1.0, 1.0, 2.0]))
    assert list(first) == [3, 2]
    assert list(mx) == [2.5, 3.0]


def test_single_value_mosum_kat():
    # pkg/tests/test_mosum.py:41-52: n=4, h=2, value 0.8 at row n-h+1 -> [0.4, 0, 0, 0]
    resid = np.zeros((8, 1))
    resid[3, 0] = 0.8
    out = bo.mosum_block(resid, 4, 2, np.array([0.5]))
    assert np.array_equal(out[:, 0], [0.4, 0.0, 0.0, 0.0])


def test_window_reach_kat():
    # pkg/tests/test_mosum.py:32-39: rows before n-h+1 never contribute
    resid = np.zeros((15, 1))
    resid[:8, 0] = np.random.default_rng(0).normal(size=8)
    assert np.array_equal(bo.mosum_block(resid, 10, 3, np.ones(1))[:, 0], np.zeros(5))


def test_tie_does_not_trigger_and_negative_counts():
    # test_mosum.py:131-140 / SPEC.md:176: MO=(0.5,-3.0), b=2.39 -> first=2, max=3.0; tie -> none
    first, mx = bo.detect_block(np.array([[0.5], [-3.0]]), np.array([2.39, 2.39]))
    assert first[0] == 2 and mx[0] == 3.0
    first, _ = bo.detect_block(np.array([[2.0]]), np.array([2.0]))
    assert first[0] == 0


def test_fill_kats():
    # pkg/tests/test_engine.py:51-70
    assert np.array_equal(bo.fill_series(np.array([np.nan, 1.0, np.nan, 3.0])), [1, 1, 1, 3])
    assert np.array_equal(bo.fill_series(np.array([2.0, np.nan, np.nan])), [2, 2, 2])
    assert np.array_equal(bo.fill_series(np.array([np.inf, 4.0, -np.inf])), [4, 4, 4])
    s = np.array([0.5, 0.25, -1.0])
    assert np.array_equal(bo.fill_series(s), s)
    with pytest.raises(ValueError):
        bo.fill_series(np.array([np.nan, np.nan]))


def test_boundary_plateau():
    # test_mosum.py:93-95: b_0 = lambda (log_plus = 1 below e)
    b = bo.boundary(100, 200, 4.9)
    assert b[0] == 4.9
    assert np.all(np.diff(b) >= 0)


def test_dead_pixel_masked():
    # test_engine.py:196-204
    rng = np.random.default_rng(3)
    y = (0.5 + 0.05 * rng.standard_normal((200, 10))).astype(np.float32)
    y[:, 3] = np.nan
    r = bo.monitor(y, np.arange(1.0, 201.0), 100, 50, 3, 23.0, 4.9)
    assert not r.valid[3] and r.first_break[3] == 0 and r.max_abs_mo[3] == 0.0


# ---- live reference cross-checks (build container only) ----------------------------------

@pytest.mark.reference
@pytest.mark.parametrize("seed", [101, 202])
def test_oracle_matches_live_reference(reference, seed):
    bw = reference
    from paper_1807_01751_b200.synth import host_stack

    t = np.arange(1.0, 229.0)
    y = host_stack(2000, t, 23.0, 114, 0.2, seed=seed)
    cfg = bw.MonitorConfig(history=114, bandwidth=28, harmonics=3, freq=23.0, crit_value=2.96519227)
    ref = bw.monitor_batch(bw.SeriesStack(y, bw.TimeAxis(t)), cfg, keep_mosum=True)
    r = bo.monitor(y, t, 114, 28, 3, 23.0, 2.96519227, keep_mosum=True)
    assert np.array_equal(r.first_break, ref.first_break)
    assert np.array_equal(r.valid, ref.valid)
    np.testing.assert_allclose(r.mosum, ref.mosum, rtol=1e-9, atol=1e-12)


@pytest.mark.reference
def test_oracle_mapping_matches_reference_irregular(reference):
    bw = reference
    t = np.cumsum(np.random.default_rng(4).uniform(8, 24, 400)) + 1.0
    X = bo.design_matrix(t, 365.25, 3)
    M = bo.mapping_matrix(X, 200)
    ref = bw.fit_mapping(bw.build_design_matrix(bw.TimeAxis(t), 365.25, 3), 200).matrix
    np.testing.assert_allclose(M, ref, rtol=1e-9, atol=1e-12)
