"""BTS1 file -> GPU streaming path (dataio.monitor_file / bwm_monitor_file), on the GPU.

monitor_file must give exactly the maps monitor_batch(read_stack(path)) gives — same kernel,
same inputs — whatever the staging geometry: whole-stack mode, the chunked pipeline
(BWM_HOST_CHUNK) and rectangles split inside a row (BWM_IO_SLOT_BYTES).  One golden case is
also checked against the reference's own outputs through the file path.
"""
import numpy as np
import pytest

from tests.golden_cases import load
from tests.test_gpu_parity import check_parity, config_for

pytestmark = pytest.mark.gpu


def _pkg():
    import paper_1807_01751_b200 as pkg

    return pkg


def _same(a, b):
    for f in ("detected", "first_break", "max_abs_mo", "valid"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    if a.mosum is not None:
        assert np.array_equal(a.mosum, b.mosum)
    if a.beta is not None:
        assert np.array_equal(a.beta, b.beta)


@pytest.mark.parametrize("name", ["c1", "irregular_h70"])
def test_file_path_matches_reference_golden(tmp_path, name):
    pkg = _pkg()
    case = load(name)
    path = tmp_path / "s.bts"
    pkg.write_stack(pkg.SeriesStack(case.y, pkg.TimeAxis(case.t)), path)
    bm = pkg.monitor_file(path, config_for(case))
    check_parity(case, bm.first_break, bm.max_abs_mo, bm.valid)


@pytest.mark.parametrize("env", [{}, {"BWM_HOST_CHUNK": "3000"}, {"BWM_IO_SLOT_BYTES": "4096"},
                                 {"BWM_HOST_CHUNK": "2600", "BWM_IO_SLOT_BYTES": "1000"}])
def test_file_equals_batch(tmp_path, monkeypatch, env):
    pkg = _pkg()
    case = load("c1")
    path = tmp_path / "s.bts"
    pkg.write_stack(pkg.SeriesStack(case.y[:, :9001], pkg.TimeAxis(case.t)), path)  # ragged tail tile
    cfg = config_for(case)
    ref = pkg.monitor_batch(pkg.read_stack(path), cfg, keep_mosum=True, return_beta=True)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    got = pkg.monitor_file(path, cfg, keep_mosum=True, return_beta=True)
    _same(got, ref)


def test_file_masked_mode(tmp_path):
    pkg = _pkg()
    case = load("c1")
    path = tmp_path / "s.bts"
    pkg.write_stack(pkg.SeriesStack(case.y, pkg.TimeAxis(case.t)), path)
    from dataclasses import replace

    cfg = replace(config_for(case), nan_mode="mask")
    _same(pkg.monitor_file(path, cfg), pkg.monitor_batch(pkg.read_stack(path), cfg))


def test_truncated_payload_raises(tmp_path):
    pkg = _pkg()
    case = load("c1")
    path = tmp_path / "s.bts"
    pkg.write_stack(pkg.SeriesStack(case.y[:, :100], pkg.TimeAxis(case.t)), path)
    raw = path.read_bytes()
    path.write_bytes(raw[:-4])
    with pytest.raises(pkg.StackFormatError, match="truncated"):
        pkg.monitor_file(path, config_for(case))


def test_profile_file_phases(tmp_path):
    pkg = _pkg()
    case = load("c1")
    path = tmp_path / "s.bts"
    pkg.write_stack(pkg.SeriesStack(case.y, pkg.TimeAxis(case.t)), path)
    bm, t = pkg.profile_file(path, config_for(case))
    assert len(bm) == case.y.shape[1]
    assert t.mosum > 0 and t.ingest > 0 and t.total >= t.mosum


@pytest.mark.parametrize("env", [{}, {"BWM_HOST_CHUNK": "3000"}, {"BWM_IO_SLOT_BYTES": "4096"},
                                 {"BWM_HOST_STAGED": "0"}])
def test_pageable_host_stack(monkeypatch, env):
    """A plain (pageable) numpy stack goes through the staged pinned-slot pipeline; the maps
    equal those of a pinned copy and of the device path, bit for bit."""
    import torch

    pkg = _pkg()
    case = load("c1")
    y = np.ascontiguousarray(case.y[:, :9001])
    cfg = config_for(case)
    pinned = torch.empty(y.shape, dtype=torch.float32, pin_memory=True)
    pinned.numpy()[...] = y
    ref = pkg.monitor_batch(pkg.SeriesStack(pinned.numpy(), pkg.TimeAxis(case.t)), cfg, return_beta=True)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    got = pkg.monitor_batch(pkg.SeriesStack(y, pkg.TimeAxis(case.t)), cfg, return_beta=True)
    _same(got, ref)
    dev = pkg.monitor_batch(pkg.SeriesStack(torch.as_tensor(y, device="cuda"), pkg.TimeAxis(case.t)), cfg)
    _same(dev, pkg.monitor_batch(pkg.SeriesStack(y, pkg.TimeAxis(case.t)), cfg))


def test_file_pixel_ranges_equal_whole(tmp_path):
    """Each rank's band of one file (monitor_file(pixels=...), bwm_monitor_file_range) gives
    exactly the corresponding slice of the whole-file maps."""
    pkg = _pkg()
    from paper_1807_01751_b200.sharding import shard_bounds

    case = load("c1")
    path = tmp_path / "s.bts"
    pkg.write_stack(pkg.SeriesStack(case.y[:, :9001], pkg.TimeAxis(case.t)), path)
    cfg = config_for(case)
    whole = pkg.monitor_file(path, cfg, keep_mosum=True)
    for a, b in shard_bounds(9001, 3, align=4):
        part = pkg.monitor_file(path, cfg, keep_mosum=True, pixels=(a, b))
        for f in ("detected", "first_break", "max_abs_mo", "valid"):
            assert np.array_equal(getattr(part, f), getattr(whole, f)[a:b]), f
        assert np.array_equal(part.mosum, whole.mosum[:, a:b])
    with pytest.raises(ValueError):
        pkg.monitor_file(path, cfg, pixels=(5, 9002))
