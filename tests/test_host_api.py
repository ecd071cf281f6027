"""Host-side API of the drop-in (CPU, no GPU): the float64 setup the package does once per
batch and its error contract — the reference's pkg/tests/test_model.py, test_mosum.py and
test_engine.py cases that apply to this layer — plus the "no CPU fallback" rule.

Where /root/reference exists (the build container) the same calls are compared with the
live reference; elsewhere the reference-pinned values below stand in.
"""
import numpy as np
import pytest

import paper_1807_01751_b200 as pkg
from paper_1807_01751_b200.errors import DegreesOfFreedomError, RankDeficiencyError
from paper_1807_01751_b200.model import kernel_basis


class TestTimeAxis:
    @pytest.mark.parametrize("v", [[1.0], [1.0, 2.0, 2.0], [1.0, np.nan, 3.0], [1.0, np.inf]])
    def test_rejects(self, v):
        with pytest.raises(ValueError):
            pkg.TimeAxis(np.array(v))

    def test_regular_axis_is_one_based(self):
        assert np.array_equal(pkg.regular_axis(4).values, [1.0, 2.0, 3.0, 4.0])


class TestDesign:
    def test_first_column_values(self):                          # test_model.py:42-45
        d = pkg.build_design_matrix(np.array([1.0, 2.0]), 23.0, 1)
        np.testing.assert_allclose(d.matrix[:, 0], [1.0, 1.0, np.sin(2 * np.pi / 23), np.cos(2 * np.pi / 23)],
                                   rtol=0, atol=1e-12)

    def test_rows_and_full_cycle(self):
        d = pkg.build_design_matrix(np.array([1.0, 23.0]), 23.0, 2)
        assert d.matrix.shape == (6, 2) and d.n_params == 6
        for j in (1, 2):
            assert abs(d.matrix[2 * j, 1]) < 1e-12 and abs(d.matrix[2 * j + 1, 1] - 1.0) < 1e-12

    def test_intercept_and_raw_trend(self):
        axis = np.array([3.0, 5.5, 9.0])
        d = pkg.build_design_matrix(axis, 10.0, 1)
        assert np.array_equal(d.matrix[0], np.ones(3)) and np.array_equal(d.matrix[1], axis)

    @pytest.mark.parametrize("axis,freq,k", [([2.0, 1.0], 23.0, 1), ([1.0, 2.0], 23.0, 0),
                                             ([1.0, 2.0], 0.0, 1), ([1.0, 2.0], -1.0, 1)])
    def test_invalid(self, axis, freq, k):
        with pytest.raises(ValueError):
            pkg.build_design_matrix(np.array(axis), freq, k)

    @pytest.mark.reference
    def test_equals_reference(self, reference):
        axis = np.cumsum(np.random.default_rng(2).uniform(1, 9, 300))
        ours = pkg.build_design_matrix(axis, 365.25, 4).matrix
        ref = reference.build_design_matrix(axis, 365.25, 4).matrix
        assert np.array_equal(ours, ref)


class TestMapping:
    def test_identity_on_history(self):                           # test_model.py:84-89
        d = pkg.build_design_matrix(pkg.regular_axis(200), 23.0, 3)
        m = pkg.fit_mapping(d, 100)
        assert np.abs(m.matrix @ d.matrix[:, :100].T - np.eye(8)).max() < 1e-9

    @pytest.mark.parametrize("n", [8, 5])
    def test_degrees_of_freedom(self, n):
        d = pkg.build_design_matrix(pkg.regular_axis(50), 23.0, 3)
        with pytest.raises(DegreesOfFreedomError):
            pkg.fit_mapping(d, n)

    def test_history_beyond_design(self):
        with pytest.raises(ValueError):
            pkg.fit_mapping(pkg.build_design_matrix(pkg.regular_axis(50), 23.0, 1), 51)

    def test_rank_deficient(self):                                 # test_model.py:112-117
        with pytest.raises(RankDeficiencyError):
            pkg.fit_mapping(pkg.build_design_matrix(pkg.regular_axis(60), 1e9, 1), 40)

    def test_matches_svd_pseudo_inverse(self):
        rng = np.random.default_rng(7)
        for _ in range(5):
            axis = np.cumsum(rng.uniform(0.3, 1.7, 200))
            d = pkg.build_design_matrix(axis, 23.0, 3)
            m = pkg.fit_mapping(d, 120).matrix
            oracle = np.linalg.pinv(d.matrix[:, :120].T)
            assert np.abs(m - oracle).max() / np.abs(oracle).max() < 1e-8

    def test_kernel_basis_is_a_reparametrisation(self):
        """The centred-trend basis handed to libbwm fits the same values as the raw one."""
        axis = pkg.TimeAxis(np.cumsum(np.random.default_rng(4).uniform(1, 9, 400)))
        raw = pkg.build_design_matrix(axis, 365.25, 3)
        m_raw = pkg.fit_mapping(raw, 200).matrix
        kb = kernel_basis(axis, 365.25, 3, 200)
        y = np.random.default_rng(5).normal(size=(200, 7))
        fit_raw = raw.matrix.T @ (m_raw @ y)
        fit_kb = kb.design.T @ (kb.mapping @ y)
        np.testing.assert_allclose(fit_kb, fit_raw, rtol=0, atol=1e-9)


class TestBoundary:
    def test_plateau_and_log(self):
        b = pkg.boundary_values(100, 400, 2.0)
        assert b[0] == 2.0 and np.all(np.diff(b) >= 0)
        j = (int(np.floor(np.e * 100)) + 1) - 101                # counts t = n+1+j; first t/n > e
        assert b[j - 1] == 2.0 and b[j] > 2.0
        assert abs(b[-1] - 2.0 * np.sqrt(np.log(4.0))) < 1e-12

    def test_log_plus(self):
        np.testing.assert_allclose(pkg.log_plus([0.5, 1.0, np.e, np.e ** 2]), [1.0, 1.0, 1.0, 2.0])

    @pytest.mark.parametrize("n,N,lam", [(100, 100, 2.0), (100, 50, 2.0), (100, 200, 0.0), (100, 200, -1.0)])
    def test_invalid(self, n, N, lam):
        with pytest.raises(ValueError):
            pkg.boundary_values(n, N, lam)

    @pytest.mark.reference
    def test_equals_reference(self, reference):
        assert np.array_equal(pkg.boundary_values(114, 228, 2.96519227),
                              reference.boundary_values(114, 228, 2.96519227))


class TestCriticalValueRequest:
    @pytest.mark.parametrize("kw", [dict(alpha=1.5), dict(alpha=0.0), dict(h_frac=0.0), dict(h_frac=1.5),
                                    dict(horizon=1.0), dict(reps=999), dict(seed=-1), dict(harmonics=0),
                                    dict(freq=0.0)])
    def test_invalid(self, kw):
        args = dict(alpha=0.05, h_frac=0.5, horizon=2.0, n_sim=100, reps=1000, seed=1)
        args.update(kw)
        with pytest.raises(ValueError):
            pkg.CriticalValueRequest(**args)

    def test_n_sim_too_short(self):
        with pytest.raises(DegreesOfFreedomError):
            pkg.CriticalValueRequest(alpha=0.05, h_frac=0.5, horizon=2.0, n_sim=8, reps=1000, seed=1)


class TestMonitorConfig:
    @pytest.mark.parametrize("kw", [dict(harmonics=0), dict(freq=0.0), dict(history=8), dict(bandwidth=0),
                                    dict(bandwidth=101), dict(alpha=1.0), dict(crit_value=0.0),
                                    dict(nan_mode="drop"), dict(backend="bogus")])
    def test_invalid(self, kw):
        args = dict(history=100, bandwidth=50, harmonics=3, freq=23.0)
        args.update(kw)
        with pytest.raises(ValueError):
            pkg.MonitorConfig(**args)

    @pytest.mark.parametrize("backend", ["fused", "naive", "cuda"])
    def test_backends_accepted(self, backend):
        # the reference's two backends (engine.py:112,129-130) plus "cuda"; all run the GPU kernel
        assert pkg.MonitorConfig(history=100, bandwidth=50, harmonics=3, freq=23.0, backend=backend).backend == backend

    def test_n_params(self):
        assert pkg.MonitorConfig(history=100, bandwidth=50, harmonics=3, freq=23.0).n_params == 8


class TestEngineContract:
    def test_resolve_threads(self, monkeypatch):
        assert pkg.resolve_threads(3) == 3
        with pytest.raises(ValueError):
            pkg.resolve_threads(0)
        monkeypatch.setenv("BREAKWATCH_THREADS", "5")
        assert pkg.resolve_threads() == 5
        monkeypatch.setenv("BREAKWATCH_THREADS", "x")
        with pytest.raises(ValueError):
            pkg.resolve_threads()

    def test_history_must_end_before_series(self):
        st = pkg.SeriesStack(np.zeros((50, 2), np.float32), pkg.regular_axis(50))
        with pytest.raises(ValueError):
            pkg.monitor_batch(st, pkg.MonitorConfig(history=60, bandwidth=10, harmonics=1, freq=23.0))

    def test_stack_validation(self):
        with pytest.raises(ValueError):
            pkg.SeriesStack(np.zeros((5, 0), np.float32), pkg.regular_axis(5))
        with pytest.raises(ValueError):
            pkg.SeriesStack(np.zeros((5, 2), np.float32), pkg.regular_axis(6))

    def test_no_cpu_fallback(self):
        """Without a CUDA device the package raises instead of computing on the CPU."""
        import torch

        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
        st = pkg.SeriesStack(np.random.default_rng(0).normal(size=(60, 4)).astype(np.float32),
                             pkg.regular_axis(60))
        with pytest.raises(RuntimeError, match="CUDA|GPU"):
            pkg.monitor_batch(st, pkg.MonitorConfig(history=30, bandwidth=10, harmonics=1, freq=23.0,
                                                    crit_value=3.0))


class TestReferenceSurface:
    """Public names of the reference package (pkg/src/breakwatch/__init__.py:52-94)."""

    # per-series CPU diagnostics of the reference that are not on the batch hot path
    # (DESIGN.md §8): fit_history/predict/mosum_process/detect/amplitude_phase and their types
    OUT_OF_SCOPE = {"HistoryModel", "MosumSeries", "amplitude_phase", "detect", "fit_history", "mosum_process",
                    "predict"}
    REFERENCE_ALL = {
        "AllNanSeriesError", "BreakMap", "BreakResult", "BreakwatchError", "CriticalValueRequest", "CsvParseError",
        "DegreesOfFreedomError", "DesignMatrix", "HistoryModel", "MappingMatrix", "MonitorConfig", "MosumSeries",
        "PhaseTimings", "RankDeficiencyError", "SeriesStack", "StackCapacityError", "StackFormatError", "SynthSpec",
        "TimeAxis", "ZeroResidualError", "amplitude_phase", "bench_scaling", "boundary_values",
        "build_design_matrix", "critical_value", "detect", "fill_gaps", "fit_history", "fit_mapping", "generate",
        "log_plus", "monitor_batch", "mosum_process", "predict", "profile_run", "read_series_csv", "read_stack",
        "regular_axis", "resolve_crit_value", "resolve_threads", "write_bench_csv", "write_break_map",
        "write_stack"}

    def test_exports(self):
        missing = self.REFERENCE_ALL - self.OUT_OF_SCOPE - set(pkg.__all__)
        assert not missing, missing
        for name in pkg.__all__:
            assert hasattr(pkg, name), name

    @pytest.mark.reference
    def test_live_reference_names(self, reference):
        assert set(reference.__all__) == self.REFERENCE_ALL

    # fill KATs of the reference (test_engine.py:52-70)
    @pytest.mark.parametrize("series, want", [
        ([np.nan, 1.0, np.nan, 3.0], [1.0, 1.0, 1.0, 3.0]),
        ([np.inf, 4.0, -np.inf], [4.0, 4.0, 4.0]),
        ([1.0, 2.0, 3.0], [1.0, 2.0, 3.0]),
        ([np.nan, np.nan, 5.0, np.nan], [5.0, 5.0, 5.0, 5.0]),
    ])
    def test_fill_gaps(self, series, want):
        np.testing.assert_array_equal(pkg.fill_gaps(np.array(series)), np.array(want))

    def test_fill_gaps_all_missing(self):
        with pytest.raises(pkg.AllNanSeriesError):
            pkg.fill_gaps(np.array([np.nan, np.inf]))

    @pytest.mark.reference
    def test_fill_gaps_matches_reference(self, reference):
        ref_fill = reference.fill_gaps
        rng = np.random.default_rng(5)
        for _ in range(50):
            v = rng.normal(size=30)
            v[rng.random(30) < 0.4] = np.nan
            if not np.isfinite(v).any():
                continue
            np.testing.assert_array_equal(pkg.fill_gaps(v), ref_fill(v))

    def test_write_bench_csv(self, tmp_path):
        import sys
        from pathlib import Path

        REFERENCE_SRC = Path("/root/reference/pkg/src")
        rows = [(16, pkg.PhaseTimings(0.5, 0.25, 0.0, 0.0, 0.125, 0.0625, 0.9375))]
        p = tmp_path / "b.csv"
        assert pkg.write_bench_csv(rows, str(p)) == 1
        assert p.read_text() == ("m,ingest,model,predictions,residuals,mosum,breaks,total\n"
                                 "16,0.500000,0.250000,0.000000,0.000000,0.125000,0.062500,0.937500\n")
        if not REFERENCE_SRC.exists():
            return
        if str(REFERENCE_SRC) not in sys.path:
            sys.path.insert(0, str(REFERENCE_SRC))
        from breakwatch.synth import write_bench_csv as ref_write

        q = tmp_path / "r.csv"
        ref_write(rows, str(q))
        assert q.read_bytes() == p.read_bytes()

    def test_bench_scaling_validation(self):
        cfg = pkg.MonitorConfig(history=100, bandwidth=50, harmonics=3, freq=23.0, crit_value=3.0)
        spec = pkg.SynthSpec(n_pixels=8, n_obs=200, freq=23.0)
        with pytest.raises(ValueError):
            pkg.bench_scaling([], cfg, spec)
        with pytest.raises(ValueError):
            pkg.bench_scaling([0], cfg, spec)
