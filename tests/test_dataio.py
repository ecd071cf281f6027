"""BTS1 stack files, the break-map CSV and the synthetic generator, on CPU.

Mirrors the reference's pkg/tests/test_dataio.py; byte-level parity is pinned against files
the REFERENCE wrote (tests/golden/make_io_golden.py) and, in this container, against the live
reference.  The native pieces (bwm_read_payload, bwm_write_break_map) need no GPU.
"""
import io
import struct
from pathlib import Path

import numpy as np
import pytest

from paper_1807_01751_b200 import (
    BreakMap,
    MonitorConfig,
    SeriesStack,
    StackCapacityError,
    StackFormatError,
    TimeAxis,
    read_series_csv,
    read_stack,
    regular_axis,
    write_break_map,
    write_stack,
)
from paper_1807_01751_b200.errors import CsvParseError
from paper_1807_01751_b200.synth import SynthSpec, generate

GOLDEN = Path(__file__).resolve().parent / "golden"


def _stack(n_obs=6, m=3, seed=0, axis=None):
    rng = np.random.default_rng(seed)
    y = rng.normal(size=(n_obs, m)).astype(np.float32)
    return SeriesStack(y, axis if axis is not None else regular_axis(n_obs))


def _bytes(stack):
    buf = io.BytesIO()
    write_stack(stack, buf)
    return buf.getvalue()


class TestWrite:
    def test_minimal_file_is_25_bytes(self):                 # test_dataio.py:41
        assert len(_bytes(SeriesStack(np.zeros((2, 1), np.float32), regular_axis(2)))) == 17 + 8

    def test_explicit_axis_adds_eight_bytes_per_observation(self):
        s = _stack(axis=TimeAxis(np.array([1.0, 2.5, 3.0, 7.0, 8.0, 9.5])))
        assert len(_bytes(s)) == 17 + 8 * 6 + 4 * 18

    def test_generate_matches_reference_file(self, tmp_path):
        stack, truth = generate(SynthSpec(n_pixels=300, n_obs=60, freq=23.0, noise_std=0.02, break_mag=0.5, seed=5))
        write_stack(stack, tmp_path / "g.bts")
        assert (tmp_path / "g.bts").read_bytes() == (GOLDEN / "io_generate.bts").read_bytes()
        assert truth.sum() == 150

    def test_generate_independent_of_threads(self):
        spec = SynthSpec(n_pixels=9000, n_obs=20, freq=10.0, seed=11)
        a, _ = generate(spec, threads=1)
        b, _ = generate(spec, threads=4)
        assert np.array_equal(a.data, b.data)


class TestRead:
    @pytest.mark.parametrize("use_path", [True, False])
    def test_round_trip_bit_exact_with_nans(self, tmp_path, use_path):
        s = _stack(n_obs=9, m=5)
        s.data[3, 2] = np.nan
        s.data[4, 1] = np.inf
        s.data[0, 0] = -0.0
        if use_path:
            write_stack(s, tmp_path / "s.bts")
            back = read_stack(tmp_path / "s.bts")
        else:
            back = read_stack(io.BytesIO(_bytes(s)))
        assert back.data.tobytes() == s.data.tobytes()
        assert np.array_equal(back.time_axis.values, s.time_axis.values)

    @pytest.mark.parametrize("use_path", [True, False])
    def test_reference_written_axis_file(self, use_path):
        path = GOLDEN / "io_axis.bts"
        st = read_stack(path if use_path else io.BytesIO(path.read_bytes()))
        assert st.data.shape == (12, 7)
        assert np.isnan(st.data[2, 1]) and np.isposinf(st.data[5, 3]) and np.isneginf(st.data[7, 0])
        assert _bytes(st) == path.read_bytes()          # rewritten bytes identical

    def test_large_payload_parallel_read(self, tmp_path):
        s = _stack(n_obs=37, m=20011, seed=4)
        write_stack(s, tmp_path / "big.bts")
        back = read_stack(tmp_path / "big.bts", threads=7)
        assert back.data.tobytes() == s.data.tobytes()

    def test_bad_magic(self):
        with pytest.raises(StackFormatError, match="magic"):
            read_stack(io.BytesIO(b"XXXX" + bytes(40)))

    def test_bad_version(self):
        with pytest.raises(StackFormatError, match="version"):
            read_stack(io.BytesIO(struct.pack("<4sIIIB", b"BTS1", 2, 2, 1, 0) + bytes(8)))

    @pytest.mark.parametrize("n_obs,m", [(1, 1), (2, 0)])
    def test_bad_dimensions(self, n_obs, m):
        with pytest.raises(StackFormatError, match="dimensions"):
            read_stack(io.BytesIO(struct.pack("<4sIIIB", b"BTS1", 1, n_obs, m, 0) + bytes(64)))

    def test_bad_axis_flag(self):
        with pytest.raises(StackFormatError, match="axis flag"):
            read_stack(io.BytesIO(struct.pack("<4sIIIB", b"BTS1", 1, 2, 1, 7) + bytes(64)))

    def test_non_increasing_axis(self):
        raw = struct.pack("<4sIIIB", b"BTS1", 1, 2, 1, 1) + np.array([2.0, 1.0]).tobytes() + bytes(8)
        with pytest.raises(StackFormatError, match="time axis"):
            read_stack(io.BytesIO(raw))

    def test_capacity_limit(self):
        with pytest.raises(StackCapacityError):
            read_stack(io.BytesIO(struct.pack("<4sIIIB", b"BTS1", 1, 2**31, 2**31, 0)))

    def test_truncations_never_crash(self, tmp_path):
        raw = _bytes(_stack(axis=TimeAxis(np.arange(6.0) + 1.5)))
        for cut in range(len(raw)):
            with pytest.raises(StackFormatError):
                read_stack(io.BytesIO(raw[:cut]))
            p = tmp_path / "t.bts"
            p.write_bytes(raw[:cut])
            with pytest.raises(StackFormatError):
                read_stack(p)

    def test_missing_file_raises_oserror(self, tmp_path):
        with pytest.raises(OSError):
            read_stack(tmp_path / "nope.bts")


class TestSeriesCsv:
    def test_blank_value_is_missing_and_header_skipped(self):
        axis, v = read_series_csv(io.StringIO("time,value\n1,0.5\n2,\n\n3,0.25\n"))
        assert np.array_equal(axis.values, [1, 2, 3])
        assert v.dtype == np.float32 and np.isnan(v[1]) and v[2] == 0.25

    def test_parse_error_names_line(self):
        with pytest.raises(CsvParseError, match="line 3"):
            read_series_csv(io.StringIO("1,2\n2,3\n3,x\n"))

    def test_wrong_field_count(self):
        with pytest.raises(CsvParseError, match="expected 2 fields"):
            read_series_csv(io.StringIO("1,2,3\n"))


def _golden_map():
    z = np.load(GOLDEN / "io_breaks.npz")
    return BreakMap(detected=z["detected"], first_break=z["first_break"], max_abs_mo=z["max_abs_mo"],
                    valid=z["valid"], config=MonitorConfig(history=100, bandwidth=50, harmonics=3, freq=23.0),
                    crit_value=4.9)


class TestBreakMapCsv:
    def test_native_writer_matches_reference_bytes(self, tmp_path):
        bm = _golden_map()
        assert write_break_map(bm, tmp_path / "b.csv") == len(bm)
        assert (tmp_path / "b.csv").read_bytes() == (GOLDEN / "io_breaks.csv").read_bytes()

    def test_python_writer_matches_reference_bytes(self):
        buf = io.StringIO()
        write_break_map(_golden_map(), buf)
        assert buf.getvalue().encode() == (GOLDEN / "io_breaks.csv").read_bytes()

    def test_native_writer_random_magnitudes(self, tmp_path):
        rng = np.random.default_rng(8)
        P = 300_000                      # several formatting blocks and threads
        mx = np.abs(rng.standard_cauchy(P)) * 10.0 ** rng.integers(-12, 12, P)
        mx[:5] = [np.inf, 0.0, 1e-320, 9.999999995, 0.1]
        fb = np.where(rng.random(P) < 0.3, rng.integers(1, 10**6, P), 0).astype(np.int64)
        bm = BreakMap(detected=fb > 0, first_break=fb, max_abs_mo=mx, valid=rng.random(P) < 0.8,
                      config=MonitorConfig(history=100, bandwidth=50, harmonics=3, freq=23.0), crit_value=1.0)
        write_break_map(bm, tmp_path / "n.csv", threads=5)
        buf = io.StringIO()
        write_break_map(bm, buf)
        assert (tmp_path / "n.csv").read_bytes() == buf.getvalue().encode()

    @pytest.mark.reference
    def test_against_live_reference(self, tmp_path, reference):
        bm = _golden_map()
        ref = reference.BreakMap(detected=bm.detected, first_break=bm.first_break, max_abs_mo=bm.max_abs_mo,
                                 valid=bm.valid, config=reference.MonitorConfig(history=100, bandwidth=50,
                                                                                harmonics=3, freq=23.0),
                                 crit_value=4.9)
        reference.write_break_map(ref, tmp_path / "r.csv")
        write_break_map(bm, tmp_path / "o.csv")
        assert (tmp_path / "r.csv").read_bytes() == (tmp_path / "o.csv").read_bytes()
