"""BTS1 stack files and the break-map CSV, feeding the GPU path.

Same file formats, function names, return values and exceptions as the reference's
pkg/src/breakwatch/dataio.py:

    magic b"BTS1" | u32 version = 1 | u32 n_obs | u32 n_pixels | u8 axis flag
    | axis flag 1: n_obs float64 time stamps
    | n_obs * n_pixels float32 samples, time-major, little-endian

The payload is already the layout the kernel reads, so nothing is transposed or converted:
  read_stack     parses the 17-byte header (and axis) here with the reference's checks and
                 messages (dataio.py:79-115), then reads the payload with libbwm's parallel
                 pread (bwm_read_payload);
  monitor_file   skips the host copy altogether: libbwm streams row blocks of the payload
                 from the page cache into pinned slots while earlier blocks are already being
                 DMA'd to HBM (bwm_monitor_file), then runs the kernel — the paper's
                 "transfer + compute" picture with the file read overlapped;
  write_break_map formats rows on all host threads in C (bwm_write_break_map), byte-identical
                 to the reference's Python loop (dataio.py:168-182).
File objects (instead of paths) take pure-Python paths with the same results.
"""

from __future__ import annotations

import os
import struct
from contextlib import contextmanager
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .engine import BreakMap, MonitorConfig, PhaseTimings, SeriesStack, _is_cuda_tensor, _run, DEFAULT_BLOCK_SIZE
from .errors import CsvParseError, StackCapacityError, StackFormatError
from .model import TimeAxis, regular_axis

MAGIC = b"BTS1"
VERSION = 1
_HEADER = struct.Struct("<4sIIIB")
PAYLOAD_LIMIT_BYTES = 1 << 40          # refuse absurd headers before allocating (dataio.py:27)


@contextmanager
def _open(target, mode):
    if hasattr(target, "read") or hasattr(target, "write"):
        yield target
    else:
        with open(target, mode) as handle:
            yield handle


def _is_path(x) -> bool:
    return isinstance(x, (str, bytes, os.PathLike))


def _read_exact(source, count: int, what: str) -> bytes:
    data = source.read(count)
    if len(data) != count:
        raise StackFormatError(f"truncated {what}: wanted {count} bytes, got {len(data)}")
    return data


@dataclass(frozen=True)
class StackHeader:
    """A parsed BTS1 header: geometry, time axis and where the payload starts."""

    n_obs: int
    n_pixels: int
    time_axis: TimeAxis
    payload_offset: int

    @property
    def payload_bytes(self) -> int:
        return 4 * self.n_obs * self.n_pixels


def read_header(handle) -> StackHeader:
    """Header + axis checks of dataio.py:87-112, in the same order with the same messages."""
    magic, version, n_obs, n_pixels, axis_flag = _HEADER.unpack(_read_exact(handle, _HEADER.size, "header"))
    if magic != MAGIC:
        raise StackFormatError(f"bad magic {magic!r}; expected {MAGIC!r}")
    if version != VERSION:
        raise StackFormatError(f"unsupported version {version}")
    if n_obs < 2 or n_pixels < 1:
        raise StackFormatError(f"invalid dimensions n_obs={n_obs}, n_pixels={n_pixels}")
    if axis_flag not in (0, 1):
        raise StackFormatError(f"unknown axis flag {axis_flag}")
    payload = 4 * n_obs * n_pixels
    if payload > PAYLOAD_LIMIT_BYTES:
        raise StackCapacityError(f"declared payload of {payload} bytes exceeds the {PAYLOAD_LIMIT_BYTES}-byte limit")
    offset = _HEADER.size
    if axis_flag:
        raw = _read_exact(handle, 8 * n_obs, "time axis")
        try:
            axis = TimeAxis(np.frombuffer(raw, dtype="<f8").copy())
        except ValueError as exc:
            raise StackFormatError(f"invalid time axis: {exc}") from exc
        offset += 8 * n_obs
    else:
        axis = regular_axis(n_obs)
    return StackHeader(int(n_obs), int(n_pixels), axis, offset)


def write_stack(stack: SeriesStack, sink) -> int:
    """Serialise a stack to a path or binary file object; returns bytes written.

    An axis equal to 1..n_obs is stored implicitly (flag 0), as dataio.py:44-71 does.
    """
    axis = stack.time_axis.values
    implicit = np.array_equal(axis, np.arange(1, stack.n_obs + 1, dtype=np.float64))
    data = stack.data.cpu().numpy() if _is_cuda_tensor(stack.data) else stack.data
    header = _HEADER.pack(MAGIC, VERSION, stack.n_obs, stack.n_pixels, 0 if implicit else 1)
    written = 0
    with _open(sink, "wb") as out:
        out.write(header)
        written += len(header)
        if not implicit:
            ab = axis.astype("<f8", copy=False).tobytes()
            out.write(ab)
            written += len(ab)
        payload = np.ascontiguousarray(data, dtype="<f4")
        out.write(memoryview(payload).cast("B"))
        written += payload.nbytes
    return written


def _payload_buffer(n_obs: int, n_pixels: int) -> np.ndarray:
    # plain memory: monitor_batch stages pageable stacks through libbwm's pinned slots at the
    # link rate, and a multi-GB page-locked allocation would cost seconds per file
    return np.empty((n_obs, n_pixels), np.float32)


def read_stack(source, *, threads: Optional[int] = None) -> SeriesStack:
    """Parse a stack from a path or binary file object (dataio.py:79-115).

    Malformed input raises StackFormatError (StackCapacityError for a plausible header that
    declares more than PAYLOAD_LIMIT_BYTES); no partial stack is returned.
    """
    if _is_path(source):
        with open(source, "rb") as handle:
            hdr = read_header(handle)
        data = _payload_buffer(hdr.n_obs, hdr.n_pixels)
        from . import _lib

        lib = _lib.load()
        _lib.check(lib.bwm_read_payload(os.fsencode(source), hdr.payload_offset, hdr.n_obs, hdr.n_pixels,
                                        data.ctypes.data, int(threads or 0)), "bwm_read_payload")
        return SeriesStack(data, hdr.time_axis)
    hdr = read_header(source)
    data = _payload_buffer(hdr.n_obs, hdr.n_pixels)
    view = memoryview(data).cast("B")
    got = 0
    while got < hdr.payload_bytes:
        n = source.readinto(view[got:]) if hasattr(source, "readinto") else None
        if n is None:
            chunk = source.read(hdr.payload_bytes - got)
            n = len(chunk)
            view[got:got + n] = chunk
        if not n:
            break
        got += n
    if got != hdr.payload_bytes:
        raise StackFormatError(f"truncated sample payload: wanted {hdr.payload_bytes} bytes, got {got}")
    if np.little_endian is False:  # pragma: no cover - big-endian hosts
        data.byteswap(inplace=True)
    return SeriesStack(data, hdr.time_axis)


@dataclass(frozen=True)
class _FileStack:
    """Geometry of a stack whose samples stay in the file (monitor_file)."""

    n_obs: int
    n_pixels: int
    time_axis: TimeAxis
    data: object = None


def _file_run(path, config, threads, keep_mosum, return_beta, return_mean, device, pixels=None):
    with open(path, "rb") as handle:
        hdr = read_header(handle)
    start, stop = (0, hdr.n_pixels) if pixels is None else (int(pixels[0]), int(pixels[1]))
    if not 0 <= start < stop <= hdr.n_pixels:
        raise ValueError(f"pixel range {pixels} outside the file's {hdr.n_pixels} pixels")
    stack = _FileStack(hdr.n_obs, stop - start, hdr.time_axis)
    return _run(stack, config, threads, DEFAULT_BLOCK_SIZE, keep_mosum, return_beta, return_mean, device,
                source=(path, hdr.payload_offset, start, hdr.n_pixels))


def monitor_file(path, config: MonitorConfig, threads: Optional[int] = None, keep_mosum: bool = False, *,
                 return_beta: bool = False, return_mean: bool = False, device=None, pixels=None) -> BreakMap:
    """monitor_batch(read_stack(path), config) without the intermediate host copy: the
    payload streams file -> pinned slots -> HBM with the reads overlapped (bwm_monitor_file).

    pixels=(start, stop) monitors one pixel band of the file — one rank's shard on a multi-GPU
    box (sharding.shard_bounds); the BreakMap then covers those pixels only."""
    return _file_run(path, config, threads, keep_mosum, return_beta, return_mean, device, pixels)[0]


def profile_file(path, config: MonitorConfig, threads: Optional[int] = None, *,
                 device=None) -> tuple[BreakMap, PhaseTimings]:
    """monitor_file plus phase timings (`ingest` = file read + H2D, `mosum` = kernel)."""
    return _file_run(path, config, threads, False, False, False, device)


def _is_number(text: str) -> bool:
    try:
        float(text)
    except ValueError:
        return False
    return True


def read_series_csv(source) -> tuple[TimeAxis, np.ndarray]:
    """Two-column time,value text -> (axis, float32 series) (dataio.py:124-165).

    An empty value field is missing (NaN); a leading non-numeric header row is skipped;
    blank lines are ignored; bad cells raise CsvParseError with the 1-based line number.
    """
    stamps: list[float] = []
    values: list[float] = []
    with _open(source, "r") as handle:
        for number, raw in enumerate(handle, start=1):
            line = raw.strip()
            if not line:
                continue
            fields = [f.strip() for f in line.split(",")]
            if len(fields) != 2:
                raise CsvParseError(f"expected 2 fields, found {len(fields)}", number)
            t_text, v_text = fields
            if number == 1 and not _is_number(t_text):
                continue
            try:
                t = float(t_text)
            except ValueError:
                raise CsvParseError(f"bad time value {t_text!r}", number) from None
            if v_text == "":
                v = float("nan")
            else:
                try:
                    v = float(v_text)
                except ValueError:
                    raise CsvParseError(f"bad sample value {v_text!r}", number) from None
            stamps.append(t)
            values.append(v)
    return TimeAxis(np.asarray(stamps, dtype=np.float64)), np.asarray(values, dtype=np.float32)


def _csv_rows(break_map: BreakMap):
    for px in range(len(break_map)):
        first = int(break_map.first_break[px])
        yield (f"{px},{int(break_map.valid[px])},{int(break_map.detected[px])},"
               f"{first if first else ''},{break_map.max_abs_mo[px]:.9g}\n")


def write_break_map(break_map: BreakMap, sink, *, threads: Optional[int] = None) -> int:
    """One CSV row per pixel, in pixel order; returns the row count (dataio.py:168-182)."""
    if _is_path(sink):
        from . import _lib

        lib = _lib.load()
        c = lambda a, dt: np.ascontiguousarray(a, dtype=dt)  # noqa: E731
        valid, det = c(break_map.valid, np.uint8), c(break_map.detected, np.uint8)
        first, mx = c(break_map.first_break, np.int64), c(break_map.max_abs_mo, np.float64)
        rows = lib.bwm_write_break_map(os.fsencode(sink), len(break_map), valid.ctypes.data, det.ctypes.data,
                                       first.ctypes.data, mx.ctypes.data, int(threads or 0))
        if rows < 0:
            _lib.check(int(rows), "bwm_write_break_map")
        return int(rows)
    rows = 0
    sink.write("pixel,valid,detected,first_break,max_abs_mo\n")
    for line in _csv_rows(break_map):
        sink.write(line)
        rows += 1
    return rows
