"""EVF1 event stream ingest: host mirror and the device decode.

EVF1 (the reference's container, `fibar/event_io.py:1-20`): a 16-byte header
("EVF1", width u16, height u16, 8 zero bytes) then 8-byte little-endian
records (dt u32 since the previous record, xp u16 with bit 15 = polarity and
bits 0..14 = x, y u16).

* ``read_header`` / ``read_blocks`` / ``read_stream`` mirror event_io.py:340-402
  (same names, block iterator, errors) and decode on the host with numpy.
* ``read_blocks_device`` is the B200 path: the raw records (8 B/event, less
  than the 13 B/event SoA packet) go to HBM and ``fibar_decode_evf1`` (a
  vectorised, coalesced kernel: two records per 16-byte load) writes the
  columns and the timestamps (device prefix sum of dt, carried across blocks
  like event_io.py:378-388).  Out-of-bounds records raise DataError with the
  record index, as the reference's decoder does.
* ``write_stream`` (event_io.py:436-475) is kept for tests and tools.
"""

from __future__ import annotations

import ctypes as C
import os
from typing import IO, Iterator

import numpy as np

from . import _native
from .core import EventArray, SensorGeometry
from .errors import DataError, FormatError, OrderError, RangeError, TruncationError

MAGIC = b"EVF1"
HEADER_BYTES = 16
RECORD_BYTES = 8
MAX_X = 0x7FFF
_REC = np.dtype([("dt", "<u4"), ("xp", "<u2"), ("y", "<u2")])


def _open(source, mode: str):
    if isinstance(source, (str, os.PathLike)):
        return open(source, mode), True
    return source, False


def read_header(fh: IO[bytes]) -> SensorGeometry:
    raw = fh.read(HEADER_BYTES)
    if len(raw) < HEADER_BYTES:
        raise TruncationError("incomplete header", len(raw))
    if raw[:4] != MAGIC:
        raise FormatError(f"bad magic {raw[:4]!r}, expected {MAGIC!r}")
    if raw[8:16] != bytes(8):
        raise FormatError("reserved header bytes must be zero")
    return SensorGeometry(int.from_bytes(raw[4:6], "little"), int.from_bytes(raw[6:8], "little"))


def _decode_host(raw: bytes, geometry: SensorGeometry, t_base: int, rec_base: int, byte_base: int) -> EventArray:
    if len(raw) % RECORD_BYTES:
        raise TruncationError("stream ends mid-record", byte_base + len(raw) - len(raw) % RECORD_BYTES)
    rec = np.frombuffer(raw, dtype=_REC)
    x = (rec["xp"] & MAX_X).astype(np.uint16)
    y = rec["y"]
    bad = np.flatnonzero((x >= geometry.width) | (y >= geometry.height))
    if bad.size:
        i = int(bad[0])
        raise DataError(f"record {rec_base + i}: pixel ({int(x[i])},{int(y[i])}) outside "
                        f"{geometry.width}x{geometry.height}")
    t = np.cumsum(rec["dt"], dtype=np.uint64)
    t += np.uint64(t_base)
    p = np.where(rec["xp"] >> 15, 1, -1).astype(np.int8)
    return EventArray(t, x, np.ascontiguousarray(y), p)


def read_blocks(source, block_events: int = 1 << 16) -> tuple[SensorGeometry, Iterator[EventArray]]:
    """Open an EVF1 stream: geometry plus a single-pass iterator of host blocks."""
    fh, owned = _open(source, "rb")
    geometry = read_header(fh)

    def gen() -> Iterator[EventArray]:
        t_base, rec_base, byte_base = 0, 0, HEADER_BYTES
        try:
            while True:
                raw = fh.read(block_events * RECORD_BYTES)
                if not raw:
                    break
                blk = _decode_host(raw, geometry, t_base, rec_base, byte_base)
                if len(blk):
                    t_base = int(blk.t[-1])
                rec_base += len(blk)
                byte_base += len(raw)
                yield blk
        finally:
            if owned:
                fh.close()

    return geometry, gen()


def read_stream(source) -> tuple[SensorGeometry, EventArray]:
    geometry, blocks = read_blocks(source)
    return geometry, EventArray.concatenate(blocks)


def decode_device(raw_dev, geometry: SensorGeometry, t_base: int = 0, rec_base: int = 0, with_t: bool = True):
    """Decode EVF1 records already on the GPU (uint8 CUDA tensor, 16-byte aligned)
    into a DeviceEventArray (t stays on the device as int64 unless with_t=False)."""
    import torch

    from .pipeline import DeviceEventArray

    n = raw_dev.numel() // RECORD_BYTES
    if raw_dev.numel() % RECORD_BYTES:
        raise TruncationError("stream ends mid-record", raw_dev.numel() - raw_dev.numel() % RECORD_BYTES)
    dev = raw_dev.device
    x = torch.empty(n, dtype=torch.int16, device=dev)
    y = torch.empty(n, dtype=torch.int16, device=dev)
    p = torch.empty(n, dtype=torch.int8, device=dev)
    t = torch.empty(n, dtype=torch.int64, device=dev) if with_t else None
    bad = C.c_int64(-1)
    lib = _native.load()
    stream = torch.cuda.current_stream(dev).cuda_stream
    _native.check(lib.fibar_decode_evf1(raw_dev.data_ptr(), n, geometry.width, geometry.height, int(t_base),
                                        x.data_ptr(), y.data_ptr(), p.data_ptr(),
                                        t.data_ptr() if t is not None else None, C.byref(bad), C.c_void_p(stream)),
                  "fibar_decode_evf1")
    if bad.value >= 0:
        i = int(bad.value)
        xi, yi = int(x[i]) & 0xFFFF, int(y[i]) & 0xFFFF
        raise DataError(f"record {rec_base + i}: pixel ({xi},{yi}) outside {geometry.width}x{geometry.height}")
    return DeviceEventArray(x, y, p, t)


def read_blocks_device(source, block_events: int = 1 << 20, device=None):
    """EVF1 stream decoded on the GPU: geometry plus an iterator of DeviceEventArray."""
    import torch

    fh, owned = _open(source, "rb")
    geometry = read_header(fh)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())

    def gen():
        t_base, rec_base, byte_base = 0, 0, HEADER_BYTES
        try:
            while True:
                raw = fh.read(block_events * RECORD_BYTES)
                if not raw:
                    break
                if len(raw) % RECORD_BYTES:
                    raise TruncationError("stream ends mid-record", byte_base + len(raw) - len(raw) % RECORD_BYTES)
                host = torch.frombuffer(bytearray(raw), dtype=torch.uint8)
                blk = decode_device(host.to(dev, non_blocking=False), geometry, t_base, rec_base)
                if len(blk):
                    t_base = int(blk.t[-1])
                rec_base += len(blk)
                byte_base += len(raw)
                yield blk
        finally:
            if owned:
                fh.close()

    return geometry, gen()


def write_stream(geometry: SensorGeometry, events: EventArray, sink) -> int:
    """Write an EventArray as EVF1 (time-ordered, gaps < 2^32 us)."""
    if geometry.width > MAX_X + 1:
        raise RangeError(f"width {geometry.width} exceeds the 15-bit x field")
    t = events.t
    if len(t) and np.any(t[1:] < t[:-1]):
        raise OrderError("event timestamps regress")
    dt = np.diff(t, prepend=np.uint64(0))
    if np.any(dt > 0xFFFFFFFF):
        raise RangeError("inter-event gap exceeds the 32-bit dt field")
    if np.any(events.x >= geometry.width) or np.any(events.y >= geometry.height):
        raise DataError("event outside declared geometry")
    rec = np.empty(len(t), dtype=_REC)
    rec["dt"] = dt
    rec["xp"] = events.x | np.where(events.p > 0, 0x8000, 0).astype(np.uint16)
    rec["y"] = events.y
    fh, owned = _open(sink, "wb")
    try:
        fh.write(MAGIC + int(geometry.width).to_bytes(2, "little") + int(geometry.height).to_bytes(2, "little")
                 + bytes(8))
        fh.write(rec.tobytes())
    finally:
        if owned:
            fh.close()
    return len(t)
