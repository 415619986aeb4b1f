"""EVF1 event-stream ingest, decoded on the GPU.

EVF1 is the reference's container (event_io.py:1-38): a 16-byte header
("EVF1", width u16, height u16, 8 zero bytes) followed by 8-byte little-endian
records -- dt u32 (us since the previous record), xp u16 (bit 15 polarity,
bits 0..14 x), y u16.

Both readers send the raw records to HBM (8 B/event, less than the 13 B/event
SoA packet they become) and decode them with ``fibar_decode_evf1``: a
coalesced kernel that loads two records per 16-byte vector load, writes the
x / y / p columns and the timestamps (a device prefix sum of dt, carried from
block to block like event_io.py:85-95), and reports the first out-of-bounds
record.

* ``read_blocks`` is the drop-in for event_io.py:79-103: same signature, same
  single-pass iterator of host ``EventArray`` blocks, same errors
  (``TruncationError`` with the byte offset of a partial record,
  ``DataError`` naming the first out-of-bounds record).  The decoded columns
  come back to pinned host memory.
* ``read_blocks_device`` yields ``DeviceEventArray`` blocks that stay in HBM
  for ``ReconstructionEngine.process_array`` (no host round trip).
* ``write_stream`` produces the reference writer's bytes (event_io.py:143-182);
  it is a tool for tests and fixtures.

There is no host decoder: without the CUDA library the readers raise
``DeviceError``.
"""

from __future__ import annotations

import ctypes as C
import os
from typing import IO, Iterable, Iterator

import numpy as np

from . import _native
from .core import EventArray, SensorGeometry
from .errors import DataError, DeviceError, FormatError, OrderError, RangeError, TruncationError

MAGIC = b"EVF1"
HEADER_BYTES = 16
RECORD_BYTES = 8
MAX_X = 0x7FFF


def _open(source, mode: str):
    if isinstance(source, (str, os.PathLike)):
        return open(source, mode), True
    return source, False


def read_header(fh: IO[bytes]) -> SensorGeometry:
    """Parse the 16-byte header (event_io.py:47-57)."""
    head = fh.read(HEADER_BYTES)
    if len(head) != HEADER_BYTES:
        raise TruncationError("incomplete header", len(head))
    magic, reserved = head[:4], head[8:]
    if magic != MAGIC:
        raise FormatError(f"bad magic {magic!r}, expected {MAGIC!r}")
    if any(reserved):
        raise FormatError("reserved header bytes must be zero")
    w, h = np.frombuffer(head, "<u2", 2, 4)
    return SensorGeometry(int(w), int(h))


class _DeviceDecoder:
    """Staging for one reader: a pinned host slab the file is read into, the
    device record buffer, and the decode call."""

    def __init__(self, geometry: SensorGeometry, block_events: int, device):
        import torch
        if not torch.cuda.is_available():
            raise DeviceError("EVF1 decoding runs on a CUDA device (no CPU fallback)")
        self.torch = torch
        self.geometry = geometry
        self.dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.cap = max(1, int(block_events))
        self.host = torch.empty(self.cap * RECORD_BYTES, dtype=torch.uint8, pin_memory=True)
        self.recs = torch.empty(self.cap * RECORD_BYTES, dtype=torch.uint8, device=self.dev)
        self.lib = _native.load()

    def read(self, fh) -> int:
        """Read up to one block of records into the pinned slab; returns the byte count."""
        view = memoryview(self.host.numpy())
        got = 0
        while got < len(view):
            k = fh.readinto(view[got:]) if hasattr(fh, "readinto") else None
            if k is None:
                chunk = fh.read(len(view) - got)
                k = len(chunk)
                view[got:got + k] = chunk
            if not k:
                break
            got += k
        return got

    def decode(self, nbytes: int, t_base: int, rec_base: int, byte_base: int):
        """Decode the slab's first nbytes on the device: (x, y, p, t) CUDA tensors."""
        torch = self.torch
        if nbytes % RECORD_BYTES:
            raise TruncationError("stream ends mid-record", byte_base + nbytes - nbytes % RECORD_BYTES)
        n = nbytes // RECORD_BYTES
        recs = self.recs[:nbytes]
        recs.copy_(self.host[:nbytes], non_blocking=True)
        x = torch.empty(n, dtype=torch.int16, device=self.dev)
        y = torch.empty(n, dtype=torch.int16, device=self.dev)
        p = torch.empty(n, dtype=torch.int8, device=self.dev)
        t = torch.empty(n, dtype=torch.int64, device=self.dev)
        _decode(self.lib, recs, n, self.geometry, t_base, rec_base, x, y, p, t)
        return x, y, p, t


def _decode(lib, recs, n, geometry, t_base, rec_base, x, y, p, t):
    import torch
    bad = C.c_int64(-1)
    stream = torch.cuda.current_stream(recs.device).cuda_stream
    _native.check(lib.fibar_decode_evf1(recs.data_ptr(), n, geometry.width, geometry.height, int(t_base),
                                        x.data_ptr(), y.data_ptr(), p.data_ptr(),
                                        t.data_ptr() if t is not None else None, C.byref(bad), C.c_void_p(stream)),
                  "fibar_decode_evf1")
    if bad.value >= 0:   # the call synchronised to report it
        i = int(bad.value)
        px, py = int(x[i]) & 0xFFFF, int(y[i]) & 0xFFFF
        raise DataError(f"record {rec_base + i}: pixel ({px},{py}) outside {geometry.width}x{geometry.height}")


def _iter_decoded(fh, owned, geometry, block_events, device):
    """Yield (x, y, p, t) CUDA tensors per block; t carried across blocks."""
    dec = _DeviceDecoder(geometry, block_events, device)
    t_base, rec_base, byte_base = 0, 0, HEADER_BYTES
    try:
        while True:
            nbytes = dec.read(fh)
            if not nbytes:
                break
            x, y, p, t = dec.decode(nbytes, t_base, rec_base, byte_base)
            n = x.numel()
            if n:
                t_base = int(t[n - 1])
            rec_base += n
            byte_base += nbytes
            yield x, y, p, t
    finally:
        if owned:
            fh.close()


def read_blocks(source, block_events: int = 1 << 16, device=None) -> tuple[SensorGeometry, Iterator[EventArray]]:
    """Open an EVF1 stream: geometry plus a single-pass iterator of host
    ``EventArray`` blocks (event_io.py:79-103), decoded on the GPU."""
    fh, owned = _open(source, "rb")
    geometry = read_header(fh)

    def blocks() -> Iterator[EventArray]:
        for x, y, p, t in _iter_decoded(fh, owned, geometry, block_events, device):
            yield EventArray(t.cpu().numpy().view(np.uint64), x.cpu().numpy().view(np.uint16),
                             y.cpu().numpy().view(np.uint16), p.cpu().numpy())

    return geometry, blocks()


def read_blocks_device(source, block_events: int = 1 << 20, device=None):
    """EVF1 stream decoded on the GPU: geometry plus an iterator of
    ``DeviceEventArray`` blocks that stay in HBM."""
    from .pipeline import DeviceEventArray

    fh, owned = _open(source, "rb")
    geometry = read_header(fh)

    def blocks():
        for x, y, p, t in _iter_decoded(fh, owned, geometry, block_events, device):
            yield DeviceEventArray(x, y, p, t)

    return geometry, blocks()


def read_stream(source) -> tuple[SensorGeometry, EventArray]:
    """A whole EVF1 stream as one host ``EventArray`` (event_io.py:106-109)."""
    geometry, blocks = read_blocks(source, block_events=1 << 20)
    return geometry, EventArray.concatenate(blocks)


def decode_device(raw_dev, geometry: SensorGeometry, t_base: int = 0, rec_base: int = 0, with_t: bool = True):
    """Decode EVF1 records already on the GPU (uint8 CUDA tensor) into a
    ``DeviceEventArray`` (t as int64 on the device unless with_t=False)."""
    import torch

    from .pipeline import DeviceEventArray

    nbytes = raw_dev.numel()
    if nbytes % RECORD_BYTES:
        raise TruncationError("stream ends mid-record", nbytes - nbytes % RECORD_BYTES)
    n = nbytes // RECORD_BYTES
    dev = raw_dev.device
    x = torch.empty(n, dtype=torch.int16, device=dev)
    y = torch.empty(n, dtype=torch.int16, device=dev)
    p = torch.empty(n, dtype=torch.int8, device=dev)
    t = torch.empty(n, dtype=torch.int64, device=dev) if with_t else None
    _decode(_native.load(), raw_dev, n, geometry, t_base, rec_base, x, y, p, t)
    return DeviceEventArray(x, y, p, t)


def _as_blocks(events) -> Iterable[EventArray]:
    if isinstance(events, EventArray):
        return [events]
    return events


def write_stream(geometry: SensorGeometry, events, sink) -> int:
    """Write an ``EventArray`` (or an iterable of them) as EVF1; returns the
    record count.  Byte-identical to the reference writer (event_io.py:143-182):
    events must be time-ordered with gaps below 2^32 us."""
    if geometry.width > MAX_X + 1:
        raise RangeError(f"width {geometry.width} exceeds the 15-bit x field")
    header = MAGIC + np.array([geometry.width, geometry.height], "<u2").tobytes() + bytes(8)
    fh, owned = _open(sink, "wb")
    try:
        fh.write(header)
        written, t_prev = 0, 0
        for blk in _as_blocks(events):
            if not len(blk):
                continue
            t = np.asarray(blk.t, np.uint64)
            if int(t[0]) < t_prev or bool(np.any(t[1:] < t[:-1])):
                raise OrderError("event timestamps regress")
            dt = np.diff(t, prepend=np.uint64(t_prev))
            if int(dt.max()) > 0xFFFFFFFF:
                raise RangeError("inter-event gap exceeds the 32-bit dt field")
            x = np.asarray(blk.x, np.uint64)
            y = np.asarray(blk.y, np.uint64)
            if bool(np.any(x >= geometry.width)) or bool(np.any(y >= geometry.height)):
                raise DataError("event outside declared geometry")
            # one little-endian u64 per record: dt | xp << 32 | y << 48
            pol = (np.asarray(blk.p) > 0).astype(np.uint64) << np.uint64(15)
            word = dt | ((x | pol) << np.uint64(32)) | (y << np.uint64(48))
            fh.write(word.astype("<u8").tobytes())
            written += len(t)
            t_prev = int(t[-1])
        return written
    finally:
        if owned:
            fh.close()
