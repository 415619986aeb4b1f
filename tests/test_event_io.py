"""EVF1 ingest: the device decoder behind read_blocks / read_blocks_device, and
the writer, pinned to the reference's own decode of a reference-written stream
(tests/golden/misc.npz)."""

import io

import numpy as np
import pytest

from conftest import golden_path
from paper_2510_20071_b200 import event_io, workloads
from paper_2510_20071_b200.core import SensorGeometry
from paper_2510_20071_b200.errors import DataError, DeviceError, FormatError, OrderError, TruncationError


def golden():
    m = dict(np.load(golden_path("misc")))
    return m["evf1"].tobytes(), m


@pytest.mark.gpu
def test_read_blocks_matches_reference():
    raw, m = golden()
    geom, blocks = event_io.read_blocks(io.BytesIO(raw), block_events=777)
    assert (geom.width, geom.height) == (100, 60)
    got = list(blocks)
    for k in ("t", "x", "y", "p"):
        assert np.array_equal(np.concatenate([getattr(b, k) for b in got]), m[f"evf1_{k}"])


def test_writer_bytes_and_header_errors():
    ev = workloads.uniform(100, 60, 5000, 3)
    buf = io.BytesIO()
    event_io.write_stream(SensorGeometry(100, 60), ev, buf)
    raw, _ = golden()
    assert buf.getvalue() == raw          # byte-identical to the reference's writer
    buf = io.BytesIO()                    # the same stream as several blocks
    event_io.write_stream(SensorGeometry(100, 60), [ev.slice(0, 1234), ev.slice(1234, 1234), ev.slice(1234, 5000)], buf)
    assert buf.getvalue() == raw
    with pytest.raises(FormatError):
        event_io.read_header(io.BytesIO(b"EVF2" + raw[4:16]))
    with pytest.raises(FormatError):
        event_io.read_header(io.BytesIO(raw[:15] + b"\x01"))
    with pytest.raises(TruncationError):
        event_io.read_header(io.BytesIO(raw[:9]))
    assert event_io.read_header(io.BytesIO(raw)) == SensorGeometry(100, 60)
    with pytest.raises(OrderError):
        event_io.write_stream(SensorGeometry(100, 60), [ev.slice(10, 20), ev.slice(0, 10)], io.BytesIO())


def test_readers_need_the_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    raw, _ = golden()
    with pytest.raises(DeviceError):
        list(event_io.read_blocks(io.BytesIO(raw))[1])


@pytest.mark.gpu
def test_read_blocks_errors():
    raw, _ = golden()
    with pytest.raises(TruncationError):
        list(event_io.read_blocks(io.BytesIO(raw[:-3]))[1])
    with pytest.raises(DataError):
        list(event_io.read_blocks(io.BytesIO(raw[:4] + (50).to_bytes(2, "little") + raw[6:]))[1])


@pytest.mark.gpu
def test_device_decode_matches_reference():
    import torch
    raw, m = golden()
    recs = torch.frombuffer(bytearray(raw[16:]), dtype=torch.uint8).cuda()
    blk = event_io.decode_device(recs, SensorGeometry(100, 60))
    assert np.array_equal(blk.x.cpu().numpy().view(np.uint16), m["evf1_x"])
    assert np.array_equal(blk.y.cpu().numpy().view(np.uint16), m["evf1_y"])
    assert np.array_equal(blk.p.cpu().numpy(), m["evf1_p"])
    assert np.array_equal(blk.t.cpu().numpy().view(np.uint64), m["evf1_t"])
    # odd record count and a carried t_base
    blk = event_io.decode_device(recs[: 8 * 4999], SensorGeometry(100, 60), t_base=1000)
    assert np.array_equal(blk.t.cpu().numpy().view(np.uint64), m["evf1_t"][:4999] + 1000)
    with pytest.raises(DataError, match="record"):
        event_io.decode_device(recs, SensorGeometry(100, 30))


@pytest.mark.gpu
def test_device_blocks_through_engine_match_host_blocks(tmp_path):
    from fractions import Fraction
    from paper_2510_20071_b200.core import compute_params
    from paper_2510_20071_b200.pipeline import ReconstructionEngine
    geom = SensorGeometry(160, 120)
    ev = workloads.moving_texture(160, 120, 200_000, seed=2)
    path = tmp_path / "s.evf1"
    event_io.write_stream(geom, ev, path)
    params = compute_params(40.0, Fraction(1, 2), geom)
    a = ReconstructionEngine(geom, params)
    for blk in event_io.read_blocks(path, block_events=30_000)[1]:
        a.process_array(blk)
    b = ReconstructionEngine(geom, params)
    for blk in event_io.read_blocks_device(path, block_events=30_000)[1]:
        b.process_array(blk)
    assert a.state_digest() == b.state_digest()
    assert a.last_t == b.last_t == int(ev.t[-1])
