"""Row-band partition of one sensor across GPUs.

SURVEY §8(e): with the spatial filter off, pixels are independent
(_kernels.py:62-73), so the sensor splits into row bands with no exchange on
the data path.  Each rank runs one native engine that owns rows
[y0, y0 + rows) and receives the *whole* packet stream (shared input, e.g.
each GPU's own copy of the camera packets); the device ingest keeps only its
band's events, in stream order, so every pixel sees exactly its reference
event sequence.  Read-out is the only collective: the bands' brightness rows
are all-gathered (NCCL over NVLink on GPUs, gloo in the CPU tests) into the
full grid, which every rank can render.  Counters are summed with all_reduce.

With the filter ON (``HaloBandEngine``) the window is one global FIFO over
the interleaved stream (_kernels.py:132-205), so every rank runs the window
pass on the whole stream, while the blur -- the reference's 3x3 Gaussian of
stale pixels (_kernels.py:173-189) -- is split by rows: each rank blurs the
items of its band plus G halo rows and takes the outermost halo row's blurred
values from the neighbour that owns it.  Those values are exchanged in rounds
(NCCL send/recv of the halo rows' values, 8 B per item) until no rank read a
value that was not final; each value carries a taint bit saying whether it
depended on one.  The fixpoint is the serial result bit for bit.
"""

from __future__ import annotations

import numpy as np

import dataclasses

from .core import FilterParams, SensorGeometry
from .errors import ConfigError


def band_rows(height: int, world: int) -> list[tuple[int, int]]:
    """(y0, rows) of each rank's band: equal heights except the last, all >= 2 rows."""
    if world < 1:
        raise ConfigError("need at least one band")
    per = -(-height // world)
    out = []
    for r in range(world):
        y0 = min(height, r * per)
        y1 = min(height, (r + 1) * per)
        out.append((y0, y1 - y0))
    if any(rows < 2 for _, rows in out):
        raise ConfigError(f"{height} rows cannot be split into {world} bands of >= 2 rows")
    return out


def band_params(params: FilterParams, width: int, rows: int) -> FilterParams:
    """The sensor's parameters for a band engine (window bounds clamped to the band;
    they are unused with the filter off)."""
    n = width * rows
    return dataclasses.replace(params, q_max=min(params.q_max, n), q_min=min(params.q_min, n))


def band_of_rows(ys: np.ndarray, height: int, world: int) -> np.ndarray:
    """Owning rank of each event row (host-side routing, used by tests and tools)."""
    per = -(-height // world)
    return np.minimum(ys.astype(np.int64) // per, world - 1)


def _all_gather_rows(mine, bands_, per, group, world, height):
    """The full (H, W) grid from every rank's (rows, W) band (all_gather of padded bands)."""
    import torch
    import torch.distributed as dist
    pad = torch.zeros((per, mine.shape[1]), dtype=torch.float32, device=mine.device)
    pad[: mine.shape[0]] = mine
    if world == 1:
        return pad[:height]
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([parts[r][: bands_[r][1]] for r in range(world)], 0)


class BandedReconstructionEngine:
    """One rank's share of a row-band partitioned engine (filter OFF)."""

    def __init__(self, geometry: SensorGeometry, params: FilterParams, *, rank: int, world: int, group=None,
                 engine_factory=None, **engine_kw):
        if params.spatial_enabled and world > 1:
            raise ConfigError("row bands need the spatial filter off (the window is one global FIFO)")
        self.geometry = geometry
        self.rank, self.world, self.group = rank, world, group
        self.bands = band_rows(geometry.height, world)
        self.y0, self.rows = self.bands[rank]
        self.per = -(-geometry.height // world)
        if engine_factory is None:
            from .pipeline import ReconstructionEngine

            def engine_factory(geom, prm, **kw):
                return ReconstructionEngine(geom, prm, row_band=(self.y0, geometry.height), **kw)
        self.engine = engine_factory(SensorGeometry(geometry.width, self.rows),
                                     band_params(params, geometry.width, self.rows), **engine_kw)

    def process_array(self, block) -> None:
        """Feed the full packet; the native ingest keeps this band's events."""
        self.engine.process_array(block)

    def local_l(self):
        """This band's brightness rows as a (rows, W) tensor (CUDA for native engines)."""
        import torch
        if hasattr(self.engine, "brightness_device"):
            return self.engine.brightness_device()
        self.engine.flush()
        return torch.from_numpy(self.engine.l.reshape(self.rows, self.geometry.width)).to(self._device())

    def _device(self):
        import torch
        return getattr(self.engine, "device", torch.device("cpu"))

    def gather_l(self):
        """The full (H, W) brightness grid on every rank (all_gather of padded bands)."""
        return _all_gather_rows(self.local_l(), self.bands, self.per, self.group, self.world, self.geometry.height)

    def render(self, scale_mode: str = "robust", fixed_bound: float = 1.0, readout_time: int = 0):
        from .pipeline import render_grid
        return render_grid(self.gather_l(), scale_mode, fixed_bound, readout_time)

    def counters(self) -> tuple[int, int]:
        """(event_count, oob_dropped) over all bands; OOB events are counted by every band, so rank 0's."""
        import torch
        import torch.distributed as dist
        ec, ob = self.engine._counters()
        if self.world == 1:
            return ec, ob
        t = torch.tensor([ec], dtype=torch.int64, device=self._device())
        dist.all_reduce(t, group=self.group)
        return int(t.item()), ob


def _slice(block, a, b):
    if hasattr(block, "slice"):
        return block.slice(a, b)
    from .pipeline import DeviceEventArray
    return DeviceEventArray(block.x[a:b], block.y[a:b], block.p[a:b], None if block.t is None else block.t[a:b])


def _concat(blocks):
    from .core import EventArray
    if all(hasattr(b, "slice") for b in blocks):
        return EventArray.concatenate(blocks)
    import torch
    from .pipeline import DeviceEventArray
    dev = next(b.x.device for b in blocks if not hasattr(b, "slice"))

    def col(b, name):   # a host packet's column as a device tensor (x, y as int16 bits)
        v = getattr(b, name)
        if hasattr(b, "slice"):
            v = torch.from_numpy(v.view(np.int16) if v.dtype == np.uint16 else v).to(dev)
        return v.to(torch.int8) if name == "p" else v.to(torch.int16) if v.dtype != torch.int16 else v

    ts = [b.t for b in blocks]
    t = None if any(v is None for v in ts) else np.concatenate(ts)
    return DeviceEventArray(torch.cat([col(b, "x") for b in blocks]), torch.cat([col(b, "y") for b in blocks]),
                            torch.cat([col(b, "p") for b in blocks]), t)


# A value word of the halo exchange: bit 63 = tainted, bits 0-31 = float32 bits.
TAINTED = -(1 << 63)


def halo_rows_for(height: int, world: int, halo: int) -> int:
    """Halo depth G actually used: at most the smallest band's rows."""
    return max(1, min(int(halo), min(r for _, r in band_rows(height, world))))


class HaloBandEngine:
    """One rank's share of a filter-ON row-band partition.

    Every rank is fed the whole packet stream.  Packets are cut into device
    batches of ``batch_events``; each batch runs the window pass, then blur
    rounds with the halo exchange until every rank's inputs were final.  With
    ``world == 1`` there is no halo and a batch takes one round.
    """

    def __init__(self, geometry: SensorGeometry, params: FilterParams, *, rank: int, world: int, group=None,
                 halo: int = 16, batch_events: int = 1 << 20, engine_factory=None, **engine_kw):
        if not params.spatial_enabled:
            raise ConfigError("halo bands are for the spatial filter (filter OFF: BandedReconstructionEngine)")
        self.geometry = geometry
        self.rank, self.world, self.group = rank, world, group
        self.bands = band_rows(geometry.height, world)
        self.y0, self.rows = self.bands[rank]
        self.y1 = self.y0 + self.rows
        self.per = -(-geometry.height // world)
        self.halo = halo_rows_for(geometry.height, world, halo)
        self.batch_events = int(batch_events)
        if engine_factory is None:
            from .pipeline import ReconstructionEngine

            def engine_factory(geom, prm, **kw):
                return ReconstructionEngine(geom, prm, **kw)
        self.engine = engine_factory(geometry, params, halo_band=(self.y0, self.y1, self.halo),
                                     batch_capacity=self.batch_events, **engine_kw)
        self._pending = []
        self._pending_n = 0
        self.rounds: list[int] = []   # exchange rounds per batch (diagnostics)

    def _device(self):
        import torch
        return getattr(self.engine, "device", torch.device("cpu"))

    # -- ingest ----------------------------------------------------------------
    def process_array(self, block) -> None:
        """Queue a packet (EventArray or DeviceEventArray); full batches run at
        once (halo rounds included)."""
        n = len(block)
        off = 0
        while off < n:
            take = min(n - off, self.batch_events - self._pending_n)
            self._pending.append(_slice(block, off, off + take) if (off or take < n) else block)
            self._pending_n += take
            off += take
            if self._pending_n == self.batch_events:
                self._run_pending()

    def flush(self) -> None:
        if self._pending_n:
            self._run_pending()

    def _run_pending(self) -> None:
        blk = self._pending[0] if len(self._pending) == 1 else _concat(self._pending)
        self._pending, self._pending_n = [], 0
        self.rounds.append(self._run_batch(blk))

    def _run_batch(self, blk) -> int:
        import torch
        import torch.distributed as dist
        eng = self.engine
        in_top, in_bot, out_top, out_bot = eng.halo_batch(blk)
        dev = self._device()
        recv = torch.full((in_top + in_bot,), TAINTED, dtype=torch.int64, device=dev)
        send = torch.empty((out_top + out_bot,), dtype=torch.int64, device=dev)
        rnd = 0
        while True:
            eng.halo_round(rnd, recv, send)
            dirty = (recv < 0).any().to(torch.int32).reshape(1)
            if self.world > 1:
                dist.all_reduce(dirty, op=dist.ReduceOp.MAX, group=self.group)
            if not int(dirty.item()):
                break
            recv = self._exchange(send, in_top, in_bot, out_top, out_bot)
            rnd += 1
        eng.halo_finish()
        return rnd + 1

    def _exchange(self, send, in_top, in_bot, out_top, out_bot):
        """Rows to the neighbours: our top rows' values up, bottom rows' down.
        Both sides derived the same item lists, so only the values travel."""
        import torch
        import torch.distributed as dist
        recv = torch.empty((in_top + in_bot,), dtype=torch.int64, device=send.device)
        ops = []
        up, down = self.rank - 1, self.rank + 1
        if out_top:
            ops.append(dist.P2POp(dist.isend, send[:out_top], up, self.group))
        if out_bot:
            ops.append(dist.P2POp(dist.isend, send[out_top:], down, self.group))
        if in_top:
            ops.append(dist.P2POp(dist.irecv, recv[:in_top], up, self.group))
        if in_bot:
            ops.append(dist.P2POp(dist.irecv, recv[in_top:], down, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return recv

    # -- read-out ----------------------------------------------------------------
    def local_l(self):
        """This band's brightness rows (rows, W)."""
        import torch
        self.flush()
        if hasattr(self.engine, "brightness_device"):
            full = self.engine.brightness_device()
        else:
            full = torch.from_numpy(self.engine.l.reshape(self.geometry.height, self.geometry.width))
        return full[self.y0:self.y1]

    def gather_l(self):
        return _all_gather_rows(self.local_l(), self.bands, self.per, self.group, self.world, self.geometry.height)

    def render(self, scale_mode: str = "robust", fixed_bound: float = 1.0, readout_time: int = 0):
        from .pipeline import render_grid
        return render_grid(self.gather_l(), scale_mode, fixed_bound, readout_time)

    def counters(self) -> tuple[int, int]:
        """(event_count, oob_dropped): every rank sees the whole stream."""
        self.flush()
        return self.engine._counters()


def run_local_halo_bands(engines: list, blk) -> int:
    """Single-process emulation of a halo-band group (tests, one-GPU
    measurements): one batch through every rank's engine, the rounds in
    lockstep and the exchange as device copies.  No kernel waits on another
    rank's kernel, so the ranks may share one GPU.  Returns the rounds."""
    import torch
    world = len(engines)
    counts = [e.halo_batch(blk) for e in engines]
    dev = getattr(engines[0], "device", torch.device("cpu"))
    recv = [torch.full((c[0] + c[1],), TAINTED, dtype=torch.int64, device=dev) for c in counts]
    send = [torch.empty((c[2] + c[3],), dtype=torch.int64, device=dev) for c in counts]
    rnd = 0
    while True:
        for e, rv, sd in zip(engines, recv, send):
            e.halo_round(rnd, rv, sd)
        if not any(bool((rv < 0).any()) for rv in recv):
            break
        for r in range(world):
            in_top, in_bot, out_top, out_bot = counts[r]
            nv = torch.empty_like(recv[r])
            if in_top:
                nv[:in_top] = send[r - 1][counts[r - 1][2]:]      # the upper band's bottom rows
            if in_bot:
                nv[in_top:] = send[r + 1][:counts[r + 1][2]]      # the lower band's top rows
            recv[r] = nv
        rnd += 1
    for e in engines:
        e.halo_finish()
    return rnd + 1
