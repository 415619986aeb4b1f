"""Row-band partition of one sensor across GPUs (filter OFF).

SURVEY §8(e): with the spatial filter off, pixels are independent
(_kernels.py:62-73), so the sensor splits into row bands with no exchange on
the data path.  Each rank runs one native engine that owns rows
[y0, y0 + rows) and receives the *whole* packet stream (shared input, e.g.
each GPU's own copy of the camera packets); the device ingest keeps only its
band's events, in stream order, so every pixel sees exactly its reference
event sequence.  Read-out is the only collective: the bands' brightness rows
are all-gathered (NCCL over NVLink on GPUs, gloo in the CPU tests) into the
full grid, which every rank can render.  Counters are summed with all_reduce.

With the filter ON the window is one global FIFO over the interleaved stream,
so bands would need a global window pass plus halo timelines; that is not
implemented and the engine refuses it.
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
        import torch
        import torch.distributed as dist
        W = self.geometry.width
        mine = self.local_l()
        pad = torch.zeros((self.per, W), dtype=torch.float32, device=mine.device)
        pad[: self.rows] = mine
        if self.world == 1:
            return pad[: self.geometry.height]
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(parts, pad, group=self.group)
        rows = [parts[r][: self.bands[r][1]] for r in range(self.world)]
        return torch.cat(rows, 0)

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
