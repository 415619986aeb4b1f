"""Row-band partition (filter OFF).

CPU: world_size-2 gloo processes run the banded engine's host logic (band
split, all_gather assembly, counter all_reduce) with an oracle-backed stand-in
for the native engine, and must reproduce the full-sensor oracle bit for bit.
GPU: several native band engines in one process, each fed the whole stream,
assemble to the full-sensor result.
"""

import os
from fractions import Fraction

import numpy as np
import pytest

from paper_2510_20071_b200 import bands, workloads
from paper_2510_20071_b200.core import SensorGeometry, compute_params


def test_band_rows_cover_the_sensor():
    for H, N in ((260, 2), (480, 8), (8, 3), (101, 4)):
        b = bands.band_rows(H, N)
        assert b[0][0] == 0 and sum(r for _, r in b) == H
        for (y0, r), (y1, _) in zip(b, b[1:]):
            assert y0 + r == y1
    with pytest.raises(Exception):
        bands.band_rows(5, 4)
    ys = np.arange(260)
    own = bands.band_of_rows(ys, 260, 3)
    for r, (y0, rows) in enumerate(bands.band_rows(260, 3)):
        assert np.all(own[y0:y0 + rows] == r)


class OracleBand:
    """Test stand-in for the native band engine: the C oracle on the band's rows."""

    def __init__(self, geom, params, y0):
        from oracle import oracle as orc
        self.y0, self.h, self.w = y0, geom.height, geom.width
        self.eng = orc.OracleEngine(geom.width, geom.height, params)
        self.n = 0

    def process_array(self, blk):
        keep = (blk.y >= self.y0) & (blk.y < self.y0 + self.h)
        self.eng.process_array(blk.t[keep], blk.x[keep], (blk.y[keep] - self.y0).astype(np.uint16), blk.p[keep])
        self.n += int(keep.sum())

    def flush(self):
        pass

    @property
    def l(self):
        return self.eng.l

    def _counters(self):
        return self.n, 0


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        geom = SensorGeometry(64, 37)
        params = compute_params(40.0, Fraction(1, 2), geom, spatial_enabled=False)
        ev = workloads.uniform(64, 37, 40000, seed=9)
        y0 = bands.band_rows(37, world)[rank][0]
        eng = bands.BandedReconstructionEngine(
            geom, params, rank=rank, world=world,
            engine_factory=lambda g, p, **kw: OracleBand(g, p, y0))
        for blk in workloads.packets(ev, 3000):
            eng.process_array(blk)
        full = eng.gather_l().numpy()
        ec, _ = eng.counters()
        q.put((rank, full, ec))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_match_full_sensor():
    import multiprocessing as mp
    from oracle import oracle as orc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    geom = SensorGeometry(64, 37)
    params = compute_params(40.0, Fraction(1, 2), geom, spatial_enabled=False)
    ev = workloads.uniform(64, 37, 40000, seed=9)
    ref = orc.OracleEngine(64, 37, params)
    for blk in workloads.packets(ev, 3000):
        ref.process_array(blk.t, blk.x, blk.y, blk.p)
    for rank, full, ec in out:
        assert np.array_equal(full.reshape(-1), ref.l), rank
        assert ec == 40000


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 8])
def test_native_bands_assemble_exactly(world):
    import torch
    from oracle import oracle as orc
    from paper_2510_20071_b200.pipeline import ReconstructionEngine, render_grid
    geom = SensorGeometry(346, 260)
    params = compute_params(40.0, Fraction(1, 2), geom, spatial_enabled=False)
    ev = workloads.texture_noise_hot(346, 260, 400_000, seed=5)
    ref = orc.OracleEngine(346, 260, params)
    engines = []
    for y0, rows in bands.band_rows(260, world):
        engines.append(ReconstructionEngine(SensorGeometry(346, rows), bands.band_params(params, 346, rows),
                                            row_band=(y0, 260)))
    for blk in workloads.packets(ev, 50_000):
        ref.process_array(blk.t, blk.x, blk.y, blk.p)
        for e in engines:
            e.process_array(blk)
    full = np.concatenate([e.l for e in engines])
    assert np.array_equal(full, ref.l)
    assert np.array_equal(np.concatenate([e.p_bar for e in engines]), ref.p_bar)
    assert sum(e.event_count for e in engines) == 400_000
    fr = render_grid(torch.from_numpy(full.reshape(260, 346)).cuda())
    px, b, d = ref.render("robust")
    assert np.array_equal(fr.pixels, px) and fr.bounds == b


@pytest.mark.gpu
def test_bands_refuse_filter_on():
    from paper_2510_20071_b200.errors import ConfigError
    from paper_2510_20071_b200.pipeline import ReconstructionEngine
    params = compute_params(40.0, Fraction(1, 2), SensorGeometry(64, 64))
    with pytest.raises(ConfigError):
        ReconstructionEngine(SensorGeometry(64, 32), bands.band_params(params, 64, 32), row_band=(32, 64))
