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


# ---------------------------------------------------------------- filter ON ---
# Halo bands: the window pass on every rank, the blur split by
# rows with G halo rows, halo values exchanged in rounds until final.

def _halo_stream():
    geom = SensorGeometry(40, 30)
    params = compute_params(40.0, Fraction(1, 2), geom, spatial_enabled=True)
    ev = workloads.moving_texture(40, 30, 12000, seed=4)
    return geom, params, ev


def _halo_reference(geom, params, ev):
    from oracle import oracle as orc
    ref = orc.OracleEngine(geom.width, geom.height, params)
    for blk in workloads.packets(ev, 1000):
        ref.process_array(blk.t, blk.x, blk.y, blk.p)
    return ref


def test_local_halo_bands_match_full_sensor_cpu():
    """Three ranks emulated in one process with the CPU stand-in engine."""
    from band_model import HaloOracleBand
    geom, params, ev = _halo_stream()
    world, G = 3, 2
    engines = [HaloOracleBand(geom, params, halo_band=(y0, y0 + r, G)) for y0, r in bands.band_rows(30, world)]
    rounds = []
    for s in range(0, len(ev), 4000):
        rounds.append(bands.run_local_halo_bands(engines, ev.slice(s, s + 4000)))
    ref = _halo_reference(geom, params, ev)
    full = np.concatenate([e.l.reshape(30, 40)[y0:y0 + r] for e, (y0, r) in zip(engines, bands.band_rows(30, world))])
    assert np.array_equal(full.reshape(-1), ref.l)
    assert max(rounds) >= 2   # the halo rows did depend on the neighbours


def _halo_worker(rank, world, port, q):
    import torch.distributed as dist
    from band_model import HaloOracleBand
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        geom, params, ev = _halo_stream()
        eng = bands.HaloBandEngine(geom, params, rank=rank, world=world, halo=2, batch_events=4000,
                                   engine_factory=lambda g, p, **kw: HaloOracleBand(g, p, **kw))
        for blk in workloads.packets(ev, 1500):
            eng.process_array(blk)
        full = eng.gather_l().numpy()
        q.put((rank, full, eng.counters()[0], eng.rounds))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_halo_bands_match_full_sensor():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 1000
    procs = [ctx.Process(target=_halo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    geom, params, ev = _halo_stream()
    ref = _halo_reference(geom, params, ev)
    for rank, full, ec, rounds in out:
        assert np.array_equal(full.reshape(-1), ref.l), rank
        assert ec == len(ev)
        assert max(rounds) >= 2


def _native_halo_group(geom, params, world, G, batch):
    from paper_2510_20071_b200.pipeline import ReconstructionEngine
    G = bands.halo_rows_for(geom.height, world, G)
    return [ReconstructionEngine(geom, params, halo_band=(y0, y0 + r, G), batch_capacity=batch)
            for y0, r in bands.band_rows(geom.height, world)]


@pytest.mark.gpu
@pytest.mark.parametrize("world,G", [(2, 1), (3, 4), (8, 2)])
def test_native_halo_bands_bit_exact(world, G):
    """Native halo-band engines, emulated ranks on one GPU: every band's rows
    (brightness and p_bar) and the global window state equal the oracle's."""
    from oracle import oracle as orc
    geom = SensorGeometry(160, 120)
    params = compute_params(40.0, Fraction(1, 2), geom, spatial_enabled=True)
    ev = workloads.moving_texture(160, 120, 300_000, seed=11)
    ref = orc.OracleEngine(160, 120, params)
    for blk in workloads.packets(ev, 10_000):
        ref.process_array(blk.t, blk.x, blk.y, blk.p)
    engines = _native_halo_group(geom, params, world, G, 40_000)
    rounds = [bands.run_local_halo_bands(engines, ev.slice(s, s + 40_000)) for s in range(0, len(ev), 40_000)]
    assert max(rounds) >= 2
    rl, rp = ref.l.reshape(120, 160), ref.p_bar.reshape(120, 160)
    for e, (y0, r) in zip(engines, bands.band_rows(120, world)):
        st = e.state_arrays()
        assert np.array_equal(st["l"].reshape(120, 160)[y0:y0 + r], rl[y0:y0 + r]), (y0, r)
        assert np.array_equal(st["p_bar"].reshape(120, 160)[y0:y0 + r], rp[y0:y0 + r])
        for k in ("active_count", "tile_count", "qx", "qy", "qs"):
            assert np.array_equal(st[k], getattr(ref, k)), k
        e.close()


@pytest.mark.gpu
def test_native_halo_bands_noise_hot_pixels():
    """Config-3-like stream (noise + hot pixels, long segments) over 4 bands."""
    from oracle import oracle as orc
    geom = SensorGeometry(256, 144)
    params = compute_params(40.0, Fraction(1, 2), geom, spatial_enabled=True)
    ev = workloads.texture_noise_hot(256, 144, 400_000, seed=2)
    ref = orc.OracleEngine(256, 144, params)
    ref.process_array(ev.t, ev.x, ev.y, ev.p)
    engines = _native_halo_group(geom, params, 4, 8, 100_000)
    for s in range(0, len(ev), 100_000):
        bands.run_local_halo_bands(engines, ev.slice(s, s + 100_000))
    full = np.concatenate([e.l.reshape(144, 256)[y0:y0 + r] for e, (y0, r) in zip(engines, bands.band_rows(144, 4))])
    assert np.array_equal(full.reshape(-1), ref.l)


@pytest.mark.gpu
def test_halo_band_engine_single_rank_and_render():
    """HaloBandEngine at world 1 (no neighbours: one round per batch) renders like the oracle."""
    import torch
    from oracle import oracle as orc
    geom = SensorGeometry(120, 90)
    params = compute_params(40.0, Fraction(1, 2), geom, spatial_enabled=True)
    ev = workloads.moving_texture(120, 90, 100_000, seed=6)
    ref = orc.OracleEngine(120, 90, params)
    eng = bands.HaloBandEngine(geom, params, rank=0, world=1, batch_events=30_000)
    from paper_2510_20071_b200.pipeline import DeviceEventArray
    for i, blk in enumerate(workloads.packets(ev, 7_000)):
        ref.process_array(blk.t, blk.x, blk.y, blk.p)
        if i % 2:   # host and device packets, split across batch boundaries
            eng.process_array(blk)
        else:
            eng.process_array(DeviceEventArray(torch.from_numpy(blk.x.view(np.int16)).cuda(),
                                               torch.from_numpy(blk.y.view(np.int16)).cuda(),
                                               torch.from_numpy(blk.p).cuda(), blk.t))
    assert torch.equal(eng.gather_l().cpu().reshape(-1), torch.from_numpy(ref.l))
    fr = eng.render("robust")
    px, b, _ = ref.render("robust")
    assert np.array_equal(fr.pixels, px) and fr.bounds == b
    assert set(eng.rounds) == {1}
    assert eng.counters()[0] == len(ev)
