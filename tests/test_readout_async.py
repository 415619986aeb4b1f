"""Asynchronous read-out (fibar_render_async) and run()'s pipelined frame loop.

Frames read out asynchronously -- after the newest blur stage on the engine's
blur stream, while the next packets' front end runs -- must equal the
synchronous render of the same state, and run() must hand the sink the same
frames in the same order as the reference's loop (pipeline.py:372-397).
"""
from fractions import Fraction

import numpy as np
import pytest

from paper_2510_20071_b200 import workloads
from paper_2510_20071_b200.core import SensorGeometry, compute_params


@pytest.mark.gpu
@pytest.mark.parametrize("spatial,packet", [(True, 20_000), (True, 100_000), (False, 50_000)])
def test_render_async_matches_render(spatial, packet):
    import torch
    from oracle import oracle as orc
    from paper_2510_20071_b200.pipeline import ReconstructionEngine
    geom = SensorGeometry(320, 240)
    params = compute_params(40.0, Fraction(1, 2), geom, spatial_enabled=spatial)
    ev = workloads.moving_texture(320, 240, 600_000, seed=8)
    eng = ReconstructionEngine(geom, params)
    ref = orc.OracleEngine(320, 240, params)
    pend = []
    for i, blk in enumerate(workloads.packets(ev, packet)):
        eng.process_array(blk)
        ref.process_array(blk.t, blk.x, blk.y, blk.p)
        mode = "robust" if i % 3 else "fixed"
        dev = bool(i % 2)
        out = torch.empty((240, 320), dtype=torch.uint8, device="cuda") if dev else None
        pend.append((eng.render_async(mode, 0.5, readout_time=i, out=out), ref.render(mode, 0.5)))
    for af, (px, bounds, deg) in pend:
        fr = af.frame()
        assert np.array_equal(fr.pixels, px), af.readout_time
        assert fr.bounds == bounds and fr.degenerate == deg
    # the synchronous read-out after them still sees the same state
    fr = eng.render("robust")
    px, bounds, _ = ref.render("robust")
    assert np.array_equal(fr.pixels, px) and fr.bounds == bounds


@pytest.mark.gpu
def test_run_pipelined_frames_match_oracle():
    from oracle import oracle as orc
    from paper_2510_20071_b200.pipeline import ReconstructionEngine, run
    geom = SensorGeometry(256, 192)
    params = compute_params(40.0, Fraction(1, 2), geom)
    ev = workloads.texture_noise_hot(256, 192, 400_000, seed=3)
    blocks = list(workloads.packets(ev, 30_000))
    times = [int(ev.t[i]) for i in range(25_000, len(ev), 25_000)] + [int(ev.t[-1]) + 10]
    got = {}
    eng = ReconstructionEngine(geom, params)
    res = run(eng, blocks, readout_times=times, frame_sink=lambda k, f: got.__setitem__(k, f))
    assert res.frames_emitted == len(times) == len(got)
    ref = orc.OracleEngine(256, 192, params)
    pos = 0
    for k, r in enumerate(times):
        idx = int(np.searchsorted(ev.t, r, side="left"))
        if idx > pos:
            ref.process_array(ev.t[pos:idx], ev.x[pos:idx], ev.y[pos:idx], ev.p[pos:idx])
            pos = idx
        px, bounds, _ = ref.render("robust")
        assert np.array_equal(got[k].pixels, px), k
        assert got[k].bounds == bounds and got[k].readout_time == r


@pytest.mark.gpu
def test_render_async_then_reset_and_reuse():
    """A read-out still in flight when the engine is reset or read: the frame is
    the pre-reset state, and the engine afterwards matches a fresh one."""
    import torch
    from oracle import oracle as orc
    from paper_2510_20071_b200.pipeline import DeviceEventArray, ReconstructionEngine
    geom = SensorGeometry(256, 192)
    params = compute_params(40.0, Fraction(1, 2), geom)
    ev = workloads.moving_texture(256, 192, 300_000, seed=21)
    xd = torch.from_numpy(ev.x.view(np.int16)).cuda()
    yd = torch.from_numpy(ev.y.view(np.int16)).cuda()
    pd = torch.from_numpy(ev.p).cuda()
    eng = ReconstructionEngine(geom, params, batch_capacity=1 << 16)
    ref = orc.OracleEngine(256, 192, params)
    for s in range(0, 200_000, 50_000):
        eng.process_array(DeviceEventArray(xd[s:s + 50_000], yd[s:s + 50_000], pd[s:s + 50_000]))
        ref.process_array(ev.t[s:s + 50_000], ev.x[s:s + 50_000], ev.y[s:s + 50_000], ev.p[s:s + 50_000])
    af = eng.render_async("robust")
    assert np.array_equal(eng.l, ref.l)        # a state read joins the read-out
    eng.reset()
    px, bounds, _ = ref.render("robust")
    fr = af.frame()
    assert np.array_equal(fr.pixels, px) and fr.bounds == bounds
    ref2 = orc.OracleEngine(256, 192, params)
    for s in range(0, 300_000, 30_000):
        eng.process_array(DeviceEventArray(xd[s:s + 30_000], yd[s:s + 30_000], pd[s:s + 30_000]))
        ref2.process_array(ev.t[s:s + 30_000], ev.x[s:s + 30_000], ev.y[s:s + 30_000], ev.p[s:s + 30_000])
        eng.render_async("fixed", 0.5)
    st = eng.state_arrays()
    for k in ("p_bar", "l", "active_count", "tile_count", "qx", "qy", "qs"):
        assert np.array_equal(st[k], getattr(ref2, k)), k
