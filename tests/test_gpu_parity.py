"""Parity of the CUDA path (through the C ABI) with the reference.

Golden vectors come from running the reference itself (tests/golden); larger
seeded streams are checked against the C oracle (pinned to the same goldens).
Bar: everything bit-exact except where noted (window/stale state is integer;
p_bar and l are replayed in stream order with separately rounded float32
multiply/add, so they are bit-exact too; the north-star tolerance
max|dl| <= 1e-4 * range(l) is asserted as a fallback message only).
"""

from fractions import Fraction

import numpy as np
import pytest

from conftest import golden_path
from test_oracle_golden import params_of, run_oracle

pytestmark = pytest.mark.gpu

STATE_KEYS = ("p_bar", "l", "active_count", "tile_count", "qx", "qy", "qs")


def make_engine(g, **kw):
    from paper_2510_20071_b200.pipeline import ReconstructionEngine
    geom, params = params_of(g)
    gain = g["gain"] if g["gain"].size else None
    return ReconstructionEngine(geom, params, threshold_map=gain, regulate_every=int(g["regulate_every"]),
                                blur_enabled=bool(g["blur"]), **kw)


def feed(eng, g, packet=None):
    from paper_2510_20071_b200.core import EventArray
    n = len(g["x"])
    P = packet or int(g["packet"])
    for a in range(0, n, P):
        b = min(n, a + P)
        eng.process_array(EventArray(g["t"][a:b], g["x"][a:b], g["y"][a:b], g["p"][a:b]))


def assert_state(eng, ref, name):
    st = eng.state_arrays()
    for k in STATE_KEYS:
        a, b = st[k], ref[k]
        if k == "l" and not np.array_equal(a, b):
            rng = float(b.max() - b.min()) or 1.0
            err = float(np.abs(a.astype(np.float64) - b).max())
            pytest.fail(f"{name}: l differs, max err {err:.3e} = {err / rng:.3e} of range")
        assert np.array_equal(a, b), (name, k, np.nonzero(a != b)[0][:10])


def test_golden_engine_state(golden_case):
    name, g = golden_case
    eng = make_engine(g)
    feed(eng, g)
    assert_state(eng, g, name)
    assert eng.event_count == int(g["event_count"])
    assert eng.oob_dropped == int(g["oob_dropped"])
    assert eng.last_t == int(g["last_t"])
    for mode in ("robust", "fixed"):
        fr = eng.render(mode, 0.5 if mode == "fixed" else 1.0)
        assert np.array_equal(fr.pixels, g[f"render_{mode}"]), (name, mode)
        assert fr.bounds == tuple(g[f"bounds_{mode}"])
        assert fr.degenerate == bool(g[f"degenerate_{mode}"])
    assert eng.state_digest() == str(g["digest"])


@pytest.mark.parametrize("cap", [97, 1000, 1 << 16])
def test_batch_capacity_invariance(cap):
    """Coalescing / splitting packets into device batches never changes state."""
    g = dict(np.load(golden_path("noise_hot_on")))
    eng = make_engine(g, batch_capacity=cap)
    feed(eng, g, packet=1234)
    assert_state(eng, g, f"cap={cap}")


def test_device_packets_match_host_packets():
    import torch
    from paper_2510_20071_b200.pipeline import DeviceEventArray
    g = dict(np.load(golden_path("texture_on")))
    eng = make_engine(g)
    n = len(g["x"])
    P = int(g["packet"])
    for a in range(0, n, P):
        b = min(n, a + P)
        eng.process_array(DeviceEventArray(torch.from_numpy(g["x"][a:b].view(np.int16)).cuda(),
                                           torch.from_numpy(g["y"][a:b].view(np.int16)).cuda(),
                                           torch.from_numpy(g["p"][a:b]).cuda(), g["t"][a:b]))
    assert_state(eng, g, "device")
    assert eng.last_t == int(g["last_t"])


def _oracle_stream(kind, w, h, n, packet, spatial=True, seed=11, **kw):
    from oracle import oracle as orc
    from paper_2510_20071_b200 import workloads
    from paper_2510_20071_b200.core import SensorGeometry, compute_params
    geom = SensorGeometry(w, h)
    ev = workloads.make(kind, geom, n, seed=seed, **kw)
    params = compute_params(40.0, Fraction(1, 2), geom, spatial_enabled=spatial)
    ref = orc.OracleEngine(w, h, params)
    for a in range(0, n, packet):
        b = min(n, a + packet)
        ref.process_array(ev.t[a:b], ev.x[a:b], ev.y[a:b], ev.p[a:b])
    return geom, params, ev, ref


@pytest.mark.parametrize("kind,w,h,n,packet,spatial", [
    ("uniform", 346, 260, 1_000_000, 1_000_000, False),
    ("texture", 640, 480, 400_000, 10_000, True),
    ("texture_noise_hot", 320, 180, 300_000, 100_000, True),
    ("uniform", 346, 260, 300_000, 50_000, True),
    ("texture_noise_hot", 320, 180, 300_000, 300_000, False),
])
def test_oracle_streams(kind, w, h, n, packet, spatial):
    from paper_2510_20071_b200.pipeline import ReconstructionEngine
    geom, params, ev, ref = _oracle_stream(kind, w, h, n, packet, spatial)
    eng = ReconstructionEngine(geom, params)
    for a in range(0, n, packet):
        eng.process_array(ev.slice(a, min(n, a + packet)))
    want = dict(p_bar=ref.p_bar, l=ref.l, active_count=ref.active_count, tile_count=ref.tile_count,
                qx=ref.qx, qy=ref.qy, qs=ref.qs)
    assert_state(eng, want, kind)
    fr = eng.render("robust")
    px, bounds, deg = ref.render("robust")
    assert np.array_equal(fr.pixels, px) and fr.bounds == bounds and fr.degenerate == deg


@pytest.mark.parametrize("spatial", [True, False])
def test_dominant_pixel_segments(spatial):
    """One pixel takes 45 % of a 400k-event batch and another 5 %: a segment
    past the tiled replay's bound (the strided-piece path) and one of several
    shared-memory tiles, beside texture events -- exact against the oracle."""
    import oracle.oracle as orc
    from paper_2510_20071_b200 import workloads
    from paper_2510_20071_b200.core import EventArray, SensorGeometry, compute_params
    from paper_2510_20071_b200.pipeline import ReconstructionEngine
    w, h, n = 240, 180, 400_000   # (43,200 pixels: the window cannot reach the reference's u16 count cap)
    geom = SensorGeometry(w, h)
    ev = workloads.make("texture", geom, n, seed=23)
    rng = np.random.default_rng(5)
    r = rng.random(n)
    x, y, p = ev.x.copy(), ev.y.copy(), ev.p.copy()
    x[r < 0.45], y[r < 0.45] = 100, 77
    x[(r >= 0.45) & (r < 0.50)], y[(r >= 0.45) & (r < 0.50)] = 7, 150
    p[r < 0.50] = rng.choice(np.array([-1, 1], np.int8), int((r < 0.50).sum()))
    params = compute_params(40.0, Fraction(1, 2), geom, spatial_enabled=spatial)
    ref = orc.OracleEngine(w, h, params)
    ref.process_array(ev.t, x, y, p)
    eng = ReconstructionEngine(geom, params, batch_capacity=1 << 19)
    eng.process_array(EventArray(ev.t, x, y, p))
    want = dict(p_bar=ref.p_bar, l=ref.l, active_count=ref.active_count, tile_count=ref.tile_count,
                qx=ref.qx, qy=ref.qy, qs=ref.qs)
    assert_state(eng, want, "dominant pixel")


@pytest.mark.parametrize("n,flag", [(60_000, False), (70_000, True)])
def test_saturation_flag(n, flag):
    """one pixel with more than 65535 events in the window reaches the
    reference's u16 cap.  The engine flags it (and, while no entry of the pixel
    has been popped yet, still matches the saturating oracle)."""
    from paper_2510_20071_b200.core import EventArray, SensorGeometry, compute_params
    from paper_2510_20071_b200.pipeline import ReconstructionEngine
    from oracle import oracle as orc
    geom = SensorGeometry(300, 300)
    params = compute_params(40.0, Fraction(1, 2), geom)
    x = np.full(n, 5, np.uint16)
    y = np.full(n, 7, np.uint16)
    p = np.where(np.arange(n) % 3 == 0, -1, 1).astype(np.int8)
    t = np.arange(n, dtype=np.uint64)
    eng = ReconstructionEngine(geom, params, batch_capacity=1 << 14)
    ref = orc.OracleEngine(300, 300, params)
    for a in range(0, n, 20_000):
        b = min(n, a + 20_000)
        eng.process_array(EventArray(t[a:b], x[a:b], y[a:b], p[a:b]))
        ref.process_array(t[a:b], x[a:b], y[a:b], p[a:b])
    assert eng.saturation_detected == flag
    want = dict(p_bar=ref.p_bar, l=ref.l, active_count=ref.active_count, tile_count=ref.tile_count,
                qx=ref.qx, qy=ref.qy, qs=ref.qs)
    assert_state(eng, want, f"single pixel n={n}")


def test_saturation_flag_after_pops():
    """Past the cap with pops the reference's counts diverge: the flag must be up."""
    from paper_2510_20071_b200.core import EventArray, SensorGeometry, compute_params
    from paper_2510_20071_b200.pipeline import ReconstructionEngine
    geom = SensorGeometry(300, 300)
    params = compute_params(40.0, Fraction(1, 2), geom)
    n = 200_000
    rng = np.random.default_rng(3)
    hot = rng.random(n) < 0.9
    x = np.where(hot, 5, rng.integers(0, 300, n)).astype(np.uint16)
    y = np.where(hot, 7, rng.integers(0, 300, n)).astype(np.uint16)
    p = rng.choice(np.array([-1, 1], np.int8), n)
    eng = ReconstructionEngine(geom, params)
    eng.process_array(EventArray(np.arange(n, dtype=np.uint64), x, y, p))
    assert eng.saturation_detected


def test_pinned_host_packets_direct_copy():
    """Large packets in pinned host memory are DMA'd without the CPU staging copy;
    mixing them with small (staged) packets and device packets changes nothing."""
    import torch
    from paper_2510_20071_b200.core import EventArray
    from paper_2510_20071_b200.pipeline import DeviceEventArray, ReconstructionEngine
    geom, params, ev, ref = _oracle_stream("texture", 320, 240, 600_000, 600_000, True, seed=5)
    pin = lambda a: torch.from_numpy(a.view(np.int16) if a.dtype == np.uint16 else a).pin_memory().numpy()
    xs, ys, ps = pin(ev.x).view(np.uint16), pin(ev.y).view(np.uint16), pin(ev.p)
    eng = ReconstructionEngine(geom, params, batch_capacity=1 << 17)
    cuts = [0, 1000, 201_000, 205_000, 405_000, 600_000]   # small, large, small, large(device), large
    for i, (a, b) in enumerate(zip(cuts[:-1], cuts[1:])):
        if i == 3:
            eng.process_array(DeviceEventArray(torch.from_numpy(ev.x[a:b].view(np.int16)).cuda(),
                                               torch.from_numpy(ev.y[a:b].view(np.int16)).cuda(),
                                               torch.from_numpy(ev.p[a:b]).cuda()))
        else:
            eng.process_array(EventArray(ev.t[a:b], xs[a:b], ys[a:b], ps[a:b]))
    want = dict(p_bar=ref.p_bar, l=ref.l, active_count=ref.active_count, tile_count=ref.tile_count,
                qx=ref.qx, qy=ref.qy, qs=ref.qs)
    assert_state(eng, want, "pinned direct")


def test_graph_and_streamed_batches_agree(monkeypatch):
    """Small batches replay captured CUDA graphs, large ones stream on two
    streams; every form gives the same (oracle-exact) state."""
    from paper_2510_20071_b200.pipeline import ReconstructionEngine
    geom, params, ev, ref = _oracle_stream("texture_noise_hot", 320, 240, 300_000, 30_000, True, seed=9)
    want = dict(p_bar=ref.p_bar, l=ref.l, active_count=ref.active_count, tile_count=ref.tile_count,
                qx=ref.qx, qy=ref.qy, qs=ref.qs)
    # graphs=1: small batches stream with their front end replayed as a graph;
    # full=1: one whole-batch graph (serial schedule); graphs=0: every kernel
    # streamed; async: read-outs behind the blur stage (render_async)
    for graphs, full, read in (("1", "0", "sync"), ("1", "1", "sync"), ("0", "0", "sync"), ("1", "0", "async")):
        monkeypatch.setenv("FIBAR_GRAPHS", graphs)
        monkeypatch.setenv("FIBAR_FULL_GRAPHS", full)
        eng = ReconstructionEngine(geom, params)
        for a in range(0, len(ev), 30_000):
            eng.process_array(ev.slice(a, min(len(ev), a + 30_000)))
            if read == "sync":
                eng.render("robust")          # a read-out per packet: one batch per packet
            else:
                eng.render_async("robust")
        assert_state(eng, want, f"graphs={graphs} full={full} {read}")
        eng.close()


def test_launch_modes_agree(monkeypatch):
    """Programmatic dependent launch, the two-stream overlap, the serial
    schedule and the blur's green-context SM partition are scheduling choices
    only: every combination is oracle-exact."""
    from paper_2510_20071_b200.pipeline import ReconstructionEngine
    geom, params, ev, ref = _oracle_stream("texture", 320, 240, 600_000, 50_000, True, seed=13)
    want = dict(p_bar=ref.p_bar, l=ref.l, active_count=ref.active_count, tile_count=ref.tile_count,
                qx=ref.qx, qy=ref.qy, qs=ref.qs)
    for pdl, serial, green in (("0", "0", "0"), ("1", "1", "16"), ("0", "1", "0"), ("1", "0", "24")):
        monkeypatch.setenv("FIBAR_PDL", pdl)
        monkeypatch.setenv("FIBAR_SERIAL", serial)
        monkeypatch.setenv("FIBAR_GREEN", green)
        eng = ReconstructionEngine(geom, params, batch_capacity=1 << 18)
        for a in range(0, len(ev), 50_000):
            eng.process_array(ev.slice(a, min(len(ev), a + 50_000)))
        assert_state(eng, want, f"pdl={pdl} serial={serial} green={green}")
        eng.close()


@pytest.mark.parametrize("env", [
    {"FIBAR_RUN_G": "0", "FIBAR_RUN_G_LARGE": "0"},          # one lane per chunk (k_window_run)
    {"FIBAR_RUN_G": "4", "FIBAR_RUN_G_LARGE": "8"},
    {"FIBAR_RUN_G": "2", "FIBAR_RUN_G_LARGE": "2", "FIBAR_REG32X": "0"},
    {"FIBAR_SORT_LANES": "1", "FIBAR_STAGE_GRAPHS": "0", "FIBAR_SNAP": "0"},
    {"FIBAR_SORT_LANES": "3", "FIBAR_GREEN_SMALL": "1", "FIBAR_LONG_GRID": "3"},
    {"FIBAR_GRAPHS": "0"},
])
def test_schedule_knobs_agree(monkeypatch, env):
    """The window run's lanes per chunk, the 32-bit regulator, the sort
    streams, the blur-stage graph, the read-out snapshot and the rest of
    DESIGN section 9 never change a result: small batches (graphs) and large
    ones mixed, a read-out after every packet, frames and final state exact."""
    from paper_2510_20071_b200.pipeline import ReconstructionEngine
    import oracle.oracle as orc
    from paper_2510_20071_b200 import workloads
    from paper_2510_20071_b200.core import SensorGeometry, compute_params
    geom = SensorGeometry(320, 240)
    ev = workloads.make("texture_noise_hot", geom, 700_000, seed=41)
    params = compute_params(40.0, Fraction(1, 2), geom)
    cuts = [0, 30_000, 60_000, 400_000, 430_000, 431_000, 700_000]   # small, large (two device batches), small, tiny, large
    ref = orc.OracleEngine(geom.width, geom.height, params)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    eng = ReconstructionEngine(geom, params, batch_capacity=1 << 18)
    pending = []
    for a, b in zip(cuts[:-1], cuts[1:]):
        blk = ev.slice(a, b)
        ref.process_array(blk.t, blk.x, blk.y, blk.p)
        eng.process_array(blk)
        pending.append((eng.render_async("robust"), ref.render("robust")))
    for af, (px, bounds, deg) in pending:
        fr = af.frame()
        assert np.array_equal(fr.pixels, px) and fr.bounds == bounds and fr.degenerate == deg, env
    want = dict(p_bar=ref.p_bar, l=ref.l, active_count=ref.active_count, tile_count=ref.tile_count,
                qx=ref.qx, qy=ref.qy, qs=ref.qs)
    assert_state(eng, want, str(env))
    eng.close()


@pytest.mark.parametrize("kind,w,h,n,packet,kw", [
    # hot pixels at config-3 geometry: long segments, several 1M-event batches
    ("texture_noise_hot", 1280, 720, 3_000_000, 100_000, dict(bcap=1 << 20)),
    # the default (non-power-of-two) 1280x720 batch of 3,735,552 events, more
    # than two of them: carried stale items and last-touch tables across batches
    ("texture_noise_hot", 1280, 720, 8_000_000, 1_000_000, {}),
    # variants at scale: tile side 3, fill 2/3, regulate_every 2, a gain map, blur off
    ("texture", 640, 480, 2_500_000, 50_000, dict(tile_side=3, fill=Fraction(2, 3), regulate_every=2, gain=True)),
    ("texture", 640, 480, 2_500_000, 250_000, dict(blur=False)),
    # config-5 geometry: a window (~1.2M events) larger than a device batch (warp-counted collapses)
    ("texture", 2560, 1440, 3_000_000, 1_000_000, dict(bcap=1 << 20)),
])
def test_large_streams_match_oracle(kind, w, h, n, packet, kw):
    from oracle import oracle as orc
    from paper_2510_20071_b200 import workloads
    from paper_2510_20071_b200.core import SensorGeometry, compute_params
    from paper_2510_20071_b200.pipeline import ReconstructionEngine
    geom = SensorGeometry(w, h)
    ev = workloads.make(kind, geom, n, seed=21)
    params = compute_params(40.0, kw.get("fill", Fraction(1, 2)), geom, tile_side=kw.get("tile_side", 2))
    gain = None
    if kw.get("gain"):
        gain = np.random.default_rng(4).uniform(0.6, 1.6, (h, w)).astype(np.float32)
    every, blur = kw.get("regulate_every", 1), kw.get("blur", True)
    eng = ReconstructionEngine(geom, params, threshold_map=gain, regulate_every=every, blur_enabled=blur,
                               batch_capacity=kw.get("bcap", 0))
    ref = orc.OracleEngine(w, h, params, gain=gain, regulate_every=every, blur_enabled=blur)
    for a in range(0, n, packet):
        b = min(n, a + packet)
        eng.process_array(ev.slice(a, b))
        ref.process_array(ev.t[a:b], ev.x[a:b], ev.y[a:b], ev.p[a:b])
    want = dict(p_bar=ref.p_bar, l=ref.l, active_count=ref.active_count, tile_count=ref.tile_count,
                qx=ref.qx, qy=ref.qy, qs=ref.qs)
    assert_state(eng, want, f"{kind} {w}x{h} {kw}")
    fr = eng.render("robust")
    px, bounds, deg = ref.render("robust")
    assert np.array_equal(fr.pixels, px) and fr.bounds == bounds


def test_golden_stale_mask_per_batch(golden_case):
    """The CUDA stale items (popping event, pixel), batch by batch, equal the
    reference's per-event blurred-pixel list (SpatialFilter.on_event,
    spatial.py:165-207) recorded in the goldens -- the stale mask bit-exact."""
    from paper_2510_20071_b200.core import EventArray
    name, g = golden_case
    if "stale_j" not in g:
        pytest.skip("filter-OFF golden")
    eng = make_engine(g)
    n = len(g["x"])
    P = int(g["packet"]) if int(g["packet"]) else n
    js, pxs = [], []
    for a in range(0, n, P):
        b = min(n, a + P)
        eng.process_array(EventArray(g["t"][a:b], g["x"][a:b], g["y"][a:b], g["p"][a:b]))
        j, pix = eng.stale_items()   # one device batch per packet
        js.append(j)
        pxs.append(pix)
    j, pix = np.concatenate(js), np.concatenate(pxs)
    assert np.array_equal(j, g["stale_j"]), (name, len(j), len(g["stale_j"]))
    assert np.array_equal(pix, g["stale_pix"]), name
    assert eng.stale_count == len(g["stale_j"])


def test_small_packets_720p_frame_by_frame():
    """600 packets of 1k events at 1280x720 (texture + noise + hot pixels), a
    robust read-out after every packet, each frame equal to the oracle's."""
    from oracle import oracle as orc
    from paper_2510_20071_b200 import workloads
    from paper_2510_20071_b200.core import SensorGeometry, compute_params
    from paper_2510_20071_b200.pipeline import ReconstructionEngine
    geom = SensorGeometry(1280, 720)
    ev = workloads.make("texture_noise_hot", geom, 600_000, seed=31)
    params = compute_params(40.0, Fraction(1, 2), geom)
    eng = ReconstructionEngine(geom, params)
    ref = orc.OracleEngine(geom.width, geom.height, params)
    bad = []
    for k, a in enumerate(range(0, len(ev), 1000)):
        blk = ev.slice(a, a + 1000)
        eng.process_array(blk)
        ref.process_array(blk.t, blk.x, blk.y, blk.p)
        fr = eng.render("robust")
        px, bounds, deg = ref.render("robust")
        if not (np.array_equal(fr.pixels, px) and fr.bounds == bounds and fr.degenerate == deg):
            bad.append(k)
    assert not bad, f"frames differ at packets {bad[:10]}"
    want = dict(p_bar=ref.p_bar, l=ref.l, active_count=ref.active_count, tile_count=ref.tile_count,
                qx=ref.qx, qy=ref.qy, qs=ref.qs)
    assert_state(eng, want, "720p 1k packets")


def test_separate_device_packets_are_gathered():
    """Device packets in separate allocations (a real device stream) are
    gathered into device batches (k_gather) instead of running one batch per
    packet, mixed with contiguous views and host packets; state stays exact."""
    import torch
    from paper_2510_20071_b200.pipeline import DeviceEventArray, ReconstructionEngine
    geom, params, ev, ref = _oracle_stream("texture_noise_hot", 320, 240, 400_000, 400_000, True, seed=13)
    eng = ReconstructionEngine(geom, params, batch_capacity=1 << 17)
    b0 = eng.stats()["batches"]
    keep = []
    cuts = list(range(0, 300_000, 7_500)) + [300_000]
    for a, b in zip(cuts[:-1], cuts[1:]):
        cols = [torch.from_numpy(ev.x[a:b].view(np.int16)).cuda(), torch.from_numpy(ev.y[a:b].view(np.int16)).cuda(),
                torch.from_numpy(ev.p[a:b].copy()).cuda()]
        keep.append(cols)   # separate allocations, so never address-contiguous
        eng.process_array(DeviceEventArray(*cols))
    big = [torch.from_numpy(ev.x[300_000:].view(np.int16)).cuda(), torch.from_numpy(ev.y[300_000:].view(np.int16)).cuda(),
           torch.from_numpy(ev.p[300_000:].copy()).cuda()]
    for a in range(0, 60_000, 20_000):   # contiguous views of one buffer, then a host packet
        eng.process_array(DeviceEventArray(big[0][a:a + 20_000], big[1][a:a + 20_000], big[2][a:a + 20_000]))
    eng.process_array(ev.slice(360_000, 400_000))
    want = dict(p_bar=ref.p_bar, l=ref.l, active_count=ref.active_count, tile_count=ref.tile_count,
                qx=ref.qx, qy=ref.qy, qs=ref.qs)
    assert_state(eng, want, "gathered device packets")
    assert eng.stats()["batches"] - b0 <= 6   # 400k events in 128k-event batches, not one per packet


def test_many_batch_sizes_cycle_the_graph_cache():
    """Small batches of 40 distinct sizes (more than the front-end graph cache
    holds): captures, evictions and replays of the two-part front end, with a
    read-out after every batch; state and frames stay oracle-exact."""
    from oracle import oracle as orc
    from paper_2510_20071_b200 import workloads
    from paper_2510_20071_b200.core import SensorGeometry, compute_params
    from paper_2510_20071_b200.pipeline import ReconstructionEngine
    geom = SensorGeometry(160, 120)
    ev = workloads.make("texture_noise_hot", geom, 240_000, seed=17)
    params = compute_params(40.0, Fraction(1, 2), geom)
    eng = ReconstructionEngine(geom, params)
    ref = orc.OracleEngine(160, 120, params)
    a = 0
    for k in range(40):
        b = min(len(ev), a + 3000 + 37 * k)
        blk = ev.slice(a, b)
        eng.process_array(blk)
        ref.process_array(blk.t, blk.x, blk.y, blk.p)
        af = eng.render_async("robust")
        px, _, _ = ref.render("robust")
        assert np.array_equal(af.frame().pixels, px), k
        a = b
    want = dict(p_bar=ref.p_bar, l=ref.l, active_count=ref.active_count, tile_count=ref.tile_count,
                qx=ref.qx, qy=ref.qy, qs=ref.qs)
    assert_state(eng, want, "graph cache cycling")


@pytest.mark.gpu
@pytest.mark.parametrize("num,den,area,q_min,q_max", [
    (1, 2, 4, 256, 921_600),        # config 3 (fill 1/2, 2x2 tiles)
    (2, 3, 9, 64, 307_200),         # fill 2/3, tile side 3
    (1, 2, 4, 1, (1 << 22) - 1),    # the largest q_max the 32-bit form takes
    (7, 127, 25, 16, 4_000_000),    # odd ratio, den * q_max just under 2^29
    (1_000_003, 3, 16, 1, 100_000),  # num * A close to 2^24: quotients far above the clamp
])
def test_regulator_32bit_form_is_the_exact_floor(num, den, area, q_min, q_max):
    """regulate32x (float quotient + 32-bit remainder fix-up, the form the window
    kernels step with) equals the reference's integer formula
    (_kernels.py:195-201) on random triples and on triples built around exact
    multiples N = k D, where a float quotient alone would be off by one."""
    import ctypes as C
    from paper_2510_20071_b200 import _native
    lib = _native.load()
    rng = np.random.default_rng(num * 31 + den)
    n = 2_000_000
    # random windows: len <= q_max + 1, 1 <= nt <= np <= len, over all magnitudes
    mag = rng.integers(0, 23, n)
    ln = np.minimum(q_max + 1, 1 + (rng.random(n) * (2.0 ** mag)).astype(np.int64)).astype(np.int64)
    npx = 1 + (rng.random(n) * ln).astype(np.int64)
    npx = np.minimum(npx, ln)
    ntl = 1 + (rng.random(n) * npx).astype(np.int64)
    ntl = np.minimum(ntl, npx)
    # adversarial third: choose len so that len * nt * numA is k * (den * np) + {-1, 0, +1} when possible
    m = n // 3
    numA = num * area
    D = den * npx[:m]
    k = 1 + (rng.random(m) * min(q_max + 4, 1 << 22)).astype(np.int64)
    target = k * D + rng.integers(-1, 2, m)
    ln_adv = np.clip(np.rint(target / (ntl[:m] * numA)).astype(np.int64), np.maximum(npx[:m], 1), q_max + 1)
    ln[:m] = ln_adv
    want = np.clip((ln * numA * ntl) // (den * npx), q_min, q_max).astype(np.uint32)
    a, b, c = (np.ascontiguousarray(v, np.uint32) for v in (ln, npx, ntl))
    fast = np.empty(n, np.uint32)
    exact = np.empty(n, np.uint32)
    rc = lib.fibar_debug_regulate(num, den, area, q_min, q_max, a.ctypes.data, b.ctypes.data, c.ctypes.data, n,
                                  fast.ctypes.data, exact.ctypes.data)
    _native.check(rc, "fibar_debug_regulate")
    assert np.array_equal(exact, want)          # the device's 64-bit reference agrees with numpy
    bad = np.nonzero(fast != want)[0]
    assert bad.size == 0, (bad[:5], ln[bad[:5]], npx[bad[:5]], ntl[bad[:5]], fast[bad[:5]], want[bad[:5]])
