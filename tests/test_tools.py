"""Calibration feeder and single-pixel traces.

Golden vectors: tests/golden/tools.npz, produced by the reference itself
(tests/golden/make_golden.py tools).  CPU tests pin the oracle and the host
helpers against them; GPU tests pin the CUDA kernels (fibar_count_events,
fibar_pixel_trace[_iir]) bit-exactly against the goldens and the oracle.
"""

import os
from fractions import Fraction

import numpy as np
import pytest

from conftest import golden_path

TCUTS = (40.0, 10.0)
DTYPES = (np.float32, np.float64)


@pytest.fixture(scope="module")
def tools():
    return dict(np.load(golden_path("tools")))


def _params(tc):
    from paper_2510_20071_b200.core import SensorGeometry, compute_params
    return compute_params(tc, Fraction(1, 2), SensorGeometry(4, 4))


def _coef(params):
    return (params.alpha, 1.0 - params.alpha, params.beta, params.half_one_plus_beta)


def _coef_iir(params):
    a, b = params.alpha, params.beta
    return (a + b, a * b, 0.5 * a * (1.0 + b))


def _tag(tc, dt):
    return f"{int(tc)}_{np.dtype(dt).name}"


# ---------------------------------------------------------------- oracle pins

@pytest.mark.parametrize("tc", TCUTS)
@pytest.mark.parametrize("dt", DTYPES)
def test_oracle_trace_matches_reference(tools, tc, dt):
    from oracle import oracle as orc
    p = _params(tc)
    pb, d, l = orc.trace(tools["trace_ps"], _coef(p), dt)
    tag = _tag(tc, dt)
    assert np.array_equal(pb, tools[f"trace_pbar_{tag}"])
    assert np.array_equal(d, tools[f"trace_delta_{tag}"])
    assert np.array_equal(l, tools[f"trace_l_{tag}"])
    assert np.array_equal(orc.trace_iir(tools["trace_ps"], _coef_iir(p), dt), tools[f"trace_iir_{tag}"])


def test_oracle_counts_match_reference(tools):
    from oracle import oracle as orc
    w, h = int(tools["cal_w"]), int(tools["cal_h"])
    on, off = orc.count_events(tools["cal_x"], tools["cal_y"], tools["cal_p"], w, w * h)
    assert np.array_equal(on.reshape(h, w), tools["cal_n_on"])
    assert np.array_equal(off.reshape(h, w), tools["cal_n_off"])
    on, off = orc.count_events(tools["wrap_x"], tools["wrap_y"], np.array([1, -1], np.int8), w, w * h)
    assert np.array_equal(on.reshape(h, w), tools["wrap_on"]) and np.array_equal(off.reshape(h, w), tools["wrap_off"])


# ------------------------------------------------------- host-side helpers

@pytest.mark.parametrize("tc", TCUTS)
def test_scalar_updates_match_reference(tools, tc):
    from paper_2510_20071_b200 import temporal
    p = _params(tc)
    st = temporal.PixelState()
    got = []
    for pol in tools["trace_ps"][:50]:
        st, d = temporal.update_pixel(st, int(pol), p)
        got.append((st.p_bar, st.l, d))
    assert np.array_equal(np.array(got), tools[f"update_{int(tc)}"])
    iir = [temporal.update_pixel_iir(0.3, -0.2, a, b, p) for a in (-1, 1) for b in (-1, 1)]
    assert np.array_equal(np.array(iir), tools[f"update_iir_{int(tc)}"])


def test_threshold_scaling_and_errors(tools):
    from paper_2510_20071_b200 import temporal
    from paper_2510_20071_b200.errors import DataError
    got = [temporal.apply_threshold_map(d, c) for d, c in zip(tools["thr_delta"], tools["thr_c"])]
    assert np.array_equal(np.array(got), tools["thr_out"])
    with pytest.raises(DataError):
        temporal.apply_threshold_map(0.5, 0.0)
    with pytest.raises(DataError):
        temporal.update_pixel(temporal.PixelState(), 0, _params(40.0))


@pytest.mark.parametrize("qtag", ["q01", "q0", "q20"])
def test_gain_grid_matches_reference(tools, qtag):
    """ThresholdMap.gain_grid (calib.py:73-78) of the reference's own thresholds."""
    from paper_2510_20071_b200 import calib
    g = calib.gain_grid(tools[f"cal_{qtag}_c"])
    assert g.dtype == np.float32 and np.array_equal(g, tools[f"cal_{qtag}_gain"])


# ------------------------------------------------------------- CUDA kernels

@pytest.mark.gpu
@pytest.mark.parametrize("tc", TCUTS)
@pytest.mark.parametrize("dt", DTYPES)
def test_gpu_stream_pixel_matches_reference(tools, tc, dt):
    from paper_2510_20071_b200 import temporal
    p = _params(tc)
    tr = temporal.stream_pixel(tools["trace_ps"], p, dtype=dt)
    tag = _tag(tc, dt)
    assert tr.l.dtype == np.dtype(dt)
    assert np.array_equal(tr.p_bar, tools[f"trace_pbar_{tag}"])
    assert np.array_equal(tr.delta, tools[f"trace_delta_{tag}"])
    assert np.array_equal(tr.l, tools[f"trace_l_{tag}"])
    assert np.array_equal(temporal.stream_pixel_iir(tools["trace_ps"], p, dtype=dt), tools[f"trace_iir_{tag}"])


@pytest.mark.gpu
def test_gpu_stream_pixels_batch_matches_oracle():
    from oracle import oracle as orc
    from paper_2510_20071_b200 import temporal
    rng = np.random.default_rng(4)
    ps = np.where(rng.random((300, 2000)) < 0.6, 1, -1).astype(np.int8)
    p = _params(40.0)
    tr = temporal.stream_pixels(ps, p)
    iir = temporal.stream_pixels_iir(ps, p, dtype=np.float64)
    for r in (0, 17, 299):
        pb, d, l = orc.trace(ps[r], _coef(p))
        assert np.array_equal(tr.p_bar[r], pb) and np.array_equal(tr.delta[r], d) and np.array_equal(tr.l[r], l)
        assert np.array_equal(iir[r], orc.trace_iir(ps[r], _coef_iir(p), np.float64))
    assert temporal.stream_pixel([], p).l.size == 0


@pytest.mark.gpu
def test_gpu_count_events_matches_reference(tools):
    import torch
    from paper_2510_20071_b200 import calib
    from paper_2510_20071_b200.core import EventArray, SensorGeometry
    from paper_2510_20071_b200.pipeline import DeviceEventArray
    w, h = int(tools["cal_w"]), int(tools["cal_h"])
    geom = SensorGeometry(w, h)
    ev = EventArray(tools["cal_t"], tools["cal_x"], tools["cal_y"], tools["cal_p"])
    blocks = [ev.slice(a, min(len(ev), a + 7000)) for a in range(0, len(ev), 7000)]
    on, off = calib.count_events(iter(blocks), geom)
    assert on.dtype == np.int64 and np.array_equal(on, tools["cal_n_on"]) and np.array_equal(off, tools["cal_n_off"])
    dev = DeviceEventArray(torch.from_numpy(ev.x.view(np.int16)).cuda(), torch.from_numpy(ev.y.view(np.int16)).cuda(),
                           torch.from_numpy(ev.p).cuda())
    on_d, off_d = calib.count_events_device(dev, geom)
    assert np.array_equal(on_d.cpu().numpy(), tools["cal_n_on"])
    wrap = EventArray(np.arange(2, dtype=np.uint64), tools["wrap_x"], tools["wrap_y"], np.array([1, -1], np.int8))
    on, off = calib.count_events(wrap, geom)
    assert np.array_equal(on, tools["wrap_on"]) and np.array_equal(off, tools["wrap_off"])


@pytest.mark.gpu
def test_gpu_count_events_hot_stream_and_errors():
    from oracle import oracle as orc
    from paper_2510_20071_b200 import calib, workloads
    from paper_2510_20071_b200.core import EventArray, SensorGeometry
    from paper_2510_20071_b200.errors import DataError
    geom = SensorGeometry(320, 180)
    ev = workloads.make("texture_noise_hot", geom, 2_000_000, seed=5)
    on, off = calib.count_events(ev, geom)
    ron, roff = orc.count_events(ev.x, ev.y, ev.p, geom.width, geom.n_pix)
    assert np.array_equal(on.reshape(-1), ron) and np.array_equal(off.reshape(-1), roff)
    bad = EventArray(np.arange(3, dtype=np.uint64), np.array([1, 2, 3], np.uint16),
                     np.array([0, 180, 0], np.uint16), np.array([1, 1, -1], np.int8))
    with pytest.raises(DataError):
        calib.count_events(bad, geom)
    empty = EventArray(np.zeros(0, np.uint64), np.zeros(0, np.uint16), np.zeros(0, np.uint16), np.zeros(0, np.int8))
    on, off = calib.count_events([empty], geom)
    assert on.sum() == 0 and off.shape == (180, 320)


@pytest.mark.gpu
def test_gpu_gain_from_calibration_feeds_engine(tools):
    """GPU counts of the reference's calibration stream -> the reference's thresholds
    -> gain_grid -> engine threshold_map, against the oracle on a longer stream."""
    from oracle import oracle as orc
    from paper_2510_20071_b200 import calib, workloads
    from paper_2510_20071_b200.core import EventArray, SensorGeometry, compute_params
    from paper_2510_20071_b200.pipeline import ReconstructionEngine
    w, h = int(tools["cal_w"]), int(tools["cal_h"])
    geom = SensorGeometry(w, h)
    cal = EventArray(tools["cal_t"], tools["cal_x"], tools["cal_y"], tools["cal_p"])
    on, off = calib.count_events(cal, geom)
    assert np.array_equal(on, tools["cal_n_on"]) and np.array_equal(off, tools["cal_n_off"])
    gain = calib.gain_grid(tools["cal_q01_c"])
    ev = workloads.make("texture_noise_hot", geom, 200_000, seed=8)
    params = compute_params(40.0, Fraction(1, 2), geom)
    eng = ReconstructionEngine(geom, params, threshold_map=gain)
    ref = orc.OracleEngine(geom.width, geom.height, params, gain=gain)
    for a in range(0, len(ev), 25_000):
        b = min(len(ev), a + 25_000)
        eng.process_array(ev.slice(a, b))
        ref.process_array(ev.t[a:b], ev.x[a:b], ev.y[a:b], ev.p[a:b])
    assert np.array_equal(eng.l, ref.l) and np.array_equal(eng.p_bar, ref.p_bar)
