"""Pin the C oracle (oracle/fibar_oracle.c) against golden vectors produced by
running the reference itself (tests/golden/make_golden.py)."""

from fractions import Fraction

import numpy as np
import pytest

from conftest import golden_path
from oracle import oracle as orc
from paper_2510_20071_b200.core import compute_params, SensorGeometry, cutoff_coefficients


def params_of(g):
    geom = SensorGeometry(int(g["width"]), int(g["height"]))
    return geom, compute_params(float(g["tcut"]), Fraction(int(g["fill_num"]), int(g["fill_den"])), geom,
                                tile_side=int(g["tile_side"]), q_min=int(g["q_min"]), q_max=int(g["q_max"]),
                                spatial_enabled=bool(g["spatial"]))


def run_oracle(g, record_stale=False):
    geom, params = params_of(g)
    gain = g["gain"] if g["gain"].size else None
    eng = orc.OracleEngine(geom.width, geom.height, params, gain=gain,
                           regulate_every=int(g["regulate_every"]), blur_enabled=bool(g["blur"]),
                           record_stale=record_stale)
    n = len(g["x"])
    P = int(g["packet"])
    for a in range(0, n, P):
        b = min(n, a + P)
        eng.process_array(g["t"][a:b], g["x"][a:b], g["y"][a:b], g["p"][a:b])
    return eng


def test_oracle_engine_bit_exact(golden_case):
    name, g = golden_case
    eng = run_oracle(g, record_stale="stale_j" in g)
    for k in ("p_bar", "l", "active_count", "tile_count", "qx", "qy", "qs"):
        assert np.array_equal(getattr(eng, k), g[k]), (name, k)
    assert eng.state_digest() == str(g["digest"])
    assert eng.event_count == int(g["event_count"])
    assert eng.oob_dropped == int(g["oob_dropped"])
    if "stale_j" in g:
        sk, sj = eng.stale_log()
        W = int(g["width"])
        keep = (g["x"] < W) & (g["y"] < int(g["height"]))
        xs, ys = g["x"][keep].astype(np.int64), g["y"][keep].astype(np.int64)
        assert np.array_equal(sj, g["stale_j"])
        assert np.array_equal(ys[sk] * W + xs[sk], g["stale_pix"])


def test_oracle_render_matches_reference(golden_case):
    name, g = golden_case
    for mode in ("robust", "fixed"):
        px, bounds, deg = orc.render(g["l"].reshape(int(g["height"]), int(g["width"])), mode,
                                     0.5 if mode == "fixed" else 1.0)
        assert np.array_equal(px, g[f"render_{mode}"]), (name, mode)
        assert bounds == tuple(g[f"bounds_{mode}"])
        assert deg == bool(g[f"degenerate_{mode}"])


def test_oracle_render_edge_grids():
    m = dict(np.load(golden_path("misc")))
    for i in range(6):
        grid = m[f"grid{i}"]
        for mode, bound in (("robust", 1.0), ("fixed", 1.0), ("fixed", 0.3)):
            px, bounds, deg = orc.render(grid.reshape(5, 8), mode, bound)
            assert np.array_equal(px, m[f"grid{i}_{mode}_{bound}_px"]), (i, mode, bound)
            assert bounds == tuple(m[f"grid{i}_{mode}_{bound}_bounds"])
            assert deg == bool(m[f"grid{i}_{mode}_{bound}_deg"])


def test_oracle_decode_evf1():
    m = dict(np.load(golden_path("misc")))
    raw = m["evf1"].tobytes()
    t, x, y, p = orc.decode_evf1(raw[16:], 100, 60)
    assert np.array_equal(t, m["evf1_t"]) and np.array_equal(x, m["evf1_x"])
    assert np.array_equal(y, m["evf1_y"]) and np.array_equal(p, m["evf1_p"])
    with pytest.raises(IndexError):
        orc.decode_evf1(raw[16:], 100, 10)


def test_coefficients_match_reference():
    m = dict(np.load(golden_path("misc")))
    for tc, (w, a, b) in zip(m["tcuts"], m["coef"]):
        assert cutoff_coefficients(float(tc)) == (w, a, b)


def test_spec_known_answers():
    # SPEC.md:226 update_pixel, :312 regulate, :322 blur of centre 16 -> 4, :381 fixed render
    lib = orc.lib()
    l = np.zeros(9, np.float32)
    l[4] = 16.0
    assert lib.oracle_blur_at(l.ctypes.data, 3, 3, 1, 1) == 4.0
    px, b, d = orc.render(np.array([[-1.0, 0.0, 1.0]], np.float32), "fixed", 1.0)
    assert px.tolist() == [[0, 128, 255]] and b == (-1.0, 1.0) and not d
