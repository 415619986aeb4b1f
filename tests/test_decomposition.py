"""The kernel decomposition (links, speculative window, stale rule, blur
dependency rules, final pass) reproduces the reference exactly on the CPU.
Runs tests/decomposition_model.py (a loop-level model of csrc/) against the
reference-generated golden vectors."""

import numpy as np
import pytest

from conftest import golden_path
from decomposition_model import DecompositionModel
from test_oracle_golden import params_of


@pytest.mark.parametrize("name", ["tiny_on", "odd_on", "noblur_on", "uniform_on", "variant_on"])
def test_model_matches_reference(name):
    g = dict(np.load(golden_path(name)))
    geom, params = params_of(g)
    gain = g["gain"] if g["gain"].size else None
    P = int(g["packet"])
    m = DecompositionModel(geom.width, geom.height, params, gain=gain, regulate_every=int(g["regulate_every"]),
                           blur_enabled=bool(g["blur"]), batch_cap=P, chunk=32, warm=32)
    n = len(g["x"])
    for a in range(0, n, P):
        m.process(g["x"][a:a + P], g["y"][a:a + P], g["p"][a:a + P])
    assert np.array_equal(m.pbar, g["p_bar"])
    assert np.array_equal(m.l, g["l"])
    assert np.array_equal(m.qs(), g["qs"])
    assert np.array_equal(m.active_count(), g["active_count"])
    assert np.array_equal(m.tile_count(), g["tile_count"])
    qx, qy = m.ring_xy()
    assert np.array_equal(qx, g["qx"]) and np.array_equal(qy, g["qy"])
    sk = np.concatenate(m.stale_k_log)
    sj = np.concatenate(m.stale_j_log)
    keep = (g["x"] < geom.width) & (g["y"] < geom.height)
    xs, ys = g["x"][keep].astype(np.int64), g["y"][keep].astype(np.int64)
    assert np.array_equal(sj, g["stale_j"])
    assert np.array_equal(ys[sk] * geom.width + xs[sk], g["stale_pix"])
