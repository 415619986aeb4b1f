"""CUDA read-out (k_readout, one cooperative kernel) against the reference's
render() (pipeline.py:247-269): the reference-generated edge grids in
golden/misc.npz and seeded grids checked against the C oracle (pinned to the
reference by tests/test_oracle_golden.py).  Bit-exact: pixels, bounds
(including the sign of zero) and the degenerate flag."""

import math

import numpy as np
import pytest

from conftest import golden_path

pytestmark = pytest.mark.gpu


def _render(grid, mode, bound):
    import torch
    from paper_2510_20071_b200.pipeline import render_grid
    return render_grid(torch.from_numpy(np.ascontiguousarray(grid, np.float32)).cuda(), mode, bound)


def _same_bounds(a, b):
    return all(x == y and math.copysign(1.0, x) == math.copysign(1.0, y) for x, y in zip(a, b))


def test_edge_grids_match_reference():
    m = dict(np.load(golden_path("misc")))
    for i in range(6):
        grid = m[f"grid{i}"].reshape(5, 8)
        for mode, bound in (("robust", 1.0), ("fixed", 1.0), ("fixed", 0.3)):
            fr = _render(grid, mode, bound)
            assert np.array_equal(fr.pixels, m[f"grid{i}_{mode}_{bound}_px"]), (i, mode, bound)
            assert _same_bounds(fr.bounds, tuple(m[f"grid{i}_{mode}_{bound}_bounds"])), (i, mode, bound, fr.bounds)
            assert fr.degenerate == bool(m[f"grid{i}_{mode}_{bound}_deg"]), (i, mode, bound)


def _grids():
    rng = np.random.default_rng(11)
    yield "laplace_720p", rng.laplace(0, 0.05, (720, 1280))
    yield "normal_vga", rng.standard_normal((480, 640)) * 1e-3
    yield "few_levels", rng.integers(-3, 4, (300, 301)) * 0.125          # heavy ties
    z = rng.laplace(0, 1, (257, 263))
    z[rng.random(z.shape) < 0.6] = 0.0
    z[rng.random(z.shape) < 0.3] *= -1.0                                 # +0/-0 mix with tails
    yield "signed_zeros", z
    yield "tiny", np.array([[0.5, -0.25], [1.0, 3.0]])
    yield "odd_len", rng.standard_normal(1001).reshape(7, 143)
    yield "big_2560x1440", rng.laplace(0, 0.02, (1440, 2560))
    yield "huge_dynamic", rng.standard_normal((333, 999)) * np.exp(rng.uniform(-60, 60, (333, 999)))


@pytest.mark.parametrize("name,grid", list(_grids()), ids=lambda v: v if isinstance(v, str) else "")
def test_seeded_grids_match_oracle(name, grid):
    from oracle import oracle as orc
    g32 = np.ascontiguousarray(grid, np.float32)
    for mode, bound in (("robust", 1.0), ("fixed", 0.7)):
        px, bounds, deg = orc.render(g32, mode, bound)
        fr = _render(g32, mode, bound)
        assert np.array_equal(fr.pixels, px), (name, mode, int((fr.pixels != px).sum()))
        assert fr.bounds == bounds, (name, mode, fr.bounds, bounds)
        assert fr.degenerate == deg


def test_engine_readouts_repeat_exactly():
    """Back-to-back read-outs of one engine alternate the kernel's histogram
    sets; every frame must equal the oracle's."""
    from fractions import Fraction

    from oracle import oracle as orc
    from paper_2510_20071_b200 import workloads
    from paper_2510_20071_b200.core import SensorGeometry, compute_params
    from paper_2510_20071_b200.pipeline import ReconstructionEngine
    geom = SensorGeometry(320, 240)
    ev = workloads.moving_texture(320, 240, 60_000, seed=5)
    params = compute_params(40.0, Fraction(1, 2), geom, spatial_enabled=True)
    eng = ReconstructionEngine(geom, params)
    ref = orc.OracleEngine(320, 240, params)
    for a in range(0, len(ev), 7_500):
        blk = ev.slice(a, a + 7_500)
        eng.process_array(blk)
        ref.process_array(blk.t, blk.x, blk.y, blk.p)
        for mode in ("robust", "fixed", "robust"):
            fr = eng.render(mode, 0.4)
            px, bounds, deg = ref.render(mode, 0.4)
            assert np.array_equal(fr.pixels, px) and fr.bounds == bounds and fr.degenerate == deg, (a, mode)
    eng.close()
