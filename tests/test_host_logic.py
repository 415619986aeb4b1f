"""Host-side logic that needs no GPU: parameter validation, workloads, run() splitting."""

from fractions import Fraction

import numpy as np
import pytest

from paper_2510_20071_b200 import workloads
from paper_2510_20071_b200.core import EventArray, SensorGeometry, compute_params, cutoff_coefficients
from paper_2510_20071_b200.errors import ConfigError, DataError, FibarError, TruncationError, raise_for_status
from paper_2510_20071_b200 import pipeline


def test_compute_params_validation_mirrors_reference():
    g = SensorGeometry(10, 10)
    with pytest.raises(ConfigError):
        compute_params(4.0, geometry=g)
    with pytest.raises(ConfigError):
        compute_params(40.0, Fraction(1, 8), g)
    with pytest.raises(ConfigError):
        compute_params(40.0, geometry=g, q_max=101)
    with pytest.raises(ConfigError):
        compute_params(40.0, geometry=g, tile_side=1)
    p = compute_params(40.0, 0.5, g)
    assert p.fill_ratio_target == Fraction(1, 2) and p.q_min == 100 and p.q_max == 100
    p = compute_params(40.0, geometry=SensorGeometry(640, 480))
    assert p.q_min == 256 and p.q_max == 307200
    w, a, b = cutoff_coefficients(40.0)
    assert np.float32(a) == np.float32(0.8540807) and np.float32(b) == np.float32(0.8549112)


def test_engine_validates_before_touching_device():
    g = SensorGeometry(8, 8)
    p = compute_params(40.0, geometry=g)
    with pytest.raises(ConfigError):
        pipeline.ReconstructionEngine(g, p, regulate_every=0)
    with pytest.raises(ConfigError):
        pipeline.ReconstructionEngine(g, p, threshold_map=np.ones((3, 3)))
    with pytest.raises(DataError):
        pipeline.ReconstructionEngine(g, p, threshold_map=np.zeros((8, 8)))


def test_status_codes_map_to_reference_exceptions():
    for code, cls in ((1, ConfigError), (2, DataError)):
        with pytest.raises(cls):
            raise_for_status(code, "x")
    raise_for_status(0, "x")
    assert issubclass(TruncationError, FibarError)


def test_workloads_are_seeded_and_ordered():
    a = workloads.uniform(346, 260, 10000, 0)
    b = workloads.uniform(346, 260, 10000, 0)
    assert np.array_equal(a.x, b.x) and np.array_equal(a.t, b.t)
    assert np.all(np.diff(a.t.astype(np.int64)) >= 1)
    t = workloads.moving_texture(64, 48, 20000, seed=1)
    assert len(t) == 20000 and t.x.max() < 64 and t.y.max() < 48
    assert np.all(np.diff(t.t.astype(np.int64)) >= 0) and set(np.unique(t.p)) <= {-1, 1}
    h = workloads.texture_noise_hot(64, 48, 20000, seed=1)
    assert len(h) == 20000 and np.all(np.diff(h.t.astype(np.int64)) >= 0)


class StubEngine:
    """Records what run() feeds and when it renders (no GPU)."""

    def __init__(self):
        self.seen = []
        self.frames = []
        self.qs = np.zeros(10, np.int64)

    def process_array(self, blk):
        self.seen.append(blk.t.copy())

    def render(self, mode, bound, readout_time=0):
        done = np.concatenate(self.seen) if self.seen else np.zeros(0, np.uint64)
        self.frames.append((readout_time, done.size, int(done.max()) if done.size else -1))
        return pipeline.Frame(np.zeros((1, 1), np.uint8), readout_time, mode, (0.0, 1.0))

    def fill_ratio(self):
        return None

    def _counters(self):
        return sum(len(s) for s in self.seen), 0

    @property
    def blur_count(self):
        return 0


def test_run_reads_out_events_strictly_before_each_time():
    ev = workloads.uniform(32, 32, 5000, 3)
    blocks = list(workloads.packets(ev, 700))
    eng = StubEngine()
    res = pipeline.run(eng, blocks, fps=400.0)
    period = 1e6 / 400.0
    for k, (r, count, tmax) in enumerate(eng.frames, start=1):
        assert r == int(k * period)
        assert count == int(np.searchsorted(ev.t, k * period, side="left"))
        assert tmax < k * period
    assert res.frames_emitted == len(eng.frames) and res.events_processed == 5000


def test_run_explicit_times_after_end_render_final_state():
    ev = workloads.uniform(16, 16, 1000, 4)
    eng = StubEngine()
    pipeline.run(eng, [ev], readout_times=[10, 10, int(ev.t[-1]) + 5, int(ev.t[-1]) + 99])
    assert [f[0] for f in eng.frames] == [10, 10, int(ev.t[-1]) + 5, int(ev.t[-1]) + 99]
    assert eng.frames[-1][1] == 1000
    with pytest.raises(ConfigError):
        pipeline.run(eng, [ev], readout_times=[5, 3])
    with pytest.raises(ConfigError):
        pipeline.run(eng, [ev], fps=0)


def test_pgm_round_trip(tmp_path):
    f = pipeline.Frame(np.arange(12, dtype=np.uint8).reshape(3, 4), 0, "robust", (0.0, 1.0))
    pipeline.write_pgm(f, tmp_path / "a.pgm")
    assert np.array_equal(pipeline.read_pgm(tmp_path / "a.pgm"), f.pixels)


def test_event_array_coercion():
    ea = EventArray([1, 2], [3, 4], [5, 6], [1, -1])
    assert ea.t.dtype == np.uint64 and ea.x.dtype == np.uint16 and ea.p.dtype == np.int8
    with pytest.raises(ConfigError):
        EventArray([1], [1, 2], [1], [1])
