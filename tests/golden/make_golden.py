"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container only (needs /root/reference; the GPU box does not
have it):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Every case feeds seeded inputs through the unmodified reference
(`fibar.pipeline.ReconstructionEngine`, `fibar.spatial.SpatialFilter`,
`fibar.event_io`, `fibar.core`) and stores inputs + outputs in
tests/golden/*.npz.  tests/test_oracle_golden.py pins the C oracle against
these files; tests/test_gpu_parity.py (engine) and tests/test_tools.py
(calibration counts, pixel traces) pin the CUDA path against them too.

    python tests/golden/make_golden.py            # every case
    python tests/golden/make_golden.py tools      # only tests/golden/tools.npz
"""

from __future__ import annotations

import io
import os
import sys
from fractions import Fraction

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from fibar import core as rcore  # noqa: E402
from fibar import event_io as rio  # noqa: E402
from fibar import pipeline as rpipe  # noqa: E402
from fibar import spatial as rspatial  # noqa: E402
from fibar import _kernels as rk  # noqa: E402
from fibar import calib as rcalib  # noqa: E402
from fibar import temporal as rtemporal  # noqa: E402

from paper_2510_20071_b200 import workloads  # noqa: E402


def _stream(kind, w, h, n, seed):
    g = rcore.SensorGeometry(w, h)
    if kind == "uniform":
        ev = workloads.uniform(w, h, n, seed)
    elif kind == "texture":
        ev = workloads.moving_texture(w, h, n, seed=seed, speed=300.0)
    elif kind == "noise_hot":
        ev = workloads.texture_noise_hot(w, h, n, seed=seed, speed=300.0)
    else:
        raise ValueError(kind)
    return g, ev


def _stale_log(geom, params, xs, ys, ps, regulate_every, gain):
    """Per-event blurred-pixel list from the reference's transparent SpatialFilter."""
    n = geom.n_pix
    p_bar = np.zeros(n, np.float32)
    l = np.zeros(n, np.float32)
    act = np.zeros(n, np.uint16)
    sf = rspatial.SpatialFilter(geom, params, regulate_every=regulate_every)
    use_gain = gain is not None
    g = np.ascontiguousarray(gain.reshape(-1), np.float32) if use_gain else np.ones(1, np.float32)
    f32 = np.float32
    j_list, pix_list = [], []
    for j in range(len(xs)):
        rk.temporal_chunk(xs[j:j + 1], ys[j:j + 1], ps[j:j + 1], geom.width, p_bar, l,
                          f32(params.alpha), f32(1.0 - params.alpha), f32(params.beta),
                          f32(params.half_one_plus_beta), g, use_gain)
        for (bx, by) in sf.on_event(l, act, int(xs[j]), int(ys[j])):
            j_list.append(j)
            pix_list.append(by * geom.width + bx)
    return np.array(j_list, np.int64), np.array(pix_list, np.int64), l


def engine_case(name, kind, w, h, n, seed, *, spatial=True, packet=None, tcut=40.0, fill=Fraction(1, 2),
                tile_side=2, q_min=None, q_max=None, regulate_every=1, blur=True, gain_seed=None, oob=0,
                stale_log=False, renders=("robust", "fixed")):
    geom, ev = _stream(kind, w, h, n, seed)
    x, y, p, t = ev.x.copy(), ev.y.copy(), ev.p.copy(), ev.t.copy()
    if oob:
        rng = np.random.default_rng(seed + 99)
        idx = rng.choice(n, oob, replace=False)
        x[idx[: oob // 2]] = w + rng.integers(0, 5, oob // 2)
        y[idx[oob // 2:]] = h + rng.integers(0, 5, oob - oob // 2)
    params = rcore.compute_params(tcut, fill, geom, tile_side=tile_side, q_min=q_min, q_max=q_max,
                                  spatial_enabled=spatial)
    gain = None
    if gain_seed is not None:
        gain = np.random.default_rng(gain_seed).uniform(0.5, 1.5, (h, w)).astype(np.float32)
    eng = rpipe.ReconstructionEngine(geom, params, threshold_map=gain, regulate_every=regulate_every,
                                     blur_enabled=blur)
    packet = packet or n
    cuts = list(range(0, n, packet)) + [n]
    for a, b in zip(cuts[:-1], cuts[1:]):
        eng.process_array(rcore.EventArray(t[a:b], x[a:b], y[a:b], p[a:b]))
    out = dict(
        kind=np.array(kind), width=w, height=h, seed=seed, spatial=spatial, packet=packet, tcut=tcut,
        fill_num=fill.numerator, fill_den=fill.denominator, tile_side=tile_side,
        q_min=params.q_min, q_max=params.q_max, regulate_every=regulate_every, blur=blur,
        t=t, x=x, y=y, p=p,
        gain=gain if gain is not None else np.zeros(0, np.float32),
        p_bar=eng.p_bar, l=eng.l, active_count=eng.active_count, tile_count=eng.tile_count,
        qx=eng.qx, qy=eng.qy, qs=eng.qs, digest=np.array(eng.state_digest()),
        event_count=eng.event_count, oob_dropped=eng.oob_dropped, last_t=eng.last_t,
        alpha=params.alpha, beta=params.beta,
    )
    for mode in renders:
        fr = eng.render(mode, 0.5 if mode == "fixed" else 1.0)
        out[f"render_{mode}"] = fr.pixels
        out[f"bounds_{mode}"] = np.array(fr.bounds)
        out[f"degenerate_{mode}"] = fr.degenerate
    if stale_log and spatial:
        keep = (x < w) & (y < h)
        sj, spix, l_sf = _stale_log(geom, params, x[keep], y[keep], p[keep], regulate_every, gain)
        if blur:
            assert np.array_equal(l_sf, eng.l), "SpatialFilter replay must match full_chunk"
        out["stale_j"] = sj
        out["stale_pix"] = spix
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: n={n} events={eng.event_count} blur={eng.blur_count} stale={eng.stale_count} "
          f"q={eng.q_target} range={eng.q_target_range_seen}")


def misc_cases():
    out = {}
    # coefficients at several cutoffs (core.py:97-115)
    tcuts = np.array([4.5, 10.0, 40.0, 100.0, 1000.0, 1e6])
    coef = np.array([rcore.cutoff_coefficients(tc) for tc in tcuts])
    out["tcuts"] = tcuts
    out["coef"] = coef
    # render edge cases (pipeline.py:247-269)
    g = rcore.SensorGeometry(8, 5)
    params = rcore.compute_params(40.0, Fraction(1, 2), g)
    rng = np.random.default_rng(5)
    grids = [
        np.zeros(40, np.float32),
        np.linspace(-1, 1, 40).astype(np.float32),
        rng.standard_normal(40).astype(np.float32),
        np.where(rng.random(40) < 0.5, -0.0, 0.0).astype(np.float32),
        np.concatenate([np.full(39, 0.25), [7.0]]).astype(np.float32),
        rng.standard_normal(40).astype(np.float32) * 1e-30,
    ]
    for i, grid in enumerate(grids):
        eng = rpipe.ReconstructionEngine(g, params)
        eng.l[:] = grid
        for mode, bound in (("robust", 1.0), ("fixed", 1.0), ("fixed", 0.3)):
            fr = eng.render(mode, bound)
            out[f"grid{i}"] = grid
            out[f"grid{i}_{mode}_{bound}_px"] = fr.pixels
            out[f"grid{i}_{mode}_{bound}_bounds"] = np.array(fr.bounds)
            out[f"grid{i}_{mode}_{bound}_deg"] = fr.degenerate
    # EVF1 round trip + decode (event_io.py:60-76, 143-182)
    geom, ev = _stream("uniform", 100, 60, 5000, 3)
    buf = io.BytesIO()
    rio.write_stream(geom, ev, buf)
    out["evf1"] = np.frombuffer(buf.getvalue(), np.uint8)
    _, blocks = rio.read_blocks(io.BytesIO(buf.getvalue()), block_events=1000)
    dec = rcore.EventArray.concatenate(list(blocks))
    out["evf1_t"], out["evf1_x"], out["evf1_y"], out["evf1_p"] = dec.t, dec.x, dec.y, dec.p
    np.savez_compressed(os.path.join(HERE, "misc.npz"), **out)
    print("misc: done")


def tools_cases():
    """Calibration feeder + single-pixel traces."""
    out = {}
    rng = np.random.default_rng(21)
    # traces: random polarities with long same-sign runs, two cutoffs, both dtypes
    ps = np.where(rng.random(6000) < 0.5, -1, 1).astype(np.int8)
    ps[1000:1600] = 1
    ps[3000:3300] = -1
    out["trace_ps"] = ps
    for tc in (40.0, 10.0):
        params = rcore.compute_params(tc, Fraction(1, 2), rcore.SensorGeometry(4, 4))
        for dt in (np.float32, np.float64):
            tr = rtemporal.stream_pixel(ps, params, dtype=dt)
            tag = f"{int(tc)}_{np.dtype(dt).name}"
            out[f"trace_pbar_{tag}"], out[f"trace_delta_{tag}"], out[f"trace_l_{tag}"] = tr.p_bar, tr.delta, tr.l
            out[f"trace_iir_{tag}"] = rtemporal.stream_pixel_iir(ps, params, dtype=dt)
        st = rtemporal.PixelState()
        seq = []
        for pol in ps[:50]:
            st, d = rtemporal.update_pixel(st, int(pol), params)
            seq.append((st.p_bar, st.l, d))
        out[f"update_{int(tc)}"] = np.array(seq)
        out[f"update_iir_{int(tc)}"] = np.array([rtemporal.update_pixel_iir(0.3, -0.2, a, b, params)
                                                 for a in (-1, 1) for b in (-1, 1)])
    out["thr_delta"] = np.array([0.5, -0.25, 1e-3])
    out["thr_c"] = np.array([1.5, 0.7, 3.0])
    out["thr_out"] = np.array([rtemporal.apply_threshold_map(d, c) for d, c in zip(out["thr_delta"], out["thr_c"])])
    # calibration: counts over several blocks of a hot-pixel stream, thresholds, histogram
    geom, ev = _stream("noise_hot", 60, 40, 30000, 9)
    blocks = [ev.slice(a, min(len(ev), a + 7000)) for a in range(0, len(ev), 7000)]
    n_on, n_off = rcalib.count_events(iter(blocks), geom)
    out["cal_t"], out["cal_x"], out["cal_y"], out["cal_p"] = ev.t, ev.x, ev.y, ev.p
    out["cal_w"], out["cal_h"] = np.int64(geom.width), np.int64(geom.height)
    out["cal_n_on"], out["cal_n_off"] = n_on, n_off
    for qtag, q in (("q01", 0.01), ("q0", 0.0), ("q20", 0.2)):
        tm = rcalib.estimate_thresholds(n_on, n_off, exclusion_quantile=q)
        out[f"cal_{qtag}_c"], out[f"cal_{qtag}_con"], out[f"cal_{qtag}_coff"] = tm.c_prime, tm.c_on_prime, tm.c_off_prime
        out[f"cal_{qtag}_excl"], out[f"cal_{qtag}_nbar"] = tm.excluded, np.float64(tm.n_bar_tot)
        out[f"cal_{qtag}_gain"] = tm.gain_grid()
        out[f"cal_{qtag}_hmean"] = np.float64(tm.harmonic_mean())
        edges, counts = rcalib.histogram(tm, "c_prime", bins=20)
        out[f"cal_{qtag}_hist_edges"], out[f"cal_{qtag}_hist_counts"] = edges, counts
        if qtag == "q01":
            path = "/tmp/_golden_map.csv"
            tm.save_csv(path)
            out[f"cal_{qtag}_csv"] = np.frombuffer(open(path, "rb").read(), np.uint8)
    # an event whose flat index y*W + x wraps into the next row still counts (x is not checked alone)
    wx = np.array([65, 3], np.uint16)
    wy = np.array([2, 39], np.uint16)
    w_on, w_off = rcalib.count_events(rcore.EventArray(np.arange(2, dtype=np.uint64), wx, wy,
                                                       np.array([1, -1], np.int8)), geom)
    out["wrap_x"], out["wrap_y"], out["wrap_on"], out["wrap_off"] = wx, wy, w_on, w_off
    np.savez_compressed(os.path.join(HERE, "tools.npz"), **out)
    print("tools: done")


def main():
    rk.warmup()
    engine_case("uniform_off", "uniform", 64, 48, 30000, 0, spatial=False, packet=7000)
    engine_case("uniform_on", "uniform", 64, 48, 30000, 1, packet=4000, stale_log=True)
    engine_case("texture_on", "texture", 96, 64, 40000, 2, packet=10000, stale_log=True)
    engine_case("texture_on_1pkt", "texture", 96, 64, 40000, 2, stale_log=True)
    engine_case("noise_hot_on", "noise_hot", 80, 60, 40000, 3, packet=3333, stale_log=True)
    engine_case("variant_on", "texture", 70, 45, 30000, 4, packet=5000, tile_side=3, fill=Fraction(2, 3),
                regulate_every=3, gain_seed=7, oob=200, q_min=64, stale_log=True)
    engine_case("noblur_on", "uniform", 40, 30, 20000, 5, packet=2500, blur=False, stale_log=True)
    engine_case("gain_off", "texture", 50, 40, 20000, 6, spatial=False, packet=1500, gain_seed=8, oob=50)
    engine_case("tiny_on", "uniform", 3, 2, 500, 7, packet=37, q_min=2, stale_log=True)
    engine_case("odd_on", "uniform", 17, 13, 8000, 8, packet=999, q_min=20, q_max=150, stale_log=True)
    misc_cases()
    tools_cases()


if __name__ == "__main__":
    if sys.argv[1:] == ["tools"]:
        rk.warmup()
        tools_cases()
    else:
        main()
