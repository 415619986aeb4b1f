"""Seeded synthetic event streams for the BASELINE.json configurations.

The reference's recordings are not available and
the reference's own generator (`fibar/synth.py`) has none of these scenes, so
these generators stand in for them.  Choices the BASELINE text leaves open
 are fixed here and repeated in DESIGN.md:

* config 1 (``uniform``): x ~ U{0..W-1}, y ~ U{0..H-1}, p = +-1 with
  probability 1/2, gaps ~ Exp(mean 1 us); integer timestamps
  t_k = t_{k-1} + max(1, round(gap_k)) so they increase strictly.  Draw order
  x, y, p, gaps from ``np.random.default_rng(seed)``.
* ``moving_texture``: N(0,1) white noise on a periodic H x W torus, Gaussian
  blurred with sigma = 3 px (in the Fourier domain) and **renormalised to unit
  standard deviation** (log-intensity).  The texture translates diagonally at
  ``speed`` px/s (equal x and y components).  Each pixel samples it bilinearly
  every ``step_px / speed`` seconds and emits one event per crossing of its
  reference level by +-``contrast``; crossing times are interpolated linearly
  inside the step; events in a step are ordered by time, ties by pixel index.
* ``texture_noise_hot`` (config 3): the texture stream plus 20 % noise
  events: half uniform-random pixels, half on 1 % "hot" pixels chosen
  uniformly, with Zipf(s=1.2) weights over hot-pixel ranks; noise polarities
  are fair coin flips and noise times uniform over the stream's span.

Timestamps never influence reconstructed state (only read-out splitting), so
these choices affect workload statistics (distinct pixels per packet, blurs per
event), not correctness.
"""

from __future__ import annotations

import numpy as np

from .core import EventArray, SensorGeometry


def uniform(width: int, height: int, n: int, seed: int = 0) -> EventArray:
    """BASELINE config 1 stream."""
    rng = np.random.default_rng(seed)
    x = rng.integers(0, width, n, dtype=np.uint16)
    y = rng.integers(0, height, n, dtype=np.uint16)
    p = np.where(rng.random(n) < 0.5, -1, 1).astype(np.int8)
    gaps = rng.exponential(1.0, n)
    steps = np.maximum(1, np.rint(gaps)).astype(np.uint64)
    t = np.cumsum(steps, dtype=np.uint64)
    return EventArray(t, x, y, p)


def _texture(width: int, height: int, sigma: float, rng) -> np.ndarray:
    noise = rng.standard_normal((height, width))
    fy = np.fft.fftfreq(height)[:, None]
    fx = np.fft.rfftfreq(width)[None, :]
    kern = np.exp(-2.0 * (np.pi ** 2) * (sigma ** 2) * (fx ** 2 + fy ** 2))
    tex = np.fft.irfft2(np.fft.rfft2(noise) * kern, s=(height, width))
    tex -= tex.mean()
    tex /= tex.std()
    return tex


def _bilinear_periodic(tex: np.ndarray, ox: float, oy: float) -> np.ndarray:
    """Texture shifted by (ox, oy) px, sampled at integer pixel centres."""
    h, w = tex.shape
    fx, ix = np.modf(-ox)
    fy, iy = np.modf(-oy)
    if fx < 0:
        fx += 1.0
        ix -= 1.0
    if fy < 0:
        fy += 1.0
        iy -= 1.0
    r0 = np.roll(tex, (-int(iy), -int(ix)), axis=(0, 1))
    r1 = np.roll(r0, -1, axis=1)
    r2 = np.roll(r0, -1, axis=0)
    r3 = np.roll(r2, -1, axis=1)
    return (1 - fy) * ((1 - fx) * r0 + fx * r1) + fy * ((1 - fx) * r2 + fx * r3)


def moving_texture(width: int, height: int, n: int, *, speed: float = 200.0, sigma: float = 3.0,
                   contrast: float = 0.2, step_px: float = 0.25, seed: int = 0) -> EventArray:
    """Translating random texture seen by an ideal log-crossing sensor (configs 2, 4, 5)."""
    rng = np.random.default_rng(seed)
    tex = _texture(width, height, sigma, rng)
    v = speed / np.sqrt(2.0)
    dt = step_px / speed
    ref = tex.copy()
    prev = tex.copy()
    pix = np.arange(width * height, dtype=np.int64)
    ts, xs, ys, ps = [], [], [], []
    total = 0
    k = 0
    while total < n:
        k += 1
        cur = _bilinear_periodic(tex, v * dt * k, v * dt * k)
        d = cur - ref
        cnt = np.floor(np.abs(d) / contrast).astype(np.int64).reshape(-1)
        hit = np.nonzero(cnt)[0]
        if hit.size:
            c = cnt[hit]
            sgn = np.sign(d.reshape(-1)[hit])
            rep = np.repeat(np.arange(hit.size), c)
            lvl_idx = np.arange(rep.size) - np.repeat(np.cumsum(c) - c, c) + 1
            base = ref.reshape(-1)[hit][rep]
            lvl = base + sgn[rep] * lvl_idx * contrast
            p0 = prev.reshape(-1)[hit][rep]
            p1 = cur.reshape(-1)[hit][rep]
            den = np.where(p1 != p0, p1 - p0, 1.0)
            frac = np.clip((lvl - p0) / den, 0.0, 1.0)
            tev = (k - 1 + frac) * dt
            order = np.lexsort((pix[hit][rep], tev))
            pid = pix[hit][rep][order]
            ts.append(np.floor(tev[order] * 1e6).astype(np.uint64))
            xs.append((pid % width).astype(np.uint16))
            ys.append((pid // width).astype(np.uint16))
            ps.append(np.where(sgn[rep][order] > 0, 1, -1).astype(np.int8))
            total += pid.size
            r = ref.reshape(-1)
            r[hit] += sgn * c * contrast
        prev = cur
    t = np.concatenate(ts)[:n]
    return EventArray(t, np.concatenate(xs)[:n], np.concatenate(ys)[:n], np.concatenate(ps)[:n])


def texture_noise_hot(width: int, height: int, n: int, *, noise_frac: float = 0.2, hot_pixel_frac: float = 0.01,
                      zipf_s: float = 1.2, seed: int = 0, **texture_kw) -> EventArray:
    """BASELINE config 3 stream: texture + uniform noise + Zipf hot pixels."""
    n_noise = int(round(n * noise_frac))
    n_tex = n - n_noise
    tex = moving_texture(width, height, n_tex, seed=seed, **texture_kw)
    rng = np.random.default_rng(seed + 1)
    n_uni = n_noise // 2
    n_hot = n_noise - n_uni
    npix = width * height
    uni = rng.integers(0, npix, n_uni)
    n_hot_pix = max(1, int(round(npix * hot_pixel_frac)))
    hot_pix = rng.choice(npix, n_hot_pix, replace=False)
    w = 1.0 / np.arange(1, n_hot_pix + 1) ** zipf_s
    hot = hot_pix[rng.choice(n_hot_pix, n_hot, p=w / w.sum())]
    noise_pix = np.concatenate([uni, hot])
    t_lo = int(tex.t[0]) if len(tex) else 0
    t_hi = int(tex.t[-1]) if len(tex) else 1
    noise_t = rng.integers(t_lo, t_hi + 1, n_noise).astype(np.uint64)
    noise_p = np.where(rng.random(n_noise) < 0.5, -1, 1).astype(np.int8)
    t = np.concatenate([tex.t, noise_t])
    pid = np.concatenate([tex.y.astype(np.int64) * width + tex.x, noise_pix])
    p = np.concatenate([tex.p, noise_p])
    order = np.argsort(t, kind="stable")
    pid = pid[order]
    return EventArray(t[order], (pid % width).astype(np.uint16), (pid // width).astype(np.uint16), p[order])


def packets(events: EventArray, size: int):
    """Split a stream into consecutive packets of ``size`` events."""
    for s in range(0, len(events), size):
        yield events.slice(s, min(s + size, len(events)))


CONFIGS = {
    1: dict(geometry=SensorGeometry(346, 260), n=1_000_000, spatial=False, packet=1_000_000, kind="uniform"),
    2: dict(geometry=SensorGeometry(640, 480), n=10_000_000, spatial=True, packet=10_000, kind="texture"),
    3: dict(geometry=SensorGeometry(1280, 720), n=100_000_000, spatial=True, packet=100_000, kind="texture_noise_hot",
            readout="packet"),
    4: dict(geometry=SensorGeometry(1280, 720), n=50_000_000, spatial=None, packet=None, kind="texture"),
    5: dict(geometry=SensorGeometry(2560, 1440), n=1_000_000_000, spatial=True, packet=1_000_000, kind="texture",
            speed=1000.0),
}


GENERATOR_VERSION = 1   # bump when a generator's output changes (invalidates cached streams)


def make_cached(kind: str, geometry: SensorGeometry, n: int, seed: int = 0, cache_dir: str | None = None,
                **kw) -> EventArray:
    """``make`` with an on-disk copy of the stream (default ``$FIBAR_STREAM_CACHE``
    or /tmp/fibar_streams), so the bench's two arms on one box generate a
    100M-event stream once.  A cache miss or an unreadable file regenerates;
    the stream itself never depends on the cache."""
    import hashlib
    import os
    cache_dir = cache_dir or os.environ.get("FIBAR_STREAM_CACHE", "/tmp/fibar_streams")
    key = hashlib.sha256(repr((GENERATOR_VERSION, kind, geometry.width, geometry.height, n, seed,
                               sorted(kw.items()))).encode()).hexdigest()[:24]
    path = os.path.join(cache_dir, f"{kind}_{geometry.width}x{geometry.height}_{n}_{seed}_{key}.npz")
    try:
        with np.load(path) as z:
            ev = EventArray(z["t"], z["x"], z["y"], z["p"])
        if len(ev) == n:
            return ev
    except (OSError, ValueError, KeyError):
        pass
    ev = make(kind, geometry, n, seed=seed, **kw)
    try:
        os.makedirs(cache_dir, exist_ok=True)
        tmp = path + f".{os.getpid()}.tmp.npz"
        np.savez(tmp, t=ev.t, x=ev.x, y=ev.y, p=ev.p)
        os.replace(tmp, path)
    except OSError:
        pass
    return ev


def make(kind: str, geometry: SensorGeometry, n: int, seed: int = 0, **kw) -> EventArray:
    if kind == "uniform":
        return uniform(geometry.width, geometry.height, n, seed)
    if kind == "texture":
        return moving_texture(geometry.width, geometry.height, n, seed=seed, **kw)
    if kind == "texture_noise_hot":
        return texture_noise_hot(geometry.width, geometry.height, n, seed=seed, **kw)
    raise ValueError(f"unknown workload kind {kind!r}")
