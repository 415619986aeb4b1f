"""ctypes front end of the CPU oracle (oracle/fibar_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs as the *checker*.  The
product package never imports this module.

``OracleEngine`` restates the reference ``ReconstructionEngine``
(`fibar/pipeline.py:63-269`): same state arrays (p_bar, l, active_count,
tile_count, ring qx/qy, qs[10]), same OOB handling and counters, and it drives
the C restatements of ``_temporal_chunk`` / ``_full_chunk`` / ``render``.
Parity of the restatement against the reference itself is pinned by
tests/test_oracle_golden.py using tests/golden/*.npz.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libfibar_oracle.so")

QS_HEAD, QS_LEN, QS_TARGET, QS_NPIX, QS_NTILES, QS_BLUR, QS_STALE, QS_QTMIN, QS_QTMAX, QS_EVCTR = range(10)
QS_SIZE = 10

_lib = None


def build() -> str:
    """Compile the oracle with its Makefile (gcc, no GPU needed)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(os.path.join(HERE, "fibar_oracle.c")):
        build()
    L = C.CDLL(LIB_PATH)
    P = C.c_void_p
    i64, f32, f64, i32 = C.c_int64, C.c_float, C.c_double, C.c_int
    L.oracle_temporal_chunk.argtypes = [P, P, P, i64, i64, P, P, f32, f32, f32, f32, P, i32]
    L.oracle_temporal_chunk.restype = None
    L.oracle_full_chunk.argtypes = (
        [P, P, P, i64, i64, i64, i64, i64, i64, P, P, P, P, P, P, i64, P, f32, f32, f32, f32, P, i32]
        + [i64, i64, i64, i64, i32, i64, i64, P, P, i64, P]
    )
    L.oracle_full_chunk.restype = None
    L.oracle_blur_at.argtypes = [P, i64, i64, i64, i64]
    L.oracle_blur_at.restype = f32
    L.oracle_render.argtypes = [P, i64, i32, f64, P, P, P]
    L.oracle_render.restype = i32
    L.oracle_decode_evf1.argtypes = [P, i64, i64, i64, C.c_uint64, P, P, P, P]
    L.oracle_trace_f32.argtypes = [P, i64, f32, f32, f32, f32, P, P, P, P]
    L.oracle_trace_f64.argtypes = [P, i64, f64, f64, f64, f64, P, P, P, P]
    L.oracle_trace_iir_f32.argtypes = [P, i64, f32, f32, f32, P, P]
    L.oracle_trace_iir_f64.argtypes = [P, i64, f64, f64, f64, P, P]
    L.oracle_count_events.argtypes = [P, P, P, i64, i64, i64, P, P]
    L.oracle_count_events.restype = i64
    L.oracle_decode_evf1.restype = i64
    _lib = L
    return L


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def render(l: np.ndarray, scale_mode: str = "robust", fixed_bound: float = 1.0):
    """(uint8 pixels, (lo, hi), degenerate) exactly as pipeline.py:247-269."""
    lf = np.ascontiguousarray(l, dtype=np.float32).reshape(-1)
    out = np.empty(lf.size, np.uint8)
    bounds = np.zeros(2, np.float64)
    deg = C.c_int(0)
    mode = {"robust": 0, "fixed": 1}.get(scale_mode, -1)
    rc = lib().oracle_render(_p(lf), lf.size, mode, float(fixed_bound), _p(out), _p(bounds), C.byref(deg))
    if rc != 0:
        raise ValueError(f"oracle render rejected mode={scale_mode!r} bound={fixed_bound}")
    return out.reshape(np.shape(l)), (float(bounds[0]), float(bounds[1])), bool(deg.value)


def decode_evf1(raw: bytes, width: int, height: int, t_base: int = 0):
    """Decode a whole number of EVF1 records; returns (t, x, y, p) or raises IndexError(first bad)."""
    buf = np.frombuffer(raw, np.uint8)
    n = buf.size // 8
    t = np.empty(n, np.uint64)
    x = np.empty(n, np.uint16)
    y = np.empty(n, np.uint16)
    p = np.empty(n, np.int8)
    bad = lib().oracle_decode_evf1(_p(buf), n, width, height, t_base, _p(t), _p(x), _p(y), _p(p))
    if bad >= 0:
        raise IndexError(int(bad))
    return t, x, y, p


def trace(ps, coef, dtype=np.float32):
    """Two-stage single-pixel trajectory (_kernels.py:219-233); coef = (a, 1-a, b, (1+b)/2) as float64."""
    ps = np.ascontiguousarray(ps, np.int8)
    dt = np.dtype(dtype)
    out = [np.empty(ps.size, dt) for _ in range(3)]
    st = np.zeros(2, dt)
    fn = lib().oracle_trace_f32 if dt == np.float32 else lib().oracle_trace_f64
    fn(_p(ps), ps.size, *[float(dt.type(c)) for c in coef], _p(st), _p(out[0]), _p(out[1]), _p(out[2]))
    return tuple(out)


def trace_iir(ps, coef, dtype=np.float32):
    """Combined recurrence (_kernels.py:236-249); coef = (a+b, a*b, a(1+b)/2) as float64."""
    ps = np.ascontiguousarray(ps, np.int8)
    dt = np.dtype(dtype)
    out = np.empty(ps.size, dt)
    st = np.zeros(3, dt)
    fn = lib().oracle_trace_iir_f32 if dt == np.float32 else lib().oracle_trace_iir_f64
    fn(_p(ps), ps.size, *[float(dt.type(c)) for c in coef], _p(st), _p(out))
    return out


def count_events(x, y, p, width: int, n_pix: int):
    """(n_on, n_off) flat int64 counts (calib.py:26-45) or raises IndexError(first bad event)."""
    x = np.ascontiguousarray(x, np.uint16)
    y = np.ascontiguousarray(y, np.uint16)
    p = np.ascontiguousarray(p, np.int8)
    on = np.zeros(n_pix, np.int64)
    off = np.zeros(n_pix, np.int64)
    bad = lib().oracle_count_events(_p(x), _p(y), _p(p), x.size, width, n_pix, _p(on), _p(off))
    if bad >= 0:
        raise IndexError(int(bad))
    return on, off


class OracleEngine:
    """CPU restatement of the reference engine (single thread, strict float32)."""

    def __init__(self, width: int, height: int, params, *, gain=None, regulate_every: int = 1,
                 blur_enabled: bool = True, record_stale: bool = False):
        self.width, self.height = int(width), int(height)
        n = self.width * self.height
        self.params = params
        self.regulate_every = int(regulate_every)
        self.blur_enabled = bool(blur_enabled)
        self.p_bar = np.zeros(n, np.float32)
        self.l = np.zeros(n, np.float32)
        self.active_count = np.zeros(n, np.uint16)
        self.tile_side = params.tile_side
        self.tiles_x = -(-self.width // self.tile_side)
        tiles_y = -(-self.height // self.tile_side)
        self.tile_count = np.zeros(self.tiles_x * tiles_y, np.uint8)
        self.qcap = n + 1
        self.qx = np.zeros(self.qcap, np.uint16)
        self.qy = np.zeros(self.qcap, np.uint16)
        self.qs = np.zeros(QS_SIZE, np.int64)
        q0 = min(max(n // 16, params.q_min), params.q_max)
        self.qs[QS_TARGET] = q0
        self.qs[QS_QTMIN] = q0
        self.qs[QS_QTMAX] = q0
        if gain is not None:
            self.gain = np.ascontiguousarray(np.asarray(gain, np.float32).reshape(-1))
            self.use_gain = 1
        else:
            self.gain = np.ones(1, np.float32)
            self.use_gain = 0
        self.alpha32 = np.float32(params.alpha)
        self.one_m_alpha32 = np.float32(1.0 - params.alpha)
        self.beta32 = np.float32(params.beta)
        self.half_1p_beta32 = np.float32(params.half_one_plus_beta)
        self.event_count = 0
        self.oob_dropped = 0
        self.last_t = None
        self.record_stale = record_stale
        self.stale_k: list[np.ndarray] = []
        self.stale_j: list[np.ndarray] = []

    def process_array(self, t, x, y, p) -> None:
        x = np.ascontiguousarray(x, np.uint16)
        y = np.ascontiguousarray(y, np.uint16)
        p = np.ascontiguousarray(p, np.int8)
        t = np.ascontiguousarray(t, np.uint64)
        if not len(x):
            return
        oob = (x >= self.width) | (y >= self.height)
        if oob.any():
            keep = ~oob
            self.oob_dropped += int(oob.sum())
            x, y, p, t = x[keep], y[keep], p[keep], t[keep]
            if not len(x):
                return
        L = lib()
        if self.params.spatial_enabled:
            n = len(x)
            cap = n * 40 + 1024 if self.record_stale else 0
            sk = np.empty(cap, np.int64)
            sj = np.empty(cap, np.int64)
            ns = C.c_int64(0)
            L.oracle_full_chunk(
                _p(x), _p(y), _p(p), n, self.width, self.height, self.tiles_x, self.tile_side,
                self.tile_side * self.tile_side, _p(self.p_bar), _p(self.l), _p(self.active_count),
                _p(self.tile_count), _p(self.qx), _p(self.qy), self.qcap, _p(self.qs),
                self.alpha32, self.one_m_alpha32, self.beta32, self.half_1p_beta32, _p(self.gain), self.use_gain,
                self.params.fill_ratio_target.numerator, self.params.fill_ratio_target.denominator,
                self.params.q_min, self.params.q_max, int(self.blur_enabled), self.regulate_every,
                self.event_count, _p(sk) if cap else None, _p(sj) if cap else None, cap, C.byref(ns),
            )
            if self.record_stale:
                if ns.value > cap:
                    raise RuntimeError("stale log overflow")
                self.stale_k.append(sk[: ns.value].copy())
                self.stale_j.append(sj[: ns.value].copy())
        else:
            L.oracle_temporal_chunk(
                _p(x), _p(y), _p(p), len(x), self.width, _p(self.p_bar), _p(self.l),
                self.alpha32, self.one_m_alpha32, self.beta32, self.half_1p_beta32, _p(self.gain), self.use_gain,
            )
        self.event_count += len(x)
        self.last_t = int(t[-1])

    def render(self, scale_mode: str = "robust", fixed_bound: float = 1.0):
        return render(self.l.reshape(self.height, self.width), scale_mode, fixed_bound)

    def stale_log(self):
        if not self.stale_k:
            return np.zeros(0, np.int64), np.zeros(0, np.int64)
        return np.concatenate(self.stale_k), np.concatenate(self.stale_j)

    def state_digest(self) -> str:
        h = hashlib.sha256()
        for a in (self.p_bar, self.l, self.active_count, self.tile_count, self.qx, self.qy, self.qs):
            h.update(a.tobytes())
        return h.hexdigest()
