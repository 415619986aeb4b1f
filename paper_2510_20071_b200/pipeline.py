"""Streaming reconstruction engine backed by the sm_100a kernels.

Drop-in for the reference's `fibar/pipeline.py`: same class and function
names, constructor arguments, properties, validation and exception types
(``ReconstructionEngine`` <- pipeline.py:63-269, ``run`` <- 640-712,
``Frame`` <- 359-375, ``write_pgm``/``read_pgm`` <- 590-610,
``RunResult`` <- 613-618).

Differences a caller can observe, all deliberate:

* State lives in device memory.  ``p_bar``, ``l``, ``active_count``,
  ``tile_count``, ``qx``, ``qy``, ``qs``, ``l_grid``, ``p_bar_grid`` return
  host *copies* (the reference returns views of its numpy state).
* ``process_array`` also accepts a :class:`DeviceEventArray` (torch CUDA
  tensors) so packets already in HBM never cross PCIe.
* Packets are coalesced on the device until the next read (render, a state
  property, or ``flush``); the reference's state is packet-size invariant, so
  results are identical (tests/test_gpu_parity.py checks it).
* ``render_device`` returns the frame as a CUDA uint8 tensor without a host copy.

Everything on the data path runs in the native library; this module only
validates arguments, moves packets, and maps status codes to exceptions.
"""

from __future__ import annotations

import collections
import ctypes as C
import hashlib
import logging
import math
import os
import weakref
from dataclasses import dataclass
from fractions import Fraction
from typing import Callable, Iterable, Iterator

import numpy as np

from . import _native
from .core import Event, EventArray, FilterParams, SensorGeometry
from .errors import ConfigError, DataError, OrderError

logger = logging.getLogger("fibar")

PERCENTILE_LO = 1.0
PERCENTILE_HI = 99.0
QS_HEAD, QS_LEN, QS_TARGET, QS_NPIX, QS_NTILES, QS_BLUR, QS_STALE, QS_QTMIN, QS_QTMAX, QS_EVCTR = range(10)
QS_SIZE = 10


@dataclass
class Frame:
    """8-bit grayscale rendering of the brightness grid."""

    pixels: np.ndarray
    readout_time: int
    scale_mode: str
    bounds: tuple[float, float]
    degenerate: bool = False

    @property
    def width(self) -> int:
        return self.pixels.shape[1]

    @property
    def height(self) -> int:
        return self.pixels.shape[0]


class AsyncFrame:
    """A read-out in flight (ReconstructionEngine.render_async)."""

    def __init__(self, out, meta, event, readout_time, scale_mode):
        self.out, self.meta, self.event = out, meta, event
        self.readout_time, self.scale_mode = readout_time, scale_mode

    def ready(self) -> bool:
        return self.event.query()

    def frame(self, copy: bool = True) -> Frame:
        """Wait for the read-out and return it as a Frame (a fresh array unless copy=False)."""
        self.event.synchronize()
        m = self.meta.cpu().numpy() if self.meta.is_cuda else self.meta.numpy()
        deg = int(np.array([m[2]], np.float64).view(np.int64)[0] & 0xFFFFFFFF)
        px = self.out.cpu().numpy() if self.out.is_cuda else self.out.numpy()
        return Frame(px.copy() if copy else px, self.readout_time, self.scale_mode, (float(m[0]), float(m[1])),
                     bool(deg))


@dataclass
class DeviceEventArray:
    """A packet whose columns are CUDA tensors (x, y: uint16/int16/int32; p: int8).

    ``t`` may stay on the host (it only feeds ``last_t`` and strict checks).
    """

    x: "object"
    y: "object"
    p: "object"
    t: np.ndarray | None = None

    def __len__(self) -> int:
        return int(self.x.shape[0])


def _torch():
    import torch

    return torch


def _addr(a: np.ndarray) -> int:
    """Data pointer of a numpy array (the buffer-protocol route is ~3x cheaper than .ctypes.data)."""
    try:
        return C.addressof(C.c_char.from_buffer(a))
    except (TypeError, ValueError, BufferError):
        return a.ctypes.data


class ReconstructionEngine:
    """Full reconstruction state for one sensor, resident on a CUDA device."""

    def __init__(
        self,
        geometry: SensorGeometry,
        params: FilterParams,
        threshold_map: np.ndarray | None = None,
        strict: bool = False,
        regulate_every: int = 1,
        blur_enabled: bool = True,
        *,
        batch_capacity: int | None = None,
        device=None,
        row_band: tuple[int, int] | None = None,
        halo_band: tuple[int, int, int] | None = None,
    ):
        if params.q_max > geometry.n_pix:
            raise ConfigError("q_max exceeds pixel count")
        if regulate_every < 1:
            raise ConfigError("regulate_every must be >= 1")
        self.geometry = geometry
        self.params = params
        self.strict = strict
        self.regulate_every = regulate_every
        self.blur_enabled = blur_enabled
        self.tiles_x = -(-geometry.width // params.tile_side)
        self.tiles_y = -(-geometry.height // params.tile_side)
        self.qcap = geometry.n_pix + 1

        gain_ptr = None
        self._gain = None
        if threshold_map is not None:
            gain = np.asarray(threshold_map, dtype=np.float32)
            if gain.shape != (geometry.height, geometry.width):
                raise ConfigError(
                    f"threshold map shape {gain.shape} does not match geometry {geometry.height}x{geometry.width}")
            if not np.all(np.isfinite(gain)) or np.any(gain <= 0):
                raise DataError("threshold map entries must be finite and positive")
            self._gain = np.ascontiguousarray(gain.reshape(-1))
            gain_ptr = self._gain.ctypes.data
        self._use_gain = self._gain is not None

        # float32 coefficients exactly as the reference casts them (pipeline.py:116-120)
        self._alpha32 = np.float32(params.alpha)
        self._one_m_alpha32 = np.float32(1.0 - params.alpha)
        self._beta32 = np.float32(params.beta)
        self._half_1p_beta32 = np.float32(params.half_one_plus_beta)

        torch = _torch()
        if not torch.cuda.is_available():
            from .errors import DeviceError
            raise DeviceError("ReconstructionEngine needs a CUDA device (no CPU fallback)")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._lib = _native.load()
        cfg = _native.FibarConfig(
            width=geometry.width, height=geometry.height, tile_side=params.tile_side,
            spatial_enabled=int(params.spatial_enabled), blur_enabled=int(blur_enabled), reserved0=0,
            regulate_every=regulate_every, fill_num=params.fill_ratio_target.numerator,
            fill_den=params.fill_ratio_target.denominator, q_min=params.q_min, q_max=params.q_max,
            alpha=float(self._alpha32), one_m_alpha=float(self._one_m_alpha32), beta=float(self._beta32),
            half_1p_beta=float(self._half_1p_beta32), gain=gain_ptr,
            batch_capacity=int(batch_capacity or 0),
            band_y0=int(row_band[0]) if row_band else 0,
            sensor_height=int(row_band[1]) if row_band else 0,
            halo_own_y0=int(halo_band[0]) if halo_band else 0,
            halo_own_y1=int(halo_band[1]) if halo_band else 0,
            halo_rows=int(halo_band[2]) if halo_band else 0,
        )
        handle = C.c_void_p()
        with torch.cuda.device(self.device):
            stream = torch.cuda.current_stream(self.device).cuda_stream
            _native.check(self._lib.fibar_create(C.byref(cfg), C.c_void_p(stream), C.byref(handle)), "fibar_create")
        self._h = handle
        self._stream_ptr = stream
        self.last_t: int | None = None
        self._held = collections.deque()   # device packets the native side still reads in place
        self._held_n = 0
        st = np.zeros(16, dtype=np.int64)
        _native.check(self._lib.fibar_stats(self._h, st.ctypes.data), "fibar_stats")
        self._bcap = int(st[7])
        self._release_at = self._bcap      # check the native pending count once this many are held
        self._dev_index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        self._raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        self._xy_ok = (torch.int16, getattr(torch, "uint16", torch.int16))
        self._i8 = torch.int8
        self._sat_warned = False

    # -- lifecycle -----------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.fibar_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _sync_stream(self) -> None:
        if self._raw_stream is not None:
            s = self._raw_stream(self._dev_index)
        else:
            s = _torch().cuda.current_stream(self.device).cuda_stream
        if s != self._stream_ptr:
            self._lib.fibar_set_stream(self._h, C.c_void_p(s))
            self._stream_ptr = s

    def reset(self) -> None:
        """Back to the freshly constructed state (zero filter, empty window)."""
        self._sync_stream()
        _native.check(self._lib.fibar_reset(self._h), "fibar_reset")
        self.last_t = None
        self._held.clear()
        self._held_n = 0
        self._release_at = self._bcap

    def flush(self) -> None:
        """Run coalesced packets now (asynchronous on the current stream)."""
        self._sync_stream()
        _native.check(self._lib.fibar_flush(self._h), "fibar_flush")
        self._release_held()

    # -- counters ------------------------------------------------------------
    def _counters(self) -> tuple[int, int]:
        ec, ob = C.c_int64(), C.c_int64()
        self._sync_stream()
        _native.check(self._lib.fibar_counters(self._h, C.byref(ec), C.byref(ob)), "fibar_counters")
        self._release_held()
        return ec.value, ob.value

    @property
    def event_count(self) -> int:
        return self._counters()[0]

    @property
    def oob_dropped(self) -> int:
        return self._counters()[1]

    @property
    def qs(self) -> np.ndarray:
        out = np.zeros(QS_SIZE, np.int64)
        self._sync_stream()
        _native.check(self._lib.fibar_read_qs(self._h, out.ctypes.data), "fibar_read_qs")
        self._release_held()
        return out

    def stats(self) -> dict:
        st = np.zeros(16, np.int64)
        self._sync_stream()
        _native.check(self._lib.fibar_stats(self._h, st.ctypes.data), "fibar_stats")
        keys = ("launches", "batches", "window_chunks", "window_reruns", "pops", "saturated", "events",
                "batch_capacity", "warm_pops", "coop_iters", "fix_rounds", "debug_window_bad")
        return dict(zip(keys, (int(v) for v in st)))

    @property
    def saturation_detected(self) -> bool:
        """True once the reference's u16 active_count (or u8 tile_count) could have
        saturated (_kernels.py:146-149).  From then on the reference's
        count-based staleness may differ from this engine's exact one; the flag is
        conservative (never missed, may fire up to one device batch early)."""
        return self.stats()["saturated"] > 0

    def _warn_saturation(self) -> None:
        if not self._sat_warned and self.params.spatial_enabled and self.saturation_detected:
            self._sat_warned = True
            logger.warning("active_count may have reached the reference's 65535 cap: results can differ "
                           "from the reference from here on (SURVEY H7)")

    def profile(self, enable: bool) -> None:
        """Per-kernel CUDA-event timing on/off (synchronises; never inside a timed region)."""
        self._sync_stream()
        _native.check(self._lib.fibar_profile(self._h, int(enable)), "fibar_profile")

    def profile_read(self) -> dict:
        """{kernel name: (total_ms, launches)} since profiling was enabled (synchronises, clears)."""
        m, L = 64, 32
        names = C.create_string_buffer(m * L)
        ms = np.zeros(m, np.float64)
        cnt = np.zeros(m, np.int64)
        k = C.c_int32(0)
        self._sync_stream()
        _native.check(self._lib.fibar_profile_read(self._h, m, names, L, ms.ctypes.data, cnt.ctypes.data, C.byref(k)),
                      "fibar_profile_read")
        raw = names.raw
        return {raw[i * L:(i + 1) * L].split(b"\0")[0].decode(): (float(ms[i]), int(cnt[i])) for i in range(k.value)}

    # -- state views (host copies) ---------------------------------------------
    def _read(self, **want) -> dict:
        n = self.geometry.n_pix
        bufs = {
            "p_bar": np.zeros(n, np.float32) if want.get("p_bar") else None,
            "l": np.zeros(n, np.float32) if want.get("l") else None,
            "active_count": np.zeros(n, np.uint16) if want.get("active_count") else None,
            "tile_count": np.zeros(self.tiles_x * self.tiles_y, np.uint8) if want.get("tile_count") else None,
            "qx": np.zeros(self.qcap, np.uint16) if want.get("qx") else None,
            "qy": np.zeros(self.qcap, np.uint16) if want.get("qy") else None,
        }
        ptr = [None if b is None else b.ctypes.data for b in bufs.values()]
        self._sync_stream()
        _native.check(self._lib.fibar_read_state(self._h, *ptr), "fibar_read_state")
        self._release_held()
        return {k: v for k, v in bufs.items() if v is not None}

    @property
    def p_bar(self) -> np.ndarray:
        return self._read(p_bar=True)["p_bar"]

    @property
    def l(self) -> np.ndarray:
        return self._read(l=True)["l"]

    @property
    def active_count(self) -> np.ndarray:
        return self._read(active_count=True)["active_count"]

    @property
    def tile_count(self) -> np.ndarray:
        return self._read(tile_count=True)["tile_count"]

    @property
    def qx(self) -> np.ndarray:
        return self._read(qx=True)["qx"]

    @property
    def qy(self) -> np.ndarray:
        return self._read(qy=True)["qy"]

    @property
    def l_grid(self) -> np.ndarray:
        return self.l.reshape(self.geometry.height, self.geometry.width)

    @property
    def p_bar_grid(self) -> np.ndarray:
        return self.p_bar.reshape(self.geometry.height, self.geometry.width)

    @property
    def queue_length(self) -> int:
        return int(self.qs[QS_LEN])

    @property
    def q_target(self) -> int:
        return int(self.qs[QS_TARGET])

    @property
    def q_target_range_seen(self) -> tuple[int, int]:
        q = self.qs
        return int(q[QS_QTMIN]), int(q[QS_QTMAX])

    @property
    def n_pix_act(self) -> int:
        return int(self.qs[QS_NPIX])

    @property
    def n_tiles_act(self) -> int:
        return int(self.qs[QS_NTILES])

    @property
    def blur_count(self) -> int:
        return int(self.qs[QS_BLUR])

    @property
    def stale_count(self) -> int:
        return int(self.qs[QS_STALE])

    def fill_ratio(self) -> Fraction | None:
        q = self.qs
        if q[QS_NTILES] < 1:
            return None
        return Fraction(int(q[QS_NPIX]), int(q[QS_NTILES]) * self.params.tile_area)

    def iap(self) -> np.ndarray:
        """Image of active pixels: per-pixel count of queued events."""
        return self.active_count.reshape(self.geometry.height, self.geometry.width)

    def state_bytes(self) -> int:
        """Bytes of the reference-layout state (pipeline.py:173-175), for parity with its report."""
        n = self.geometry.n_pix
        b = n * 4 * 2 + n * 2 + self.tiles_x * self.tiles_y + self.qcap * 4 + QS_SIZE * 8
        return b + (self._gain.nbytes if self._use_gain else 0)

    def state_arrays(self) -> dict:
        """All reference-layout state arrays as host copies (one synchronisation)."""
        d = self._read(p_bar=True, l=True, active_count=True, tile_count=True, qx=True, qy=True)
        d["qs"] = self.qs
        return d

    def stale_items(self) -> tuple[np.ndarray, np.ndarray]:
        """Stale episodes of the most recent device batch (runs pending packets
        first): (in-bounds event index, pixel) in pop order, the reference's
        per-event blurred-pixel list (spatial.py:165-207) for that batch."""
        cap = max(1024, self._bcap + self.geometry.n_pix)
        j = np.empty(cap, np.int64)
        pix = np.empty(cap, np.uint32)
        n = C.c_int64(0)
        self._sync_stream()
        _native.check(self._lib.fibar_debug_stale_items(self._h, j.ctypes.data, pix.ctypes.data, cap, C.byref(n)),
                      "fibar_debug_stale_items")
        return j[: n.value].copy(), pix[: n.value].astype(np.int64)

    def state_digest(self) -> str:
        d = self.state_arrays()
        h = hashlib.sha256()
        for k in ("p_bar", "l", "active_count", "tile_count", "qx", "qy", "qs"):
            h.update(d[k].tobytes())
        return h.hexdigest()

    # -- event intake --------------------------------------------------------
    def process(self, event: Event) -> None:
        """Apply one event (wraps the block path)."""
        self.process_array(EventArray(np.array([event.t], np.uint64), np.array([event.x], np.uint16),
                                      np.array([event.y], np.uint16), np.array([event.polarity], np.int8)))

    def process_array(self, block) -> None:
        """Apply a packet of events in order (host EventArray or DeviceEventArray)."""
        if isinstance(block, DeviceEventArray):
            self._process_device(block)
            return
        n = len(block)
        if not n:
            return
        xs, ys, ps, ts = block.x, block.y, block.p, block.t
        W, H = self.geometry.width, self.geometry.height
        if self.strict:
            oob = (xs >= W) | (ys >= H)
            if oob.any():
                i = int(np.nonzero(oob)[0][0])
                raise DataError(f"event {self.event_count + i} at ({int(xs[i])},{int(ys[i])}) outside {W}x{H}")
            if self.last_t is not None and int(ts[0]) < self.last_t:
                raise OrderError("event timestamps regress across blocks")
            if np.any(ts[1:] < ts[:-1]):
                raise OrderError("event timestamps regress within a block")
        # host packets are copied on the engine's stream (no cross-stream hazard),
        # so the per-packet path skips the current-stream check
        rc = self._lib.fibar_process(self._h, _addr(xs), _addr(ys), _addr(ps), n, _native.FIBAR_MEM_HOST)
        if rc:
            _native.check(rc, "fibar_process")
        self._note_last_t(xs, ys, ts)

    # -- halo-band batches (filter-ON row bands, bands.HaloBandEngine) ----------
    def halo_batch(self, block) -> tuple[int, int, int, int]:
        """Front end of one batch (<= batch capacity events) on a halo-band engine:
        window pass, stale items, temporal replay, blur-tap resolution.  Returns
        (in_top, in_bot, out_top, out_bot): how many blur values this band
        receives from / sends to its neighbours per round (fibar_halo_batch)."""
        counts = np.zeros(4, np.int64)
        self._sync_stream()
        if isinstance(block, DeviceEventArray):
            torch = _torch()
            x = block.x.to(torch.int16).contiguous() if block.x.dtype not in self._xy_ok else block.x.contiguous()
            y = block.y.to(torch.int16).contiguous() if block.y.dtype not in self._xy_ok else block.y.contiguous()
            p = block.p.to(torch.int8).contiguous()
            if self.strict:
                self._check_device_packet(block, x, y)
            rc = self._lib.fibar_halo_batch(self._h, x.data_ptr(), y.data_ptr(), p.data_ptr(), int(x.shape[0]),
                                            _native.FIBAR_MEM_DEVICE, counts.ctypes.data)
            _native.check(rc, "fibar_halo_batch")
            if block.t is not None and len(block.t):
                self._note_last_t(block.x.cpu().numpy(), block.y.cpu().numpy(), block.t)
        else:
            xs = np.ascontiguousarray(block.x, np.uint16)
            ys = np.ascontiguousarray(block.y, np.uint16)
            ps = np.ascontiguousarray(block.p, np.int8)
            rc = self._lib.fibar_halo_batch(self._h, xs.ctypes.data, ys.ctypes.data, ps.ctypes.data, len(xs),
                                            _native.FIBAR_MEM_HOST, counts.ctypes.data)
            _native.check(rc, "fibar_halo_batch")
            if len(xs):
                self._note_last_t(xs, ys, block.t)
        return tuple(int(v) for v in counts)

    def halo_round(self, rnd: int, in_words, out_words) -> None:
        """One blur round: in_words / out_words are int64 CUDA tensors (bit 63 =
        tainted, bits 0-31 = float32 bits), laid out [top | bottom]."""
        self._sync_stream()
        rc = self._lib.fibar_halo_round(self._h, int(rnd), in_words.data_ptr() if in_words.numel() else None,
                                        out_words.data_ptr() if out_words.numel() else None)
        _native.check(rc, "fibar_halo_round")

    def halo_finish(self) -> None:
        self._sync_stream()
        _native.check(self._lib.fibar_halo_finish(self._h), "fibar_halo_finish")

    def _note_last_t(self, xs, ys, ts) -> None:
        # the reference keeps the time of the last *in-bounds* event (pipeline.py:243)
        if ts is None:
            return
        W, H = self.geometry.width, self.geometry.height
        i = len(xs) - 1
        if int(xs[i]) < W and int(ys[i]) < H:
            self.last_t = int(ts[i])
            return
        keep = np.nonzero((xs < W) & (ys < H))[0]
        if keep.size:
            self.last_t = int(ts[keep[-1]])

    def _process_device(self, block: DeviceEventArray) -> None:
        x, y, p = block.x, block.y, block.p
        n = x.shape[0]
        if not n:
            return
        xy_ok = self._xy_ok
        if not (x.dtype in xy_ok and y.dtype in xy_ok and p.dtype is self._i8 and x.is_contiguous()
                and y.is_contiguous() and p.is_contiguous()):
            torch = _torch()
            x = x.contiguous()
            y = y.contiguous()
            p = p.contiguous()
            if x.dtype not in xy_ok:
                x = x.to(torch.int16)
            if y.dtype not in xy_ok:
                y = y.to(torch.int16)
            if p.dtype != torch.int8:
                p = p.to(torch.int8)
        if self.strict:
            self._check_device_packet(block, x, y)
        self._sync_stream()
        rc = self._lib.fibar_process(self._h, x.data_ptr(), y.data_ptr(), p.data_ptr(), n, _native.FIBAR_MEM_DEVICE)
        if rc:
            _native.check(rc, "fibar_process")
        self._held.append((n, x, y, p))
        self._held_n += n
        if self._held_n >= self._release_at:
            self._release_held()
            self._release_at = self._held_n + self._bcap
        if block.t is not None:
            if self.strict:
                self.last_t = int(block.t[-1])
            else:
                # in-bounds test on the host would need the columns; the last event is the
                # common case, resolved lazily on the device copy only when it is out of bounds
                self._pending_last = (x, y, block.t)
                self.last_t = self._resolve_last_t()

    def _check_device_packet(self, block, x, y) -> None:
        torch = _torch()
        W, H = self.geometry.width, self.geometry.height
        xi, yi = x.to(torch.int32) & 0xFFFF, y.to(torch.int32) & 0xFFFF
        oob = (xi >= W) | (yi >= H)
        if bool(oob.any()):
            i = int(torch.nonzero(oob)[0, 0])
            raise DataError(f"event {self.event_count + i} at ({int(xi[i])},{int(yi[i])}) outside {W}x{H}")
        if block.t is not None:
            ts = block.t
            if self.last_t is not None and int(ts[0]) < self.last_t:
                raise OrderError("event timestamps regress across blocks")
            if bool((ts[1:] < ts[:-1]).any()):
                raise OrderError("event timestamps regress within a block")

    def _release_held(self) -> None:
        """Drop references to device packets the native side no longer reads in place."""
        if not self._held:
            return
        pend = C.c_int64(0)
        _native.check(self._lib.fibar_pending(self._h, C.byref(pend), None), "fibar_pending")
        while self._held and self._held_n - self._held[0][0] >= pend.value:
            self._held_n -= self._held.popleft()[0]
        if pend.value == 0:
            self._held.clear()
            self._held_n = 0

    def _resolve_last_t(self):
        x, y, t = self._pending_last
        W, H = self.geometry.width, self.geometry.height
        xi = int(x[-1]) & 0xFFFF
        yi = int(y[-1]) & 0xFFFF
        if xi < W and yi < H:
            return int(t[-1])
        xs = (x.to(_torch().int32) & 0xFFFF).cpu().numpy()
        ys = (y.to(_torch().int32) & 0xFFFF).cpu().numpy()
        keep = np.nonzero((xs < W) & (ys < H))[0]
        return int(t[keep[-1]]) if keep.size else self.last_t

    # -- read-out ------------------------------------------------------------
    def render(self, scale_mode: str = "robust", fixed_bound: float = 1.0, readout_time: int = 0) -> Frame:
        """Map brightness to 8-bit gray (robust 1..99th percentile stretch or fixed +-bound)."""
        mode = self._mode(scale_mode, fixed_bound)
        g = self.geometry
        out = np.empty(g.n_pix, np.uint8)
        bounds = np.zeros(2, np.float64)
        deg = C.c_int32(0)
        self._sync_stream()
        _native.check(self._lib.fibar_render(self._h, mode, float(fixed_bound), out.ctypes.data, _native.FIBAR_MEM_HOST,
                                             bounds.ctypes.data, C.byref(deg)), "fibar_render")
        self._release_held()
        self._warn_saturation()
        return Frame(out.reshape(g.height, g.width), readout_time, scale_mode, (float(bounds[0]), float(bounds[1])),
                     bool(deg.value))

    def render_async(self, scale_mode: str = "robust", fixed_bound: float = 1.0, readout_time: int = 0,
                     out=None, meta=None) -> "AsyncFrame":
        """Enqueue a read-out without waiting (fibar_render_async): the frame of
        the current state, written into ``out`` (a pinned host or CUDA uint8
        (H, W) tensor; pinned host by default) once ``AsyncFrame.event`` fires.
        The next packets' front end overlaps it on the GPU."""
        torch = _torch()
        mode = self._mode(scale_mode, fixed_bound)
        g = self.geometry
        if out is None:
            out = torch.empty((g.height, g.width), dtype=torch.uint8, pin_memory=True)
        dev = out.is_cuda
        if meta is None:
            meta = torch.empty(4, dtype=torch.float64, device=self.device) if dev else \
                torch.empty(4, dtype=torch.float64, pin_memory=True)
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()   # creates the CUDA event (torch makes it lazily); the engine re-records it
        self._sync_stream()
        mem = _native.FIBAR_MEM_DEVICE if dev else _native.FIBAR_MEM_HOST
        _native.check(self._lib.fibar_render_async(self._h, mode, float(fixed_bound), out.data_ptr(), mem,
                                                   meta.data_ptr(), C.c_void_p(ev.cuda_event)), "fibar_render_async")
        self._release_held()
        return AsyncFrame(out, meta, ev, readout_time, scale_mode)

    def brightness_device(self, out=None):
        """The brightness grid as a CUDA float32 (H, W) tensor (device copy, no sync)."""
        torch = _torch()
        g = self.geometry
        if out is None:
            out = torch.empty((g.height, g.width), dtype=torch.float32, device=self.device)
        self._sync_stream()
        _native.check(self._lib.fibar_copy_brightness(self._h, out.data_ptr(), _native.FIBAR_MEM_DEVICE),
                      "fibar_copy_brightness")
        self._release_held()
        return out

    def render_device(self, scale_mode: str = "robust", fixed_bound: float = 1.0, out=None):
        """Render into a CUDA uint8 tensor (H, W) without synchronising; returns the tensor."""
        torch = _torch()
        mode = self._mode(scale_mode, fixed_bound)
        g = self.geometry
        if out is None:
            out = torch.empty((g.height, g.width), dtype=torch.uint8, device=self.device)
        self._sync_stream()
        _native.check(self._lib.fibar_render(self._h, mode, float(fixed_bound), out.data_ptr(), _native.FIBAR_MEM_DEVICE,
                                             None, None), "fibar_render")
        self._release_held()
        return out

    @staticmethod
    def _mode(scale_mode: str, fixed_bound: float) -> int:
        if scale_mode == "robust":
            return _native.FIBAR_RENDER_ROBUST
        if scale_mode == "fixed":
            if not (fixed_bound > 0):
                raise ConfigError("fixed scale bound must be positive")
            return _native.FIBAR_RENDER_FIXED
        raise ConfigError(f"unknown scale mode {scale_mode!r}")


def render_grid(l, scale_mode: str = "robust", fixed_bound: float = 1.0, readout_time: int = 0) -> Frame:
    """Read out any CUDA float32 (H, W) brightness grid (e.g. assembled from row bands)."""
    torch = _torch()
    mode = ReconstructionEngine._mode(scale_mode, fixed_bound)
    lib = _native.load()
    g = l.contiguous()
    if g.dtype != torch.float32 or not g.is_cuda:
        raise ConfigError("render_grid needs a CUDA float32 tensor")
    out = np.empty(g.numel(), np.uint8)
    bounds = np.zeros(2, np.float64)
    deg = C.c_int32(0)
    stream = torch.cuda.current_stream(g.device).cuda_stream
    _native.check(lib.fibar_render_grid(g.data_ptr(), g.numel(), mode, float(fixed_bound), out.ctypes.data,
                                        _native.FIBAR_MEM_HOST, bounds.ctypes.data, C.byref(deg), C.c_void_p(stream)),
                  "fibar_render_grid")
    return Frame(out.reshape(g.shape), readout_time, scale_mode, (float(bounds[0]), float(bounds[1])), bool(deg.value))


# -- frame output ----------------------------------------------------------------


def write_pgm(frame: Frame, path) -> None:
    """Binary PGM (P5, maxval 255)."""
    with open(path, "wb") as fh:
        fh.write(f"P5\n{frame.width} {frame.height}\n255\n".encode("ascii"))
        fh.write(frame.pixels.tobytes())


def read_pgm(path) -> np.ndarray:
    with open(path, "rb") as fh:
        magic = fh.readline().strip()
        if magic != b"P5":
            raise ConfigError(f"not a binary PGM: {magic!r}")
        line = fh.readline()
        while line.startswith(b"#"):
            line = fh.readline()
        w, h = (int(v) for v in line.split())
        if int(fh.readline()) != 255:
            raise ConfigError("only maxval 255 PGM supported")
        return np.frombuffer(fh.read(w * h), dtype=np.uint8).reshape(h, w)


@dataclass
class RunResult:
    frames_emitted: int
    events_processed: int
    oob_dropped: int
    blur_count: int


def _readout_times(fps: float | None, explicit) -> tuple[Iterator[float], bool]:
    if explicit is not None:
        times = list(explicit)
        if any(b < a for a, b in zip(times, times[1:])):
            raise ConfigError("explicit readout times must be non-decreasing")
        return iter(times), True
    if fps is None or not (fps > 0):
        raise ConfigError("need fps > 0 or explicit readout times")
    period = 1e6 / fps

    def grid():
        k = 1
        while True:
            yield k * period
            k += 1

    return grid(), False


_RUN_ZERO_COPY_MAX = 32   # frames handed out as views of pinned buffers at a time
_RUN_DEPTH = 8   # read-outs in flight in run() (the device pipeline holds about five batches)


def _time_key(r, dtype):
    """A read-out time as a scalar of the timestamp dtype with the same 'left'
    split: for integer timestamps t < r <=> t < ceil(r).  (A Python int or
    float against a uint64 array would make numpy convert the whole array.)"""
    if np.issubdtype(dtype, np.integer):
        c = math.ceil(r)
        info = np.iinfo(dtype)
        return dtype.type(min(max(c, info.min), info.max))
    return r


def run(
    engine: ReconstructionEngine,
    blocks: Iterable[EventArray],
    *,
    fps: float | None = 40.0,
    readout_times=None,
    scale_mode: str = "robust",
    fixed_bound: float = 1.0,
    frame_sink: Callable[[int, Frame], None] | None = None,
    out_dir=None,
    diagnostics_path=None,
    async_frames: bool = True,
) -> RunResult:
    """Stream packets through the engine, reading out frames on a time grid.

    A frame at time r reflects exactly the events with t < r (packets are
    split with ``searchsorted(..., 'left')`` as in pipeline.py:379-384);
    explicit read-out times after the stream end render the final state.

    With ``async_frames`` (default, and only without diagnostics) frames are
    rendered asynchronously and handed to ``frame_sink`` in order up to
    ``_RUN_DEPTH`` read-outs late, i.e. after later packets were submitted: the
    frame's pixels are exact, but a sink that reads engine state (counters,
    ``l``) sees a later state than the reference's loop would show.  Pass
    ``async_frames=False`` for the reference's call order (render, then sink).
    """
    if frame_sink is None and out_dir is not None:
        os.makedirs(out_dir, exist_ok=True)

        def frame_sink(index: int, frame: Frame) -> None:
            write_pgm(frame, os.path.join(out_dir, f"frame_{index:06d}.pgm"))

    diag = None
    if diagnostics_path is not None:
        diag = open(diagnostics_path, "w")
        diag.write("frame,readout_us,q_target,fill_ratio,n_pix_act,n_tiles_act,blur_count\n")
    times, explicit = _readout_times(fps, readout_times)
    next_r = next(times, None)
    frame_index = 0
    # Without diagnostics (which read the state at each frame), frames are read
    # out asynchronously (render_async into a small ring of pinned buffers) and
    # handed to the sink in order as they land, so the GPU runs the next
    # packets while earlier frames are copied back.
    pipelined = async_frames and diag is None and hasattr(engine, "render_async")
    pending = collections.deque()
    # pinned frame buffers, kept on the engine across run() calls
    ring = engine.__dict__.setdefault("_run_frame_pool", []) if pipelined else []

    lent = engine.__dict__.setdefault("_run_frames_lent", [0]) if pipelined else [0]

    def give_back(buf) -> None:
        ring.append(buf)
        lent[0] -= 1

    def deliver(af) -> None:
        # the frame's pixels are the pinned buffer itself (no copy); the buffer
        # goes back to the ring once nothing refers to the array any more.  A
        # sink that keeps its frames gets copies from the 33rd on, so the
        # pinned memory lent out stays bounded.
        if lent[0] < _RUN_ZERO_COPY_MAX:
            frame = af.frame(copy=False)
            lent[0] += 1
            weakref.finalize(frame.pixels, give_back, (af.out, af.meta))
        else:
            frame = af.frame()
            ring.append((af.out, af.meta))
        if frame_sink is not None:
            frame_sink(af.index, frame)
        del frame

    def emit(readout) -> None:
        nonlocal frame_index
        if pipelined:
            while pending and (len(pending) >= _RUN_DEPTH or pending[0].ready()):
                deliver(pending.popleft())
            out, meta = ring.pop() if ring else (None, None)
            af = engine.render_async(scale_mode, fixed_bound, readout_time=int(readout), out=out, meta=meta)
            af.index = frame_index
            pending.append(af)
            frame_index += 1
            return
        frame = engine.render(scale_mode, fixed_bound, readout_time=int(readout))
        if frame_sink is not None:
            frame_sink(frame_index, frame)
        if diag is not None:
            q = engine.qs
            r = engine.fill_ratio()
            diag.write(f"{frame_index},{int(readout)},{int(q[QS_TARGET])},"
                       f"{float(r) if r is not None else math.nan:.6f},"
                       f"{int(q[QS_NPIX])},{int(q[QS_NTILES])},{int(q[QS_BLUR])}\n")
        frame_index += 1

    try:
        for block in blocks:
            if not len(block):
                continue
            ts = block.t
            pos = 0
            while next_r is not None and next_r <= ts[-1]:
                idx = int(np.searchsorted(ts, _time_key(next_r, ts.dtype), side="left"))
                if idx > pos:
                    engine.process_array(block.slice(pos, idx))
                    pos = idx
                emit(next_r)
                next_r = next(times, None)
            if pos < len(block):
                engine.process_array(block.slice(pos, len(block)))
        if explicit:
            while next_r is not None:
                emit(next_r)
                next_r = next(times, None)
        while pending:
            deliver(pending.popleft())
    finally:
        # on an error, frames still in flight are copying into pinned buffers
        # that torch does not track: wait for them before the buffers go
        while pending:
            pending.popleft().event.synchronize()
        if diag is not None:
            diag.close()
    ec, ob = engine._counters()
    logger.info("run complete: %d frames, %d events", frame_index, ec)
    return RunResult(frame_index, ec, ob, engine.blur_count)
